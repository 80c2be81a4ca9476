"""Where the synchronous host call's time goes (diagnostics).  On the C2 cache, per fixed
N: wall time of argus_route_batch through the Python binding, of the bare ctypes call
with preallocated outputs, of argus_route_batch_dev + argus_sync (device prompts), and
the GPU stage times of the same serial calls (argus_profile_*)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_06724_b200 import argus  # noqa: E402
from paper_2511_06724_b200.argus import _lib, _p  # noqa: E402
from synth import argus_inputs as gen  # noqa: E402


def best_of(f, reps=40):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2] * 1e6, ts[0] * 1e6


def main():
    cfg = gen.CONFIGS["C2"]
    d, k = cfg.d, cfg.k
    opts = gen.option_table(cfg.models, cfg.ks)
    L = len(opts)
    W1, b1, W2, b2 = gen.mlp_weights(d, k, cfg.hidden, L)
    fr = gen.load_fractions(L, cfg.frac_base)
    cg = gen.CacheGen(cfg.M, d, cfg.seed)
    rows = cg.all(threads=os.cpu_count() or 1)
    ns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16,48,91,128,320").split(",")]
    with argus.Router(d, k, opts, W1, b1, W2, b2, capacity=cfg.M, max_batch=512, pipeline=True) as r:
        for a in range(0, cfg.M, gen.CHUNK):
            r.argus_cache_insert(rows[a:a + gen.CHUNK])
        for N in ns:
            X = torch.from_numpy(gen.queries(cg, N, cfg.seed, 3, cache_rows=rows)).pin_memory()
            Xn = X.numpy()
            q = argus.argus_quota_from_fractions(fr, N)
            qa = np.ascontiguousarray(q, np.int32)
            pin = lambda s, dt: torch.empty(s, dtype=dt).pin_memory().numpy()  # noqa: E731
            o = [pin((N,), torch.int32), pin((N, k), torch.int32), pin((N, k), torch.float32),
                 pin((N, L), torch.float32), pin((N,), torch.uint8)]
            Xd = X.cuda()
            od = [torch.empty(N, dtype=torch.int32, device="cuda"), torch.empty((N, k), dtype=torch.int32, device="cuda"),
                  torch.empty((N, k), dtype=torch.float32, device="cuda"),
                  torch.empty((N, L), dtype=torch.float32, device="cuda"),
                  torch.empty(N, dtype=torch.uint8, device="cuda")]
            ptrs = [_p(Xn), N, _p(qa)] + [_p(x) for x in o]

            def py():
                r.argus_route_batch(Xn, q, N=N)

            def raw():
                _lib.argus_route_batch(r._h, *ptrs)

            def dev():
                r.argus_route_batch_dev(Xd, q, *od)
                r.argus_sync()

            for f in (py, raw, dev):
                for _ in range(5):
                    f()
            res = {n: best_of(f) for n, f in (("py", py), ("raw", raw), ("dev", dev))}
            r.argus_profile_enable(True)
            for _ in range(20):
                raw()
            pr = r.argus_profile_read()
            r.argus_profile_enable(False)
            st = {s: v[0] * 1e3 / max(v[1], 1) for s, v in pr.items() if v[1]}
            print(f"N={N}: sync call median/min us: py {res['py'][0]:.1f}/{res['py'][1]:.1f}  "
                  f"raw {res['raw'][0]:.1f}/{res['raw'][1]:.1f}  dev+sync {res['dev'][0]:.1f}/{res['dev'][1]:.1f}  "
                  f"| gpu us/launch " + " ".join(f"{s} {v:.1f}" for s, v in st.items()), flush=True)


if __name__ == "__main__":
    main()
