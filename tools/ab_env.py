"""In-process A/B of a router environment knob (diagnostics, one GPU).

    python tools/ab_env.py VAR VALUE_A VALUE_B [--n 320] [--steps 40] [--rounds 8] [--config C2]

Two routers over the same cache, one initialised with VAR=VALUE_A, the other with
VAR=VALUE_B (the knobs are read at argus_route_init), then timed windows of --steps
pipelined device calls alternating A, B, A, B ... so both arms see the same power
state (the board's 1000 W cap moves the SM clock between ~1.0 and 1.97 GHz from run
to run, which swamps a few-percent effect between separate bench runs).  --n 0 plays
the C2 trace in order.  Prints one JSON line: per-round ms per step of each arm and
the median B / A ratio.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import argus_inputs as gen  # noqa: E402
from paper_2511_06724_b200 import argus  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("var")
    ap.add_argument("a")
    ap.add_argument("b")
    ap.add_argument("--n", type=int, default=320)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--rounds", type=int, default=8)
    ap.add_argument("--config", default="C2")
    args = ap.parse_args()
    cfg = gen.CONFIGS[args.config]
    d, k = cfg.d, cfg.k
    opts = gen.option_table(cfg.models, cfg.ks)
    L = len(opts)
    W1, b1, W2, b2 = gen.mlp_weights(d, k, cfg.hidden, L, stress=cfg.stress)
    fr = gen.load_fractions(L, cfg.frac_base)
    NT = 64
    if args.n:
        sizes = [args.n] * NT
    else:
        import bench
        NT = bench.N_TRACE
        sizes = bench.batch_sizes(cfg, NT)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    cg = gen.CacheGen(cfg.M, d, cfg.seed)
    rows = cg.all(threads=os.cpu_count() or 1)
    routers = []
    for val in (args.a, args.b):
        os.environ[args.var] = val
        r = argus.Router(d, k, opts, W1, b1, W2, b2, capacity=cfg.M, max_batch=max(sizes), stream=stream.cuda_stream,
                         pipeline=True)
        for a0 in range(0, cfg.M, gen.CHUNK):
            r.argus_cache_insert(rows[a0:a0 + gen.CHUNK])
        routers.append(r)
    os.environ.pop(args.var, None)
    Xd = [torch.from_numpy(gen.queries(cg, n, cfg.seed, b, cache_rows=rows)).to(dev) for b, n in enumerate(sizes)]
    quotas = [argus.argus_quota_from_fractions(fr, n) for n in sizes]
    mb = max(sizes)
    out = dict(option=torch.empty(mb, dtype=torch.int32, device=dev),
               topk_idx=torch.empty((mb, k), dtype=torch.int32, device=dev),
               topk_score=torch.empty((mb, k), dtype=torch.float32, device=dev),
               quality=torch.empty((mb, L), dtype=torch.float32, device=dev),
               status=torch.empty(mb, dtype=torch.uint8, device=dev))

    def window(r, t0):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for t in range(t0, t0 + args.steps):
                b = t % NT
                r.argus_route_batch_dev(Xd[b], quotas[b], out["option"], out["topk_idx"], out["topk_score"],
                                        out["quality"], out["status"], N=sizes[b])
            r.argus_route_join()
            e1.record(stream)
        e1.synchronize()
        r.argus_sync()
        return e0.elapsed_time(e1) / args.steps

    for r in routers:  # warm-up (and a clock ramp)
        for _ in range(3):
            window(r, 0)
    ms = [[], []]
    for rd in range(args.rounds):
        t0 = (rd * args.steps) % NT
        order = (0, 1) if rd % 2 == 0 else (1, 0)
        for i in order:
            ms[i].append(window(routers[i], t0))
    ratio = [b / a for a, b in zip(ms[0], ms[1])]
    print(json.dumps({"var": args.var, "a": args.a, "b": args.b, "n": args.n or "C2 trace", "steps": args.steps,
                      "ms_a": [round(x, 4) for x in ms[0]], "ms_b": [round(x, 4) for x in ms[1]],
                      "median_ratio_b_over_a": round(statistics.median(ratio), 4)}), flush=True)


if __name__ == "__main__":
    main()
