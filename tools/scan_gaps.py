"""Per-CTA timestamps of consecutive pipelined scans (diagnostics, one GPU).

    python tools/scan_gaps.py [--n 48] [--batches 64] [--config C2]

The one-slice scan (k_scan_tc) stamps %globaltimer per CTA at entry, after its
grid-dependency wait, at its first accumulator read and at exit into a buffer this
script owns (ARGUS_SCAN_STAMP).  Prints, per consecutive pair of scans, medians over
the batches of: the drain (first to last CTA exit), the gap from the last exit of scan
b to the first entry / last dependency wait / median first accumulator of scan b+1,
and the batch period (entry to entry).
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=48)
    ap.add_argument("--batches", type=int, default=64)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--pipeline", type=int, default=1)
    args = ap.parse_args()
    cap = args.batches
    stamps = torch.zeros((cap, 256, 4), dtype=torch.int64, device="cuda")
    os.environ["ARGUS_SCAN_STAMP"] = f"{stamps.data_ptr():x},{cap}"
    from paper_2511_06724_b200 import argus
    cfg = gen.CONFIGS[args.config]
    d, k = cfg.d, cfg.k
    opts = gen.option_table(cfg.models, cfg.ks)
    L = len(opts)
    W1, b1, W2, b2 = gen.mlp_weights(d, k, cfg.hidden, L, stress=cfg.stress)
    fr = gen.load_fractions(L, cfg.frac_base)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    cg = gen.CacheGen(cfg.M, d, cfg.seed)
    rows = cg.all(threads=os.cpu_count() or 1)
    r = argus.Router(d, k, opts, W1, b1, W2, b2, capacity=cfg.M, max_batch=args.n, stream=stream.cuda_stream,
                     pipeline=bool(args.pipeline))
    for a0 in range(0, cfg.M, gen.CHUNK):
        r.argus_cache_insert(rows[a0:a0 + gen.CHUNK])
    NT = 16
    Xd = [torch.from_numpy(gen.queries(cg, args.n, cfg.seed, b, cache_rows=rows)).to(dev) for b in range(NT)]
    quota = argus.argus_quota_from_fractions(fr, args.n)
    out = dict(option=torch.empty(args.n, dtype=torch.int32, device=dev),
               topk_idx=torch.empty((args.n, k), dtype=torch.int32, device=dev),
               topk_score=torch.empty((args.n, k), dtype=torch.float32, device=dev),
               quality=torch.empty((args.n, L), dtype=torch.float32, device=dev),
               status=torch.empty(args.n, dtype=torch.uint8, device=dev))

    def run(nb):
        with torch.cuda.stream(stream):
            for t in range(nb):
                r.argus_route_batch_dev(Xd[t % NT], quota, out["option"], out["topk_idx"], out["topk_score"],
                                        out["quality"], out["status"], N=args.n)
            r.argus_route_join()
        r.argus_sync()

    run(2 * cap)  # warm-up + clock ramp; leaves the stamp index at 0
    torch.cuda.synchronize()
    stamps.zero_()
    torch.cuda.synchronize()
    run(cap)
    st = stamps.cpu().numpy().astype(np.float64)
    res = []
    for i in range(cap):
        live = st[i, :, 0] > 0
        res.append(dict(entry=st[i, live, 0], wait=st[i, live, 1], acc=st[i, live, 2], exit=st[i, live, 3]))
    ctas = int(sum(st[0, :, 0] > 0))
    drain, g_entry, g_wait, g_acc, period, dur = [], [], [], [], [], []
    for i in range(cap - 1):
        a, b = res[i], res[i + 1]
        drain.append((a["exit"].max() - a["exit"].min()) / 1e3)
        g_entry.append((b["entry"].min() - a["exit"].max()) / 1e3)
        g_wait.append((b["wait"].max() - a["exit"].max()) / 1e3)
        g_acc.append((np.median(b["acc"]) - a["exit"].max()) / 1e3)
        period.append((b["entry"].min() - a["entry"].min()) / 1e3)
        dur.append((a["exit"].max() - a["wait"].max()) / 1e3)
    med = lambda x: round(statistics.median(x), 2)  # noqa: E731
    print(json.dumps({"n": args.n, "pipeline": args.pipeline, "ctas": ctas, "batches": cap,
                      "us_drain_first_to_last_exit": med(drain),
                      "us_last_exit_to_next_first_entry": med(g_entry),
                      "us_last_exit_to_next_last_wait": med(g_wait),
                      "us_last_exit_to_next_median_first_acc": med(g_acc),
                      "us_last_wait_to_last_exit": med(dur),
                      "us_period_entry_to_entry": med(period)}), flush=True)


if __name__ == "__main__":
    main()
