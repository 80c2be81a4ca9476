"""Diagnostics: where the host-API call's time goes (C2 cache, fixed N).  Not a bench."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_06724_b200 import argus  # noqa: E402
from synth import argus_inputs as gen  # noqa: E402

cfg = gen.CONFIGS["C2"]
d, k = cfg.d, cfg.k
opts = gen.option_table(cfg.models, cfg.ks)
L = len(opts)
W1, b1, W2, b2 = gen.mlp_weights(d, k, cfg.hidden, L)
fr = gen.load_fractions(L, cfg.frac_base)
cg = gen.CacheGen(cfg.M, d, cfg.seed)
rows = cg.all(threads=16)
for N in [int(x) for x in (sys.argv[1:] or ["96"])]:
    for pipe in (False, True):
        r = argus.Router(d, k, opts, W1, b1, W2, b2, capacity=cfg.M, max_batch=512, pipeline=pipe)
        for a in range(0, cfg.M, 65536):
            r.argus_cache_insert(rows[a:a + 65536])
        X = gen.queries(cg, N, cfg.seed, 0, cache_rows=rows)
        Xp = torch.from_numpy(X).pin_memory().numpy()
        Xd = torch.from_numpy(X).cuda()
        q = argus.argus_quota_from_fractions(fr, N)
        o = dict(option=torch.empty(N, dtype=torch.int32, device="cuda"),
                 topk_idx=torch.empty((N, k), dtype=torch.int32, device="cuda"),
                 topk_score=torch.empty((N, k), dtype=torch.float32, device="cuda"),
                 quality=torch.empty((N, L), dtype=torch.float32, device="cuda"),
                 status=torch.empty(N, dtype=torch.uint8, device="cuda"))
        for _ in range(20):
            r.argus_route_batch(Xp, q)
        reps = 200
        t0 = time.perf_counter()
        for _ in range(reps):
            r.argus_route_batch(Xp, q)
        host = (time.perf_counter() - t0) / reps * 1e6
        t0 = time.perf_counter()
        for _ in range(reps):
            r.argus_route_batch_dev(Xd, q, o["option"], o["topk_idx"], o["topk_score"], o["quality"], o["status"])
            r.argus_sync()
        devsync = (time.perf_counter() - t0) / reps * 1e6
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            r.argus_route_batch_dev(Xd, q, o["option"], o["topk_idx"], o["topk_score"], o["quality"], o["status"])
        r.argus_sync()
        devpipe = (time.perf_counter() - t0) / reps * 1e6
        # asynchronous host call (the bench's e2e): host enqueue cost vs wall time per batch
        outs = [dict(option=torch.empty(N, dtype=torch.int32).pin_memory().numpy(),
                     topk_idx=torch.empty((N, k), dtype=torch.int32).pin_memory().numpy().view(np.uint32),
                     topk_score=torch.empty((N, k), dtype=torch.float32).pin_memory().numpy(),
                     quality=torch.empty((N, L), dtype=torch.float32).pin_memory().numpy(),
                     status=torch.empty(N, dtype=torch.uint8).pin_memory().numpy()) for _ in range(8)]
        for i in range(8):
            r.argus_route_wait(r.argus_route_batch_async(Xp, q, outs[i]))
        enq = 0.0
        t0 = time.perf_counter()
        last = None
        for i in range(reps):
            t1 = time.perf_counter()
            last = r.argus_route_batch_async(Xp, q, outs[i % 8])
            enq += time.perf_counter() - t1
        r.argus_route_wait(last)
        asyn = (time.perf_counter() - t0) / reps * 1e6
        print(f"N={N} pipeline={pipe}: async call wall {asyn:.1f} us/batch, host enqueue {enq / reps * 1e6:.1f} us/call",
              flush=True)
        # again after the device-buffer runs (separates power / clock state from the call path)
        t0 = time.perf_counter()
        for i in range(reps):
            last = r.argus_route_batch_async(Xp, q, outs[i % 8])
        r.argus_route_wait(last)
        torch.cuda.synchronize()
        t0b = time.perf_counter()
        for _ in range(reps):
            r.argus_route_batch_dev(Xd, q, o["option"], o["topk_idx"], o["topk_score"], o["quality"], o["status"])
        r.argus_sync()
        devpipe2 = (time.perf_counter() - t0b) / reps * 1e6
        print(f"N={N} pipeline={pipe}: async again {(t0b - t0) / reps * 1e6:.1f} us/batch, then dev pipelined "
              f"{devpipe2:.1f} us/batch", flush=True)
        r.argus_profile_enable(True)
        r.argus_profile_read()
        for _ in range(50):
            r.argus_route_batch_dev(Xd, q, o["option"], o["topk_idx"], o["topk_score"], o["quality"], o["status"])
        pr = r.argus_profile_read()
        r.argus_profile_enable(False)
        stages = {kk: round(v[0] / 50 * 1e3, 1) for kk, v in pr.items() if v[1]}
        t0 = time.perf_counter()
        for _ in range(10000):
            r.argus_cache_size()
        ctypes_us = (time.perf_counter() - t0) / 10000 * 1e6
        print(f"N={N} pipeline={pipe}: host call {host:.1f} us | dev+sync {devsync:.1f} us | dev pipelined "
              f"{devpipe:.1f} us/batch | kernels(us) {stages} | ctypes call {ctypes_us:.2f} us", flush=True)
        r.close()
