"""GPU parity at BASELINE.json's FULL sizes, in the launch configuration bench.py
times (pipelined router, device-buffer ABI call, batches back to back).

The oracle scans the full cache for a seeded sample of prompts of every batch
(first, last and random ones: they span every 128-prompt slice's position) and
replays the predictor (M1) and the assignment (A1, bit-exact) on EVERY prompt.  The
16-prompt C2 batch also runs the whole oracle route over the 1M-row cache (T3 on every
prompt, M2, A2 end to end).

  C2  M = 1M,  d = 768,  L = 12, bursty sizes 357 / 16 / 512 back to back
  C3  M = 10M, d = 768,  L = 12, N = 256 (one GPU holds all 10M rows: 15.4 GB)
  C4  M = 4M,  d = 1024, L = 16, N = 8192 (the tensor-bound regime, A tail in smem)
  C5  M = 2M,  d = 768,  L = 24, N = 4096, skewed predictor + a batch with
      sum(c) = N - 8 (overflow)
"""
import os

import numpy as np
import pytest

import oracle
from synth import argus_inputs as gen
from tests import parity

pytestmark = [pytest.mark.gpu, pytest.mark.full]

CASES = {
    "C2": dict(sizes=[357, 16, 512], sample=32, e2e_max=16),
    "C3": dict(sizes=[256], sample=16),
    "C4": dict(sizes=[8192], sample=16),
    "C5": dict(sizes=[4096, 4096], sample=16, short_quota_batch=1),
}


def _threads():
    return max(1, os.cpu_count() or 1)


@pytest.mark.parametrize("name", list(CASES))
def test_full_size(name):
    import torch
    from paper_2511_06724_b200 import argus
    assert torch.cuda.is_available()
    case = CASES[name]
    cfg = gen.CONFIGS[name]
    d, k = cfg.d, cfg.k
    opts = gen.option_table(cfg.models, cfg.ks)
    L = len(opts)
    W1, b1, W2, b2 = gen.mlp_weights(d, k, cfg.hidden, L, stress=cfg.stress)
    fr = gen.load_fractions(L, cfg.frac_base)
    cg = gen.CacheGen(cfg.M, d, cfg.seed)
    cache = cg.all(threads=_threads())
    sizes = case["sizes"]
    Xs = [gen.queries(cg, n, cfg.seed, b, cache_rows=cache) for b, n in enumerate(sizes)]
    quotas = [oracle.quota_from_fractions(fr, n) for n in sizes]
    if case.get("short_quota_batch") is not None:   # sum(c) = N - 8: eight prompts overflow
        q = quotas[case["short_quota_batch"]]
        for _ in range(8):
            q[int(np.argmax(q))] -= 1
    stream = torch.cuda.Stream()
    with argus.Router(d, k, opts, W1, b1, W2, b2, capacity=cfg.M, max_batch=max(sizes), device=0,
                      stream=stream.cuda_stream, pipeline=True) as r:
        for a, chunk in cg.chunks():
            assert r.argus_cache_insert(chunk) == a   # first global id of the chunk
        Xd = [torch.from_numpy(x).cuda() for x in Xs]
        outs = [dict(option=torch.empty(n, dtype=torch.int32, device="cuda"),
                     topk_idx=torch.empty((n, k), dtype=torch.int32, device="cuda"),
                     topk_score=torch.empty((n, k), dtype=torch.float32, device="cuda"),
                     quality=torch.empty((n, L), dtype=torch.float32, device="cuda"),
                     status=torch.empty(n, dtype=torch.uint8, device="cuda")) for n in sizes]
        torch.cuda.synchronize()
        for x, q, o in zip(Xd, quotas, outs):
            r.argus_route_batch_dev(x, q, o["option"], o["topk_idx"], o["topk_score"], o["quality"], o["status"])
        rc = r.argus_sync()
        torch.cuda.synchronize()
    assert rc in (0, 1)
    rng = np.random.default_rng(2024)
    for b, (X, q, o) in enumerate(zip(Xs, quotas, outs)):
        n = X.shape[0]
        g = {kk: v.cpu().numpy() for kk, v in o.items()}
        g["topk_idx"] = g["topk_idx"].view(np.uint32)
        rows = sorted(set([0, n - 1] + list(rng.choice(n, min(case["sample"], n) - min(2, n), replace=False))))
        tk = parity.check_topk(X, cache, k, g["topk_idx"], g["topk_score"], rows=rows)     # T1 + T3 (sample)
        assert tk["max_score_err"] < 1e-4
        # every returned score is the oracle cosine of the returned id (all prompts)
        ids = g["topk_idx"][:, 0].astype(np.int64)
        probe = rng.choice(n, min(n, 256), replace=False)
        for i in probe:
            assert abs(oracle.cosine(X[i], cache[ids[i]]) - g["topk_score"][i, 0]) <= 1e-4
        err = float(np.abs(oracle.mlp(X, g["topk_score"].astype(np.float64), W1, b1, W2, b2,
                                      threads=_threads()) - g["quality"]).max())      # M1 (all prompts)
        assert err <= parity.SCORE_TOL, err
        rep = parity.check_replay(g, opts, q)                                           # A1 (all prompts)
        parity.invariants(g, opts, q)
        if n <= case.get("e2e_max", 0):  # small batch: the whole oracle route over the full cache
            ores = oracle.route(X, cache, k, W1, b1, W2, b2, opts, q, threads=_threads())
            parity.check_topk(X, cache, k, g["topk_idx"], g["topk_score"])              # T3, every prompt
            np.testing.assert_allclose(g["quality"], ores["rhat"], atol=parity.SCORE_TOL)  # M2
            parity.check_e2e(ores, g, opts, q)                                              # A2
        if case.get("short_quota_batch") == b:
            assert rep["rc"] == 1 and int(np.sum(g["status"] & oracle.OVERFLOW)) > 0
