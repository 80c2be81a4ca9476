"""GPU parity of the opt-in transposed small-N scan (csrc/k_scan_t.cu, ARGUS_SCAN_T=1):
cache rows as the MMA's M, the batch's prompts as its N.  Same checks as the default scan:
T2 (the oracle's O4 on the scan's own captured fp32 scores reproduces the GPU top-k exactly,
every prompt), T1 on the whole score matrix, T3 against the fp64 oracle, A1 replay; and the
outputs equal the default one-slice scan's (k_scan_tc) on the same batch.

Run on a B200 via gpurun: ``python -m pytest tests -m gpu``.
"""
import os

import numpy as np
import pytest

import oracle
from synth import argus_inputs as gen
from tests import parity
from tests.test_gpu_parity_exact import make_router, route_captured

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def argus_mod():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2511_06724_b200 import argus
    return argus


def router_with(argus, p, scan_t):
    """The knob is read once, at argus_route_init."""
    old = os.environ.get("ARGUS_SCAN_T")
    os.environ["ARGUS_SCAN_T"] = "1" if scan_t else "0"
    try:
        return make_router(argus, p)
    finally:
        if old is None:
            os.environ.pop("ARGUS_SCAN_T", None)
        else:
            os.environ["ARGUS_SCAN_T"] = old


# N = 1 / 16 / 33 / 48 / 64 (every B width 16..64), ragged M (last 128-row tile partial),
# k = 1 / 3 / 4 / 8, many tiles per CTA
CASES = [(1, 300, 4, 401), (16, 4133, 4, 402), (33, 9000, 3, 403), (48, 20000, 4, 404), (64, 6001, 8, 405),
         (47, 70000, 1, 406)]


@pytest.mark.parametrize("N,M,k,seed", CASES)
def test_scan_t_exact(argus_mod, N, M, k, seed):
    p = gen.small_problem("C1", N=N, M=M, k=k, seed=seed)
    quota = oracle.quota_from_fractions(p.fractions, N)
    with router_with(argus_mod, p, True) as r:
        r.argus_cache_insert(p.cache)
        rc, g, S = route_captured(argus_mod, r, p.X, quota, M)
    parity.check_topk_replay(S, g["topk_idx"], g["topk_score"], k)          # T2, every row
    if N * M <= 2_000_000:
        So = oracle.score_matrix(p.X, p.cache)
        err = float(np.abs(So - S).max())
        assert err <= parity.SCORE_TOL, err
        parity.report("T1_matrix_scan_t", rows=N, M=M, max_abs_err=err)
    rows = None if N * M <= 5_000_000 else list(range(0, N, 5))
    parity.check_topk(p.X, p.cache, k, g["topk_idx"], g["topk_score"], rows=rows)
    rep = parity.check_replay(g, p.opts, quota)
    assert rc == rep["rc"]
    # the default scan on the same batch: identical outputs
    with router_with(argus_mod, p, False) as r0:
        r0.argus_cache_insert(p.cache)
        rc0, g0 = r0.argus_route_batch(p.X, quota)
    assert rc0 == rc
    for key in ("option", "topk_idx", "topk_score", "quality", "status"):
        np.testing.assert_array_equal(g[key], g0[key], err_msg=key)
