"""GPU parity of the control-plane steps fused into the tail kernel (through the C
ABI): the optimal option o_i, PASM sampling, the
affinity window and Eq. 3 worker selection, replayed bit-exactly
by the oracle on the GPU's own fp32 r and s_1 (decisions in the kernel's
precision, widened exactly)."""
import numpy as np
import pytest

import oracle
from oracle import control as oc
from synth import argus_inputs as gen
from tests import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def argus_mod():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2511_06724_b200 import argus
    return argus


def make_router(argus, p, max_batch, **kw):
    return argus.Router(p.X.shape[1], p.k, p.opts, p.W1, p.b1, p.W2, p.b2,
                        capacity=max(p.cache.shape[0], 1) + 1024, max_batch=max_batch, **kw)


def _pth(opts):
    return [o["p_th_qpm"] for o in opts]


def _replay_optimal(g, opts):
    rep = oracle.assign(g["quality"].astype(np.float64), g["topk_score"][:, 0].astype(np.float64), opts,
                        np.full(len(opts), 10 ** 6, np.int32))
    p_th = _pth(opts)
    return np.array([oc.optimal_option(g["quality"][i].astype(np.float64), int(rep["adm"][i]), p_th)
                     for i in range(g["quality"].shape[0])], np.int32)


def test_optimal_option_under_sd(argus_mod):
    p = gen.small_problem("C2", N=300, M=20000, seed=201)
    q = oracle.quota_from_fractions(p.fractions, 300)
    with make_router(argus_mod, p, 300) as r:
        r.argus_cache_insert(p.cache)
        rc, g = r.argus_route_batch_ex(p.X, q)
    parity.check_replay(g, p.opts, q)
    np.testing.assert_array_equal(g["optimal"], _replay_optimal(g, p.opts))
    assert len(np.unique(g["optimal"])) > 2


@pytest.mark.parametrize("name,N,M,seed", [("C2", 300, 20000, 202), ("C5", 700, 9000, 203), ("C1", 64, 4096, 204)])
def test_pasm_policy_bit_exact(argus_mod, name, N, M, seed):
    """ODA from the batch's own optimal-option histogram and the allocator's shares;
    every sampled option (and status) equals the oracle's counter-based draw; the
    counter advances per routing call."""
    argus = argus_mod
    p = gen.small_problem(name, N=N, M=M, seed=seed)
    L = len(p.opts)
    q = oracle.quota_from_fractions(p.fractions, N)
    with make_router(argus, p, N) as r:
        r.argus_cache_insert(p.cache)
        _, g0 = r.argus_route_batch_ex(p.X, q)
        H, n = r.argus_affinity_histogram()
        assert n == min(N, 1000)
        np.testing.assert_array_equal(H, oc.affinity_histogram(g0["optimal"], L))
        P = argus.argus_oda_pasm(H.astype(np.float64) + 1e-3, p.fractions)
        seed_ = 0x1234_5678_9ABC
        r.argus_set_policy(argus.POLICY_PASM, P, seed_)
        outs = [r.argus_route_batch_ex(p.X, None)[1] for _ in range(3)]
    for b, g in enumerate(outs):
        ref = oc.pasm_assign(g["quality"], g["topk_score"][:, 0], p.opts, P, seed_, b)
        np.testing.assert_array_equal(g["optimal"], ref["optimal"])
        np.testing.assert_array_equal(g["option"], ref["option"])
        np.testing.assert_array_equal(g["status"], ref["status"])
    assert not np.array_equal(outs[0]["option"], outs[1]["option"])      # batch counter enters the draw
    # the served mix follows the PASM push-forward (loose: one batch of samples)
    counts = np.bincount(np.concatenate([g["option"] for g in outs]), minlength=L)
    assert counts.sum() == 3 * N


def test_affinity_window_wraps(argus_mod):
    p = gen.small_problem("C2", N=450, M=5000, seed=205)
    L = len(p.opts)
    q = oracle.quota_from_fractions(p.fractions, 450)
    hist = []
    with make_router(argus_mod, p, 450) as r:
        r.argus_cache_insert(p.cache)
        for b in range(4):   # 1800 prompts through a 1000-prompt window
            X = p.X[np.random.default_rng(b).permutation(450)]
            _, g = r.argus_route_batch_ex(X, q)
            hist.extend(g["optimal"].tolist())
        H, n = r.argus_affinity_histogram()
    assert n == 1000
    np.testing.assert_array_equal(H, oc.affinity_histogram(hist, L, 1000))


@pytest.mark.parametrize("policy", [0, 1])
def test_worker_selection_bit_exact(argus_mod, policy):
    """Eq. 3 over two batches (queues carried on the device) equals the oracle's
    sequential argmin on the GPU's assignments; options nobody serves get -1."""
    argus = argus_mod
    p = gen.small_problem("C2", N=257, M=8000, seed=206)
    L = len(p.opts)
    q = oracle.quota_from_fractions(p.fractions, 257)
    rng = np.random.default_rng(7)
    n_w = 40
    wo = rng.integers(-1, L - 1, n_w).astype(np.int32)     # option L-1 is served by nobody
    t = rng.choice([2.18, 3.0, 4.2], n_w).astype(np.float32)
    q0 = rng.integers(0, 5, n_w).astype(np.int32)
    with make_router(argus, p, 257) as r:
        r.argus_cache_insert(p.cache)
        if policy == 1:
            r.argus_set_policy(argus.POLICY_PASM, argus.argus_oda_pasm(np.ones(L), p.fractions), 99)
        r.argus_set_workers(wo, t, q0)
        outs = [r.argus_route_batch_ex(p.X[::-1] if b else p.X, q, want_workers=True)[1] for b in range(2)]
        qf = r.argus_get_queues()
    queue = q0
    for g in outs:
        w, queue = oc.select_workers(g["option"], wo, t, queue)
        np.testing.assert_array_equal(g["worker"], w)
    np.testing.assert_array_equal(qf, queue)
    assert (outs[0]["worker"] >= 0).any()


def test_pasm_pipelined_matches_serial(argus_mod):
    import torch
    argus = argus_mod
    p = gen.small_problem("C2", N=300, M=30000, seed=207)
    L, k = len(p.opts), p.k
    P = argus.argus_oda_pasm(np.ones(L), p.fractions)
    sizes = [64, 300, 129, 1, 200]
    batches = [p.X[:n] for n in sizes]
    wo = np.arange(L, dtype=np.int32) % L
    t = np.full(L, 3.0, np.float32)
    with make_router(argus, p, 300) as r:
        r.argus_cache_insert(p.cache)
        r.argus_set_policy(argus.POLICY_PASM, P, 5)
        r.argus_set_workers(wo, t, np.zeros(L, np.int32))
        ref = [r.argus_route_batch_ex(x, None, want_workers=True)[1] for x in batches]
    with make_router(argus, p, 300, pipeline=True) as r:
        r.argus_cache_insert(p.cache)
        r.argus_set_policy(argus.POLICY_PASM, P, 5)
        r.argus_set_workers(wo, t, np.zeros(L, np.int32))
        outs = []
        for x in batches:
            n = x.shape[0]
            o = dict(option=torch.empty(n, dtype=torch.int32, device="cuda"),
                     topk_idx=torch.empty((n, k), dtype=torch.int32, device="cuda"),
                     topk_score=torch.empty((n, k), dtype=torch.float32, device="cuda"),
                     optimal=torch.empty(n, dtype=torch.int32, device="cuda"),
                     worker=torch.empty(n, dtype=torch.int32, device="cuda"))
            r.argus_route_batch_ex_dev(torch.from_numpy(x).cuda(), None, o["option"], o["topk_idx"],
                                       o["topk_score"], None, None, o["optimal"], o["worker"])
            outs.append(o)
        r.argus_sync()
    for a, b in zip(ref, outs):
        for key in ("option", "optimal", "worker"):
            np.testing.assert_array_equal(b[key].cpu().numpy(), a[key])
