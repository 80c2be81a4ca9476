"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Run on a B200 via gpurun: ``python -m pytest tests -m gpu``.
Sizes: C1 (N=64, M=4096, d=768) plus ragged variants that span several scan
tiles and a ragged tail; edge cases (empty cache, M < k, duplicates, invalid
inputs, overflow); G-invariance with striped shards on one GPU.
"""
import numpy as np
import pytest

import oracle
from synth import argus_inputs as gen
from tests import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def argus_mod():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2511_06724_b200 import argus
    return argus


def make_router(argus, p, max_batch=None, capacity=None, **kw):
    N = p.X.shape[0]
    return argus.Router(p.X.shape[1], p.k, p.opts, p.W1, p.b1, p.W2, p.b2,
                        capacity=capacity or max(p.cache.shape[0], 1) + 1024,
                        max_batch=max_batch or max(N, 1), **kw)


def run_case(argus, p, quota=None, check_e2e=True):
    N = p.X.shape[0]
    quota = oracle.quota_from_fractions(p.fractions, N) if quota is None else np.asarray(quota, np.int32)
    with make_router(argus, p) as r:
        if p.cache.shape[0]:
            assert r.argus_cache_insert(p.cache) == 0
        rc, g = r.argus_route_batch(p.X, quota)
    tk = parity.check_topk(p.X, p.cache, p.k, g["topk_idx"], g["topk_score"])
    parity.check_mlp_replay(p.X, g, p.W1, p.b1, p.W2, p.b2)
    rep = parity.check_replay(g, p.opts, quota)
    assert rc == rep["rc"]
    parity.invariants(g, p.opts, quota)
    frac = None
    if check_e2e and p.cache.shape[0]:
        ores = oracle.route(p.X, p.cache, p.k, p.W1, p.b1, p.W2, p.b2, p.opts, quota)
        np.testing.assert_allclose(g["quality"], ores["rhat"], atol=parity.SCORE_TOL)   # M2
        frac = parity.check_e2e(ores, g, p.opts, quota)
    return g, tk, frac


def test_c1_parity(argus_mod):
    p = gen.small_problem("C1")
    g, tk, frac = run_case(argus_mod, p)
    assert tk["max_score_err"] < 1e-4
    assert frac is not None and frac <= 2   # exempt (fragile) prompts
    # 30 % exact repeats: self-similarity 1 within the bf16/fp32 error
    assert np.sum(g["topk_score"][:, 0] > 0.9999) >= 5


@pytest.mark.parametrize("N,M,k,seed", [(77, 4133, 4, 11), (1, 300, 4, 12), (200, 9000, 8, 13),
                                        (129, 2048 + 63, 2, 14), (300, 5000, 1, 15),
                                        # odd N * k: candidate lists start 8 bytes off a 16-byte line
                                        (77, 4133, 3, 16), (33, 9000, 7, 17), (75, 9000, 1, 18),
                                        (257, 20000, 5, 19)])
def test_ragged_parity(argus_mod, N, M, k, seed):
    p = gen.small_problem("C1", N=N, M=M, k=k, seed=seed)
    run_case(argus_mod, p)


def test_gates_off_and_stress(argus_mod):
    p = gen.small_problem("C1", N=150, M=3000, seed=21, gates=False)
    run_case(argus_mod, p)
    p = gen.small_problem("C5", N=400, M=6000, seed=22)
    quota = oracle.quota_from_fractions(p.fractions, 400)
    g, _, _ = run_case(argus_mod, p, quota)
    assert len(np.unique(g["option"])) > 3


@pytest.mark.parametrize("N", [10, 200, 300])
def test_empty_cache_and_m_less_than_k(argus_mod, N):
    """N = 200 runs the CTA-pair scan, N = 300 three single-CTA slices."""
    p = gen.small_problem("C1", N=N, M=0, seed=31)
    g, _, _ = run_case(argus_mod, p, check_e2e=False)
    assert np.all(g["topk_idx"] == 0xFFFFFFFF) and np.all(g["topk_score"] == -1.0)
    p = gen.small_problem("C1", N=N, M=3, seed=32)
    g, _, _ = run_case(argus_mod, p)
    assert np.all(g["topk_idx"][:, 3] == 0xFFFFFFFF)


def test_duplicates_tie_to_lower_id(argus_mod):
    p = gen.small_problem("C1", N=8, M=1000, seed=33)
    p.cache[700] = p.cache[5]
    p.cache[900] = p.cache[5]
    p.X[0] = p.cache[5]
    g, _, _ = run_case(argus_mod, p)
    assert list(g["topk_idx"][0, :3]) == [5, 700, 900]
    assert g["topk_score"][0, 0] == g["topk_score"][0, 1] == g["topk_score"][0, 2]


def test_overflow_warning(argus_mod):
    p = gen.small_problem("C1", N=50, M=2000, seed=41)
    quota = np.zeros(len(p.opts), np.int32)
    quota[0] = 20
    quota[-1] = 5
    g, _, _ = run_case(argus_mod, p, quota)
    assert int(((g["status"] & 1) != 0).sum()) >= 25


def test_invalid_inputs(argus_mod):
    argus = argus_mod
    p = gen.small_problem("C1", N=4, M=100, seed=51)
    quota = oracle.quota_from_fractions(p.fractions, 4)
    with make_router(argus, p, capacity=150) as r:
        r.argus_cache_insert(p.cache)
        bad = p.X.copy()
        bad[2, 5] = np.nan
        with pytest.raises(argus.ArgusError) as e:
            r.argus_route_batch(bad, quota)
        assert e.value.code == argus.ARGUS_E_INVALID
        bad = p.X.copy()
        bad[1] = 0
        with pytest.raises(argus.ArgusError):
            r.argus_route_batch(bad, quota)
        with pytest.raises(argus.ArgusError):
            r.argus_route_batch(p.X, np.full(len(p.opts), -1, np.int32))
        with pytest.raises(argus.ArgusError) as e:
            r.argus_cache_insert(p.cache)          # 100 + 100 > 150
        assert e.value.code == argus.ARGUS_E_CAPACITY
        zero = np.zeros((3, p.X.shape[1]), np.float32)
        with pytest.raises(argus.ArgusError):
            r.argus_cache_insert(zero)
        assert r.argus_cache_size() == 100         # failed inserts leave M unchanged
        rc, g = r.argus_route_batch(p.X, quota)    # router still usable
        assert g["topk_idx"].shape == (4, p.k)


def test_determinism(argus_mod):
    p = gen.small_problem("C1", N=90, M=5000, seed=61)
    quota = oracle.quota_from_fractions(p.fractions, 90)
    outs = []
    for _ in range(2):
        with make_router(argus_mod, p) as r:
            r.argus_cache_insert(p.cache[:2500])
            r.argus_cache_insert(p.cache[2500:])
            outs.append(r.argus_route_batch(p.X, quota)[1])
    for key in ("option", "topk_idx", "topk_score", "quality", "status"):
        np.testing.assert_array_equal(outs[0][key], outs[1][key])


@pytest.mark.parametrize("N", [70, 256])
def test_g_invariance_striped_shards(argus_mod, N):
    """Outputs are bit-identical for G = 1, 2, 3, 4, 8 striped shards:
    G routers on one GPU in external-collective mode, keys concatenated here.
    N = 256 runs the CTA-pair scan on every shard."""
    import torch
    argus = argus_mod
    p = gen.small_problem("C1", N=N, M=6001, seed=71)
    k, L = p.k, len(p.opts)
    quota = oracle.quota_from_fractions(p.fractions, N)
    X = torch.from_numpy(p.X).cuda()
    ref = None
    for G in (1, 2, 3, 4, 8):
        routers = [make_router(argus, p, rank=rk, world=G) for rk in range(G)]
        for r in routers:
            r.argus_cache_insert(p.cache)
        keys = torch.zeros((G, N, k), dtype=torch.int64, device="cuda")
        for rk, r in enumerate(routers):
            r.argus_route_partial_dev(X, keys[rk])
        for r in routers:
            r.argus_sync()
        outs = []
        for r in routers:
            o = dict(option=torch.empty(N, dtype=torch.int32, device="cuda"),
                     topk_idx=torch.empty((N, k), dtype=torch.int32, device="cuda"),
                     topk_score=torch.empty((N, k), dtype=torch.float32, device="cuda"),
                     quality=torch.empty((N, L), dtype=torch.float32, device="cuda"),
                     status=torch.empty(N, dtype=torch.uint8, device="cuda"))
            r.argus_route_finish_dev(keys, G, N, quota, o["option"], o["topk_idx"], o["topk_score"],
                                     o["quality"], o["status"])
            r.argus_sync()
            outs.append({kk: v.cpu().numpy() for kk, v in o.items()})
        for o in outs[1:]:
            for kk in o:
                np.testing.assert_array_equal(o[kk], outs[0][kk])
        if ref is None:
            ref = outs[0]
        else:
            for kk in ref:
                np.testing.assert_array_equal(outs[0][kk], ref[kk])
        for r in routers:
            r.close()
    g = dict(ref)
    g["topk_idx"] = g["topk_idx"].view(np.uint32)
    parity.check_topk(p.X, p.cache, k, g["topk_idx"], g["topk_score"])
    parity.check_replay(g, p.opts, quota)


def test_dev_path_matches_host_path(argus_mod):
    import torch
    p = gen.small_problem("C1", N=100, M=4500, seed=81)
    N, k, L = 100, p.k, len(p.opts)
    quota = oracle.quota_from_fractions(p.fractions, N)
    with make_router(argus_mod, p) as r:
        r.argus_cache_insert_dev(torch.from_numpy(p.cache).cuda())
        rc, g = r.argus_route_batch(p.X, quota)
        X = torch.from_numpy(p.X).cuda()
        o = dict(option=torch.empty(N, dtype=torch.int32, device="cuda"),
                 topk_idx=torch.empty((N, k), dtype=torch.int32, device="cuda"),
                 topk_score=torch.empty((N, k), dtype=torch.float32, device="cuda"),
                 quality=torch.empty((N, L), dtype=torch.float32, device="cuda"),
                 status=torch.empty(N, dtype=torch.uint8, device="cuda"))
        r.argus_route_batch_dev(X, quota, o["option"], o["topk_idx"], o["topk_score"], o["quality"], o["status"])
        assert r.argus_sync() == rc
    np.testing.assert_array_equal(o["option"].cpu().numpy(), g["option"])
    np.testing.assert_array_equal(o["topk_idx"].cpu().numpy().view(np.uint32), g["topk_idx"])
    np.testing.assert_array_equal(o["quality"].cpu().numpy(), g["quality"])


@pytest.mark.parametrize("N,M,seed", [(70, 60000, 91), (300, 30000, 92), (129, 40000, 93)])
def test_many_tiles_per_cta(argus_mod, N, M, seed):
    """Every CTA walks many cache tiles (buffer / accumulator / barrier phases wrap
    several times), including the multi-slice (N > 128) launch."""
    p = gen.small_problem("C2", N=N, M=M, seed=seed)
    quota = oracle.quota_from_fractions(p.fractions, N)
    with make_router(argus_mod, p) as r:
        r.argus_cache_insert(p.cache)
        rc, g = r.argus_route_batch(p.X, quota)
    parity.check_topk(p.X, p.cache, p.k, g["topk_idx"], g["topk_score"])
    parity.check_replay(g, p.opts, quota)
    parity.invariants(g, p.opts, quota)


def test_pipelined_matches_serial(argus_mod):
    """argus_config.pipeline = 1: the tail of batch b runs on the internal stream
    while batch b+1 is scanned; outputs of every batch are bit-identical to the
    serial router's, for a mix of batch sizes (1 and several slices) and after
    joins on the router's stream, a foreign stream and argus_sync."""
    import torch
    argus = argus_mod
    p = gen.small_problem("C2", N=300, M=30000, seed=101)
    k, L = p.k, len(p.opts)
    sizes = [64, 200, 1, 129, 300, 77, 128, 256, 33, 300]
    rng = np.random.default_rng(5)
    batches = [p.X[rng.choice(300, n, replace=False)] for n in sizes]
    quotas = [oracle.quota_from_fractions(p.fractions, n) for n in sizes]
    with make_router(argus, p) as r:
        r.argus_cache_insert(p.cache)
        ref = [r.argus_route_batch(x, q) for x, q in zip(batches, quotas)]
    with make_router(argus, p, pipeline=True) as r:
        r.argus_cache_insert(p.cache)
        Xd = [torch.from_numpy(x).cuda() for x in batches]
        outs = [dict(option=torch.full((n,), -7, dtype=torch.int32, device="cuda"),
                     topk_idx=torch.empty((n, k), dtype=torch.int32, device="cuda"),
                     topk_score=torch.empty((n, k), dtype=torch.float32, device="cuda"),
                     quality=torch.empty((n, L), dtype=torch.float32, device="cuda"),
                     status=torch.empty(n, dtype=torch.uint8, device="cuda")) for n in sizes]
        torch.cuda.synchronize()
        for x, q, o in zip(Xd, quotas, outs):   # back to back: tails overlap the next scans
            r.argus_route_batch_dev(x, q, o["option"], o["topk_idx"], o["topk_score"], o["quality"], o["status"])
        side = torch.cuda.Stream()
        r.argus_route_join(side.cuda_stream)      # a foreign stream sees every batch's outputs
        with torch.cuda.stream(side):
            got = [{kk: v.to("cpu", non_blocking=False) for kk, v in o.items()} for o in outs]
        side.synchronize()
        rc_dev = r.argus_sync()
        # the host API on a pipelined router stays synchronous and identical
        rc_h, gh = r.argus_route_batch(batches[3], quotas[3])
    for (rc, g), o in zip(ref, got):
        np.testing.assert_array_equal(o["option"].numpy(), g["option"])
        np.testing.assert_array_equal(o["topk_idx"].numpy().view(np.uint32), g["topk_idx"])
        np.testing.assert_array_equal(o["topk_score"].numpy(), g["topk_score"])
        np.testing.assert_array_equal(o["quality"].numpy(), g["quality"])
        np.testing.assert_array_equal(o["status"].numpy(), g["status"])
    assert rc_dev == max(rc for rc, _ in ref)
    for kk in gh:
        np.testing.assert_array_equal(gh[kk], ref[3][1][kk])
    assert rc_h == ref[3][0]


@pytest.mark.parametrize("N,M,d,seed", [(64, 4096, 1024, 111), (200, 20000, 1024, 112), (77, 9000, 832, 113),
                                        (129, 5000, 960, 114), (33, 3000, 64, 115), (256, 6000, 64, 116),
                                        (200, 7000, 128, 117), (512, 5000, 192, 118)])
def test_wide_and_narrow_embeddings(argus_mod, N, M, d, seed):
    """d > 768 (OpenCLIP-H d = 1024, C4): k-blocks 12.. of the prompt slice are read by
    the MMA from shared memory, cache tiles stream through quarter-tile slots; d = 832
    / 960 split unevenly over the quarters; d = 64 is a single k-block (one of the two
    half-tile slots of a tile is then empty), also on CTA pairs (N = 200, 256, 512)."""
    p = gen.small_problem("C4", N=N, M=M, d=d, seed=seed)
    g, tk, _ = run_case(argus_mod, p)
    assert tk["max_score_err"] < 1e-4


@pytest.mark.parametrize("seed", [131, 132, 133, 134])
def test_assignment_random_quotas(argus_mod, seed):
    """The tail's parallel deferred-acceptance rounds must equal the oracle's serial
    dictatorship (O10) bit-exactly under arbitrary quotas: zeros, a few large ones,
    sum below N (overflow) and far above N."""
    p = gen.small_problem("C5", N=700, M=6000, seed=seed)
    rng = np.random.default_rng(seed)
    L = len(p.opts)
    with make_router(argus_mod, p) as r:
        r.argus_cache_insert(p.cache)
        for trial in range(6):
            q = rng.integers(0, 80, L).astype(np.int32)
            q[rng.random(L) < 0.3] = 0
            if trial == 0:
                q[:] = 0
                q[0] = 700                    # everything on the full model
            if trial == 1:
                q = (q * 10).astype(np.int32)  # slack everywhere
            rc, g = r.argus_route_batch(p.X, q)
            rep = parity.check_replay(g, p.opts, q)
            assert rc == rep["rc"]
            parity.invariants(g, p.opts, q)


@pytest.mark.parametrize("pipeline", [False, True])
def test_async_host_calls_match_sync(argus_mod, pipeline):
    """argus_route_batch_async (pinned host buffers, H2D + path + D2H enqueued, up to
    two calls in flight) returns exactly what the synchronous host call returns, and
    each ticket carries its own result code (overflow, invalid prompt)."""
    import torch
    argus = argus_mod
    p = gen.small_problem("C2", N=300, M=20000, seed=141)
    k, L = p.k, len(p.opts)
    sizes = [64, 300, 1, 129, 300, 77, 200, 33]
    rng = np.random.default_rng(9)
    batches = [np.ascontiguousarray(p.X[rng.choice(300, n, replace=False)]) for n in sizes]
    quotas = [oracle.quota_from_fractions(p.fractions, n) for n in sizes]
    quotas[3] = np.maximum(quotas[3] - 20, 0).astype(np.int32)     # overflow in call 3
    bad = 5
    batches[bad] = batches[bad].copy()
    batches[bad][3, 7] = np.nan                                       # invalid prompt in call 5
    with make_router(argus, p, max_batch=300, pipeline=pipeline) as r:
        r.argus_cache_insert(p.cache)
        ref = []
        for b, (x, q) in enumerate(zip(batches, quotas)):
            if b == bad:
                with pytest.raises(argus.ArgusError):
                    r.argus_route_batch(x, q)
                ref.append(None)
            else:
                ref.append(r.argus_route_batch(x, q))
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        tickets, outs = [], []
        for x, q in zip(batches, quotas):
            n = x.shape[0]
            o = dict(option=pin(np.full(n, -7, np.int32)), topk_idx=pin(np.zeros((n, k), np.uint32)),
                     topk_score=pin(np.zeros((n, k), np.float32)), quality=pin(np.zeros((n, L), np.float32)),
                     status=pin(np.zeros(n, np.uint8)))
            tickets.append(r.argus_route_batch_async(pin(x), q, o))
            outs.append(o)
        rcs = []
        for t in tickets:
            try:
                rcs.append(r.argus_route_wait(t))
            except argus.ArgusError as e:
                rcs.append(e.code)
    for b, (rf, o, rc) in enumerate(zip(ref, outs, rcs)):
        if b == bad:
            assert rc == argus.ARGUS_E_INVALID
            continue
        assert rc == rf[0], (b, rc, rf[0])
        for key in ("option", "topk_idx", "topk_score", "quality", "status"):
            np.testing.assert_array_equal(o[key], rf[1][key])
    assert rcs[3] == 1   # ARGUS_W_OVERFLOW


@pytest.mark.parametrize("N,M,k,seed", [(768, 90000, 4, 151), (1300, 80000, 4, 152), (768, 85000, 8, 153)])
def test_pair_scan_migration(argus_mod, N, M, k, seed):
    """More pair slices than divide the 74 TPC pairs evenly (N = 768: 3 pair slices;
    N = 1300: 6): every TPC runs a pair, pairs whose slice runs dry reload another
    slice's prompts and continue its tiles.  Top-k and assignment must be exact."""
    p = gen.small_problem("C2", N=N, M=M, k=k, seed=seed)
    quota = oracle.quota_from_fractions(p.fractions, N)
    with make_router(argus_mod, p) as r:
        r.argus_cache_insert(p.cache)
        rc, g = r.argus_route_batch(p.X, quota)
        rc2, g2 = r.argus_route_batch(p.X, quota)
    np.testing.assert_array_equal(g["topk_idx"], g2["topk_idx"])    # migration timing never changes results
    rows = list(range(0, N, 3))
    parity.check_topk(p.X, p.cache, p.k, g["topk_idx"], g["topk_score"], rows=rows)
    parity.check_replay(g, p.opts, quota)
    parity.invariants(g, p.opts, quota)


def test_largest_shapes(argus_mod):
    """The ABI's largest shapes at once: max_batch 8192, d = 1024, k = 8, L = 32
    (4 models x 8 skip levels) -- the CTA-pair scan with floating pairs, 8-key
    lists, a 32-lane option table in the tail."""
    N, M, d, k = 8192, 50000, 1024, 8
    p = gen.small_problem("C4", N=N, M=M, d=d, k=k, seed=181)
    opts = gen.option_table(("SD-XL", "SD-2.1", "SD-Small", "Tiny-SD"), (0, 3, 6, 9, 12, 15, 18, 21))
    assert len(opts) == 32
    W1, b1, W2, b2 = gen.mlp_weights(d, k, 256, 32)
    quota = oracle.quota_from_fractions(gen.load_fractions(32, 1.1), N)
    with argus_mod.Router(d, k, opts, W1, b1, W2, b2, capacity=M, max_batch=N) as r:
        r.argus_cache_insert(p.cache)
        rc, g = r.argus_route_batch(p.X, quota)
    rows = list(range(0, N, 128)) + [N - 1]
    parity.check_topk(p.X, p.cache, k, g["topk_idx"], g["topk_score"], rows=rows)
    err = float(np.abs(oracle.mlp(p.X, g["topk_score"].astype(np.float64), W1, b1, W2, b2) - g["quality"]).max())
    assert err <= parity.SCORE_TOL
    rep = parity.check_replay(g, opts, quota)
    assert rc == rep["rc"]
    parity.invariants(g, opts, quota)


@pytest.mark.parametrize("pipeline", [False, True])
def test_bf16_device_prompts_match_fp32(argus_mod, pipeline):
    """argus_route_batch_bf16_dev (SURVEY §8(b)'s bf16 device prompts): the fp32 batch
    rounded to bf16 by torch (RNE, pinned against the oracle's O1) routes bit-identically
    to the fp32 call; a NaN row fails with ARGUS_E_INVALID at argus_sync."""
    import torch
    argus = argus_mod
    p = gen.small_problem("C1", N=200, M=7000, seed=191)
    N, k, L = 200, p.k, len(p.opts)
    quota = oracle.quota_from_fractions(p.fractions, N)
    X = torch.from_numpy(p.X).cuda()
    Xh = X.to(torch.bfloat16)
    outs = []
    with make_router(argus, p, pipeline=pipeline) as r:
        r.argus_cache_insert(p.cache)
        for bf in (False, True):
            o = dict(option=torch.empty(N, dtype=torch.int32, device="cuda"),
                     topk_idx=torch.empty((N, k), dtype=torch.int32, device="cuda"),
                     topk_score=torch.empty((N, k), dtype=torch.float32, device="cuda"),
                     quality=torch.empty((N, L), dtype=torch.float32, device="cuda"),
                     status=torch.empty(N, dtype=torch.uint8, device="cuda"),
                     optimal=torch.empty(N, dtype=torch.int32, device="cuda"))
            fn = r.argus_route_batch_bf16_dev if bf else r.argus_route_batch_ex_dev
            fn(Xh if bf else X, quota, o["option"], o["topk_idx"], o["topk_score"], o["quality"], o["status"],
               optimal=o["optimal"])
            r.argus_sync()
            outs.append({kk: v.cpu().numpy() for kk, v in o.items()})
        bad = Xh.clone()
        bad[5, 3] = float("nan")
        o = outs[0]
        r.argus_route_batch_bf16_dev(bad, quota, *(torch.empty_like(torch.from_numpy(v)).cuda() for v in
                                                   (o["option"], o["topk_idx"], o["topk_score"])))
        with pytest.raises(argus.ArgusError) as e:
            r.argus_sync()
        assert e.value.code == argus.ARGUS_E_INVALID
    for kk in outs[0]:
        np.testing.assert_array_equal(outs[0][kk], outs[1][kk], err_msg=kk)
    g = dict(outs[1])
    g["topk_idx"] = g["topk_idx"].view(np.uint32)
    parity.check_topk(p.X, p.cache, k, g["topk_idx"], g["topk_score"], rows=range(0, N, 9))
    parity.check_replay(g, p.opts, quota)
