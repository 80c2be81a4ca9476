"""GPU parity of the second workload: SM mode (k = 0: model
variants only, no cache retrieval) and the cache lifecycle
(insert-after-generate with latent handles, and ring eviction at capacity)."""
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


@pytest.mark.parametrize("N,d,seed", [(333, 768, 301), (64, 1024, 302), (1, 768, 303)])
def test_sm_mode_parity(argus_mod, N, d, seed):
    """k = 0: the predictor sees the prompt only (w1 [H][d]); no scan; the option
    table is the six SM variants, all with k_skip = 0; assignment as usual."""
    opts = gen.option_table(("SD-XL", "SD-2.1", "SD-Small", "Tiny-SD"), (0,))
    L = len(opts)
    W1, b1, W2, b2 = gen.mlp_weights(d, 0, 256, L)
    X = gen.small_problem("C1", N=N, M=0, d=d, seed=seed).X
    quota = oracle.quota_from_fractions(gen.load_fractions(L, 1.3), N)
    with argus_mod.Router(d, 0, opts, W1, b1, W2, b2, capacity=0, max_batch=N) as r:
        rc, g = r.argus_route_batch_ex(X, quota)
    S = np.zeros((N, 0))
    ref = oracle.mlp(X, S, W1, b1, W2, b2)
    assert float(np.abs(ref - g["quality"]).max()) <= parity.SCORE_TOL
    g["topk_score"] = np.zeros((N, 1), np.float32)   # s_1 is unused: no option is gated
    parity.check_replay(g, opts, quota)
    parity.invariants(g, opts, quota)


def test_sm_mode_rejects_cache_options(argus_mod):
    p = gen.small_problem("C1", N=4, M=0)
    W1 = p.W1[:, :768]
    with pytest.raises(argus_mod.ArgusError):   # an AC option (k_skip > 0) needs the cache
        argus_mod.Router(768, 0, p.opts, W1, p.b1, p.W2, p.b2, capacity=0, max_batch=4)


@pytest.mark.parametrize("world", [1])
def test_ring_eviction_and_handles(argus_mod, world):
    """Capacity 5000, 8500 rows inserted in three calls: the live set is the last
    5000 (ids 3500..8499, positions wrapped); top-k over exactly those rows with
    their global ids (ties -> older), and every returned id carries its handle."""
    argus = argus_mod
    p = gen.small_problem("C2", N=200, M=8500, seed=304)
    cap, k = 5000, p.k
    handles = (np.arange(8500, dtype=np.uint64) * np.uint64(7919) + np.uint64(11))
    quota = oracle.quota_from_fractions(p.fractions, 200)
    with argus.Router(768, k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=cap, max_batch=200, evict=True) as r:
        for a, b in [(0, 3000), (3000, 6000), (6000, 8500)]:
            assert r.argus_cache_insert_h(p.cache[a:b], handles[a:b]) == a
        assert r.argus_cache_size() == 8500
        # a rejected insert leaves the (full, wrapped) cache unchanged
        bad = p.cache[:10].copy()
        bad[4, 3] = np.nan
        with pytest.raises(argus.ArgusError):
            r.argus_cache_insert_h(bad, None)
        rc, g = r.argus_route_batch_ex(p.X, quota, want_handles=True)
    live_ids = np.arange(3500, 8500, dtype=np.uint32)
    parity.check_topk(p.X, p.cache[3500:8500], k, g["topk_idx"], g["topk_score"], ids=live_ids)
    assert (g["topk_idx"] >= 3500).all() and (g["topk_idx"] < 8500).all()
    np.testing.assert_array_equal(g["topk_handle"], handles[g["topk_idx"].astype(np.int64)])
    parity.check_replay(g, p.opts, quota)


def test_ring_before_wrap_matches_plain_cache(argus_mod):
    """An evicting cache that has not wrapped is the plain cache (bit-identical)."""
    argus = argus_mod
    p = gen.small_problem("C2", N=100, M=3000, seed=305)
    quota = oracle.quota_from_fractions(p.fractions, 100)
    outs = []
    for ev in (False, True):
        with argus.Router(768, p.k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=4096, max_batch=100, evict=ev) as r:
            r.argus_cache_insert(p.cache)
            outs.append(r.argus_route_batch(p.X, quota)[1])
    for key in ("option", "topk_idx", "topk_score", "quality"):
        np.testing.assert_array_equal(outs[0][key], outs[1][key])


def test_ring_eviction_g_invariance(argus_mod):
    """A wrapped ring cache striped over G = 1, 2, 4 routers (external collective
    mode, one GPU): bit-identical outputs, top-k over the live ids, handles."""
    import torch
    argus = argus_mod
    p = gen.small_problem("C2", N=90, M=7000, seed=306)
    N, k, L, cap = 90, p.k, len(p.opts), 4096
    quota = oracle.quota_from_fractions(p.fractions, N)
    handles = np.arange(7000, dtype=np.uint64) + np.uint64(1 << 40)
    X = torch.from_numpy(p.X).cuda()
    ref = None
    for G in (1, 2, 4):
        routers = [argus.Router(768, k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=cap, max_batch=N, rank=rk,
                                world=G, evict=True) for rk in range(G)]
        for r in routers:
            r.argus_cache_insert_h(p.cache[:5000], handles[:5000])
            r.argus_cache_insert_h(p.cache[5000:], handles[5000:])
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
            r.close()
        for o in outs[1:]:
            for kk in o:
                np.testing.assert_array_equal(o[kk], outs[0][kk])
        if ref is None:
            ref = outs[0]
        else:
            for kk in ref:
                np.testing.assert_array_equal(outs[0][kk], ref[kk])
    live = np.arange(7000 - cap, 7000, dtype=np.uint32)
    ref["topk_idx"] = ref["topk_idx"].view(np.uint32)
    parity.check_topk(p.X, p.cache[7000 - cap:], k, ref["topk_idx"], ref["topk_score"], ids=live)
