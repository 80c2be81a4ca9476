"""The multi-GPU data path on one GPU: a router built with world = 1 and an NCCL
unique id runs every collective of the G-GPU path through a one-rank NCCL
communicator (rank 0's rows and prompts broadcast, the per-shard K5 merge, the
all-gather of the N x k candidate keys, the handle broadcast) and must return
exactly what the single-GPU router returns."""
import numpy as np
import pytest

import oracle
from synth import argus_inputs as gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def argus_mod():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2511_06724_b200 import argus
    return argus


@pytest.mark.parametrize("N,M,evict", [(300, 20000, False), (200, 9000, True), (77, 4133, False)])
def test_one_rank_nccl_path_matches_single_gpu(argus_mod, N, M, evict):
    import torch
    argus = argus_mod
    p = gen.small_problem("C2", N=N, M=M, seed=171)
    quota = oracle.quota_from_fractions(p.fractions, N)
    cap = M - M // 3 if evict else M + 64
    handles = np.arange(M, dtype=np.uint64) * np.uint64(3) + np.uint64(5)
    outs = []
    for uid in (None, argus.argus_nccl_unique_id()):
        with argus.Router(768, p.k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=cap, max_batch=N, evict=evict,
                          nccl_unique_id=uid) as r:
            r.argus_cache_insert_h(p.cache[: M // 2], handles[: M // 2])
            r.argus_cache_insert_h(p.cache[M // 2:], handles[M // 2:])
            rc, g = r.argus_route_batch_ex(p.X, quota, want_handles=True)
            X = torch.from_numpy(p.X).cuda()
            o = dict(option=torch.empty(N, dtype=torch.int32, device="cuda"),
                     topk_idx=torch.empty((N, p.k), dtype=torch.int32, device="cuda"),
                     topk_score=torch.empty((N, p.k), dtype=torch.float32, device="cuda"))
            r.argus_route_batch_dev(X, quota, o["option"], o["topk_idx"], o["topk_score"])
            r.argus_sync()
            g["dev_option"] = o["option"].cpu().numpy()
            g["dev_idx"] = o["topk_idx"].cpu().numpy().view(np.uint32)
            outs.append((rc, g))
    (rc0, a), (rc1, b) = outs
    assert rc0 == rc1
    for key in ("option", "topk_idx", "topk_score", "quality", "status", "optimal", "topk_handle", "dev_option",
                "dev_idx"):
        np.testing.assert_array_equal(a[key], b[key], err_msg=key)


def test_nccl_path_quota_broadcast_checks_negative(argus_mod):
    """Under NCCL the tail reads rank 0's broadcast quotas from the device: a negative
    quota fails the call (ARGUS_E_INVALID, on every rank) without poisoning the router,
    and the next valid call matches the single-GPU router."""
    argus = argus_mod
    N, M = 150, 6000
    p = gen.small_problem("C2", N=N, M=M, seed=173)
    quota = oracle.quota_from_fractions(p.fractions, N)
    bad = quota.copy()
    bad[1] = -1
    outs = []
    for uid in (None, argus.argus_nccl_unique_id()):
        with argus.Router(768, p.k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=M, max_batch=N,
                          nccl_unique_id=uid) as r:
            r.argus_cache_insert(p.cache)
            with pytest.raises(argus.ArgusError):
                r.argus_route_batch(p.X, bad)
            outs.append(r.argus_route_batch(p.X, quota))
    (rc0, a), (rc1, b) = outs
    assert rc0 == rc1
    for key in a:
        np.testing.assert_array_equal(a[key], b[key], err_msg=key)


def test_nccl_path_async_and_pasm(argus_mod):
    """The asynchronous host call and the PASM policy (no quotas: nothing to broadcast)
    through the one-rank NCCL communicator match the single-GPU router bit for bit."""
    import torch
    argus = argus_mod
    N, M = 140, 7000
    p = gen.small_problem("C2", N=N, M=M, seed=175)
    L = len(p.opts)
    quota = oracle.quota_from_fractions(p.fractions, N)
    P = argus.argus_oda_pasm(np.ones(L), p.fractions)

    def pinned(shape, dt):
        return torch.empty(shape, dtype=dt).pin_memory().numpy()

    results = []
    for uid in (None, argus.argus_nccl_unique_id()):
        with argus.Router(768, p.k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=M, max_batch=N,
                          nccl_unique_id=uid) as r:
            r.argus_cache_insert(p.cache)
            outs = []
            for policy in (argus.POLICY_SD, argus.POLICY_PASM):
                if policy == argus.POLICY_PASM:
                    r.argus_set_policy(argus.POLICY_PASM, P, 77)
                tickets = []
                for b in range(3):
                    o = dict(option=pinned((N,), torch.int32), topk_idx=pinned((N, p.k), torch.int32).view(np.uint32),
                             topk_score=pinned((N, p.k), torch.float32), quality=pinned((N, L), torch.float32),
                             status=pinned((N,), torch.uint8))
                    Xb = torch.from_numpy(np.roll(p.X, b, axis=0).copy()).pin_memory().numpy()
                    q = quota if policy == argus.POLICY_SD else None
                    tickets.append((r.argus_route_batch_async(Xb, q, o), o))
                for t, o in tickets:
                    outs.append((r.argus_route_wait(t), o))
            results.append(outs)
    for (rc0, a), (rc1, b) in zip(*results):
        assert rc0 == rc1
        for key in a:
            np.testing.assert_array_equal(a[key], b[key], err_msg=key)


@pytest.mark.parametrize("k", [4, 0])
def test_pipelined_nccl_path_matches_serial(argus_mod, k):
    """Pipelined NCCL mode (one comm stream: bcast(b), AG(b-1), bcast(b+1), ...; the
    all-gather and tail of batch b deferred until call b+1 has issued its broadcast):
    a bursty sequence of batches through the device API and the asynchronous host API is
    bit-identical to the serial single-GPU router, including the PASM counter and the
    Eq. 3 queues carried across batches.  k = 0 is the SM mode (no scan)."""
    import torch
    argus = argus_mod
    M = 9000
    p = gen.small_problem("C2", N=300, M=M, seed=177)
    if k == 0:
        p = gen.small_problem("C2", N=300, M=M, k=0, seed=177)
        for o in p.opts:
            o["k_skip"] = 0
    L = len(p.opts)
    sizes = [48, 300, 17, 129, 256, 64]
    workers = np.arange(2 * L) % L
    tproc = np.linspace(1.0, 3.0, 2 * L).astype(np.float32)
    runs = []
    for uid, pipe in ((None, False), (argus.argus_nccl_unique_id(), True)):
        with argus.Router(768, k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=M, max_batch=300,
                          nccl_unique_id=uid, pipeline=pipe) as r:
            if k:
                r.argus_cache_insert(p.cache)
            r.argus_set_workers(workers, tproc, np.zeros(2 * L, np.int32))
            res = []
            outs = []
            for b, n in enumerate(sizes):
                X = torch.from_numpy(np.roll(p.X, 7 * b, axis=0)[:n].copy()).cuda()
                quota = oracle.quota_from_fractions(p.fractions, n)
                o = dict(option=torch.empty(n, dtype=torch.int32, device="cuda"),
                         topk_idx=torch.empty((n, max(k, 1)), dtype=torch.int32, device="cuda"),
                         topk_score=torch.empty((n, max(k, 1)), dtype=torch.float32, device="cuda"),
                         quality=torch.empty((n, L), dtype=torch.float32, device="cuda"),
                         status=torch.empty(n, dtype=torch.uint8, device="cuda"),
                         optimal=torch.empty(n, dtype=torch.int32, device="cuda"),
                         worker=torch.empty(n, dtype=torch.int32, device="cuda"))
                r.argus_route_batch_ex_dev(X, quota, o["option"], o["topk_idx"] if k else None,
                                           o["topk_score"] if k else None, o["quality"], o["status"],
                                           optimal=o["optimal"], worker=o["worker"])
                outs.append(o)
                if b == 2:
                    r.argus_set_policy(argus.POLICY_PASM, argus.argus_oda_pasm(np.ones(L), p.fractions), 5)
            r.argus_sync()
            for o in outs:
                res.append({kk: v.cpu().numpy() for kk, v in o.items()})
            res.append({"queues": r.argus_get_queues()})
            runs.append(res)
    for a, b in zip(*runs):
        for kk in a:
            if k == 0 and kk in ("topk_idx", "topk_score"):
                continue
            np.testing.assert_array_equal(a[kk], b[kk], err_msg=kk)


def test_pipelined_nccl_async_host_calls(argus_mod):
    """The asynchronous host call in pipelined NCCL mode (the result copy of call b is
    issued with its deferred tail) returns what the serial single-GPU router returns."""
    import torch
    argus = argus_mod
    N, M = 200, 8000
    p = gen.small_problem("C2", N=N, M=M, seed=179)
    L = len(p.opts)
    quota = oracle.quota_from_fractions(p.fractions, N)

    def pinned(shape, dt):
        return torch.empty(shape, dtype=dt).pin_memory().numpy()

    results = []
    for uid, pipe in ((None, False), (argus.argus_nccl_unique_id(), True)):
        with argus.Router(768, p.k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=M, max_batch=N,
                          nccl_unique_id=uid, pipeline=pipe) as r:
            r.argus_cache_insert(p.cache)
            tickets = []
            for b in range(6):
                o = dict(option=pinned((N,), torch.int32), topk_idx=pinned((N, p.k), torch.int32).view(np.uint32),
                         topk_score=pinned((N, p.k), torch.float32), quality=pinned((N, L), torch.float32),
                         status=pinned((N,), torch.uint8))
                Xb = torch.from_numpy(np.roll(p.X, 3 * b, axis=0).copy()).pin_memory().numpy()
                tickets.append((r.argus_route_batch_async(Xb, quota, o), o))
                if b == 3:   # collect the oldest ticket while later ones are in flight
                    tickets[0] = (r.argus_route_wait(tickets[0][0]), tickets[0][1], True)
            outs = []
            for t in tickets:
                rc = t[0] if len(t) == 3 else r.argus_route_wait(t[0])
                outs.append((rc, t[1]))
            results.append(outs)
    for (rc0, a), (rc1, b) in zip(*results):
        assert rc0 == rc1
        for key in a:
            np.testing.assert_array_equal(a[key], b[key], err_msg=key)
