"""Two processes, one GPU: the multi-GPU protocol with real libargus instances.

Each process loads libargus.so and builds a router with world = 2 in external
collective mode (no NCCL: one GPU cannot host two NCCL ranks); gloo carries the
N*k candidate keys between the processes, exactly where the library's all-gather
sits (P:381's one-process-per-GPU deployment).  Both processes'
outputs must be bit-identical to each other and to a single-GPU router, and the
top-k / assignment must pass the oracle checks.  A NaN prompt must fail the call
on both ranks.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from synth import argus_inputs as gen
        from paper_2511_06724_b200 import argus
        torch.cuda.set_device(0)
        res = {}
        for N, M, seed in ((70, 6001, 251), (256, 9001, 252)):
            p = gen.small_problem("C1", N=N, M=M, seed=seed)
            k, L = p.k, len(p.opts)
            quota = oracle.quota_from_fractions(p.fractions, N)
            with argus.Router(p.X.shape[1], k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=M + 64, max_batch=N,
                              rank=rank, world=world) as r:
                r.argus_cache_insert(p.cache)       # every rank keeps its stripe
                X = torch.from_numpy(p.X).cuda()
                keys = torch.zeros((N, k), dtype=torch.int64, device="cuda")
                r.argus_route_partial_dev(X, keys)
                r.argus_sync()
                parts = [torch.zeros((N, k), dtype=torch.int64) for _ in range(world)]
                dist.all_gather(parts, keys.cpu())       # the exchange step, over gloo
                keys_all = torch.stack(parts).cuda()
                o = dict(option=torch.empty(N, dtype=torch.int32, device="cuda"),
                         topk_idx=torch.empty((N, k), dtype=torch.int32, device="cuda"),
                         topk_score=torch.empty((N, k), dtype=torch.float32, device="cuda"),
                         quality=torch.empty((N, L), dtype=torch.float32, device="cuda"),
                         status=torch.empty(N, dtype=torch.uint8, device="cuda"))
                r.argus_route_finish_dev(keys_all, world, N, quota, o["option"], o["topk_idx"], o["topk_score"],
                                         o["quality"], o["status"])
                rc = r.argus_sync()
                res[N] = dict(rc=rc, **{kk: v.cpu().numpy() for kk, v in o.items()})
                # a NaN prompt: the call fails on this rank too
                bad = X.clone()
                bad[3, 7] = float("nan")
                def code(f):
                    try:
                        return f()
                    except argus.ArgusError as e:
                        return e.code
                r.argus_route_partial_dev(bad, keys)
                rcb = code(r.argus_sync)
                r.argus_route_finish_dev(keys_all, world, N, quota, o["option"], o["topk_idx"], o["topk_score"],
                                         o["quality"], o["status"])
                res[N]["rc_nan"] = min(rcb, code(r.argus_sync))
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_processes_one_gpu_external_mode(tmp_path):
    import torch.multiprocessing as mp
    import oracle
    from synth import argus_inputs as gen
    from tests import parity
    from paper_2511_06724_b200 import argus
    world = 2
    mp.start_processes(_rank_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    res = [np.load(os.path.join(tmp_path, f"rank{r}.npy"), allow_pickle=True).item() for r in range(world)]
    for N, M, seed in ((70, 6001, 251), (256, 9001, 252)):
        a, b = res[0][N], res[1][N]
        for kk in ("option", "topk_idx", "topk_score", "quality", "status", "rc"):
            np.testing.assert_array_equal(a[kk], b[kk])
        assert a["rc_nan"] == b["rc_nan"] == argus.ARGUS_E_INVALID
        p = gen.small_problem("C1", N=N, M=M, seed=seed)
        quota = oracle.quota_from_fractions(p.fractions, N)
        with argus.Router(p.X.shape[1], p.k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=M + 64, max_batch=N) as r:
            r.argus_cache_insert(p.cache)
            rc1, g1 = r.argus_route_batch(p.X, quota)
        g = {kk: a[kk] for kk in ("option", "topk_score", "quality", "status")}
        g["topk_idx"] = a["topk_idx"].view(np.uint32)
        for kk in g:
            np.testing.assert_array_equal(g[kk], g1[kk], err_msg=kk)   # G = 2 == G = 1
        assert a["rc"] == rc1
        parity.check_topk(p.X, p.cache, p.k, g["topk_idx"], g["topk_score"])
        parity.check_replay(g, p.opts, quota)


def _rank_main_p2p(rank, world, port, out_dir):
    """External mode with the fused exchange: each process maps the other's inbox (CUDA
    IPC handles swapped over gloo) and routes with argus_route_batch: the merge kernels
    store their keys into both inboxes and the tails wait on the arrival flags."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from synth import argus_inputs as gen
        from paper_2511_06724_b200 import argus
        torch.cuda.set_device(0)
        N, M = 256, 9001
        p = gen.small_problem("C1", N=N, M=M, seed=261)
        res = []
        with argus.Router(p.X.shape[1], p.k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=M + 64, max_batch=N,
                          rank=rank, world=world) as r:
            r.argus_cache_insert(p.cache)
            h = r.argus_p2p_export()
            hs = [None] * world
            dist.all_gather_object(hs, h)
            r.argus_p2p_connect(hs)
            dist.barrier()
            for b, n in enumerate((256, 77, 130, 48, 256)):   # five batches: both inbox parities, reused
                X = np.roll(p.X, 5 * b, axis=0)[:n].copy()
                quota = oracle.quota_from_fractions(p.fractions, n)
                rc, g = r.argus_route_batch(X, quota)
                res.append(dict(rc=rc, **g))
        np.save(os.path.join(out_dir, f"p2p_rank{rank}.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_processes_fused_peer_exchange(tmp_path):
    import torch.multiprocessing as mp
    import oracle
    from synth import argus_inputs as gen
    from tests import parity
    from paper_2511_06724_b200 import argus
    world = 2
    mp.start_processes(_rank_main_p2p, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    res = [np.load(os.path.join(tmp_path, f"p2p_rank{r}.npy"), allow_pickle=True) for r in range(world)]
    N, M = 256, 9001
    p = gen.small_problem("C1", N=N, M=M, seed=261)
    with argus.Router(p.X.shape[1], p.k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=M + 64, max_batch=N) as r:
        r.argus_cache_insert(p.cache)
        for b, n in enumerate((256, 77, 130, 48, 256)):
            X = np.roll(p.X, 5 * b, axis=0)[:n].copy()
            quota = oracle.quota_from_fractions(p.fractions, n)
            rc1, g1 = r.argus_route_batch(X, quota)
            a, c = res[0][b], res[1][b]
            for kk in ("option", "topk_idx", "topk_score", "quality", "status", "rc"):
                np.testing.assert_array_equal(a[kk], c[kk], err_msg=f"batch {b} {kk}")
            assert a["rc"] == rc1
            for kk in g1:
                np.testing.assert_array_equal(a[kk], g1[kk], err_msg=f"batch {b} {kk} vs one GPU")
            parity.check_topk(X, p.cache, p.k, a["topk_idx"], a["topk_score"], rows=range(0, n, 5))
