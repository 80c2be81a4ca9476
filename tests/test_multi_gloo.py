"""world_size=2 gloo tests (CPU) of the multi-GPU host protocol.

The GPU data path cannot run here; what is checked is the decomposition the
library relies on: striping the cache by g mod G, taking a top-k
per shard with global ids, exchanging the N*k candidates and merging by
(score desc, id asc) yields exactly the global top-k (the oracle computes each
shard's candidates); plus unique-id distribution and max-over-ranks timing from
paper_2511_06724_b200/dist.py, which bench.py uses under torchrun.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_06724_b200 import dist as adist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from synth import argus_inputs as gen
        from paper_2511_06724_b200 import argus
        p = gen.small_problem("C1", N=24, M=1037, seed=7)
        M, k = p.cache.shape[0], p.k
        # shard by stripe; candidates with global ids from this shard only
        ids = np.array([g for g in range(M) if adist.stripe_owner(g, world) == rank], np.uint32)
        assert ids.size == adist.local_rows(M, world, rank)
        assert all(adist.stripe_slot(int(g), world) == j for j, g in enumerate(ids))
        sc, ix = oracle.scan_topk(p.X, p.cache[ids], k, ids=ids)
        gathered = [None] * world
        dist.all_gather_object(gathered, (sc, ix))
        # merge: top-k of the union by (score desc, id asc)
        allsc = np.concatenate([g[0] for g in gathered], axis=1)
        allix = np.concatenate([g[1] for g in gathered], axis=1)
        merged = np.empty((p.X.shape[0], k), np.uint32)
        for i in range(p.X.shape[0]):
            o = np.lexsort((allix[i].astype(np.int64), -allsc[i]))[:k]
            merged[i] = allix[i][o]
        ref_sc, ref_ix = oracle.scan_topk(p.X, p.cache, k)
        ok_topk = bool(np.array_equal(merged, ref_ix))
        # ring-evicting cache (capacity 600 < M, wrapped): each rank holds the live ids
        # whose position g mod 600 is in its stripe; merging the shards' candidates by
        # (score desc, id asc) is the top-k over exactly the live set
        cap = 600
        live = np.array(list(adist.live_ids(M, cap, True)), np.uint32)
        mine = np.array([g for g in live if adist.stripe_owner(int(g), world, cap, True) == rank], np.uint32)
        slots = sorted(adist.stripe_slot(int(g), world, cap, True) for g in mine)
        assert slots == list(range(len(mine)))              # dense local slots 0..cap/G-1
        sc, ix = oracle.scan_topk(p.X, p.cache[mine], k, ids=mine)
        gathered = [None] * world
        dist.all_gather_object(gathered, (sc, ix))
        allsc = np.concatenate([g[0] for g in gathered], axis=1)
        allix = np.concatenate([g[1] for g in gathered], axis=1)
        ref_sc, ref_ix = oracle.scan_topk(p.X, p.cache[live], k, ids=live)
        for i in range(p.X.shape[0]):
            o = np.lexsort((allix[i].astype(np.int64), -allsc[i]))[:k]
            ok_topk = ok_topk and bool(np.array_equal(allix[i][o], ref_ix[i]))
        uid = adist.share_nccl_id(dist, rank, argus.argus_nccl_unique_id)
        uids = [None] * world
        dist.all_gather_object(uids, uid)
        mx = adist.max_over_ranks(dist, 10.0 + rank)
        q.put((rank, ok_topk, len(uid), uids[0] == uids[1], mx))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(240)
def test_world2_gloo_protocol():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=200) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, ok_topk, ulen, same_uid, mx in res:
        assert ok_topk, rank
        assert ulen == 128 and same_uid
        assert mx == 11.0


def test_stripe_layout_covers_cache():
    for M in (0, 1, 7, 1000, 1001):
        for G in (1, 2, 3, 8):
            assert sum(adist.local_rows(M, G, r) for r in range(G)) == M
            seen = {(adist.stripe_owner(g, G), adist.stripe_slot(g, G)) for g in range(M)}
            assert len(seen) == M
            for r in range(G):
                assert max([s for (o, s) in seen if o == r], default=-1) == adist.local_rows(M, G, r) - 1
