"""Host cost of one routing call (enqueue only): time of 32 back-to-back
argus_route_batch_dev calls before any synchronisation, C2-shaped batches on a small
cache (the GPU work per call is short, so the queue never fills).  Diagnostics."""
import time

import numpy as np
import torch

from paper_2511_06724_b200 import argus
from synth import argus_inputs as gen


def main():
    p = gen.small_problem("C2", N=512, M=20000, seed=5)
    L, k = len(p.opts), p.k
    for pipe, uid in ((True, None), (False, None), (True, argus.argus_nccl_unique_id())):
        with argus.Router(768, k, p.opts, p.W1, p.b1, p.W2, p.b2, capacity=20000, max_batch=512, pipeline=pipe,
                          nccl_unique_id=uid) as r:
            r.argus_cache_insert(p.cache)
            X = torch.from_numpy(p.X[:48].copy()).cuda()
            q = argus.argus_quota_from_fractions(p.fractions, 48)
            o = [torch.empty(48, dtype=torch.int32, device="cuda"), torch.empty((48, k), dtype=torch.int32, device="cuda"),
                 torch.empty((48, k), dtype=torch.float32, device="cuda")]
            for _ in range(8):
                r.argus_route_batch_dev(X, q, *o)
            r.argus_sync()
            best = 1e9
            for rep in range(5):
                t0 = time.perf_counter()
                for _ in range(32):
                    r.argus_route_batch_dev(X, q, *o)
                t1 = time.perf_counter()
                r.argus_sync()
                best = min(best, (t1 - t0) / 32 * 1e6)
            print(f"pipeline={pipe} nccl={uid is not None}: {best:.1f} us host time per argus_route_batch_dev call")


if __name__ == "__main__":
    main()
