"""Thin ctypes binding of libargus.so (include/argus.h), same names as the C ABI.

Argument marshalling only: every step of the routing path runs in the CUDA
kernels of libargus.so.  PyTorch is used by callers for device memory, streams
and process groups; this module accepts numpy arrays (host calls) or torch CUDA
tensors (``*_dev`` calls) and passes raw pointers.  If the shared library is
missing the import fails loudly -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libargus.so")

ARGUS_OK = 0
ARGUS_W_OVERFLOW = 1
ARGUS_E_INVALID = -1
ARGUS_E_CAPACITY = -2
ARGUS_E_CUDA = -3
ARGUS_E_NCCL = -4
ARGUS_E_STATE = -5
ARGUS_E_UNIMPLEMENTED = -6
ST_OVERFLOW, ST_NONCOMPLIANT, ST_GATED_ALL = 1, 2, 4

# every symbol include/argus.h declares
SYMBOLS = (
    "argus_nccl_unique_id", "argus_route_init", "argus_cache_insert", "argus_cache_insert_dev",
    "argus_route_batch", "argus_route_batch_dev", "argus_route_partial_dev", "argus_route_finish_dev",
    "argus_route_join", "argus_sync", "argus_quota_from_fractions", "argus_cache_size", "argus_launch_count",
    "argus_get_stream", "argus_profile_enable", "argus_profile_read", "argus_route_destroy",
    "argus_strerror", "argus_solve_allocation", "argus_oda_pasm", "argus_pasm_degradation", "argus_set_policy",
    "argus_affinity_histogram", "argus_set_workers", "argus_get_queues", "argus_route_batch_ex",
    "argus_route_batch_ex_dev", "argus_cache_insert_h", "argus_route_batch_async", "argus_route_wait",
    "argus_debug_capture", "argus_p2p_export", "argus_p2p_connect", "argus_route_batch_bf16_dev",
)
STAGES = ("prep", "scan", "merge_local", "unused3", "tail", "unused5", "insert")


class argus_option(C.Structure):
    _fields_ = [("model_id", C.c_int32), ("k_skip", C.c_int32),
                ("p_th_qpm", C.c_float), ("sim_gate", C.c_float)]


class argus_config(C.Structure):
    _fields_ = [("d", C.c_int32), ("k", C.c_int32), ("L", C.c_int32), ("hidden", C.c_int32),
                ("max_batch", C.c_int32), ("capacity", C.c_int64), ("delta", C.c_float),
                ("rank", C.c_int32), ("world", C.c_int32), ("device", C.c_int32),
                ("nccl_unique_id", C.c_void_p), ("stream", C.c_void_p), ("pipeline", C.c_int32),
                ("evict", C.c_int32)]


class argus_route_extra(C.Structure):
    _fields_ = [("optimal", C.c_void_p), ("worker", C.c_void_p), ("topk_handle", C.c_void_p)]


class ArgusError(RuntimeError):
    def __init__(self, code, what=""):
        self.code = code
        super().__init__(f"{what}: argus error {code}: {strerror(code)}")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2511_06724_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "argus_nccl_unique_id": [P],
        "argus_route_init": [P, P, P, P, P, P, P],
        "argus_cache_insert": [P, P, I64, P],
        "argus_cache_insert_dev": [P, P, I64, P],
        "argus_route_batch": [P, P, I32, P, P, P, P, P, P],
        "argus_route_batch_dev": [P, P, I32, P, P, P, P, P, P],
        "argus_route_partial_dev": [P, P, I32, P],
        "argus_route_finish_dev": [P, P, I32, I32, P, P, P, P, P, P],
        "argus_route_join": [P, P],
        "argus_sync": [P],
        "argus_quota_from_fractions": [P, I32, I32, P],
        "argus_cache_size": [P, P],
        "argus_launch_count": [P, P],
        "argus_get_stream": [P, P],
        "argus_profile_enable": [P, C.c_int],
        "argus_profile_read": [P, C.c_int, P, P],
        "argus_route_destroy": [P],
        "argus_strerror": [C.c_int],
        "argus_solve_allocation": [I32, I32, I32, P, P, P, P, P, P, P],
        "argus_oda_pasm": [P, P, I32, P],
        "argus_pasm_degradation": [P, P, P, P, I32, P],
        "argus_set_policy": [P, I32, P, C.c_uint64],
        "argus_affinity_histogram": [P, P, P],
        "argus_set_workers": [P, I32, P, P, P],
        "argus_get_queues": [P, P],
        "argus_route_batch_ex": [P, P, I32, P, P, P, P, P, P, P],
        "argus_route_batch_ex_dev": [P, P, I32, P, P, P, P, P, P, P],
        "argus_cache_insert_h": [P, P, P, I64, P],
        "argus_route_batch_async": [P, P, I32, P, P, P, P, P, P, P],
        "argus_route_wait": [P, I64],
        "argus_debug_capture": [P, P, I64],
        "argus_p2p_export": [P, P],
        "argus_route_batch_bf16_dev": [P, P, I32, P, P, P, P, P, P, P],
        "argus_p2p_connect": [P, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    lib.argus_strerror.restype = C.c_char_p
    return lib


_lib = _load()


def strerror(code: int) -> str:
    return _lib.argus_strerror(int(code)).decode()


def _p(a):
    """Raw pointer of a numpy array or a torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    return C.c_void_p(a.data_ptr())  # torch tensor


def _check(rc, what):
    if rc < 0:
        raise ArgusError(rc, what)
    return rc


# ------------------------------------------------------------------ raw ABI (same names)
def argus_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.argus_nccl_unique_id(buf), "argus_nccl_unique_id")
    return buf.raw


def argus_quota_from_fractions(f, N: int) -> np.ndarray:
    f = np.ascontiguousarray(f, np.float64)
    c = np.empty(f.size, np.int32)
    _check(_lib.argus_quota_from_fractions(_p(f), f.size, int(N), _p(c)), "argus_quota_from_fractions")
    return c


def argus_strerror(code: int) -> str:
    return strerror(code)


POLICY_SD, POLICY_PASM = 0, 1
AFFINITY_WINDOW = 1000


def argus_solve_allocation(W: int, n_workers: int, Q, p_th):
    """Eq. 1 allocator (host).  Returns dict(levels, loads, F, objective, feasible)."""
    Q = np.ascontiguousarray(Q, np.float64)
    p_th = np.ascontiguousarray(p_th, np.float32)
    L = Q.size
    lv = np.empty(n_workers, np.int32)
    ld = np.empty(n_workers, np.int32)
    F = np.empty(L, np.float64)
    obj, feas = C.c_double(), C.c_int32()
    _check(_lib.argus_solve_allocation(int(W), int(n_workers), L, _p(Q), _p(p_th), _p(lv), _p(ld), _p(F),
                                       C.byref(obj), C.byref(feas)), "argus_solve_allocation")
    return dict(levels=lv, loads=ld, F=F, objective=obj.value, feasible=bool(feas.value))


def argus_oda_pasm(H, F) -> np.ndarray:
    """Algorithm 1 (host): PASM [L][L], row = optimal level, column = served level."""
    H = np.ascontiguousarray(H, np.float64)
    F = np.ascontiguousarray(F, np.float64)
    P = np.empty((H.size, H.size), np.float64)
    _check(_lib.argus_oda_pasm(_p(H), _p(F), H.size, _p(P)), "argus_oda_pasm")
    return P


def argus_pasm_degradation(pasm, H, p_th, D) -> float:
    pasm = np.ascontiguousarray(pasm, np.float64)
    H = np.ascontiguousarray(H, np.float64)
    p_th = np.ascontiguousarray(p_th, np.float32)
    D = np.ascontiguousarray(D, np.float64)
    dq = C.c_double()
    _check(_lib.argus_pasm_degradation(_p(pasm), _p(H), _p(p_th), _p(D), H.size, C.byref(dq)),
           "argus_pasm_degradation")
    return dq.value


class Router:
    """Owner of one ``argus_router*``.  Methods map 1:1 onto the C ABI."""

    def __init__(self, d, k, opts, W1, b1, W2, b2, capacity, max_batch, hidden=None,
                 delta=0.9, rank=0, world=1, device=0, nccl_unique_id=None, stream=None, pipeline=False,
                 evict=False):
        L = len(opts)
        self.d, self.k, self.L = int(d), int(k), L
        W1 = np.ascontiguousarray(W1, np.float32)
        H = W1.shape[0] if hidden is None else int(hidden)
        self.H = H
        self.max_batch = int(max_batch)
        oa = (argus_option * L)()
        for i, o in enumerate(opts):
            oa[i] = argus_option(int(o["model_id"]), int(o["k_skip"]), float(o["p_th_qpm"]),
                                 float(o["sim_gate"]))
        self._uid = None
        if nccl_unique_id is not None:
            self._uid = C.create_string_buffer(bytes(nccl_unique_id), 128)
        cfg = argus_config(self.d, self.k, L, H, self.max_batch, int(capacity), float(delta),
                           int(rank), int(world), int(device),
                           C.cast(self._uid, C.c_void_p) if self._uid is not None else None,
                           C.c_void_p(stream) if stream else None, int(bool(pipeline)), int(bool(evict)))
        self._keep = [np.ascontiguousarray(x, np.float32) for x in (W1, b1, W2, b2)]
        h = C.c_void_p()
        _check(_lib.argus_route_init(C.byref(cfg), oa, *[_p(x) for x in self._keep], C.byref(h)),
               "argus_route_init")
        self._h = h

    # lifecycle
    def close(self):
        if getattr(self, "_h", None):
            _lib.argus_route_destroy(self._h)
            self._h = None

    argus_route_destroy = close

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # cache
    def argus_cache_insert(self, emb, n=None) -> int:
        """emb host fp32 [n][d]; emb = None with n rows on a non-root rank of an NCCL
        router (rank 0's rows are broadcast by the library)."""
        if emb is None:
            first = C.c_int64(-1)
            _check(_lib.argus_cache_insert(self._h, None, int(n), C.byref(first)), "argus_cache_insert")
            return first.value
        emb = np.ascontiguousarray(emb, np.float32)
        first = C.c_int64(-1)
        _check(_lib.argus_cache_insert(self._h, _p(emb), emb.shape[0] if emb.size else 0, C.byref(first)),
               "argus_cache_insert")
        return first.value

    def argus_cache_insert_dev(self, emb_dev) -> int:
        first = C.c_int64(-1)
        _check(_lib.argus_cache_insert_dev(self._h, _p(emb_dev), int(emb_dev.shape[0]), C.byref(first)),
               "argus_cache_insert_dev")
        return first.value

    def argus_cache_size(self) -> int:
        m = C.c_int64()
        _check(_lib.argus_cache_size(self._h, C.byref(m)), "argus_cache_size")
        return m.value

    def argus_launch_count(self) -> int:
        n = C.c_int64()
        _check(_lib.argus_launch_count(self._h, C.byref(n)), "argus_launch_count")
        return n.value

    def argus_get_stream(self) -> int:
        s = C.c_void_p()
        _check(_lib.argus_get_stream(self._h, C.byref(s)), "argus_get_stream")
        return s.value or 0

    # routing
    def argus_route_batch(self, prompts, quota, want_quality=True, want_status=True, N=None):
        """Host-buffer route.  Returns (rc, dict of numpy outputs).  Non-root ranks of an
        NCCL router may pass prompts = None (and quota = None) with N."""
        prompts = None if prompts is None else np.ascontiguousarray(prompts, np.float32)
        quota = None if quota is None else np.ascontiguousarray(quota, np.int32)
        N = prompts.shape[0] if prompts is not None else int(N)
        out = dict(option=np.empty(N, np.int32), topk_idx=np.empty((N, self.k), np.uint32),
                   topk_score=np.empty((N, self.k), np.float32),
                   quality=np.empty((N, self.L), np.float32) if want_quality else None,
                   status=np.empty(N, np.uint8) if want_status else None)
        rc = _check(_lib.argus_route_batch(self._h, _p(prompts), N, _p(quota), _p(out["option"]),
                                           _p(out["topk_idx"]), _p(out["topk_score"]), _p(out["quality"]),
                                           _p(out["status"])), "argus_route_batch")
        return rc, out

    def argus_route_batch_dev(self, prompts_dev, quota, option, topk_idx, topk_score, quality=None,
                              status=None, N=None):
        quota = None if quota is None else np.ascontiguousarray(quota, np.int32)
        N = int(prompts_dev.shape[0]) if N is None else int(N)
        return _check(_lib.argus_route_batch_dev(self._h, _p(prompts_dev), N, _p(quota), _p(option),
                                                 _p(topk_idx), _p(topk_score), _p(quality), _p(status)),
                      "argus_route_batch_dev")

    def argus_route_batch_ex(self, prompts, quota, want_workers=False, want_handles=False):
        """Host-buffer route with the optimal options (and Eq. 3 workers, latent
        handles).  quota may be None under the PASM policy.  Returns (rc, outputs)."""
        prompts = np.ascontiguousarray(prompts, np.float32)
        quota = None if quota is None else np.ascontiguousarray(quota, np.int32)
        N = prompts.shape[0]
        out = dict(option=np.empty(N, np.int32), topk_idx=np.empty((N, self.k), np.uint32),
                   topk_score=np.empty((N, self.k), np.float32), quality=np.empty((N, self.L), np.float32),
                   status=np.empty(N, np.uint8), optimal=np.empty(N, np.int32),
                   worker=np.empty(N, np.int32) if want_workers else None,
                   topk_handle=np.empty((N, self.k), np.uint64) if want_handles else None)
        ex = argus_route_extra(_p(out["optimal"]), _p(out["worker"]), _p(out["topk_handle"]))
        rc = _check(_lib.argus_route_batch_ex(self._h, _p(prompts), N, _p(quota), _p(out["option"]),
                                              _p(out["topk_idx"]), _p(out["topk_score"]), _p(out["quality"]),
                                              _p(out["status"]), C.byref(ex)), "argus_route_batch_ex")
        return rc, out

    def argus_route_batch_ex_dev(self, prompts_dev, quota, option, topk_idx, topk_score, quality=None,
                                 status=None, optimal=None, worker=None, topk_handle=None, N=None):
        quota = None if quota is None else np.ascontiguousarray(quota, np.int32)
        N = int(prompts_dev.shape[0]) if N is None else int(N)
        ex = argus_route_extra(_p(optimal), _p(worker), _p(topk_handle))
        return _check(_lib.argus_route_batch_ex_dev(self._h, _p(prompts_dev), N, _p(quota), _p(option),
                                                    _p(topk_idx), _p(topk_score), _p(quality), _p(status),
                                                    C.byref(ex)), "argus_route_batch_ex_dev")

    def argus_route_batch_bf16_dev(self, prompts_bf16_dev, quota, option, topk_idx, topk_score, quality=None,
                                   status=None, optimal=None, worker=None, topk_handle=None, N=None):
        """Device route with bf16 prompts [N][d] (a torch.bfloat16 CUDA tensor)."""
        quota = None if quota is None else np.ascontiguousarray(quota, np.int32)
        N = int(prompts_bf16_dev.shape[0]) if N is None else int(N)
        ex = argus_route_extra(_p(optimal), _p(worker), _p(topk_handle))
        return _check(_lib.argus_route_batch_bf16_dev(self._h, _p(prompts_bf16_dev), N, _p(quota), _p(option),
                                                      _p(topk_idx), _p(topk_score), _p(quality), _p(status),
                                                      C.byref(ex)), "argus_route_batch_bf16_dev")

    def argus_route_batch_async(self, prompts, quota, out, N=None):
        """Enqueue one batch from (pinned) host memory; outputs land in the arrays of
        `out` (option, topk_idx, topk_score, optional quality / status), which must
        stay alive until argus_route_wait(ticket).  Returns the ticket.  Non-root
        ranks of an NCCL router may pass prompts = None (and quota = None) with N."""
        N = int(prompts.shape[0]) if prompts is not None else int(N)
        quota = None if quota is None else np.ascontiguousarray(quota, np.int32)
        t = C.c_int64(-1)
        _check(_lib.argus_route_batch_async(self._h, _p(prompts), N, _p(quota), _p(out["option"]),
                                            _p(out["topk_idx"]), _p(out["topk_score"]), _p(out.get("quality")),
                                            _p(out.get("status")), C.byref(t)), "argus_route_batch_async")
        self._async_keep = getattr(self, "_async_keep", {})
        self._async_keep[t.value] = (prompts, quota, out)   # keep the buffers alive
        return t.value

    def argus_route_wait(self, ticket) -> int:
        rc = _check(_lib.argus_route_wait(self._h, C.c_int64(int(ticket))), "argus_route_wait")
        keep = getattr(self, "_async_keep", {})
        for t in [x for x in keep if x <= ticket]:
            del keep[t]
        return rc

    def argus_cache_insert_h(self, emb, handles=None) -> int:
        emb = np.ascontiguousarray(emb, np.float32).reshape(-1, self.d)
        h = None if handles is None else np.ascontiguousarray(handles, np.uint64)
        first = C.c_int64(-1)
        _check(_lib.argus_cache_insert_h(self._h, _p(emb), _p(h), emb.shape[0], C.byref(first)),
               "argus_cache_insert_h")
        return first.value

    def argus_set_policy(self, policy, pasm=None, seed=0):
        pasm = None if pasm is None else np.ascontiguousarray(pasm, np.float64)
        _check(_lib.argus_set_policy(self._h, int(policy), _p(pasm), C.c_uint64(int(seed))), "argus_set_policy")

    def argus_affinity_histogram(self):
        """(counts [L] int64, prompts counted)."""
        h = np.empty(self.L, np.int64)
        n = C.c_int64()
        _check(_lib.argus_affinity_histogram(self._h, _p(h), C.byref(n)), "argus_affinity_histogram")
        return h, n.value

    def argus_set_workers(self, option_of_worker, t_proc, queue):
        ow = np.ascontiguousarray(option_of_worker, np.int32)
        t = np.ascontiguousarray(t_proc, np.float32)
        q = np.ascontiguousarray(queue, np.int32)
        self._n_workers = int(ow.size)
        _check(_lib.argus_set_workers(self._h, ow.size, _p(ow), _p(t), _p(q)), "argus_set_workers")

    def argus_get_queues(self) -> np.ndarray:
        q = np.empty(getattr(self, "_n_workers", 0), np.int32)
        _check(_lib.argus_get_queues(self._h, _p(q)), "argus_get_queues")
        return q

    def argus_route_partial_dev(self, prompts_dev, keys_dev, N=None):
        N = int(prompts_dev.shape[0]) if N is None else int(N)
        return _check(_lib.argus_route_partial_dev(self._h, _p(prompts_dev), N, _p(keys_dev)),
                      "argus_route_partial_dev")

    def argus_route_finish_dev(self, keys_all_dev, G, N, quota, option, topk_idx, topk_score,
                               quality=None, status=None):
        quota = np.ascontiguousarray(quota, np.int32)
        return _check(_lib.argus_route_finish_dev(self._h, _p(keys_all_dev), int(G), int(N), _p(quota),
                                                  _p(option), _p(topk_idx), _p(topk_score), _p(quality),
                                                  _p(status)), "argus_route_finish_dev")

    def argus_debug_capture(self, scores_dev=None, ld=None):
        """Parity test T2: later scans also write every exact score they compare into
        scores_dev (device fp32 [N][ld], ld >= this shard's live rows); None switches off."""
        if scores_dev is None:
            _check(_lib.argus_debug_capture(self._h, None, 0), "argus_debug_capture")
            self._dbg_keep = None
            return
        ld = int(scores_dev.shape[-1]) if ld is None else int(ld)
        self._dbg_keep = scores_dev
        _check(_lib.argus_debug_capture(self._h, _p(scores_dev), ld), "argus_debug_capture")

    def argus_p2p_export(self) -> bytes:
        """External mode: this rank's 64-byte inbox handle (to be exchanged by the caller)."""
        buf = C.create_string_buffer(64)
        _check(_lib.argus_p2p_export(self._h, buf), "argus_p2p_export")
        return buf.raw

    def argus_p2p_connect(self, handles):
        """External mode: map every rank's inbox (handles: list of 64-byte handles in rank order)."""
        blob = C.create_string_buffer(b"".join(bytes(h) for h in handles), 64 * len(handles))
        _check(_lib.argus_p2p_connect(self._h, blob), "argus_p2p_connect")

    def argus_profile_enable(self, on=True):
        _check(_lib.argus_profile_enable(self._h, int(bool(on))), "argus_profile_enable")

    def argus_profile_read(self):
        """{stage: (total_ms, launches)} since the last read (resets)."""
        out = {}
        for i, name in enumerate(STAGES):
            ms, n = C.c_double(), C.c_int64()
            _check(_lib.argus_profile_read(self._h, i, C.byref(ms), C.byref(n)), "argus_profile_read")
            out[name] = (ms.value, n.value)
        return out

    def argus_route_join(self, stream=None):
        """Make ``stream`` (raw cudaStream_t int; None = the router's) wait for all enqueued work."""
        _check(_lib.argus_route_join(self._h, C.c_void_p(stream) if stream else None), "argus_route_join")

    def argus_sync(self) -> int:
        return _check(_lib.argus_sync(self._h), "argus_sync")
