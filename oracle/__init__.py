"""ARGUS routing oracle -- TEST INFRASTRUCTURE ONLY.

A ctypes wrapper around ``argus_oracle.c``: the plain fp64 CPU implementation
of SURVEY.md §8(c) steps O1..O11.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2511_06724_b200`` never imports it and
shares no code with it.

Parity pins: tests/test_oracle_pins.py.  Functions without a pin are marked
"parity unpinned" in their docstring (none at present; the *meaning* of the
predictor weights is unpinned).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "argus_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

OVERFLOW, NONCOMPLIANT, GATED_ALL = 1, 2, 4
DELTA = 0.9  # P:140 "We use delta = 0.9"


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no fast-math, OpenMP over prompts)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Opt(C.Structure):
    _fields_ = [("model_id", C.c_int32), ("k_skip", C.c_int32),
                ("p_th_qpm", C.c_float), ("sim_gate", C.c_float)]


def _load():
    global _lib
    if _lib is None:
        lib = C.CDLL(build())
        P = C.c_void_p
        lib.orc_bf16.restype = C.c_double
        lib.orc_bf16.argtypes = [C.c_float]
        lib.orc_bf16_array.argtypes = [P, P, C.c_int64]
        lib.orc_cosine.restype = C.c_double
        lib.orc_cosine.argtypes = [P, P, C.c_int32]
        lib.orc_scan_topk.restype = C.c_int
        lib.orc_scan_topk.argtypes = [P, C.c_int32, P, C.c_int64, C.c_int32, C.c_int32, P, C.c_int, P, P]
        lib.orc_score_matrix.restype = C.c_int
        lib.orc_score_matrix.argtypes = [P, C.c_int32, P, C.c_int64, C.c_int32, C.c_int, P]
        lib.orc_topk_of_scores.restype = C.c_int
        lib.orc_topk_of_scores.argtypes = [P, C.c_int32, C.c_int64, C.c_int64, C.c_int32, P, P, P]
        lib.orc_mlp.restype = C.c_int
        lib.orc_mlp.argtypes = [P, P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                P, P, P, P, C.c_int, P]
        lib.orc_assign.restype = C.c_int
        lib.orc_assign.argtypes = [P, P, C.c_int32, C.c_int32, P, P, C.c_float, P, P, P, P, P, P]
        lib.orc_quota_from_fractions.restype = C.c_int
        lib.orc_quota_from_fractions.argtypes = [P, C.c_int32, C.c_int32, P]
        lib.orc_max_threads.restype = C.c_int
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def max_threads() -> int:
    return int(_load().orc_max_threads())


def bf16(a) -> np.ndarray:
    """O1: fp32 -> bf16 (RNE), returned as float64 values."""
    a = _f32(a)
    out = np.empty(a.shape, np.float64)
    _load().orc_bf16_array(_p(a), _p(out), a.size)
    return out


def cosine(x, c) -> float:
    """O2/O3 for one pair."""
    x, c = _f32(x), _f32(c)
    return float(_load().orc_cosine(_p(x), _p(c), x.size))


def scan_topk(X, Cache, k: int, ids=None, threads: int = 0):
    """O1..O4: (topk_score f64 [N,k], topk_idx u32 [N,k]) over all cache rows."""
    X, Cache = _f32(X), _f32(Cache)
    N, d = X.shape
    M = Cache.shape[0]
    sc = np.empty((N, k), np.float64)
    ix = np.empty((N, k), np.uint32)
    idp = None
    if ids is not None:
        ids = np.ascontiguousarray(ids, np.uint32)
        idp = _p(ids)
    rc = _load().orc_scan_topk(_p(X), N, _p(Cache) if M else None, M, d, k, idp, threads, _p(sc), _p(ix))
    if rc != 0:
        raise ValueError("oracle scan: invalid input (zero norm or non-finite)")
    return sc, ix


def score_matrix(X, Cache, threads: int = 0) -> np.ndarray:
    """O1..O3 for every pair: cos(x_i, c_j) f64 [N, M] (NaN for a zero-norm row)."""
    X, Cache = _f32(X), _f32(Cache)
    N, d = X.shape
    M = Cache.shape[0]
    S = np.empty((N, M), np.float64)
    if N and M:
        _load().orc_score_matrix(_p(X), N, _p(Cache), M, d, threads, _p(S))
    return S


def topk_of_scores(S, k: int, ids=None):
    """O4 alone on a given score matrix S [N, M] (widened to fp64): the k best
    (s desc, g asc) per row.  Parity test T2 replays it on the GPU's fp32 scores."""
    S = np.ascontiguousarray(S, np.float64)
    N, M = S.shape
    sc = np.empty((N, k), np.float64)
    ix = np.empty((N, k), np.uint32)
    idp = None
    if ids is not None:
        ids = np.ascontiguousarray(ids, np.uint32)
        idp = _p(ids)
    rc = _load().orc_topk_of_scores(_p(S), N, M, M, k, idp, _p(sc), _p(ix))
    if rc != 0:
        raise ValueError("oracle topk: invalid shapes")
    return sc, ix


def mlp(X, S, W1, b1, W2, b2, threads: int = 0) -> np.ndarray:
    """O5: predicted relative quality rhat f64 [N, L] with rhat[:, 0] = 1."""
    X = _f32(X)
    S = np.ascontiguousarray(S, np.float64)
    W1, b1, W2, b2 = _f32(W1), _f32(b1), _f32(W2), _f32(b2)
    N, d = X.shape
    k = S.shape[1]
    H = W1.shape[0]
    L = W2.shape[0]
    assert W1.shape == (H, d + k) and W2.shape == (L, H)
    out = np.empty((N, L), np.float64)
    rc = _load().orc_mlp(_p(X), _p(S), N, d, k, H, L, _p(W1), _p(b1), _p(W2), _p(b2), threads, _p(out))
    if rc != 0:
        raise ValueError("oracle mlp: invalid shapes")
    return out


def _opts_array(opts):
    arr = (_Opt * len(opts))()
    for i, o in enumerate(opts):
        arr[i] = _Opt(int(o["model_id"]), int(o["k_skip"]), float(o["p_th_qpm"]), float(o["sim_gate"]))
    return arr


def assign(rhat, s1, opts, quota, delta: float = DELTA):
    """O6..O10.  Returns dict(option, status, adm, cmp, pref, order, rc)."""
    rhat = np.ascontiguousarray(rhat, np.float64)
    s1 = np.ascontiguousarray(s1, np.float64)
    quota = np.ascontiguousarray(quota, np.int32)
    N, L = rhat.shape
    oa = _opts_array(opts)
    out = dict(option=np.empty(N, np.int32), status=np.empty(N, np.uint8),
               adm=np.empty(N, np.uint32), cmp=np.empty(N, np.uint32),
               pref=np.empty((N, L), np.uint8), order=np.empty(N, np.int32))
    rc = _load().orc_assign(_p(rhat), _p(s1), N, L, C.cast(oa, C.c_void_p), _p(quota), C.c_float(delta),
                            _p(out["option"]), _p(out["status"]), _p(out["adm"]), _p(out["cmp"]),
                            _p(out["pref"]), _p(out["order"]))
    if rc < 0:
        raise ValueError("oracle assign: invalid input")
    out["rc"] = rc
    return out


def quota_from_fractions(f, N: int) -> np.ndarray:
    f = np.ascontiguousarray(f, np.float64)
    c = np.empty(f.size, np.int32)
    rc = _load().orc_quota_from_fractions(_p(f), f.size, int(N), _p(c))
    if rc != 0:
        raise ValueError("oracle quota: invalid fractions")
    return c


def route(X, Cache, k, W1, b1, W2, b2, opts, quota, delta=DELTA, threads=0):
    """End-to-end oracle: O1..O10 on the oracle's own fp64 values."""
    sc, ix = scan_topk(X, Cache, k, threads=threads)
    rhat = mlp(X, sc, W1, b1, W2, b2, threads=threads)
    a = assign(rhat, sc[:, 0], opts, quota, delta)
    a.update(topk_score=sc, topk_idx=ix, rhat=rhat)
    return a
