"""Pins for the CPU oracle (oracle/argus_oracle.c) against things other than itself.

Each test checks the oracle against what the paper or mathematics fixes: hand
computed golden values (tests/golden/, each with its citation), closed forms,
brute force on tiny inputs, invariants, or special cases that reduce to a
library routine (torch's bf16 conversion, math.fsum).  A plausible slip in the
oracle -- a dropped term, a wrong sign or index, a transposed operand, a reversed
tie-break -- fails at least one of these.
"""
import itertools
import math
import struct

import numpy as np
import pytest

import oracle
from synth import argus_inputs as gen


def f32_from_bits(h):
    return struct.unpack("<f", struct.pack("<I", int(h, 16)))[0]


# ------------------------------------------------------------------ O1 bf16
def test_bf16_golden(golden):
    g = golden("bf16_rne.json")
    for c in g["cases"]:
        x = f32_from_bits(c["in_bits"])
        got = oracle.bf16(np.array([x], np.float32))[0]
        want = float(c["out"]) if c["out"] != "inf" else math.inf
        assert got == want, c
        assert math.copysign(1.0, got) == math.copysign(1.0, want), c


def test_bf16_matches_torch_library_rne():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32),
                        (rng.standard_normal(20000) * 1e-30).astype(np.float32),
                        (rng.standard_normal(20000) * 1e30).astype(np.float32)])
    want = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(oracle.bf16(x), want)


# ------------------------------------------------------------------ O2/O3 cosine
def test_cosine_golden(golden):
    for c in golden("cosine_hand.json")["cases"]:
        got = oracle.cosine(np.array(c["x"], np.float32), np.array(c["c"], np.float32))
        assert abs(got - c["cos"]) <= 1e-15, c


def test_cosine_closed_forms():
    rng = np.random.default_rng(1)
    d = 64
    # orthonormal basis rows: exactly 0 / 1
    E = np.eye(d, dtype=np.float32)
    sc, ix = oracle.scan_topk(E[:5], E, k=3)
    for i in range(5):
        assert sc[i, 0] == 1.0 and ix[i, 0] == i
        assert sc[i, 1] == 0.0 and sc[i, 2] == 0.0
        # all others tie at 0 -> lowest ids that are not i
        assert list(ix[i, 1:]) == [j for j in range(d) if j != i][:2]
    # self-similarity ~ 1, antipodal ~ -1, |s| <= 1
    X = rng.standard_normal((8, d)).astype(np.float32)
    for x in X:
        assert abs(oracle.cosine(x, x) - 1.0) < 1e-14
        assert abs(oracle.cosine(x, -x) + 1.0) < 1e-14
    sc, _ = oracle.scan_topk(X, rng.standard_normal((200, d)).astype(np.float32), k=200)
    assert np.all(np.abs(sc) <= 1.0 + 1e-15)


def test_cosine_power_of_two_scale_is_exact():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((6, 96)).astype(np.float32)
    Cc = rng.standard_normal((300, 96)).astype(np.float32)
    s0, i0 = oracle.scan_topk(X, Cc, k=5)
    for e in (-7, 3, 11):
        s1, i1 = oracle.scan_topk(X * np.float32(2.0 ** e), Cc, k=5)
        np.testing.assert_array_equal(s0, s1)
        np.testing.assert_array_equal(i0, i1)
        s2, i2 = oracle.scan_topk(X, Cc * np.float32(2.0 ** -e), k=5)
        np.testing.assert_array_equal(s0, s2)


def _fsum_cos(xb, cb):
    """Exactly-rounded cosine of bf16 values with math.fsum (independent of order)."""
    dot = math.fsum(float(a) * float(b) for a, b in zip(xb, cb))
    nx = math.sqrt(math.fsum(float(a) * float(a) for a in xb))
    nc = math.sqrt(math.fsum(float(a) * float(a) for a in cb))
    return dot / (nx * nc)


# ------------------------------------------------------------------ O4 top-k
def test_topk_brute_force_with_duplicates():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    d, M, N, k = 24, 60, 7, 5
    Cc = rng.standard_normal((M, d)).astype(np.float32)
    Cc[17] = Cc[3]       # exact duplicates: ties -> lower id first
    Cc[40] = Cc[3]
    Cc[41] = 2.0 * Cc[9]  # parallel row: same cosine as row 9
    X = rng.standard_normal((N, d)).astype(np.float32)
    X[0] = Cc[3]
    X[1] = Cc[9]
    bf = lambda a: torch.from_numpy(a).to(torch.bfloat16).to(torch.float64).numpy()
    Xb, Cb = bf(X), bf(Cc)
    sc, ix = oracle.scan_topk(X, Cc, k)
    for i in range(N):
        s = np.array([_fsum_cos(Xb[i], Cb[j]) for j in range(M)])
        order = np.lexsort((np.arange(M), -s))  # primary: -s, secondary: id
        assert list(ix[i]) == list(order[:k]), i
        np.testing.assert_allclose(sc[i], s[order[:k]], rtol=0, atol=1e-14)
    assert list(ix[0, :3]) == [3, 17, 40]
    assert set(ix[1, :2]) == {9, 41} and ix[1, 0] == 9


def test_topk_k_at_least_m_pads():
    rng = np.random.default_rng(4)
    Cc = rng.standard_normal((3, 16)).astype(np.float32)
    X = rng.standard_normal((2, 16)).astype(np.float32)
    sc, ix = oracle.scan_topk(X, Cc, k=5)
    for i in range(2):
        assert sorted(ix[i, :3].tolist()) == [0, 1, 2]
        assert np.all(np.diff(sc[i, :3]) <= 0)
        assert list(ix[i, 3:]) == [0xFFFFFFFF] * 2 and list(sc[i, 3:]) == [-1.0, -1.0]
    sc, ix = oracle.scan_topk(X, np.zeros((0, 16), np.float32), k=2)
    assert np.all(ix == 0xFFFFFFFF) and np.all(sc == -1.0)


def test_topk_permutation_relabels():
    rng = np.random.default_rng(5)
    Cc = rng.standard_normal((120, 32)).astype(np.float32)
    X = rng.standard_normal((5, 32)).astype(np.float32)
    s0, i0 = oracle.scan_topk(X, Cc, 6)
    perm = rng.permutation(120)
    s1, i1 = oracle.scan_topk(X, Cc[perm], 6, ids=perm.astype(np.uint32))
    np.testing.assert_array_equal(i0, i1)
    np.testing.assert_array_equal(s0, s1)


def test_topk_of_scores_brute_force():
    """O4 alone (the T2 replay): np.lexsort by (-s, id) on scores with many exact ties
    (two-decimal values), -0.0 tying with +0.0 by id, ids relabelling, k > M padding."""
    rng = np.random.default_rng(44)
    for trial in range(40):
        N, M = int(rng.integers(1, 6)), int(rng.integers(0, 40))
        k = int(rng.integers(1, 9))
        S = np.round(rng.uniform(-1, 1, (N, M)), 1 + trial % 2)
        if M > 3:
            S[:, 1], S[:, 3] = -0.0, 0.0   # lower id holds -0.0: must still come first
        ids = rng.permutation(1000)[:M].astype(np.uint32) if trial % 3 == 0 else None
        sc, ix = oracle.topk_of_scores(S, k, ids=ids)
        g = np.arange(M) if ids is None else ids.astype(np.int64)
        for i in range(N):
            order = np.lexsort((g, -S[i]))[:k]
            n = min(k, M)
            assert list(ix[i, :n]) == [int(g[j]) for j in order], (trial, i)
            assert list(sc[i, :n]) == [float(S[i, j]) for j in order]
            assert list(ix[i, n:]) == [0xFFFFFFFF] * (k - n) and list(sc[i, n:]) == [-1.0] * (k - n)


def test_topk_of_scores_agrees_with_scan():
    """The scan's O4 and the standalone O4 agree on the oracle's own cosines."""
    rng = np.random.default_rng(45)
    Cc = rng.standard_normal((70, 16)).astype(np.float32)
    Cc[30] = Cc[7]
    X = rng.standard_normal((4, 16)).astype(np.float32)
    X[0] = Cc[7]
    S = np.array([[oracle.cosine(x, c) for c in Cc] for x in X])
    np.testing.assert_array_equal(oracle.score_matrix(X, Cc), S)
    s0, i0 = oracle.scan_topk(X, Cc, 6)
    s1, i1 = oracle.topk_of_scores(S, 6)
    np.testing.assert_array_equal(i0, i1)
    np.testing.assert_array_equal(s0, s1)
    assert list(i0[0, :2]) == [7, 30]


def test_topk_rejects_zero_norm():
    with pytest.raises(ValueError):
        oracle.scan_topk(np.zeros((1, 8), np.float32), np.ones((2, 8), np.float32), 1)
    with pytest.raises(ValueError):
        oracle.scan_topk(np.ones((1, 8), np.float32), np.zeros((2, 8), np.float32), 1)


# ------------------------------------------------------------------ O5 predictor
def _sig(z):
    return 1.0 / (1.0 + math.exp(-z))


def test_mlp_hand_example():
    # d=2, k=1, H=2, L=2 with bf16-exact values
    X = np.array([[1.0, 2.0]], np.float32)
    S = np.array([[0.5]])
    W1 = np.array([[1.0, -1.0, 2.0],    # 1 - 2 + 1 = 0 + b1(0.25) -> 0.25
                   [0.5, 0.25, -4.0]], np.float32)  # .5 + .5 - 2 = -1 + b1(0.5) -> relu 0
    b1 = np.array([0.25, 0.5], np.float32)
    W2 = np.array([[9.0, 9.0], [2.0, -3.0]], np.float32)
    b2 = np.array([0.0, -0.25], np.float32)
    r = oracle.mlp(X, S, W1, b1, W2, b2)
    assert r[0, 0] == 1.0                       # full model reference
    assert abs(r[0, 1] - _sig(2.0 * 0.25 - 0.25)) < 1e-15


def test_mlp_closed_forms_and_numpy_forward():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(6)
    N, d, k, H, L = 9, 32, 4, 16, 5
    X = rng.standard_normal((N, d)).astype(np.float32)
    S = rng.uniform(-1, 1, (N, k))
    W1 = rng.standard_normal((H, d + k)).astype(np.float32)
    b1 = rng.standard_normal(H).astype(np.float32)
    W2 = rng.standard_normal((L, H)).astype(np.float32)
    b2 = rng.standard_normal(L).astype(np.float32)
    # W1 = 0 -> identical rows sigma(W2 relu(b1) + b2)
    r = oracle.mlp(X, S, np.zeros_like(W1), b1, W2, b2)
    want = 1 / (1 + np.exp(-(W2.astype(np.float64) @ np.maximum(b1.astype(np.float64), 0) + b2)))
    np.testing.assert_allclose(r[:, 1:], np.tile(want[1:], (N, 1)), rtol=0, atol=1e-14)
    # W2 = 0 -> sigma(b2)
    r = oracle.mlp(X, S, W1, b1, np.zeros_like(W2), b2)
    np.testing.assert_allclose(r[:, 1:], np.tile(1 / (1 + np.exp(-b2[1:].astype(np.float64))), (N, 1)), atol=1e-15)
    # library forward (numpy fp64 on torch-rounded bf16 operands)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(torch.float64).numpy()
    h = np.maximum(bf(X) @ bf(W1[:, :d]).T + S @ W1[:, d:].astype(np.float64).T + b1, 0)
    want = 1 / (1 + np.exp(-(h @ W2.astype(np.float64).T + b2)))
    want[:, 0] = 1.0
    np.testing.assert_allclose(oracle.mlp(X, S, W1, b1, W2, b2), want, rtol=1e-12, atol=1e-13)


def test_mlp_sm_mode_numpy_forward():
    """k = 0 (SM mode: a classifier on the prompt alone): numpy fp64 forward."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(61)
    N, d, H, L = 7, 64, 32, 6
    X = rng.standard_normal((N, d)).astype(np.float32)
    W1 = rng.standard_normal((H, d)).astype(np.float32)
    b1 = rng.standard_normal(H).astype(np.float32)
    W2 = rng.standard_normal((L, H)).astype(np.float32)
    b2 = rng.standard_normal(L).astype(np.float32)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(torch.float64).numpy()
    h = np.maximum(bf(X) @ bf(W1).T + b1, 0)
    want = 1 / (1 + np.exp(-(h @ W2.astype(np.float64).T + b2)))
    want[:, 0] = 1.0
    np.testing.assert_allclose(oracle.mlp(X, np.zeros((N, 0)), W1, b1, W2, b2), want, rtol=1e-12, atol=1e-13)


# ------------------------------------------------------------------ O6..O8 compliance
def _opts(L, pth=None, gates=None, kskip=None):
    pth = list(range(10, 10 + L)) if pth is None else pth
    return [dict(model_id=0, k_skip=(0 if kskip is None else kskip[v]), p_th_qpm=float(pth[v]),
                 sim_gate=(float("-inf") if gates is None else gates[v])) for v in range(L)]


def test_s67_worked_example(golden):
    g = golden("s67_compliance.json")
    q = np.array(g["q"])
    r = (q / q.max())[None, :]           # relative to the best (= full model) image
    lat = g["latency_s"]
    opts = _opts(4, pth=[math.floor(60 / x) for x in lat])
    res = oracle.assign(r, np.array([1.0]), opts, quota=[0, 0, 1, 1], delta=g["delta"])
    assert [v for v in range(4) if res["cmp"][0] >> v & 1] == g["eligible"]
    # the fastest compliant option is the paper's optimal model
    assert max(v for v in range(4) if res["cmp"][0] >> v & 1) == g["fastest_eligible"]
    assert res["option"][0] == 2 and res["status"][0] == 0
    res = oracle.assign(r, np.array([1.0]), opts, quota=[0, 0, 0, 1], delta=g["delta"])
    assert res["option"][0] == 3 and res["status"][0] == oracle.NONCOMPLIANT
    # threshold 19.8 / 22 = 0.9 exactly at the boundary of v3?  19/22 < 0.9 < 20/22
    assert 19 / 22 < g["threshold"] / 22 <= 20 / 22


def test_preference_tie_breaks():
    # equal quality -> faster (higher p_th) first, then lower index
    r = np.array([[1.0, 0.95, 0.95, 0.95]])
    opts = _opts(4, pth=[10, 20, 30, 30])
    res = oracle.assign(r, np.array([1.0]), opts, quota=[1, 1, 1, 1])
    assert list(res["pref"][0]) == [0, 2, 3, 1]


def test_gates():
    r = np.array([[1.0, 0.99, 0.98, 0.97]] * 3)
    opts = _opts(4, gates=[0.99, 0.5, 0.8, 0.9], kskip=[0, 5, 10, 15])
    s1 = np.array([0.95, 0.85, 0.1])
    res = oracle.assign(r, s1, opts, quota=[0, 3, 3, 3])
    assert list(res["adm"]) == [0b1111, 0b0111, 0b0001]
    # option 0 carries a gate value but is never gated
    assert res["option"].tolist() == [1, 1, 0]
    assert res["status"][2] == oracle.OVERFLOW | oracle.GATED_ALL


# ------------------------------------------------------------------ O9/O10 assignment
def _indep_pref_and_priority(r, s1, opts, delta):
    """Re-derive A_i, C_i, pi_i and the priority order with plain Python sorts."""
    N, L = r.shape
    d64 = float(np.float32(delta))
    A = [[v for v in range(L) if v == 0 or opts[v]["k_skip"] == 0 or s1[i] >= float(np.float32(opts[v]["sim_gate"]))]
         for i in range(N)]
    Cs = [[v for v in A[i] if r[i, v] >= d64] for i in range(N)]
    pi = [sorted(A[i], key=lambda v: (-r[i, v], -opts[v]["p_th_qpm"], v)) for i in range(N)]
    order = sorted(range(N), key=lambda i: (len(Cs[i]), i))
    return A, Cs, pi, order


def _brute_sd(r, s1, opts, quota, delta=0.9):
    """Serial dictatorship characterised as the lexicographically best assignment
    (preference ranks compared in priority order), found by enumeration.  A prompt
    may also be left unserved (OVF, ranked after all of pi_i, consumes no quota);
    SD maps it to option 0 with the OVERFLOW bit."""
    A, Cs, pi, order = _indep_pref_and_priority(r, s1, opts, delta)
    N = len(A)
    OVF = -1
    best, best_key = None, None
    for a in itertools.product(*[pi[i] + [OVF] for i in range(N)]):
        served = [x for x in a if x != OVF]
        cnt = np.bincount(served, minlength=len(quota)) if served else np.zeros(len(quota), int)
        if np.any(cnt > quota):
            continue
        key = tuple(len(pi[i]) if a[i] == OVF else pi[i].index(a[i]) for i in order)
        if best_key is None or key < best_key:
            best, best_key = a, key
    return best


def _random_instance(rng, N, L, gates=True):
    r = rng.uniform(0.8, 1.0, (N, L))
    r[:, 0] = 1.0
    if rng.random() < 0.5:   # coarse values to create quality ties
        r = np.round(r * 20) / 20
        r[:, 0] = 1.0
    pth = np.sort(rng.integers(10, 14, L)).astype(float)
    kskip = [0] + [int(x) for x in rng.integers(0, 2, L - 1) * 5]
    g = [float(x) for x in rng.uniform(0.3, 0.9, L)] if gates else None
    opts = _opts(L, pth=pth, gates=g, kskip=kskip)
    s1 = rng.uniform(0.2, 1.0, N)
    return r, s1, opts


def test_serial_dictatorship_brute_force():
    rng = np.random.default_rng(7)
    n_checked = 0
    for _ in range(300):
        N = int(rng.integers(1, 7))
        L = int(rng.integers(1, 5))
        r, s1, opts = _random_instance(rng, N, L)
        quota = rng.integers(0, N + 1, L)
        quota[0] = max(quota[0], N - quota[1:].sum())  # sum c >= N: no overflow possible
        want = _brute_sd(r, s1, opts, quota)
        got = oracle.assign(r, s1, opts, quota)
        ovf = [x == -1 for x in want]
        assert ((got["status"] & oracle.OVERFLOW) != 0).tolist() == ovf
        assert got["option"].tolist() == [0 if x == -1 else x for x in want]
        assert got["rc"] == int(any(ovf))
        A, Cs, pi, order = _indep_pref_and_priority(r, s1, opts, 0.9)
        assert got["order"].tolist() == order
        for i in range(N):
            assert [int(x) for x in got["pref"][i][:len(pi[i])]] == pi[i]
        n_checked += 1
    assert n_checked == 300


def test_assignment_invariants():
    rng = np.random.default_rng(8)
    for t in range(400):
        N = int(rng.integers(1, 40))
        L = int(rng.integers(1, 9))
        gates = t % 2 == 0
        r, s1, opts = _random_instance(rng, N, L, gates)
        quota = rng.integers(0, max(2, N // 2), L)
        res = oracle.assign(r, s1, opts, quota)
        a, st = res["option"], res["status"]
        ok = (st & oracle.OVERFLOW) == 0
        cnt = np.bincount(a[ok], minlength=L)
        assert np.all(cnt <= quota)                                  # I1
        rem = quota - cnt
        for i in range(N):
            assert res["cmp"][i] & 1                                 # I3
            if r[i, a[i]] < 0.9 and ok[i]:                           # I2
                for v in range(L):
                    if res["cmp"][i] >> v & 1:
                        assert rem[v] == 0
            assert bool(st[i] & oracle.NONCOMPLIANT) == (r[i, a[i]] < float(np.float32(0.9)))
        assert a.size == N                                           # I6
        if not gates:
            assert int((~ok).sum()) == max(0, N - int(quota.sum()))  # overflow count
        assert (res["rc"] == 1) == bool((~ok).any())
    # I4: ample quotas -> each prompt gets the head of its preference list
    r, s1, opts = _random_instance(rng, 12, 5)
    res = oracle.assign(r, s1, opts, [12] * 5)
    assert res["option"].tolist() == [int(p[0]) for p in res["pref"]]
    # I5: the whole quota on one option -> every prompt admitted to it gets it
    res = oracle.assign(r, s1, opts, [0, 0, 12, 0, 0])
    for i in range(12):
        assert res["option"][i] == (2 if res["adm"][i] >> 2 & 1 else 0)


def test_p_oda_monotone_pin():
    """With gates off, r strictly decreasing in v and sum c = N, |C_i| - 1 is the
    paper's optimal model o_i (fastest compliant) and SD minimises the
    Eq.-2-style cost sum_i D(a_i, o_i) for any convex non-decreasing D with
    D = 0 for slower shifts.  Brute force with D = max(0,gap)^2."""
    rng = np.random.default_rng(9)
    for _ in range(400):
        N = int(rng.integers(1, 7))
        L = int(rng.integers(2, 5))
        r = np.sort(rng.uniform(0.8, 1.0, (N, L)), axis=1)[:, ::-1].copy()
        r[:, 0] = 1.0
        r[:, 1:] = np.minimum(r[:, 1:], 0.9999)
        opts = _opts(L)
        cuts = np.sort(rng.integers(0, N + 1, L - 1))
        quota = np.diff(np.concatenate([[0], cuts, [N]]))
        res = oracle.assign(r, np.ones(N), opts, quota)
        o = np.array([bin(int(m)).count("1") - 1 for m in res["cmp"]])
        assert np.all(o == (r >= float(np.float32(0.9))).sum(1) - 1)
        D = lambda a, oi: max(0, a - oi) ** 2
        got = sum(D(a, oi) for a, oi in zip(res["option"], o))
        best = min(sum(D(a, oi) for a, oi in zip(asg, o))
                   for asg in itertools.product(range(L), repeat=N)
                   if np.all(np.bincount(asg, minlength=L) == quota))
        assert got == best


# ------------------------------------------------------------------ quotas
def test_quota_golden(golden):
    for c in golden("quota_ties.json")["cases"]:
        assert oracle.quota_from_fractions(c["f"], c["N"]).tolist() == c["c"], c


def test_quota_properties():
    rng = np.random.default_rng(10)
    for _ in range(500):
        L = int(rng.integers(1, 25))
        N = int(rng.integers(0, 9000))
        f = rng.random(L) * (rng.random(L) < 0.8)
        if f.sum() == 0:
            f[0] = 1
        c = oracle.quota_from_fractions(f, N)
        assert c.sum() == N and np.all(c >= 0)
        assert np.all(np.abs(c - f / f.sum() * N) < 1.0 + 1e-9)
    c = oracle.quota_from_fractions([1, 3, 4], 16)   # F*N integer -> exact
    assert c.tolist() == [2, 6, 8]
    with pytest.raises(ValueError):
        oracle.quota_from_fractions([0, 0], 4)
    with pytest.raises(ValueError):
        oracle.quota_from_fractions([1, -1], 4)


# ------------------------------------------------------------------ end to end on C1
def test_oracle_route_c1_invariants():
    p = gen.small_problem("C1")
    quota = oracle.quota_from_fractions(p.fractions, p.X.shape[0])
    res = oracle.route(p.X, p.cache, p.cfg.k, p.W1, p.b1, p.W2, p.b2, p.opts, quota)
    N = p.X.shape[0]
    assert res["topk_idx"].shape == (N, p.cfg.k)
    # 30 % of C1 prompts are exact repeats: top-1 cosine == 1 up to rounding
    assert np.sum(res["topk_score"][:, 0] > 1 - 1e-12) >= 5
    assert np.all(np.diff(res["topk_score"], axis=1) <= 0)
    assert res["option"].size == N and np.all(res["rhat"][:, 0] == 1.0)
    cnt = np.bincount(res["option"][(res["status"] & 1) == 0], minlength=len(p.opts))
    assert np.all(cnt <= quota)


def test_delta_boundary_is_inclusive():
    """r >= delta (P:189 'q >= 0.9 q_1'), delta compared as the fp32 value 0.9f."""
    d32 = float(np.float32(0.9))
    r = np.array([[1.0, d32, np.nextafter(d32, 0)]])
    res = oracle.assign(r, np.ones(1), _opts(3), quota=[0, 1, 1])
    assert res["cmp"][0] == 0b011
    assert res["option"][0] == 1 and res["status"][0] == 0


def test_gate_boundary_is_inclusive():
    """Similarity gate s_i1 >= tau_v, tau compared as fp32."""
    tau = float(np.float32(0.8))
    opts = _opts(2, gates=[float("-inf"), 0.8], kskip=[0, 10])
    r = np.array([[1.0, 0.95], [1.0, 0.95]])
    res = oracle.assign(r, np.array([tau, np.nextafter(tau, 0)]), opts, quota=[0, 2])
    assert res["adm"].tolist() == [0b11, 0b01]
    assert res["option"].tolist() == [1, 0]
