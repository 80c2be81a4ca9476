"""Pins for the control-plane oracle (oracle/control.py): ODA/PASM (Algorithm 1,
Eq. 2), Philox sampling, the optimal option, Eq. 3 worker selection and the
Eq. 1 allocator, each checked against something other than itself: the SPEC's
hand traces, known-answer vectors, a linear-programming solver, closed forms,
exhaustive search and invariants."""
import itertools

import numpy as np
import pytest

from oracle import control as oc


def hx(s):
    return int(s, 16)


# ------------------------------------------------------------------ Philox (R20)
def test_philox_known_answers(golden):
    for c in golden("philox_kat.json")["cases"]:
        got = oc.philox4x32_10([hx(x) for x in c["ctr"]], [hx(x) for x in c["key"]])
        assert list(got) == [hx(x) for x in c["out"]]


def test_uniform24_exact_and_in_range():
    us = [oc.uniform24(7, 3, i) for i in range(2000)]
    assert all(0.0 <= float(u) < 1.0 for u in us)
    assert all(float(u) * 16777216.0 == int(float(u) * 16777216.0) for u in us)   # multiples of 2^-24
    assert len(set(float(u) for u in us)) > 1990                                   # counter-based, not constant
    assert oc.uniform24(7, 3, 5) != oc.uniform24(7, 4, 5) != oc.uniform24(8, 3, 5)


def test_uniform24_golden_counter_layout(golden):
    """R20's draw against cuRAND's independent Philox4x32-10 (tests/golden/pasm_uniform.json,
    tools/gen_pasm_golden.cu): pins the counter layout {i, seq lo, seq hi, 0}, the key
    {seed lo, seed hi}, the use of word x0 (not x1) and the >> 8 scaling.  Case 0 is also
    the Random123 zero KAT: x0 = 0x6627e8d5."""
    g = golden("pasm_uniform.json")["cases"]
    assert g[0]["x0"] == "6627e8d5"
    for c in g:
        u = oc.uniform24(c["seed"], c["seq"], c["i"])
        assert u.dtype == np.float32
        assert float(u) == c["u_m"] / 16777216.0, c
        assert c["u_m"] == hx(c["x0"]) >> 8
        assert float(u) != (hx(c["x1"]) >> 8) / 16777216.0   # word x0, not x1


def test_pasm_sample_strict_boundary(golden):
    """u == cdf_j exactly selects j + 1 (a = first j with u < cdf_j, R20): the row
    (u, 1 - u) for prompt 0 of call 0 under seed 0 must land on option 1."""
    c = golden("pasm_uniform.json")["cases"][0]
    u = np.float32(c["u_m"] / 16777216.0)
    P = np.array([[float(u), 1.0 - float(u)], [0.0, 1.0]])
    cdf = oc.pasm_cdf32(P)
    assert cdf[0][0] == u
    assert oc.pasm_sample(P[0], cdf[0], u) == 1
    # one ulp (2^-24 steps are exact here) below the boundary stays on option 0
    assert oc.pasm_sample(P[0], cdf[0], np.float32(u - np.float32(2 ** -24))) == 0
    # the same through the per-batch sampler: o_0 = 0 (option 1 non-compliant)
    opts = [dict(model_id=0, k_skip=0, p_th_qpm=10.0, sim_gate=0.0), dict(model_id=1, k_skip=0, p_th_qpm=20.0, sim_gate=0.0)]
    res = oc.pasm_assign(np.array([[1.0, 0.5]]), np.array([0.3]), opts, P, 0, 0)
    assert res["optimal"][0] == 0 and res["option"][0] == 1


# ------------------------------------------------------------------ ODA (Alg. 1)
def test_oda_spec_traces(golden):
    for c in golden("oda_spec.json")["cases"]:
        P = oc.oda_pasm(c["H"], c["F"])
        np.testing.assert_allclose(P, np.array(c["pasm"], float), atol=1e-12)
        n = len(c["H"])
        D = np.zeros((n, n))
        D[1][0] = c["D_v1_v0"]
        p_th = list(range(n))
        assert abs(oc.eq2_degradation(P, c["H"], p_th, D) - c["D_Q"]) < 1e-12


def _rand_hf(rng, n):
    H = rng.random(n) * (rng.random(n) < 0.8)
    F = rng.random(n) * (rng.random(n) < 0.8)
    if H.sum() == 0:
        H[0] = 1
    if F.sum() == 0:
        F[-1] = 1
    return H / H.sum(), F / F.sum()


def test_oda_row_stochastic_and_pushforward():
    """every PASM row sums to 1, entries >= 0, and sum_i H_i P(j|i) = F_j."""
    rng = np.random.default_rng(1)
    for _ in range(3000):
        n = int(rng.integers(2, 9))
        H, F = _rand_hf(rng, n)
        P = oc.oda_pasm(H, F)
        assert (P >= -1e-12).all()
        np.testing.assert_allclose(P.sum(1), 1.0, atol=1e-9)
        np.testing.assert_allclose(H @ P, F, atol=1e-9)


@pytest.mark.parametrize("p", [2.0, 1.5, 3.0])
def test_oda_minimises_eq2(p):
    """The paper's optimality claim: for a degradation that grows
    super-linearly with the speed gap, ODA's Eq. 2 cost equals the minimum over ALL
    transport plans, found by an independent LP solver (scipy/HiGHS)."""
    rng = np.random.default_rng(int(p * 10))
    for _ in range(150):
        n = int(rng.integers(2, 7))
        H, F = _rand_hf(rng, n)
        D = oc.superlinear_D(n, p)
        p_th = list(range(n))
        dq = oc.eq2_degradation(oc.oda_pasm(H, F), H, p_th, D)
        best = oc.min_degradation_transport(H, F, p_th, D)
        assert abs(dq - best) <= 1e-9 * max(1.0, best), (H, F, dq, best)


def test_oda_only_slower_shifts_when_fast_levels_oversubscribed():
    """S:329 slower-shift purity: if H_i >= F_i at every level but the slowest, no
    mass moves to a faster level (D_Q = 0 for any D)."""
    rng = np.random.default_rng(3)
    for _ in range(500):
        n = int(rng.integers(2, 8))
        F = rng.random(n)
        F /= F.sum()
        extra = rng.random(n) * 0.3
        H = F + extra
        H[0] = 0.0
        H = H / H.sum()
        if not all(H[i] >= F[i] for i in range(1, n)):
            continue
        P = oc.oda_pasm(H, F)
        assert all(P[i][j] == 0 for i in range(n) for j in range(i + 1, n))


def test_oda_reverses_nothing_when_equal():
    for n in range(1, 9):
        h = np.arange(1, n + 1, dtype=float)
        h /= h.sum()
        np.testing.assert_array_equal(oc.oda_pasm(h, h), np.eye(n))


# ------------------------------------------------------------------ sampling
def test_pasm_sampling_frequency():
    """row {v0: 5/7, v1: 2/7}, 70k counter-based samples -> v1 frequency
    within [0.27, 0.30] (binomial concentration)."""
    P = oc.oda_pasm([0.7, 0.3], [0.5, 0.5])
    cdf = oc.pasm_cdf32(P)
    hits = sum(oc.pasm_sample(P[0], cdf[0], oc.uniform24(11, 0, i)) for i in range(70000))
    assert 0.27 <= hits / 70000 <= 0.30


def test_pasm_sampling_degenerate_rows():
    P = np.array([[0.0, 0.0, 1.0], [0, 1, 0], [0, 0, 1]])
    cdf = oc.pasm_cdf32(P)
    for i in range(500):
        u = oc.uniform24(5, 1, i)
        assert oc.pasm_sample(P[0], cdf[0], u) == 2
        assert oc.pasm_sample(P[1], cdf[1], u) == 1
    # rounding leaves u above the last cdf entry -> the last option with mass
    P = np.array([[0.5, 0.49999, 0.0], [0, 1, 0], [0, 0, 1]])
    c = oc.pasm_cdf32(P)
    assert c[0][2] < np.float32(1.0 - 2 ** -24)
    assert oc.pasm_sample(P[0], c[0], np.float32(1.0 - 2 ** -24)) == 1


# ------------------------------------------------------------------ optimal option
def test_optimal_option_spec_example(golden):
    """q = {22, 21, 20, 19}, delta = 0.9 -> eligible {v0, v1, v2}, fastest = v2."""
    g = golden("s67_compliance.json")
    r = np.array(g["q"]) / g["q"][0]
    p_th = [60.0 / x for x in g["latency_s"]]
    assert oc.optimal_option(r, 0b1111, p_th, g["delta"]) == g["fastest_eligible"]
    # gating v2 out leaves v1 the fastest compliant option
    assert oc.optimal_option(r, 0b1011, p_th, g["delta"]) == 1


def test_optimal_option_ties_and_full_model():
    p_th = [10.0, 20.0, 20.0, 30.0]
    assert oc.optimal_option([1, .95, .97, .5], 0b1111, p_th) == 2     # equal p_th: higher r
    assert oc.optimal_option([1, .95, .95, .5], 0b1111, p_th) == 1     # then lower v
    assert oc.optimal_option([1, .1, .1, .1], 0b1111, p_th) == 0       # only the full model complies
    assert oc.optimal_option([1, .95, .95, .95], 0b0001, p_th) == 0    # gates leave option 0


def test_pasm_assign_identity_and_gate_fallback():
    opts = [dict(model_id=0, k_skip=0, p_th_qpm=10.0, sim_gate=-np.inf),
            dict(model_id=0, k_skip=5, p_th_qpm=12.0, sim_gate=0.8),
            dict(model_id=0, k_skip=10, p_th_qpm=14.0, sim_gate=0.9)]
    rhat = np.array([[1, .95, .93], [1, .95, .5], [1, .5, .5], [1, .95, .95]])
    s1 = np.array([0.95, 0.95, 0.95, 0.85])
    res = oc.pasm_assign(rhat, s1, opts, np.eye(3), seed=1, batch_seq=0)
    np.testing.assert_array_equal(res["optimal"], [2, 1, 0, 1])
    np.testing.assert_array_equal(res["option"], [2, 1, 0, 1])
    # PASM sends every v2-optimal prompt to v2, but prompt 3 fails v2's gate -> v1
    P = np.array([[0, 0, 1.0], [0, 0, 1.0], [0, 0, 1.0]])
    res = oc.pasm_assign(rhat, s1, opts, P, seed=1, batch_seq=0)
    np.testing.assert_array_equal(res["option"], [2, 2, 2, 1])
    assert res["status"][1] & 2 and res["status"][2] & 2 and not res["status"][0] & 2


# ------------------------------------------------------------------ Eq. 3
def test_select_worker_spec_examples(golden):
    for c in golden("control_spec.json")["workers"]:
        w, _ = oc.select_workers(c["assigned"], c["option_of_worker"], c["t_proc"], c["queue"])
        assert list(w) == c["worker"]


def test_select_worker_exhaustive_argmin():
    """each choice is the exhaustive argmin of R_w * t_w over the eligible
    workers at that moment (ties -> lowest id); queues grow by the batch's counts."""
    rng = np.random.default_rng(4)
    for _ in range(300):
        W = int(rng.integers(1, 9))
        L = int(rng.integers(1, 4))
        wo = rng.integers(0, L, W)
        t = rng.choice([1.0, 2.5, 4.2], W).astype(np.float32)
        q0 = rng.integers(0, 4, W)
        assigned = rng.integers(0, L, int(rng.integers(1, 20)))
        w, q1 = oc.select_workers(assigned, wo, t, q0)
        q = list(q0)
        for a, got in zip(assigned, w):
            elig = [x for x in range(W) if wo[x] == a]
            if not elig:
                assert got == -1
                continue
            costs = {x: np.float32(q[x]) * np.float32(t[x]) for x in elig}
            m = min(costs.values())
            assert got == min(x for x in elig if costs[x] == m)
            q[got] += 1
        np.testing.assert_array_equal(q1, q)


# ------------------------------------------------------------------ Eq. 1
def test_allocation_spec_examples(golden):
    for c in golden("control_spec.json")["allocation"]:
        r = oc.allocation_bruteforce(c["W"], c["workers"], c["Q"], c["P_th"])
        assert abs(r["objective"] - c["objective"]) < 1e-12
        assert tuple(c["Y"]) in r["optimal_Y"]


def test_allocation_closed_forms():
    # enough slow capacity: everything on the slowest (highest-Q) level
    for W in range(1, 4 * 14 + 1, 5):
        r = oc.allocation_bruteforce(W, 4, [1.0, 0.8, 0.6], [14, 27, 40])
        assert r["optimal_Y"] == {(W, 0, 0)} and r["objective"] == 1.0
    # above every capacity: saturated on the fastest level, flagged
    r = oc.allocation_bruteforce(200, 2, [1.0, 0.8], [14, 27])
    assert not r["feasible"] and r["optimal_Y"] == {(0, 54)}


def test_allocation_monotone_in_load():
    """the objective is non-increasing in W for a fixed cluster."""
    prev = None
    for W in range(1, 3 * 27 + 1):
        r = oc.allocation_bruteforce(W, 3, [1.0, 0.85, 0.7], [14, 20, 27])
        assert r["feasible"]
        if prev is not None:
            assert r["objective"] <= prev + 1e-12
        prev = r["objective"]


def test_allocation_matches_lp_relaxation_bound():
    """Eq. 1 with integer loads can never beat its LP relaxation over the same
    composition (independent solver), and reaches it when P_th are integers."""
    from scipy.optimize import linprog
    rng = np.random.default_rng(6)
    for _ in range(40):
        Lv = int(rng.integers(2, 4))
        n = int(rng.integers(1, 4))
        Q = sorted(rng.random(Lv) * 0.5 + 0.5, reverse=True)
        P = sorted(rng.integers(5, 30, Lv))
        W = int(rng.integers(1, n * P[-1] + 1))
        r = oc.allocation_bruteforce(W, n, Q, P)
        best = -1.0
        for comp in itertools.product(range(n + 1), repeat=Lv):
            if sum(comp) > n:
                continue
            caps = [comp[v] * P[v] for v in range(Lv)]
            if sum(caps) < W:
                continue
            res = linprog(-np.array(Q), A_eq=[np.ones(Lv)], b_eq=[W], bounds=[(0, c) for c in caps], method="highs")
            best = max(best, -res.fun / W)
        assert abs(best - r["objective"]) < 1e-9


def test_affinity_histogram_window():
    """H(v) over the last 1000 prompts' optimal options (hand-countable)."""
    hist = [0] * 700 + [3] * 500 + [1] * 300
    h = oc.affinity_histogram(hist, 4)
    assert list(h) == [200, 300, 0, 500]          # the first 500 zeros fell out of the window
    assert list(oc.affinity_histogram([2, 2, 1], 4)) == [0, 1, 2, 0]
    assert list(oc.affinity_histogram(hist, 4, window=10)) == [0, 10, 0, 0]
