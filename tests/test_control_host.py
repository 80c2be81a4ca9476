"""Host-side control plane of libargus (no GPU needed: plain host functions of the
C ABI) against the control-plane oracle: ODA / PASM (Algorithm 1), Eq. 2 and the
Eq. 1 allocator.  The oracle is pinned in test_oracle_control.py."""
import numpy as np
import pytest

from oracle import control as oc


@pytest.fixture(scope="module")
def argus():
    from paper_2511_06724_b200 import argus
    return argus


def _rand_hf(rng, n):
    H = rng.random(n) * (rng.random(n) < 0.8)
    F = rng.random(n) * (rng.random(n) < 0.8)
    if H.sum() == 0:
        H[0] = 1
    if F.sum() == 0:
        F[-1] = 1
    return H / H.sum(), F / F.sum()


def test_oda_matches_oracle(argus):
    rng = np.random.default_rng(10)
    for _ in range(2000):
        n = int(rng.integers(1, 33 if rng.random() < 0.1 else 9))
        H, F = _rand_hf(rng, n)
        np.testing.assert_allclose(argus.argus_oda_pasm(H, F), oc.oda_pasm(H, F), atol=1e-12)


def test_oda_counts_are_normalised(argus):
    H = np.array([70.0, 30.0])   # counts from the affinity window
    P = argus.argus_oda_pasm(H, [0.5, 0.5])
    np.testing.assert_allclose(P, [[5 / 7, 2 / 7], [0, 1]], atol=1e-15)


def test_eq2_matches_oracle(argus):
    rng = np.random.default_rng(11)
    for _ in range(200):
        n = int(rng.integers(2, 9))
        H, F = _rand_hf(rng, n)
        P = oc.oda_pasm(H, F)
        p_th = np.sort(rng.integers(5, 40, n)).astype(np.float32)
        D = rng.random((n, n))
        assert abs(argus.argus_pasm_degradation(P, H, p_th, D) - oc.eq2_degradation(P, H, p_th, D)) < 1e-12


def _check_plan(res, W, n, Q, P_th):
    caps = [int(p) for p in P_th]
    lv, ld = res["levels"], res["loads"]
    assert len(lv) == n and all(0 <= v < len(Q) for v in lv)
    assert all(0 <= ld[w] <= caps[lv[w]] for w in range(n))
    Y = np.zeros(len(Q), np.int64)
    for w in range(n):
        Y[lv[w]] += ld[w]
    return Y


def test_allocation_matches_bruteforce(argus):
    rng = np.random.default_rng(12)
    for _ in range(150):
        Lv = int(rng.integers(1, 4))
        n = int(rng.integers(1, 4))
        Q = list(np.round(rng.random(Lv) * 0.5 + 0.5, 3))
        P = sorted(rng.integers(4, 25, Lv).tolist())
        W = int(rng.integers(0, n * P[-1] + 8))
        ref = oc.allocation_bruteforce(W, n, Q, P)
        res = argus.argus_solve_allocation(W, n, Q, P)
        assert res["feasible"] == ref["feasible"]
        Y = _check_plan(res, W, n, Q, P)
        if ref["feasible"]:
            assert Y.sum() == W
            assert res["objective"] >= ref["objective"] - 1e-12, (W, n, Q, P, res, ref)
            assert abs(res["objective"] - ref["objective"]) <= 1e-12
            if W > 0:
                np.testing.assert_allclose(res["F"], Y / W, atol=0)
        else:
            assert tuple(Y) in ref["optimal_Y"]
            assert res["objective"] == ref["objective"]


def test_allocation_spec_examples(argus, golden):
    for c in golden("control_spec.json")["allocation"]:
        res = argus.argus_solve_allocation(c["W"], c["workers"], c["Q"], c["P_th"])
        assert abs(res["objective"] - c["objective"]) < 1e-12
        Y = _check_plan(res, c["W"], c["workers"], c["Q"], c["P_th"])
        assert list(Y) == c["Y"]


def test_allocation_paper_cluster(argus):
    """8 workers, the AC levels K = 0..25 of SD-XL: quality falls as
    load rises and the plan always carries exactly W (or saturates)."""
    lat = [(50 - K) / 50 * 4.2 + 0.05 for K in (0, 5, 10, 15, 20, 25)]
    p_th = [float(np.floor(60 / x)) for x in lat]
    Q = [1.0, 0.97, 0.94, 0.9, 0.86, 0.8]
    prev = 2.0
    for W in range(0, 8 * int(p_th[-1]) + 20, 7):
        res = argus.argus_solve_allocation(W, 8, Q, p_th)
        Y = _check_plan(res, W, 8, Q, p_th)
        if res["feasible"]:
            assert Y.sum() == W
            if W:
                assert res["objective"] <= prev + 1e-12
                prev = res["objective"]
        else:
            assert W > 8 * int(p_th[-1]) and Y.sum() == 8 * int(p_th[-1])


def test_control_rejects_bad_inputs(argus):
    with pytest.raises(argus.ArgusError):
        argus.argus_oda_pasm([0.0, 0.0], [0.5, 0.5])
    with pytest.raises(argus.ArgusError):
        argus.argus_oda_pasm([np.nan, 1.0], [0.5, 0.5])
    with pytest.raises(argus.ArgusError):
        argus.argus_solve_allocation(-1, 2, [1.0], [10.0])
