"""Parity helpers: compare the CUDA path with the oracle.

Test infrastructure (imports oracle/).  Tolerances come from BASELINE.json
north_star: "similarity and predictor outputs within 2e-2 absolute (bf16 inputs,
fp32 accumulate); top-k index sets and final assignments bit-exact, except where
the oracle's score gap at the boundary is below 1e-3".
"""
from __future__ import annotations

import json
import os

import numpy as np

import oracle

SCORE_TOL = 2e-2    # T1, M1, M2
GAP_TOL = 1e-3      # T3 boundary-gap exemption, A2 fragility
# Bounds on the loosely checked share (SURVEY §8(c).iii "report the exemption rate"):
# clustered caches put several rows within 1e-3 of a prompt's k-th score, so T3 leaves
# 30-80 % of rows to its tie-group rule at these sizes (T2 checks them exactly); a rate
# above this bound means the synthetic workload degenerated (e.g. all-duplicate rows)
# and the top-k parity would be checking little.
MAX_T3_EXEMPT_RATE = 0.9
DELTA32 = float(np.float32(oracle.DELTA))

# Per-test parity statistics (T3 exemption rates, A2 matched-prefix fractions, T2
# replays), printed at the end of the session by tests/conftest.py and written to
# $ARGUS_PARITY_REPORT (JSON lines) when that is set.
REPORT = []


def report(kind, **kw):
    rec = dict(test=os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], kind=kind, **kw)
    REPORT.append(rec)
    path = os.environ.get("ARGUS_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
    return rec


def check_topk(X, cache, k, gpu_idx, gpu_score, ids=None, rows=None):
    """T1 + T3.  Returns dict(exempt_rows, max_score_err).  Raises AssertionError.

    For each row the oracle's top-(k+1) fixes tie groups (maximal runs of
    consecutive oracle scores closer than GAP_TOL).  Entries whose group is fully
    inside the top-k must appear (as a set per group, in group order); the group
    straddling position k may be filled by any of its members.  Every returned id
    must score (in the oracle) >= s_(k) - GAP_TOL, and |gpu - oracle| <= SCORE_TOL
    for every returned (id, score)."""
    rows = range(X.shape[0]) if rows is None else rows
    Xs = X[list(rows)]
    M = cache.shape[0]
    kk = min(k + 1, max(M, 1))
    osc, oix = oracle.scan_topk(Xs, cache, kk, ids=ids)
    row_of = (lambda g: g) if ids is None else {int(g): j for j, g in enumerate(ids)}.__getitem__
    exempt, max_err = 0, 0.0
    for r, i in enumerate(rows):
        gi = [int(x) for x in gpu_idx[i]]
        gs = [float(x) for x in gpu_score[i]]
        nreal = min(k, M)
        # padding
        assert gi[nreal:] == [0xFFFFFFFF] * (k - nreal), (i, gi)
        assert all(s == -1.0 for s in gs[nreal:]), (i, gs)
        if nreal == 0:
            continue
        o_s = osc[r]
        o_i = [int(x) for x in oix[r]]
        # scores of the GPU's ids, in the oracle
        g_true = np.array([oracle.cosine(X[i], cache[row_of(g)]) for g in gi[:nreal]])
        err = np.abs(g_true - np.array(gs[:nreal]))
        max_err = max(max_err, float(err.max()))
        assert err.max() <= SCORE_TOL, (i, err.max())
        # tie groups over the oracle's k(+1) list
        groups, cur = [], [0]
        for t in range(1, len(o_i)):
            if o_s[t - 1] - o_s[t] < GAP_TOL:
                cur.append(t)
            else:
                groups.append(cur)
                cur = [t]
        groups.append(cur)
        kth = o_s[nreal - 1]
        boundary_tie = len(o_i) > nreal and (o_s[nreal - 1] - o_s[nreal] < GAP_TOL)
        if boundary_tie:
            exempt += 1
        pos = 0
        for grp in groups:
            if pos >= nreal:
                break
            members = [o_i[t] for t in grp if t < len(o_i)]
            take = min(len(members), nreal - pos)
            got = gi[pos:pos + take]
            if take == len(members) and not (boundary_tie and grp[-1] >= nreal - 1):
                assert sorted(got) == sorted(members), (i, got, members, o_s)
            else:   # the straddling group: any members with score >= s_k - GAP_TOL
                for g, sg in zip(got, g_true[pos:pos + take]):
                    assert sg >= kth - GAP_TOL - 1e-12, (i, g, sg, kth)
            pos += take
        # order: GPU list sorted by its own scores, descending (ties -> lower id)
        for t in range(nreal - 1):
            assert (gs[t] > gs[t + 1]) or (gs[t] == gs[t + 1] and gi[t] < gi[t + 1]), (i, gs, gi)
    nrows = len(list(rows))
    report("T3", rows=nrows, exempt_rows=exempt, exempt_rate=round(exempt / max(1, nrows), 4), M=int(M), k=int(k),
           max_score_err=max_err)
    if nrows >= 20:
        assert exempt / nrows <= MAX_T3_EXEMPT_RATE, (exempt, nrows)
    return dict(exempt_rows=exempt, max_score_err=max_err, rows=nrows)


def check_topk_replay(S_gpu, gpu_idx, gpu_score, k, ids=None):
    """T2: oracle O4 run on the GPU's own fp32 scores (S_gpu [N, M], captured from the
    scan by argus_debug_capture) must give the GPU's top-k exactly -- ids, scores and
    order.  This checks the fused filter / top-k / merges independently of rounding."""
    S_gpu = np.asarray(S_gpu, np.float32)
    assert np.isfinite(S_gpu).all(), "capture left unwritten (NaN) entries"
    sc, ix = oracle.topk_of_scores(S_gpu.astype(np.float64), k, ids=ids)
    np.testing.assert_array_equal(np.asarray(gpu_idx, np.uint32), ix)
    np.testing.assert_array_equal(np.asarray(gpu_score, np.float32).astype(np.float64), sc)
    report("T2", rows=int(S_gpu.shape[0]), M=int(S_gpu.shape[1]), k=int(k), exact=True)


def check_replay(gpu, opts, quota, delta=oracle.DELTA):
    """A1: O6..O10 in fp64 on the GPU's own fp32 r and s_1 -> bit-exact options/status."""
    rhat = gpu["quality"].astype(np.float64)
    s1 = gpu["topk_score"][:, 0].astype(np.float64)
    rep = oracle.assign(rhat, s1, opts, quota, delta)
    np.testing.assert_array_equal(gpu["option"], rep["option"])
    np.testing.assert_array_equal(gpu["status"], rep["status"])
    return rep


def check_mlp_replay(X, gpu, W1, b1, W2, b2):
    """M1: oracle O5 on the GPU's top-k scores vs the GPU's r (<= 2e-2)."""
    r = oracle.mlp(X, gpu["topk_score"].astype(np.float64), W1, b1, W2, b2)
    err = float(np.abs(r - gpu["quality"]).max())
    assert err <= SCORE_TOL, err
    return err


def invariants(gpu, opts, quota, delta=oracle.DELTA):
    """A3: I1 (quotas), I2 (no below-threshold option while a compliant one is
    free), I3 (full model compliant), I6 (everyone assigned)."""
    a, st, rq = gpu["option"], gpu["status"], gpu["quality"]
    L = len(opts)
    ok = (st & oracle.OVERFLOW) == 0
    cnt = np.bincount(a[ok], minlength=L)
    assert np.all(cnt <= quota), (cnt, quota)
    rem = np.asarray(quota) - cnt
    s1 = gpu["topk_score"][:, 0]
    for i in range(a.size):
        assert rq[i, 0] == 1.0
        if ok[i] and rq[i, a[i]] < np.float32(delta):
            for v in range(L):
                adm = v == 0 or opts[v]["k_skip"] == 0 or s1[i] >= np.float32(opts[v]["sim_gate"])
                if adm and rq[i, v] >= np.float32(delta):
                    assert rem[v] == 0, (i, v)
    assert a.size == rq.shape[0]


def check_e2e(ores, gpu, opts, quota):
    """A2: end-to-end decisions.  The GPU's decisions (A_i, C_i, pi_i from its own
    fp32 r and s_1) must equal the oracle's (from fp64) for every prompt whose
    oracle margins are all >= GAP_TOL; a differing prompt must be fragile (some
    r within GAP_TOL of delta, s_1 within GAP_TOL of a gate, or two options whose
    order flipped within GAP_TOL of each other).  If no prompt differs, the final
    assignments must be identical.  Returns the number of exempt prompts."""
    rep = oracle.assign(gpu["quality"].astype(np.float64), gpu["topk_score"][:, 0].astype(np.float64),
                        opts, quota)
    r, s1 = ores["rhat"], ores["topk_score"][:, 0]
    N, L = r.shape
    exempt = 0
    for i in range(N):
        same = (ores["adm"][i] == rep["adm"][i] and ores["cmp"][i] == rep["cmp"][i]
                and np.array_equal(ores["pref"][i], rep["pref"][i]))
        if same:
            continue
        exempt += 1
        near_delta = any(abs(r[i, v] - DELTA32) < GAP_TOL for v in range(1, L))
        near_gate = any(opts[v]["k_skip"] != 0 and abs(s1[i] - float(np.float32(opts[v]["sim_gate"]))) < GAP_TOL
                        for v in range(L))
        po, pg = list(ores["pref"][i]), list(rep["pref"][i])
        flips = [(u, v) for a_, u in enumerate(po) for b_, v in enumerate(po)
                 if a_ < b_ and u != 0xFF and v != 0xFF and u in pg and v in pg and pg.index(u) > pg.index(v)]
        near_tie = bool(flips) and all(abs(r[i, u] - r[i, v]) < GAP_TOL for u, v in flips)
        assert near_delta or near_gate or near_tie, (i, ores["pref"][i], rep["pref"][i])
    if exempt == 0:
        np.testing.assert_array_equal(gpu["option"], ores["option"])
        np.testing.assert_array_equal(gpu["status"], ores["status"])
    prefix = matched_prefix(ores, rep, gpu, opts, quota)
    full = bool(np.array_equal(gpu["option"], ores["option"]) and np.array_equal(gpu["status"], ores["status"]))
    report("A2", prompts=int(N), exempt=int(exempt), matched_prefix=prefix,
           matched_prefix_frac=round(prefix / max(1, N), 4), all_assignments_equal=full)
    return exempt


def fragile_mask(ores, opts, quota):
    """prompt i is fragile when, in the oracle's fp64 values,
    min(min_{v>=1} |r_iv - delta|, min_{v gated} |s_i1 - tau_v|,
        min_{v in A_i free at its turn, v != a_i} |r_{i,a_i} - r_iv|) < GAP_TOL,
    with "free at its turn" replayed along the oracle's priority order."""
    r, s1 = ores["rhat"], ores["topk_score"][:, 0]
    N, L = r.shape
    rem = np.array(quota, np.int64).copy()
    frag = np.zeros(N, bool)
    for i in ores["order"]:
        a = int(ores["option"][i])
        m = min([abs(r[i, v] - DELTA32) for v in range(1, L)] or [1.0])
        for v in range(L):
            if opts[v]["k_skip"] != 0:
                m = min(m, abs(s1[i] - float(np.float32(opts[v]["sim_gate"]))))
            if v != a and (ores["adm"][i] >> v) & 1 and rem[v] > 0:
                m = min(m, abs(r[i, a] - r[i, v]))
        frag[i] = m < GAP_TOL
        if not (ores["status"][i] & oracle.OVERFLOW):
            rem[a] -= 1
    return frag


def matched_prefix(ores, rep, gpu, opts, quota):
    """A2 matched prefix: the longest prefix of the oracle's priority order that (a)
    the GPU's own priority order (replayed from its fp32 values) shares and (b)
    holds no fragile prompt.  Along it both serial dictatorships see the same
    prompts with the same preference lists and quotas, so every assignment and
    status there must be identical (asserted).  Returns its length."""
    frag = fragile_mask(ores, opts, quota)
    oo, go = np.asarray(ores["order"]), np.asarray(rep["order"])
    t = 0
    while t < len(oo) and oo[t] == go[t] and not frag[oo[t]]:
        t += 1
    idx = oo[:t]
    np.testing.assert_array_equal(gpu["option"][idx], ores["option"][idx])
    np.testing.assert_array_equal(gpu["status"][idx], ores["status"][idx])
    return int(t)
