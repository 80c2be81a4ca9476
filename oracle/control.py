"""ARGUS control-plane oracle -- TEST INFRASTRUCTURE ONLY.

Plain Python / numpy fp64 implementations, written from PAPER.md, of the steps
around the routing path that SURVEY.md §8(f) ranks "next":

  F1  optimal option o_i ............ P:140-142 §3 ("Optimal Model: ... the one that
                                        generates an optimal quality image with the
                                        lowest inference time")
      ODA -> PASM ................... P:313-343 §4.3, Algorithm 1 + the chain rule
                                        P(v'_j|v_i) = P(v'_j|v'_{j-1}) ... P(v'_{j-n}|v_i)
      Eq. 2 expected degradation .... P:307
      PASM sampling ................. P:299 ("probabilistically redistributed")
                                        counter-based Philox4x32-10 (Salmon et al., SC'11)
  F2  allocator (Eq. 1) ............. P:279-289 §4.2, brute force over worker
                                        assignments and integer loads
  F3  worker selector (Eq. 3) ....... P:353-357 §4.4, w = argmin_w R_queue,w * t_proc

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module.  It shares no code with paper_2511_06724_b200/ (which never imports it).
Readings of the paper taken here are DESIGN.md R18-R24.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

M32 = 0xFFFFFFFF


# ----------------------------------------------------------------------------- F1
def optimal_option(rhat_row, adm_mask, p_th, delta=0.9):
    """o_i: among the compliant options C_i = {v in A_i : r_v >= delta}
    the fastest (largest P_th); equal P_th -> higher r (S:79 breaks latency ties by
    quality), then lower v (DESIGN R18).  Option 0 (r := 1) is always compliant.
    delta is compared as the float32 value (DESIGN R6)."""
    d64 = float(np.float32(delta))
    best = None
    for v in range(len(p_th)):
        if not (adm_mask >> v) & 1:
            continue
        r = float(rhat_row[v])
        if r < d64:
            continue
        key = (float(p_th[v]), r, -v)
        if best is None or key > best[0]:
            best = (key, v)
    return best[1]


def oda_pasm(H, F):
    """Algorithm 1 -> PASM P[i][j] = P(v'_j | v_i), rows = optimal option
    (source), columns = assigned option (target); levels ordered slow (0) -> fast.

    Mass is tracked per origin (DESIGN R19): every step moves `amount` from node a
    to node b, and the moved mass is made of each origin's share of what sits at a
    at that moment ("a fraction of shift divided by the total at v_i").  The
    PASM row of an origin is where its mass ends up, which is the paper's chain
    composition of step probabilities.  Lines refer to Algorithm 1."""
    H = [float(x) for x in H]
    F = [float(x) for x in F]
    n = len(H)
    assert len(F) == n and n >= 1
    # mass[o][node]: mass of origin o currently at node
    mass = [[0.0] * n for _ in range(n)]
    for o in range(n):
        mass[o][o] = H[o]
    h = list(H)  # line 1: H (current totals per node)

    def move(a, b, amount):
        tot = h[a]
        if amount <= 0.0 or tot <= 0.0:
            return
        frac = amount / tot
        for o in range(n):
            m = mass[o][a] * frac
            mass[o][a] -= m
            mass[o][b] += m
        h[a] -= amount
        h[b] += amount

    for i in range(n - 1, -1, -1):          # line 2: fastest -> slowest
        if h[i] > F[i]:                      # line 3
            if i > 0:                        # lines 4-6: excess to the immediately slower level
                move(i, i - 1, h[i] - F[i])
        else:
            m = 1
            while h[i] < F[i] and i - m >= 0:   # lines 8-16: pull from progressively slower levels
                shift = min(h[i - m], F[i] - h[i])   # line 10
                move(i - m, i, shift)                 # lines 11-14
                m += 1
    P = np.zeros((n, n))
    for o in range(n):
        if H[o] > 0.0:
            for j in range(n):
                P[o][j] = mass[o][j] / H[o]
        else:
            P[o][o] = 1.0      # an option nobody prefers: identity row (never sampled)
    return P


def eq2_degradation(P, H, p_th, D):
    """Eq. 2: D_Q = sum_i sum_{j : P_th(v'_j) > P_th(v_i)} P(v'_j|v_i) H(v_i) D(v'_j, v_i).
    D[j][i] = degradation of serving a v_i-optimal prompt on v'_j."""
    n = len(H)
    dq = 0.0
    for i in range(n):
        for j in range(n):
            if p_th[j] > p_th[i]:
                dq += P[i][j] * H[i] * D[j][i]
    return dq


def _mulhilo(a, b):
    p = a * b
    return (p >> 32) & M32, p & M32


def philox4x32_10(ctr, key):
    """Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy
    as 1, 2, 3", SC'11): 10 rounds of the 4x32 S-box with multipliers 0xD2511F53,
    0xCD9E8D57 and Weyl key increments 0x9E3779B9, 0xBB67AE85."""
    c0, c1, c2, c3 = [x & M32 for x in ctr]
    k0, k1 = [x & M32 for x in key]
    for r in range(10):
        if r > 0:
            k0 = (k0 + 0x9E3779B9) & M32
            k1 = (k1 + 0xBB67AE85) & M32
        hi0, lo0 = _mulhilo(0xD2511F53, c0)
        hi1, lo1 = _mulhilo(0xCD9E8D57, c2)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def uniform24(seed, batch_seq, i):
    """u_i = (x0 >> 8) * 2^-24 in [0, 1), exact in float32, with
    (x0..x3) = Philox4x32-10(counter = (i, batch_seq lo, batch_seq hi, 0),
    key = (seed lo, seed hi)) (DESIGN R20)."""
    x0 = philox4x32_10((i, batch_seq & M32, (batch_seq >> 32) & M32, 0), (seed & M32, (seed >> 32) & M32))[0]
    return np.float32((x0 >> 8) * (1.0 / 16777216.0))


def pasm_cdf32(P):
    """Per row, the float32 running sums cdf[o][j] = fl32(cdf[o][j-1] + fl32(P[o][j]))
    (the sampling decision is taken in float32 on both sides, DESIGN R20)."""
    n = P.shape[0]
    cdf = np.zeros((n, n), np.float32)
    for o in range(n):
        c = np.float32(0.0)
        for j in range(n):
            c = np.float32(c + np.float32(P[o][j]))
            cdf[o][j] = c
    return cdf


def pasm_sample(P_row, cdf_row, u):
    """First j with u < cdf[j]; if rounding leaves u >= cdf[n-1], the last j with
    P[j] > 0."""
    for j in range(len(cdf_row)):
        if u < cdf_row[j]:
            return j
    return max(j for j in range(len(P_row)) if np.float32(P_row[j]) > 0)


def pasm_assign(rhat, s1, opts, P, seed, batch_seq, delta=0.9):
    """F1 per batch: o_i = optimal option, a_i ~ PASM row o_i (counter-based), then
    the gate: an inadmissible a_i falls back to the nearest slower admissible option
    (option 0 is always admissible; DESIGN R21).  Returns dict(option, optimal,
    status) with status bits NONCOMPLIANT (2) and GATED_ALL (4) as in O10."""
    rhat = np.asarray(rhat, np.float64)
    s1 = np.asarray(s1, np.float64)
    N, L = rhat.shape
    p_th = [o["p_th_qpm"] for o in opts]
    d64 = float(np.float32(delta))
    cdf = pasm_cdf32(np.asarray(P, np.float64))
    any_gate = any(o["k_skip"] != 0 for o in opts)
    out_a = np.zeros(N, np.int32)
    out_o = np.zeros(N, np.int32)
    st = np.zeros(N, np.uint8)
    for i in range(N):
        adm = 0
        npass = 0
        for v, o in enumerate(opts):
            g_ok = s1[i] >= float(np.float32(o["sim_gate"]))
            if v == 0 or o["k_skip"] == 0 or g_ok:
                adm |= 1 << v
            if o["k_skip"] != 0 and g_ok:
                npass += 1
        oi = optimal_option(rhat[i], adm, p_th, delta)
        a = pasm_sample(P[oi], cdf[oi], uniform24(seed, batch_seq, i))
        while not (adm >> a) & 1:
            a -= 1
        out_o[i] = oi
        out_a[i] = a
        s = 4 if (any_gate and npass == 0) else 0
        if rhat[i][a] < d64:
            s |= 2
        st[i] = s
    return dict(option=out_a, optimal=out_o, status=st)


def affinity_histogram(optimal_history, L, window=1000):
    """H(v) over the last `window` prompts' optimal options ("a look-back
    window of 1000 prompts"), as counts."""
    h = np.zeros(L, np.int64)
    for o in list(optimal_history)[-window:]:
        h[o] += 1
    return h


# ----------------------------------------------------------------------------- F3
def select_workers(assigned, worker_option, t_proc, queue):
    """Eq. 3 for the prompts of a batch in arrival order: prompt i (assigned
    option a_i) goes to w = argmin over workers hosting a_i of R_queue,w * t_proc,w,
    the product taken in float32, ties to the lowest worker id; R_queue,w
    then grows by one (DESIGN R22).  No worker hosts a_i -> -1.  Returns
    (worker [N], queue after the batch)."""
    q = [int(x) for x in queue]
    out = np.full(len(assigned), -1, np.int32)
    for i, a in enumerate(assigned):
        best = None
        for w in range(len(worker_option)):
            if worker_option[w] != a:
                continue
            cost = np.float32(np.float32(q[w]) * np.float32(t_proc[w]))
            if best is None or cost < best[0]:
                best = (cost, w)
        if best is not None:
            out[i] = best[1]
            q[best[1]] += 1
    return out, np.array(q, np.int32)


# ----------------------------------------------------------------------------- F2
def allocation_bruteforce(W, n_workers, Q, P_th):
    """Eq. 1 by exhaustive search over every assignment of levels to
    workers (x_{v,w} in {0,1}, sum_v x_{v,w} <= 1; -1 = idle) and every integer
    per-level load vector Y (Y_v = sum of y_w over the workers at v, 0 <= Y_v <=
    n_v * P_th(v), sum_v Y_v = W; any such Y splits over the n_v workers within
    y_w <= P_th(v)).  Objective sum_v Q_v F(v) with F(v) = Y_v / W, evaluated as
    (sum_{v ascending} Q_v * Y_v) / W in double (DESIGN R23).  Tiny instances only.

    Returns dict(objective, feasible, optimal_Y = set of every maximising Y tuple).
    W > capacity of every assignment -> feasible False, objective of the all-fastest
    saturated plan, optimal_Y = {that plan's Y}.  W = 0 -> objective 0, Y = 0."""
    Lv = len(Q)
    P_th = [int(p) for p in P_th]
    if W == 0:
        return dict(objective=0.0, feasible=True, optimal_Y={tuple([0] * Lv)})
    best_obj, best_Y = None, set()
    seen = set()
    for levels in itertools.product(range(-1, Lv), repeat=n_workers):
        n_v = tuple(sum(1 for x in levels if x == v) for v in range(Lv))
        if n_v in seen:
            continue
        seen.add(n_v)
        caps = [n_v[v] * P_th[v] for v in range(Lv)]
        if sum(caps) < W:
            continue
        for Y in itertools.product(*[range(0, c + 1) for c in caps]):
            if sum(Y) != W:
                continue
            num = 0.0
            for v in range(Lv):
                num += Q[v] * Y[v]
            obj = num / W
            if best_obj is None or obj > best_obj:
                best_obj, best_Y = obj, {Y}
            elif obj == best_obj:
                best_Y.add(Y)
    if best_obj is None:
        fast = max(range(Lv), key=lambda v: (P_th[v], v))
        Y = [0] * Lv
        Y[fast] = n_workers * P_th[fast]
        return dict(objective=float(Q[fast]), feasible=False, optimal_Y={tuple(Y)})
    return dict(objective=best_obj, feasible=True, optimal_Y=best_Y)


def min_degradation_transport(H, F, p_th, D):
    """Minimum of Eq. 2 over ALL transport plans T >= 0 with row sums H and column
    sums F (the plan need not come from Algorithm 1), by linear programming
    (scipy.optimize.linprog, HiGHS).  Used to pin ODA's optimality claim."""
    from scipy.optimize import linprog
    n = len(H)
    c = np.zeros(n * n)
    for i in range(n):
        for j in range(n):
            if p_th[j] > p_th[i]:
                c[i * n + j] = D[j][i]
    A_eq, b_eq = [], []
    for i in range(n):
        row = np.zeros(n * n)
        row[i * n:(i + 1) * n] = 1
        A_eq.append(row)
        b_eq.append(H[i])
    for j in range(n):
        col = np.zeros(n * n)
        col[j::n] = 1
        A_eq.append(col)
        b_eq.append(F[j])
    res = linprog(c, A_eq=np.array(A_eq), b_eq=np.array(b_eq), bounds=(0, None), method="highs")
    assert res.status == 0, res.message
    return float(res.fun)


def superlinear_D(n, p=2.0):
    """D(v'_j, v_i) = (j - i)^p for faster targets (index gap; "D increases
    super-linearly with the model speed gap"), 0 otherwise."""
    D = np.zeros((n, n))
    for j in range(n):
        for i in range(n):
            if j > i:
                D[j][i] = float(j - i) ** p
    return D


__all__ = [n for n in dir() if not n.startswith("_")]
_ = math
