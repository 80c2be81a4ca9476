// control.cu -- host-side control plane of libargus: the
// Optimized Distribution Aligner that turns the affinity histogram H and the
// allocator's load shares F into the PASM (Algorithm 1), the
// Eq. 2 expected degradation, and the Eq. 1 allocator.
//
// These run once per re-solve tick ("Every minute"), off the per-batch
// path, so they are plain host code; their outputs feed the per-batch kernels
// (quotas c_v by largest remainder for the serial-dictatorship policy, the PASM
// cumulative table for the sampling policy; see argus.cu / k_tail.cu).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "argus.h"

namespace {

constexpr int LMAX = 32;

bool finite_nonneg(const double* x, int n, double* sum) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!std::isfinite(x[i]) || x[i] < 0.0) return false;
    s += x[i];
  }
  *sum = s;
  return s > 0.0;
}

}  // namespace

extern "C" {

// Algorithm 1.  Levels are ordered slow (0) -> fast (L-1).  The flow is simulated
// with per-origin bookkeeping: at[o][v] = share of origin o's mass sitting at level
// v.  A step that moves `amt` out of level a takes the same fraction amt / tot(a)
// of every origin present at a ("the probability is computed using a fraction of
// shift divided by the total at v_i"), so an origin's final distribution is
// the paper's chain product of step probabilities (DESIGN R19).
int argus_oda_pasm(const double* H, const double* F, int32_t L, double* pasm_out) {
  if (!H || !F || !pasm_out || L < 1 || L > LMAX) return ARGUS_E_INVALID;
  double sh = 0.0, sf = 0.0;
  if (!finite_nonneg(H, L, &sh) || !finite_nonneg(F, L, &sf)) return ARGUS_E_INVALID;
  double h[LMAX], f[LMAX], h0[LMAX];
  double at[LMAX][LMAX];
  for (int v = 0; v < L; ++v) {
    h[v] = h0[v] = H[v] / sh;  // both as distributions (H may be counts)
    f[v] = F[v] / sf;
    for (int u = 0; u < L; ++u) at[v][u] = (u == v) ? h[v] : 0.0;
  }
  auto flow = [&](int from, int to, double amt) {
    const double tot = h[from];
    if (!(amt > 0.0) || !(tot > 0.0)) return;
    const double frac = amt / tot;
    for (int o = 0; o < L; ++o) {
      const double m = at[o][from] * frac;
      at[o][from] -= m;
      at[o][to] += m;
    }
    h[from] -= amt;
    h[to] += amt;
  };
  for (int i = L - 1; i >= 0; --i) {      // line 2: right to left (fastest first)
    if (h[i] > f[i]) {                     // line 3: oversubscribed -> the next slower level
      if (i > 0) flow(i, i - 1, h[i] - f[i]);
    } else {                               // lines 8-16: fill the gap from slower levels,
      for (int m = 1; h[i] < f[i] && i - m >= 0; ++m) {   // nearest first
        const double need = f[i] - h[i];
        flow(i - m, i, h[i - m] < need ? h[i - m] : need);
      }
    }
  }
  for (int o = 0; o < L; ++o)
    for (int v = 0; v < L; ++v)
      pasm_out[o * L + v] = h0[o] > 0.0 ? at[o][v] / h0[o] : (o == v ? 1.0 : 0.0);
  return ARGUS_OK;
}

// Eq. 2: D_Q = sum_i sum_{j: P_th(j) > P_th(i)} P(j|i) H(i) D(j, i); D row-major [j][i].
int argus_pasm_degradation(const double* pasm, const double* H, const float* p_th, const double* D, int32_t L,
                           double* dq_out) {
  if (!pasm || !H || !p_th || !D || !dq_out || L < 1 || L > LMAX) return ARGUS_E_INVALID;
  double dq = 0.0;
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < L; ++j)
      if (p_th[j] > p_th[i]) dq += pasm[i * L + j] * H[i] * D[j * L + i];
  *dq_out = dq;
  return ARGUS_OK;
}

// Eq. 1 for homogeneous workers.  For a fixed number of workers per level the best
// integer loads fill levels in decreasing profiled quality Q (a fractional knapsack
// with unit weights, exact for integer capacities n_v * P_th(v)); the composition is
// chosen by dynamic programming over (levels taken in that order, workers used,
// load placed), which covers every composition without enumerating them.
int argus_solve_allocation(int32_t W, int32_t n_workers, int32_t L, const double* Q, const float* p_th,
                           int32_t* level_out, int32_t* load_out, double* F_out, double* objective_out,
                           int32_t* feasible_out) {
  if (W < 0 || n_workers < 1 || n_workers > 1024 || L < 1 || L > LMAX || !Q || !p_th) return ARGUS_E_INVALID;
  if ((int64_t)(L + 1) * (n_workers + 1) * ((int64_t)W + 1) > ((int64_t)1 << 24)) return ARGUS_E_INVALID;  // DP table
  int cap[LMAX];
  for (int v = 0; v < L; ++v) {
    if (!std::isfinite(Q[v]) || !std::isfinite(p_th[v]) || p_th[v] < 0.f) return ARGUS_E_INVALID;
    cap[v] = (int)std::floor(p_th[v]);  // integer QPM per worker ("integer decision variables")
  }
  std::vector<int> nv(L, 0), Y(L, 0);
  int feasible = 1;
  if (W == 0) {
    nv[0] = n_workers;  // no load: every worker on the slowest (highest quality) level
  } else {
    int fast = 0;
    for (int v = 1; v < L; ++v)
      if (cap[v] >= cap[fast]) fast = v;
    if ((int64_t)cap[fast] * n_workers < W) {  // above every plan's capacity: saturate
      feasible = 0;
      nv[fast] = n_workers;
      Y[fast] = cap[fast] * n_workers;
    } else {
      // levels in decreasing Q (ties: slower first, then lower index)
      int ord[LMAX];
      for (int v = 0; v < L; ++v) ord[v] = v;
      for (int a = 1; a < L; ++a)
        for (int b = a; b > 0; --b) {
          const int x = ord[b - 1], y = ord[b];
          const bool swap = Q[y] > Q[x] || (Q[y] == Q[x] && (p_th[y] < p_th[x] || (p_th[y] == p_th[x] && y < x)));
          if (swap) std::swap(ord[b - 1], ord[b]);
        }
      const int NW = n_workers, WW = W;
      const double NEG = -INFINITY;
      // best[t][j][y]: max sum Q*Y over the first t levels of `ord`, j workers, y placed
      std::vector<double> best((size_t)(L + 1) * (NW + 1) * (WW + 1), NEG);
      std::vector<int16_t> pick((size_t)(L + 1) * (NW + 1) * (WW + 1), -1);   // workers given to level t-1
      std::vector<int32_t> prev((size_t)(L + 1) * (NW + 1) * (WW + 1), -1);   // load placed before it
      auto at = [&](int t, int j, int y) { return ((size_t)t * (NW + 1) + j) * (WW + 1) + y; };
      best[at(0, 0, 0)] = 0.0;
      for (int t = 0; t < L; ++t) {
        const int v = ord[t];
        for (int j = 0; j <= NW; ++j)
          for (int y = 0; y <= WW; ++y) {
            const double b0 = best[at(t, j, y)];
            if (b0 == NEG) continue;
            for (int n = 0; j + n <= NW; ++n) {
              const int64_t room = (int64_t)n * cap[v];
              const int add = (int)(room < WW - y ? room : WW - y);
              const double val = b0 + Q[v] * add;
              const size_t dst = at(t + 1, j + n, y + add);
              if (val > best[dst]) {
                best[dst] = val;
                pick[dst] = (int16_t)n;
                prev[dst] = y;
              }
              if (y + add == WW && n > 0) break;  // more workers add no load
            }
          }
      }
      int bj = -1;
      for (int j = 0; j <= NW; ++j)
        if (best[at(L, j, WW)] != NEG && (bj < 0 || best[at(L, j, WW)] > best[at(L, bj, WW)])) bj = j;
      if (bj < 0) return ARGUS_E_INVALID;  // unreachable: capacity was checked
      int j = bj, y = WW;
      for (int t = L; t > 0; --t) {  // walk the choices back
        const size_t c = at(t, j, y);
        const int n = pick[c], yprev = prev[c];
        nv[ord[t - 1]] = n;
        Y[ord[t - 1]] = y - yprev;
        j -= n;
        y = yprev;
      }
      nv[ord[0]] += n_workers - bj;  // spare workers run the top-quality level, idle
    }
  }
  // per-worker plan: workers take levels in ascending order; a level's load fills
  // its workers one after another up to P_th
  double num = 0.0;
  int w = 0;
  for (int v = 0; v < L; ++v) {
    int left = Y[v];
    for (int c = 0; c < nv[v]; ++c, ++w) {
      const int y = left < cap[v] ? left : cap[v];
      if (level_out) level_out[w] = v;
      if (load_out) load_out[w] = y;
      left -= y;
    }
    num += Q[v] * Y[v];
  }
  int64_t served = 0;
  for (int v = 0; v < L; ++v) served += Y[v];
  if (F_out)
    for (int v = 0; v < L; ++v) F_out[v] = served > 0 ? (double)Y[v] / (double)served : (v == 0 ? 1.0 : 0.0);
  if (objective_out) *objective_out = !feasible ? Q[std::max_element(Y.begin(), Y.end()) - Y.begin()]
                                                : (served > 0 ? num / (double)served : 0.0);
  if (feasible_out) *feasible_out = feasible;
  return ARGUS_OK;
}

}  // extern "C"
