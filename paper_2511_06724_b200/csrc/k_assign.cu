// k_assign.cu -- K4: quota-capped assignment.
//
// Priority (|C_i| asc, i asc) by a stable block-wide counting sort (histogram,
// exclusive scan, match_any ranks), then serial dictatorship (P:289 F(v) as
// integer quotas; §4.3 redistribution; north_star "assign each prompt
// the highest-quality option that the allocator's per-option throughput quota
// still admits, with a fixed deterministic tie-break"):
//   rem <- c;  for i in priority order: a_i <- first v in pi_i with rem_v > 0;
//   rem_{a_i} -= 1;  none -> a_i = 0, OVERFLOW.
// The walk is one warp: lane r holds pi_i[r], lane v holds rem_v, the
// availability mask is a ballot, the choice is ffs(ballot).
#include "common.cuh"
#include "kernels.h"

namespace argus {

constexpr int ASSIGN_THREADS = 1024;
constexpr int NB = 33;  // |C_i| in [1, 32]

__global__ void __launch_bounds__(ASSIGN_THREADS) k_assign(AssignArgs a) {
  extern __shared__ int32_t order_s[];           // [N]
  __shared__ int32_t base[NB];
  __shared__ int32_t tot[NB];
  __shared__ int32_t wcnt[ASSIGN_THREADS / 32][NB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = a.N, L = a.L;

  // ---- stable counting sort of prompts by |C_i|
  if (tid < NB) base[tid] = 0;
  __syncthreads();
  for (int i = tid; i < N; i += ASSIGN_THREADS) atomicAdd(&base[a.ccount[i]], 1);
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int b = 0; b < NB; ++b) { const int c = base[b]; base[b] = run; run += c; }
  }
  __syncthreads();
  for (int c0 = 0; c0 < N; c0 += ASSIGN_THREADS) {
    const int i = c0 + tid;
    const int b = i < N ? a.ccount[i] : -1;
    for (int x = tid; x < (ASSIGN_THREADS / 32) * NB; x += ASSIGN_THREADS) (&wcnt[0][0])[x] = 0;
    __syncthreads();
    const uint32_t peers = __match_any_sync(0xffffffffu, b);
    const int wrank = __popc(peers & ((1u << lane) - 1u));
    if (b >= 0 && wrank == 0) wcnt[warp][b] = __popc(peers);
    __syncthreads();
    if (tid < NB) {  // exclusive prefix over warps for bucket tid
      int run = 0;
      for (int w = 0; w < ASSIGN_THREADS / 32; ++w) { const int c = wcnt[w][tid]; wcnt[w][tid] = run; run += c; }
      tot[tid] = run;
    }
    __syncthreads();
    if (b >= 0) order_s[base[b] + wcnt[warp][b] + wrank] = i;
    __syncthreads();
    if (tid < NB) base[tid] += tot[tid];  // advance bucket bases by this chunk's counts
    __syncthreads();
  }

  // ---- serial dictatorship, one warp
  if (warp != 0) return;
  int rem = lane < L ? a.quota[lane] : 0;
  uint32_t avail = __ballot_sync(0xffffffffu, rem > 0);
  bool any_overflow = false;
  int nxt_i = N > 0 ? order_s[0] : 0;
  uint32_t nxt_pv = (N > 0 && lane < L) ? a.pref[(int64_t)nxt_i * L + lane] : 0xFFu;
  for (int t = 0; t < N; ++t) {
    const int i = nxt_i;
    const uint32_t pv = nxt_pv;
    if (t + 1 < N) {  // prefetch the next prompt's preference row
      nxt_i = order_s[t + 1];
      nxt_pv = lane < L ? a.pref[(int64_t)nxt_i * L + lane] : 0xFFu;
    }
    const bool ok = pv != 0xFFu && ((avail >> pv) & 1u);
    const uint32_t b = __ballot_sync(0xffffffffu, ok);
    int opt = 0;
    bool ovf = (b == 0);
    if (!ovf) {
      opt = (int)__shfl_sync(0xffffffffu, pv, __ffs(b) - 1);
      if (lane == opt) --rem;
      avail = __ballot_sync(0xffffffffu, rem > 0);
    }
    if (lane == 0) {
      const uint32_t cm = a.cmask[i];
      uint8_t st = a.status[i];
      if (ovf) st |= 1u;                      // ARGUS_ST_OVERFLOW
      if (!((cm >> opt) & 1u)) st |= 2u;      // ARGUS_ST_NONCOMPLIANT
      a.status[i] = st;
      a.option_out[i] = opt;
    }
    any_overflow |= ovf;
  }
  if (lane == 0 && any_overflow) atomicOr(a.flags, FLAG_OVERFLOW);
}

void launch_assign(const AssignArgs& a, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 4);
    attr_set = true;
  }
  k_assign<<<1, ASSIGN_THREADS, sizeof(int32_t) * (a.N > 0 ? a.N : 1), s>>>(a);
}

}  // namespace argus
