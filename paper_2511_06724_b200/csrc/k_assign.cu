// k_assign.cu -- K4: quota-capped assignment.
//
// Priority (|C_i| asc, i asc) by a stable block-wide counting sort (histogram,
// exclusive scan, match_any ranks), then serial dictatorship (P:289 F(v) as
// integer quotas; §4.3 redistribution; north_star "assign each prompt
// the highest-quality option that the allocator's per-option throughput quota
// still admits, with a fixed deterministic tie-break"):
//   rem <- c;  for i in priority order: a_i <- first v in pi_i with rem_v > 0;
//   rem_{a_i} -= 1;  none -> a_i = 0, OVERFLOW.
// "First v in pi_i with quota" = the admissible option with quota whose position
// in pi_i is smallest, so the walk is one warp with lane v holding rem_v and the
// position of v in pi_i: one REDUX.MIN picks the option, the chosen lane
// decrements.  The loop-carried chain is compare -> redux -> compare -> add.
// Each chunk of position rows is staged (in priority order) into shared memory by
// the whole block first, so the serial walk never waits on global memory.
#include "common.cuh"
#include "kernels.h"

namespace argus {

constexpr int ASSIGN_THREADS = 256;
constexpr int AW = ASSIGN_THREADS / 32;
constexpr int NB = 33;      // |C_i| in [1, 32]
constexpr int CH = 2048;    // prompts per staged chunk

size_t assign_smem_bytes(int max_batch, int L) {
  const int Lw = (L + 3) / 4 * 4;
  return sizeof(int32_t) * (size_t)max_batch + (size_t)CH * Lw + sizeof(uint32_t) * CH + CH;
}

__global__ void __launch_bounds__(ASSIGN_THREADS) k_assign(AssignArgs a) {
  extern __shared__ __align__(16) uint8_t smraw[];
  const int N = a.N, L = a.L;
  const int Lw = (L + 3) / 4 * 4;
  int32_t* order_s = reinterpret_cast<int32_t*>(smraw);                  // [N]
  uint8_t* rk_s = smraw + sizeof(int32_t) * (size_t)N;                   // [CH][Lw]
  uint32_t* cm_s = reinterpret_cast<uint32_t*>(rk_s + (size_t)CH * Lw);  // [CH]
  uint8_t* opt_s = reinterpret_cast<uint8_t*>(cm_s + CH);                 // [CH] (option | 0x80 overflow)
  __shared__ int32_t base[NB];
  __shared__ int32_t tot[NB];
  __shared__ int32_t wcnt[AW][NB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_wait();

  // ---- stable counting sort of prompts by |C_i|
  if (tid < NB) base[tid] = 0;
  __syncthreads();
  for (int i0 = 0; i0 < N; i0 += ASSIGN_THREADS) {  // warp-aggregated histogram
    const int i = i0 + tid;
    const int b = i < N ? a.ccount[i] : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, b);
    if (b >= 0 && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&base[b], __popc(peers));
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 33 bucket counts (one warp, shuffles)
    const int c0 = lane < NB ? base[lane] : 0;
    int x = c0;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, m);
      if (lane >= m) x += y;
    }
    const int tot31 = __shfl_sync(0xffffffffu, x, 31);
    if (lane < 32) base[lane] = x - c0;
    if (lane == 0) base[32] = tot31;  // bucket 32 (|C| = 32) starts after buckets 0..31
  }
  __syncthreads();
  for (int c0 = 0; c0 < N; c0 += ASSIGN_THREADS) {
    const int i = c0 + tid;
    const int b = i < N ? a.ccount[i] : -1;
    for (int x = tid; x < AW * NB; x += ASSIGN_THREADS) (&wcnt[0][0])[x] = 0;
    __syncthreads();
    const uint32_t peers = __match_any_sync(0xffffffffu, b);
    const int wrank = __popc(peers & ((1u << lane) - 1u));
    if (b >= 0 && wrank == 0) wcnt[warp][b] = __popc(peers);
    __syncthreads();
    if (tid < NB) {  // exclusive prefix over warps for bucket tid
      int run = 0;
#pragma unroll
      for (int w = 0; w < AW; ++w) { const int c = wcnt[w][tid]; wcnt[w][tid] = run; run += c; }
      tot[tid] = run;
    }
    __syncthreads();
    if (b >= 0) order_s[base[b] + wcnt[warp][b] + wrank] = i;
    __syncthreads();
    if (tid < NB) base[tid] += tot[tid];
  }
  __syncthreads();

  // ---- serial dictatorship over staged chunks
  int rem = lane < L ? a.quota[lane] : 0;       // warp 0 only
  bool any_overflow = false;
  for (int c0 = 0; c0 < N; c0 += CH) {
    const int n = min(CH, N - c0);
    // gather rows in priority order; 4 rows per thread in flight (the loads are independent)
    const int W = Lw / 4;
    const uint32_t* rk32 = reinterpret_cast<const uint32_t*>(a.rankof);
    for (int t0 = tid; t0 < n; t0 += 4 * ASSIGN_THREADS) {
      int ii[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u * ASSIGN_THREADS;
        ii[u] = t < n ? order_s[c0 + t] : -1;
      }
      uint32_t cm[4];
      uint32_t wd[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        cm[u] = ii[u] >= 0 ? __ldg(a.cmask + ii[u]) : 0u;
#pragma unroll
        for (int w = 0; w < 8; ++w) wd[u][w] = (ii[u] >= 0 && w < W) ? __ldg(rk32 + (int64_t)ii[u] * W + w) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u * ASSIGN_THREADS;
        if (t < n) {
          cm_s[t] = cm[u];
#pragma unroll
          for (int w = 0; w < 8; ++w)
            if (w < W) reinterpret_cast<uint32_t*>(rk_s + (size_t)t * Lw)[w] = wd[u][w];
        }
      }
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t nxt = lane < L ? rk_s[lane] : 0xFFu;
      for (int t = 0; t < n; ++t) {
        const uint32_t rk = nxt;
        if (t + 1 < n) nxt = lane < L ? rk_s[(size_t)(t + 1) * Lw + lane] : 0xFFu;
        const uint32_t cand = (rk != 0xFFu && rem > 0) ? rk : 0xFFu;
        const uint32_t best = __reduce_min_sync(0xffffffffu, cand);
        const bool mine = best != 0xFFu && cand == best;   // positions are distinct: one lane
        rem -= mine ? 1 : 0;
        const uint32_t who = __ballot_sync(0xffffffffu, mine);   // off the loop-carried chain
        if (lane == 0) opt_s[t] = who ? (uint8_t)(__ffs(who) - 1) : (uint8_t)0x80;
        any_overflow |= (who == 0);
      }
    }
    __syncthreads();
    for (int t = tid; t < n; t += ASSIGN_THREADS) {
      const int i = order_s[c0 + t];
      const int o = opt_s[t] & 0x7F;
      uint8_t st = a.status[i];
      if (opt_s[t] & 0x80) st |= 1u;                  // ARGUS_ST_OVERFLOW (option 0)
      if (!((cm_s[t] >> o) & 1u)) st |= 2u;           // ARGUS_ST_NONCOMPLIANT
      a.status[i] = st;
      a.option_out[i] = o;
    }
    __syncthreads();
  }
  if (tid == 0 && any_overflow) atomicOr(a.flags, FLAG_OVERFLOW);
  pdl_launch();
}

void launch_assign(const AssignArgs& a, cudaStream_t s) {
  const size_t smem = assign_smem_bytes(a.N > 0 ? a.N : 1, a.L);
  static size_t attr_set = 0;
  if (smem > attr_set) {
    cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = smem;
  }
  launch_pdl(k_assign, dim3(1), dim3(ASSIGN_THREADS), smem, s, a);
}

}  // namespace argus
