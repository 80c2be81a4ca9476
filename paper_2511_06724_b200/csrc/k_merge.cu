// k_merge.cu -- K5: merge per-range / per-shard top-k candidate lists
// (SURVEY §8(a) row A3, steps 5-6).  Keys are unique (the global id is in the
// low word), so the merged result is independent of the order of the inputs:
// the same keys come out whether the cache was scanned by 1 CTA range or 296,
// on 1 GPU or 8 (G-invariance).
//
// One CTA of 4 warps per prompt: each warp folds a quarter of the P*k candidate
// keys into per-lane register lists (loads batched 8 deep so the L2 latency
// overlaps), reduces them to its top-k, and warp 0 merges the 4 warp lists.
#include "common.cuh"
#include "kernels.h"

namespace argus {

constexpr int MERGE_WARPS = 4;

template <int KMAX>
__global__ void __launch_bounds__(MERGE_WARPS * 32) k_merge_topk(const uint64_t* __restrict__ in, int P, int N, int k,
                                                               uint64_t* __restrict__ keys_out,
                                                               uint32_t* __restrict__ idx_out,
                                                               float* __restrict__ score_out) {
  const int i = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ uint64_t wl[MERGE_WARPS][KMAX];
  pdl_wait();
  TopList<KMAX> l;
  l.clear();
  const int total = P * k;
  const int per = (total + MERGE_WARPS - 1) / MERGE_WARPS;
  const int e0 = warp * per, e1 = min(total, e0 + per);
  constexpr int B = 8;
  for (int e = e0 + lane; e < e1; e += 32 * B) {
    uint64_t buf[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int ee = e + u * 32;
      uint64_t key = 0;
      if (ee < e1) {
        const int p = ee / k, t = ee - p * k;
        key = __ldg(reinterpret_cast<const unsigned long long*>(in) + ((int64_t)p * N + i) * k + t);
      }
      buf[u] = key;
    }
#pragma unroll
    for (int u = 0; u < B; ++u) l.insert(buf[u]);
  }
  warp_merge_topk<KMAX>(l, k, wl[warp]);
  __syncthreads();
  pdl_launch();
  if (warp == 0) {
    TopList<KMAX> m;
    m.clear();
    if (lane < MERGE_WARPS * k) m.insert(wl[lane / k][lane % k]);
    __shared__ uint64_t out_s[KMAX];
    warp_merge_topk<KMAX>(m, k, out_s);
    __syncwarp();
    if (lane < k) {
      const uint64_t key = out_s[lane];
      if (keys_out) keys_out[(int64_t)i * k + lane] = key;
      if (idx_out) idx_out[(int64_t)i * k + lane] = key_id(key);
      if (score_out) score_out[(int64_t)i * k + lane] = key_score(key);
    }
  }
}

void launch_merge_topk(const uint64_t* in, int32_t P, int32_t N, int32_t k, uint64_t* keys_out,
                       uint32_t* idx_out, float* score_out, cudaStream_t s) {
  if (k <= 4)
    launch_pdl(k_merge_topk<4>, dim3(N), dim3(MERGE_WARPS * 32), 0, s, in, P, N, k, keys_out, idx_out, score_out);
  else
    launch_pdl(k_merge_topk<8>, dim3(N), dim3(MERGE_WARPS * 32), 0, s, in, P, N, k, keys_out, idx_out, score_out);
}

}  // namespace argus
