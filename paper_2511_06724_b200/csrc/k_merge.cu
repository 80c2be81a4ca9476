// k_merge.cu -- K5: merge per-range / per-shard top-k candidate lists
// (SURVEY §8(a) row A3, steps 5-6).  Keys are unique (the global id is in the
// low word), so the merged result is independent of the order of the inputs:
// the same keys come out whether the cache was scanned by 1 CTA range or 148,
// on 1 GPU or 8 (G-invariance).
#include "common.cuh"
#include "kernels.h"

namespace argus {

template <int KMAX>
__global__ void k_merge_topk(const uint64_t* __restrict__ in, int P, int N, int k,
                             uint64_t* __restrict__ keys_out, uint32_t* __restrict__ idx_out,
                             float* __restrict__ score_out) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= N) return;
  TopList<KMAX> l;
  l.clear();
  const int total = P * k;
  for (int e = lane; e < total; e += 32) {
    const int p = e / k, t = e - p * k;
    l.insert(in[((int64_t)p * N + i) * k + t]);
  }
  __shared__ uint64_t out_s[8][KMAX];
  uint64_t* o = out_s[(threadIdx.x >> 5) & 7];
  warp_merge_topk<KMAX>(l, k, o);
  __syncwarp();
  if (lane < k) {
    const uint64_t key = o[lane];
    if (keys_out) keys_out[(int64_t)i * k + lane] = key;
    if (idx_out) idx_out[(int64_t)i * k + lane] = key_id(key);
    if (score_out) score_out[(int64_t)i * k + lane] = key_score(key);
  }
}

void launch_merge_topk(const uint64_t* in, int32_t P, int32_t N, int32_t k, uint64_t* keys_out,
                       uint32_t* idx_out, float* score_out, cudaStream_t s) {
  const int threads = 256;  // 8 warps = 8 prompts per block
  const int blocks = (N + 7) / 8;
  if (k <= 4)
    k_merge_topk<4><<<blocks, threads, 0, s>>>(in, P, N, k, keys_out, idx_out, score_out);
  else
    k_merge_topk<8><<<blocks, threads, 0, s>>>(in, P, N, k, keys_out, idx_out, score_out);
}

}  // namespace argus
