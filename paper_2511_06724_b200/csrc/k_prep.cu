// k_prep.cu -- K0 (cache insert) and K6 (query preparation), SURVEY §8(a) row A1.
//
// Both kernels round fp32 -> bf16 (RNE, the canonical tensor-core operand) and
// compute the fp32 inverse norm of the ROUNDED values, so the cosine of row A2
// is the cosine of the stored bf16 vectors (reading R2).  Warp per
// row; lanes stride the row in bf16x2 pairs; the sum of squares is reduced by
// xor-shuffles in a fixed order (deterministic, independent of sharding).
#include "common.cuh"
#include "kernels.h"

namespace argus {

__device__ __forceinline__ float row_to_bf16(const float* __restrict__ src, __nv_bfloat162* dst,
                                             int d, bool* bad) {
  const int lane = threadIdx.x & 31;
  const float2* s2 = reinterpret_cast<const float2*>(src);
  float acc = 0.f;
  bool b = false;
  for (int j = lane; j < d / 2; j += 32) {
    float2 v = s2[j];
    __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
    float2 r = __bfloat1622float2(h);
    b |= !isfinite(r.x) || !isfinite(r.y);
    acc = __fmaf_rn(r.x, r.x, acc);
    acc = __fmaf_rn(r.y, r.y, acc);
    if (dst) dst[j] = h;
  }
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, m));
  b = __any_sync(0xffffffffu, b);
  *bad = b || !(acc > 0.f) || !isfinite(acc);
  return acc;
}

// The same for a row that is already bf16 (argus_route_batch_bf16_dev): copied as is, the
// norm from the same values in the same order, so inv_q is bit-identical to what the fp32
// path computes for inputs that round to these bf16 values.
__device__ __forceinline__ float row_bf16(const __nv_bfloat162* __restrict__ src, __nv_bfloat162* dst, int d,
                                          bool* bad) {
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  bool b = false;
  for (int j = lane; j < d / 2; j += 32) {
    const __nv_bfloat162 h = src[j];
    const float2 r = __bfloat1622float2(h);
    b |= !isfinite(r.x) || !isfinite(r.y);
    acc = __fmaf_rn(r.x, r.x, acc);
    acc = __fmaf_rn(r.y, r.y, acc);
    dst[j] = h;
  }
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, m));
  b = __any_sync(0xffffffffu, b);
  *bad = b || !(acc > 0.f) || !isfinite(acc);
  return acc;
}

__global__ void k_insert_rows(const float* __restrict__ rows, int64_t n, int64_t g0, int d,
                              int rank, int world, int64_t cap, int dry, __nv_bfloat16* __restrict__ Cb,
                              float* __restrict__ inv_c, uint32_t* flags) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    const int64_t g = g0 + i;
    // cache position g mod capacity (ring eviction; g < capacity otherwise), striped:
    // rank pos % world holds it at slot pos / world (capacity % world == 0 when evicting)
    const int64_t pos = cap > 0 ? g % cap : g;
    if (!dry && pos % world != rank) continue;
    const int64_t slot = pos / world;
    bool bad;
    float ss = row_to_bf16(rows + i * d, dry ? nullptr : reinterpret_cast<__nv_bfloat162*>(Cb + slot * d), d, &bad);
    if ((threadIdx.x & 31) == 0) {
      if (!dry) inv_c[slot] = bad ? 0.f : __fdiv_rn(1.0f, __fsqrt_rn(ss));
      if (bad) atomicOr(flags, FLAG_INVALID_INPUT);
    }
  }
}

__global__ void k_prep_queries(const void* __restrict__ X, int in_bf16, int N, int n_pad, int d,
                               __nv_bfloat16* __restrict__ Xb, float* __restrict__ inv_q,
                               uint64_t* __restrict__ gthr, int32_t* __restrict__ ctr, uint32_t* flags,
                               QuotaVec quota, int32_t* __restrict__ quota_dev) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  pdl_wait();  // the previous batch's kernels may still read Xb / inv_q / the quotas
  if (blockIdx.x == 0 && threadIdx.x < CTR_WORDS) ctr[threadIdx.x] = 0;  // scan work / visit counters
  // multi-GPU: the root stages its quotas c_v next to the batch for the C-1 broadcast
  if (quota_dev && blockIdx.x == 0 && threadIdx.x < 32) quota_dev[threadIdx.x] = quota.v[threadIdx.x];
  if (warp >= n_pad) return;
  if (lane == 0) gthr[warp] = 0;  // the scan's shared per-prompt threshold starts empty
  if (warp >= N) {  // zero padding rows: score 0, never reported
    uint32_t* z = reinterpret_cast<uint32_t*>(Xb + (int64_t)warp * d);
    for (int j = lane; j < d / 2; j += 32) z[j] = 0u;
    if (lane == 0) inv_q[warp] = 0.f;
    return;
  }
  bool bad;
  __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(Xb + (int64_t)warp * d);
  const float ss = in_bf16 ? row_bf16(reinterpret_cast<const __nv_bfloat162*>(X) + (int64_t)warp * d / 2, dst, d, &bad)
                           : row_to_bf16(reinterpret_cast<const float*>(X) + (int64_t)warp * d, dst, d, &bad);
  if (lane == 0) {
    inv_q[warp] = bad ? 0.f : __fdiv_rn(1.0f, __fsqrt_rn(ss));
    if (bad) atomicOr(flags, FLAG_INVALID_INPUT);
  }
  pdl_launch();
}

__global__ void k_publish(uint32_t* flag, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}

void launch_publish(uint32_t* flag, uint32_t v, cudaStream_t s) { k_publish<<<1, 1, 0, s>>>(flag, v); }

void launch_insert_rows(const float* rows, int64_t n, int64_t g0, int32_t d, int32_t rank, int32_t world,
                        int64_t cap, bool dry, __nv_bfloat16* Cb, float* inv_c, uint32_t* flags, cudaStream_t s) {
  if (n <= 0) return;
  const int threads = 256;
  int64_t warps = n;
  int64_t blocks = (warps * 32 + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_insert_rows<<<(unsigned)blocks, threads, 0, s>>>(rows, n, g0, d, rank, world, cap, dry ? 1 : 0, Cb, inv_c,
                                                     flags);
}

void launch_prep_queries(const void* X, bool in_bf16, int32_t N, int32_t n_pad, int32_t d, __nv_bfloat16* Xb,
                         float* inv_q, uint64_t* gthr, int32_t* ctr, uint32_t* flags, cudaStream_t s, bool pdl,
                         const int32_t* quota, int32_t L, int32_t* quota_dev) {
  const int threads = 256;
  int blocks = (n_pad * 32 + threads - 1) / threads;
  QuotaVec qv{};
  for (int v = 0; v < 32; ++v) qv.v[v] = (quota && v < L) ? quota[v] : 0;
  launch_pdl_opt(pdl, k_prep_queries, dim3(blocks), dim3(threads), 0, s, X, (int)in_bf16, N, n_pad, d, Xb, inv_q, gthr,
                 ctr, flags,
                 qv, quota ? quota_dev : nullptr);
}

}  // namespace argus
