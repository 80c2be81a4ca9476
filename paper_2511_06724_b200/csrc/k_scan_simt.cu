// k_scan_simt.cu -- K1 v0: a plain SIMT cosine scan with the fused top-k
// epilogue (SURVEY §8(a) rows A2+A3).  First correct CUDA path; superseded by
// the tcgen05/TMA kernel for the benchmarked sizes.
//
// CTA = 256 threads x 8 prompts (prompt block in shared memory as fp32) x one
// contiguous range of cache rows.  Thread = cache row (strided); each thread
// keeps a register top-k per prompt; every warp then merges its 32 lists and
// writes one partial list per (range, warp).  Scores never leave registers.
#include "common.cuh"
#include "kernels.h"

namespace argus {

constexpr int SIMT_PB = 8;
constexpr int SIMT_THREADS = 256;
constexpr int SIMT_WARPS = SIMT_THREADS / 32;
constexpr int SIMT_MAX_RANGES = 18;  // P = ranges * warps <= 148

template <int KMAX>
__global__ void __launch_bounds__(SIMT_THREADS) k_scan_simt(ScanArgs a, int ranges, int64_t rows_per_range) {
  extern __shared__ float xs[];  // [d][PB]
  const int d = a.d;
  const int pb = blockIdx.y;
  const int r = blockIdx.x;
  const int i0 = pb * SIMT_PB;
  for (int idx = threadIdx.x; idx < d * SIMT_PB; idx += SIMT_THREADS) {
    const int p = idx / d, l = idx - p * d;
    xs[l * SIMT_PB + p] = (i0 + p < a.n_pad) ? __bfloat162float(a.Xb[(int64_t)(i0 + p) * d + l]) : 0.f;
  }
  __syncthreads();
  float iq[SIMT_PB];
#pragma unroll
  for (int p = 0; p < SIMT_PB; ++p) iq[p] = (i0 + p < a.N) ? a.inv_q[i0 + p] : 0.f;
  TopList<KMAX> tl[SIMT_PB];
#pragma unroll
  for (int p = 0; p < SIMT_PB; ++p) tl[p].clear();

  const int64_t j0 = (int64_t)r * rows_per_range;
  const int64_t j1 = min(a.m_local, j0 + rows_per_range);
  for (int64_t j = j0 + threadIdx.x; j < j1; j += SIMT_THREADS) {
    float acc[SIMT_PB];
#pragma unroll
    for (int p = 0; p < SIMT_PB; ++p) acc[p] = 0.f;
    const uint4* row = reinterpret_cast<const uint4*>(a.Cb + j * d);
    for (int l8 = 0; l8 < d / 8; ++l8) {
      uint4 u = row[l8];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 c = __bfloat1622float2(h[q]);
        const int l = l8 * 8 + q * 2;
        const float4 xa0 = *reinterpret_cast<const float4*>(xs + l * SIMT_PB);
        const float4 xa1 = *reinterpret_cast<const float4*>(xs + l * SIMT_PB + 4);
        const float4 xb0 = *reinterpret_cast<const float4*>(xs + (l + 1) * SIMT_PB);
        const float4 xb1 = *reinterpret_cast<const float4*>(xs + (l + 1) * SIMT_PB + 4);
        acc[0] = __fmaf_rn(c.x, xa0.x, acc[0]); acc[0] = __fmaf_rn(c.y, xb0.x, acc[0]);
        acc[1] = __fmaf_rn(c.x, xa0.y, acc[1]); acc[1] = __fmaf_rn(c.y, xb0.y, acc[1]);
        acc[2] = __fmaf_rn(c.x, xa0.z, acc[2]); acc[2] = __fmaf_rn(c.y, xb0.z, acc[2]);
        acc[3] = __fmaf_rn(c.x, xa0.w, acc[3]); acc[3] = __fmaf_rn(c.y, xb0.w, acc[3]);
        acc[4] = __fmaf_rn(c.x, xa1.x, acc[4]); acc[4] = __fmaf_rn(c.y, xb1.x, acc[4]);
        acc[5] = __fmaf_rn(c.x, xa1.y, acc[5]); acc[5] = __fmaf_rn(c.y, xb1.y, acc[5]);
        acc[6] = __fmaf_rn(c.x, xa1.z, acc[6]); acc[6] = __fmaf_rn(c.y, xb1.z, acc[6]);
        acc[7] = __fmaf_rn(c.x, xa1.w, acc[7]); acc[7] = __fmaf_rn(c.y, xb1.w, acc[7]);
      }
    }
    const float ic = a.inv_c[j];
    const uint32_t g = (uint32_t)(j * a.world + a.rank);
#pragma unroll
    for (int p = 0; p < SIMT_PB; ++p) {
      const float s = __fmul_rn(__fmul_rn(acc[p], ic), iq[p]);
      const uint64_t key = pack_key(s, g);
      tl[p].insert(key);
    }
  }
  __shared__ uint64_t outk[SIMT_WARPS][KMAX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int prow = r * SIMT_WARPS + warp;  // partial list index
#pragma unroll
  for (int p = 0; p < SIMT_PB; ++p) {
    warp_merge_topk<KMAX>(tl[p], a.k, outk[warp]);
    __syncwarp();
    if (i0 + p < a.N && lane < a.k)
      a.partial[((int64_t)prow * a.N + (i0 + p)) * a.k + lane] = outk[warp][lane];
    __syncwarp();
  }
}

int scan_plan_ranges_simt(int64_t m_local, int32_t N, int num_sms) {
  const int nb = (N + SIMT_PB - 1) / SIMT_PB;
  int ranges = (4 * num_sms + nb - 1) / nb;
  if (ranges > SIMT_MAX_RANGES) ranges = SIMT_MAX_RANGES;
  const int64_t min_rows = 256;
  const int64_t by_rows = (m_local + min_rows - 1) / min_rows;
  if (ranges > by_rows) ranges = (int)(by_rows > 0 ? by_rows : 1);
  return ranges * SIMT_WARPS;
}

void launch_scan_simt(const ScanArgs& a, cudaStream_t s) {
  const int ranges = a.P / SIMT_WARPS;
  const int64_t rows_per_range = (a.m_local + ranges - 1) / ranges;
  dim3 grid(ranges, (a.N + SIMT_PB - 1) / SIMT_PB);
  const size_t smem = sizeof(float) * (size_t)a.d * SIMT_PB;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_scan_simt<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_scan_simt<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    attr = true;
  }
  if (a.k <= 4)
    k_scan_simt<4><<<grid, SIMT_THREADS, smem, s>>>(a, ranges, rows_per_range);
  else
    k_scan_simt<8><<<grid, SIMT_THREADS, smem, s>>>(a, ranges, rows_per_range);
}

}  // namespace argus
