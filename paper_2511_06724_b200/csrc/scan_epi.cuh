// scan_epi.cuh -- the per-prompt top-k epilogue shared by the scan kernels
// (k_scan_tc.cu, k_scan_pair.cu): SURVEY §8(a) row A3, fused into row A2.
#pragma once
#include "common.cuh"
#include "tc.cuh"

namespace argus {

// Epilogue on 32 accumulator columns (cache rows c0 .. c0+31 of the tile) of one
// prompt.  Fast path (2 instructions per score): x_c = acc_c * inv_c[c] and a
// running max; since rounding is monotone, max_c fl(x_c * inv_q) = fl(max_c x_c *
// inv_q), so the chunk holds a candidate iff fl(max * inv_q) >= thr.  Slow path
// (warp-uniform entry, compact code): the warp parks its 32x32 x values in shared
// memory (column-major, conflict-free) and each lane rescans its own 32 with the
// exact score s = fl(x * inv_q) and inserts into its register top-k.
template <int KMAX>
__device__ __forceinline__ void epi_chunk(uint32_t (&v)[32], uint32_t icp, float iq, int cmax, uint32_t g0,
                                          uint32_t world, uint32_t head, uint32_t capg, TopList<KMAX>& tl,
                                          float& thr, uint32_t scratch) {
  const int lane = threadIdx.x & 31;
  float m = -INFINITY;
#pragma unroll
  for (int c4 = 0; c4 < 8; ++c4) {
    const float4 ic = tc::lds_f32x4(icp + c4 * 16);   // shared memory, same address in every lane (broadcast)
    // x = fl(acc * inv_c): packed fp32x2 multiplies (FMUL2, round-to-nearest per lane,
    // the same bits as two __fmul_rn) halve the epilogue's multiply issue slots
    uint64_t p01, p23;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p01)
        : "l"(((uint64_t)v[c4 * 4 + 1] << 32) | v[c4 * 4 + 0]),
          "l"(((uint64_t)__float_as_uint(ic.y) << 32) | __float_as_uint(ic.x)));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p23)
        : "l"(((uint64_t)v[c4 * 4 + 3] << 32) | v[c4 * 4 + 2]),
          "l"(((uint64_t)__float_as_uint(ic.w) << 32) | __float_as_uint(ic.z)));
    v[c4 * 4 + 0] = (uint32_t)p01;
    v[c4 * 4 + 1] = (uint32_t)(p01 >> 32);
    v[c4 * 4 + 2] = (uint32_t)p23;
    v[c4 * 4 + 3] = (uint32_t)(p23 >> 32);
    const float x0 = __uint_as_float(v[c4 * 4 + 0]), x1 = __uint_as_float(v[c4 * 4 + 1]);
    const float x2 = __uint_as_float(v[c4 * 4 + 2]), x3 = __uint_as_float(v[c4 * 4 + 3]);
    m = fmaxf(m, fmaxf(fmaxf(x0, x1), fmaxf(x2, x3)));
  }
  const bool cand = __fmul_rn(m, iq) >= thr;
  if (__any_sync(0xffffffffu, cand)) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {   // 16 columns at a time: 2 KB of scratch per warp
      uint32_t mask = 0;
      if (cand) {  // exact scores of this half, candidate bits (columns past the shard excluded)
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const float sc = __fmul_rn(__uint_as_float(v[half * 16 + c]), iq);
          mask |= (sc >= thr && half * 16 + c < cmax) ? (1u << c) : 0u;
        }
      }
      if (__any_sync(0xffffffffu, mask != 0)) {
        if (mask) {
#pragma unroll
          for (int c = 0; c < 16; ++c)
            tc::sts_f32(scratch + (uint32_t)(c * 32 + lane) * 4, __uint_as_float(v[half * 16 + c]));
          while (mask) {  // only the candidate columns (typically one or two)
            const int c = __ffs(mask) - 1;
            mask &= mask - 1;
            const float sc = __fmul_rn(tc::lds_f32(scratch + (uint32_t)(c * 32 + lane) * 4), iq);
            if (sc >= thr) {
              // key id = age of the entry (0 = oldest live): the cache position itself
              // unless a ring-evicting cache has wrapped (head > 0)
              const uint32_t pos = g0 + (uint32_t)(half * 16 + c) * world;
              tl.insert(pack_key(sc, pos >= head ? pos - head : pos + capg - head));
              if (tl.v[KMAX - 1] != 0) thr = fmaxf(thr, key_score(tl.v[KMAX - 1]));
            }
          }
        }
        __syncwarp();
      }
    }
  }
}

}  // namespace argus
