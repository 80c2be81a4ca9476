// scan_epi.cuh -- the per-prompt top-k epilogue shared by the scan kernels
// (k_scan_tc.cu, k_scan_pair.cu): SURVEY §8(a) row A3, fused into row A2.
#pragma once
#include "common.cuh"
#include "tc.cuh"

namespace argus {

// Epilogue on 32 accumulator columns (cache rows c0 .. c0+31 of the tile) of one
// prompt.  The exact score is s_c = fl(fl(acc_c * inv_c[c]) * inv_q).
// Fast path (about one instruction per score): a bound on the chunk.  With m = max_c
// acc_c and inv_c in [lo, hi] (lo >= 0), every acc_c * inv_c[c] <= m * (m >= 0 ? hi : lo)
// as real numbers, and rounding is monotone, so no s_c can reach thr unless
// fl(fl(m * hi|lo) * inv_q) >= thr: the filter never drops a candidate.  The chunk's
// inv_c range is one shared load per lane and two integer warp reductions (inv_c >= 0,
// so its bits order like the floats).  Slow path (warp-uniform entry, compact code):
// x_c = fl(acc_c * inv_c[c]) with packed fp32x2 multiplies, then the warp parks its
// 32x32 x values in shared memory (column-major, conflict-free) and each lane rescans
// its own 32 with the exact score and inserts into its register top-k.
template <int KMAX>
__device__ __forceinline__ void epi_chunk(uint32_t (&v)[32], uint32_t icp, float iq, int cmax, uint32_t g0,
                                          uint32_t world, uint32_t head, uint32_t capg, TopList<KMAX>& tl,
                                          float& thr, uint32_t scratch) {
  const int lane = threadIdx.x & 31;
  float m = -INFINITY;
#pragma unroll
  for (int c = 0; c < 32; c += 4)
    m = fmaxf(m, fmaxf(fmaxf(__uint_as_float(v[c]), __uint_as_float(v[c + 1])),
                       fmaxf(__uint_as_float(v[c + 2]), __uint_as_float(v[c + 3]))));
  const uint32_t icu = __float_as_uint(tc::lds_f32(icp + lane * 4));
  const float ic_hi = __uint_as_float(__reduce_max_sync(0xffffffffu, icu));
  const float ic_lo = __uint_as_float(__reduce_min_sync(0xffffffffu, icu));
  const bool cand = __fmul_rn(__fmul_rn(m, m >= 0.f ? ic_hi : ic_lo), iq) >= thr;
  if (__any_sync(0xffffffffu, cand)) {
    // x = fl(acc * inv_c) for the whole chunk (packed multiplies, same bits as __fmul_rn)
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4) {
      const float4 ic = tc::lds_f32x4(icp + c4 * 16);  // broadcast
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
    }
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

// argus_debug_capture (parity test T2): the chunk's exact scores, computed exactly as
// epi_chunk computes them (fl(fl(acc * inv_c) * inv_q)), to row[c] for c < cmax.  Must
// run before epi_chunk, which overwrites v with the scaled values.
__device__ __forceinline__ void epi_dump(const uint32_t (&v)[32], uint32_t icp, float iq, int cmax, float* row) {
#pragma unroll
  for (int c = 0; c < 32; ++c)  // unrolled: v stays in registers
    if (c < cmax) row[c] = __fmul_rn(__fmul_rn(__uint_as_float(v[c]), tc::lds_f32(icp + c * 4)), iq);
}

}  // namespace argus
