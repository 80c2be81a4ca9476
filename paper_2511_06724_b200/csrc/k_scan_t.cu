// k_scan_t.cu -- K1+K2 for small batches (N <= 64) with exact tensor work: the cosine scan
// with the fused per-prompt top-k (SURVEY §8(a) rows A2 + A3; §2.1, §4.5).
//
// Same scores, keys and top-k as k_scan_tc.cu (s = fl(fl(acc * inv_c) * inv_q), top-k by
// (s desc, age asc), the same epilogue code), with the MMA transposed: the cache tile is the
// UMMA A operand (M = 128 cache rows, shared memory) and the batch's prompts are B (N = the
// batch rounded up to 16, resident in shared memory for the whole kernel).  k_scan_tc computes
// 128 prompt rows per MMA whatever N is (62 % padding at C2's N = 48); here the tensor work is
// N / 128 of that, which at small N measured as HBM time (halving the MMAs of
// the N = 48 scan was worth 8 % at equal clock).
//
// Roles: warp 0 = TMA producer (prompts once, then 128-row cache tiles one k-block per ring
// slot), warp 1 = MMA issuer, warp 2 = TMEM allocator, warps 4..7 = row warps (TMEM lane
// quarter q: cache rows 32q .. 32q+31 of the tile), warps 8..11 = column warps (lane = prompt:
// the per-prompt top-k in registers).  Per tile the row warps read the accumulator (lane =
// cache row, column = prompt) and park the raw fp32 values transposed in shared memory, 64
// rows at a time; the column warps then run k_scan_tc's chunk epilogue (epi_chunk) on 32-row
// chunks of their prompt's column -- the same code, the same bound filter, the same keys.
//
// Measured (DESIGN.md §9 item 0, profiles/r02/sched/scan_t/): parity-green, mainloop 7.08 TB/s
// at N = 48 (+3 % over k_scan_tc) but slower overall with the column epilogue, so it is opt-in
// (ARGUS_SCAN_T=1) and k_scan_tc serves N <= 128 by default.
#include <cstddef>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "scan_epi.cuh"
#include "tc.cuh"

#ifndef ARGUS_SCANT_EXP
#define ARGUS_SCANT_EXP 0  // diagnostics only (scores wrong): 1 = column warps skip the top-k, 2 = and the
                           // row warps skip the transposed stores (mainloop + accumulator reads only)
#endif

namespace argus {

namespace {
constexpr int TR = 128;                      // cache rows per tile (UMMA M)
constexpr int KBLK = 64;                     // bf16 per 128-byte swizzle row
constexpr int KB = 12;                       // k-blocks (d = 768)
constexpr int SLOT_BYTES = TR * KBLK * 2;    // one k-block of a tile: two 64-row boxes, 16 KB
constexpr int NP_MAX = 64;                   // prompts (UMMA N) at most
constexpr int THREADS = 384;                 // 4 control + 4 row + 4 column warps
constexpr int COLW = 4;                      // column warps: 2 prompt groups x 2 row chunks
constexpr int INV_SLOTS = 8;
constexpr int CHUNK = 4;                     // tiles per dynamically scheduled work unit
constexpr int TSTRIDE = 64 + 4;              // transposed half tile: [prompt][64 rows], padded
constexpr uint32_t TMEM_COLS = 128;          // two accumulators of NP <= 64 columns
constexpr size_t SMEM_CAP = 227 * 1024;
}  // namespace

struct TSmem {
  uint64_t full[16];             // ring slot s landed
  uint64_t empty[16];            // MMAs reading slot s complete
  uint64_t afull[2];             // accumulator b final
  uint64_t tempty[2];            // row warps have read accumulator b
  uint64_t bfull;                // prompts landed
  uint64_t invfull[INV_SLOTS];   // inv_c / tile id of tile l % 8 landed
  uint64_t invempty[INV_SLOTS];  // column warps finished tile l % 8
  int64_t tile_id[INV_SLOTS];
  uint32_t tmem_base;
  uint32_t pad_[3];
  alignas(16) float invc[INV_SLOTS][TR];
};

template <int KMAX>
__global__ void __launch_bounds__(THREADS, 1)
    k_scan_t(const __grid_constant__ CUtensorMap tmap_c, const __grid_constant__ CUtensorMap tmap_q16, ScanArgs a,
             int NP, int nsl, int64_t n_tiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // layout: [B: KB x NP rows x 128 B][ring: nsl x 16 KB][transposed half tile][scratch][TSmem]
  const uint32_t b_s = tc::smem_u32(base);
  const uint32_t bbytes = (uint32_t)(KB * NP * 128);
  const uint32_t ring_s = b_s + bbytes;
  float* ttile = reinterpret_cast<float*>(base + bbytes + (size_t)nsl * SLOT_BYTES);  // [NP][TSTRIDE]
  uint8_t* after = reinterpret_cast<uint8_t*>(ttile) + 2 * sizeof(float) * (size_t)NP_MAX * TSTRIDE;  // 2 halves
  const uint32_t scratch0 = tc::smem_u32(after);  // 2 column warps x 16 x 32 fp32
  TSmem* sm = reinterpret_cast<TSmem*>(after + COLW * 16 * 32 * 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int range = blockIdx.x;  // one slice: CTA = candidate list

  if (a.stamp != nullptr && threadIdx.x == 0) a.stamp[4 * blockIdx.x] = gtimer();
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmap_c);
    tc::prefetch_tmap(&tmap_q16);
    for (int s = 0; s < nsl; ++s) {
      tc::mbar_init(tc::smem_u32(&sm->full[s]), 1);
      tc::mbar_init(tc::smem_u32(&sm->empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(tc::smem_u32(&sm->afull[b]), 1);
      tc::mbar_init(tc::smem_u32(&sm->tempty[b]), 4 * 32);
    }
    tc::mbar_init(tc::smem_u32(&sm->bfull), 1);
    for (int s = 0; s < INV_SLOTS; ++s) {
      tc::mbar_init(tc::smem_u32(&sm->invfull[s]), 1);
      tc::mbar_init(tc::smem_u32(&sm->invempty[s]), COLW * 32);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) {
    tc::tmem_alloc(tc::smem_u32(&sm->tmem_base), TMEM_COLS);
    tc::tmem_relinquish();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = sm->tmem_base;
  pdl_wait();
  if (a.stamp != nullptr && threadIdx.x == 0) a.stamp[4 * blockIdx.x + 1] = gtimer();

  if (warp == 0) {
    // ======================= TMA producer
    if (lane == 0) {
      {  // the prompts (B operand): KB k-blocks of NP rows, 16-row boxes, once
        const uint32_t bb = tc::smem_u32(&sm->bfull);
        tc::mbar_arrive_expect_tx(bb, bbytes);
        for (int kb = 0; kb < KB; ++kb)
          for (int r = 0; r < NP; r += 16)
            tc::tma_load_2d(b_s + (uint32_t)(kb * NP * 128 + r * 128), &tmap_q16, bb, kb * KBLK, r);
      }
      const uint64_t pol = tc::policy_evict_first();
      int* ctr = a.ctr;
      int64_t l = 0, u = 0;  // tile and slot sequence numbers
      const int64_t tail_tiles = (int64_t)gridDim.x * CHUNK * 2;
      int csz = n_tiles > tail_tiles ? CHUNK : 1;
      int64_t c = atomicAdd(ctr, csz);
      for (;;) {
        const int64_t t0 = c;
        if (t0 >= n_tiles) break;
        const int64_t t1 = t0 + csz < n_tiles ? t0 + csz : n_tiles;
        csz = n_tiles - t1 > tail_tiles ? CHUNK : 1;
        c = atomicAdd(ctr, csz);
        for (int64_t t = t0; t < t1; ++t, ++l) {
          // tile id + inverse norms of its 128 rows (the column warps release the slot)
          const int li = (int)(l & (INV_SLOTS - 1));
          tc::mbar_wait(tc::smem_u32(&sm->invempty[li]), (uint32_t)(((l >> 3) & 1) ^ 1));
          sm->tile_id[li] = t;
          const uint32_t ib = tc::smem_u32(&sm->invfull[li]);
          tc::mbar_arrive_expect_tx(ib, TR * 4);
          tc::bulk_load_hint(tc::smem_u32(&sm->invc[li][0]), a.inv_c + t * TR, TR * 4, ib, pol);
          for (int kb = 0; kb < KB; ++kb, ++u) {
            const int sl = (int)(u % nsl);
            const uint32_t ph = (uint32_t)((u / nsl) & 1);
            tc::mbar_wait(tc::smem_u32(&sm->empty[sl]), ph ^ 1u);
            const uint32_t fb = tc::smem_u32(&sm->full[sl]);
            tc::mbar_arrive_expect_tx(fb, SLOT_BYTES);
            const uint32_t dst = ring_s + (uint32_t)(sl * SLOT_BYTES);
            tc::tma_load_2d_hint(dst, &tmap_c, fb, kb * KBLK, (int32_t)(t * TR), pol);
            tc::tma_load_2d_hint(dst + SLOT_BYTES / 2, &tmap_c, fb, kb * KBLK, (int32_t)(t * TR + 64), pol);
          }
        }
      }
      // end marker in the next tile entry (after the column warps released it)
      const int li = (int)(l & (INV_SLOTS - 1));
      tc::mbar_wait(tc::smem_u32(&sm->invempty[li]), (uint32_t)(((l >> 3) & 1) ^ 1));
      sm->tile_id[li] = -1;
      tc::mbar_arrive(tc::smem_u32(&sm->invfull[li]));
    }
  } else if (warp == 1) {
    // ======================= MMA issuer: D[row][prompt] (+)= A[row][k] . B[prompt][k]
    const uint32_t idesc = tc::idesc_bf16_f32(TR, NP);
    tc::mbar_wait(tc::smem_u32(&sm->bfull), 0);
    tc::fence_after();
    const uint64_t adesc0 = tc::desc_kmajor_sw128(ring_s);
    const uint64_t bdesc0 = tc::desc_kmajor_sw128(b_s);
    int64_t u = 0;
    for (int64_t l = 0;; ++l) {
      tc::mbar_wait(tc::smem_u32(&sm->invfull[l & (INV_SLOTS - 1)]), (uint32_t)((l >> 3) & 1));
      if (sm->tile_id[l & (INV_SLOTS - 1)] < 0) break;
      const int b = (int)(l & 1);
      tc::mbar_wait(tc::smem_u32(&sm->tempty[b]), (uint32_t)(((l >> 1) & 1) ^ 1));
      tc::fence_after();
      const uint32_t d_tmem = tmem + (uint32_t)(b * NP_MAX);
      for (int kb = 0; kb < KB; ++kb, ++u) {
        const int sl = (int)(u % nsl);
        tc::mbar_wait(tc::smem_u32(&sm->full[sl]), (uint32_t)((u / nsl) & 1));
        tc::fence_after();
        const uint64_t ad = adesc0 + (uint64_t)((sl * SLOT_BYTES) >> 4);
        const uint64_t bd = bdesc0 + (uint64_t)((kb * NP * 128) >> 4);
#pragma unroll
        for (int kk = 0; kk < KBLK / 16; ++kk)
          tc::mma_ss_warp(d_tmem, ad + (uint64_t)((kk * 32) >> 4), bd + (uint64_t)((kk * 32) >> 4), idesc,
                          (kb | kk) != 0);
        tc::mma_commit_warp(tc::smem_u32(&sm->empty[sl]));
      }
      tc::mma_commit_warp(tc::smem_u32(&sm->afull[b]));
    }
  } else if (warp >= 4 && warp < 8) {
    // ======================= row warps: accumulator -> transposed half tiles
    const int q = warp & 3;                              // TMEM lane quarter = cache rows 32q..
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const int half = q >> 1;                             // rows 0..63 (half 0) or 64..127
    const int r = (q & 1) * 32 + lane;                   // row within the half
    int64_t l = 0;
    for (;; ++l) {
      tc::mbar_wait(tc::smem_u32(&sm->invfull[l & (INV_SLOTS - 1)]), (uint32_t)((l >> 3) & 1));
      if (sm->tile_id[l & (INV_SLOTS - 1)] < 0) break;
      const int b = (int)(l & 1);
      tc::mbar_wait(tc::smem_u32(&sm->afull[b]), (uint32_t)((l >> 1) & 1));
      tc::fence_after();
      uint32_t v0[32], v1[32];
      tc::tmem_ld32(tmem + lane_base + (uint32_t)(b * NP_MAX), v0);
      if (NP > 32) tc::tmem_ld32(tmem + lane_base + (uint32_t)(b * NP_MAX + 32), v1);
      tc::tmem_wait_ld();
      tc::fence_before();
      tc::mbar_arrive(tc::smem_u32(&sm->tempty[b]));
      // half hh goes to buffer hh (named barriers 1 + hh: stored, 3 + hh: read); the row warps
      // wait only for the column warps' release of the same half of the previous tile, so
      // they store half 1 while the column warps work through half 0
      for (int hh = 0; hh < 2; ++hh) {
        float* tb = ttile + (size_t)hh * NP_MAX * TSTRIDE;
        if (l > 0) asm volatile("bar.sync %0, %1;" ::"r"(3 + hh), "n"(8 * 32) : "memory");
        if (half == hh && ARGUS_SCANT_EXP < 2) {
#pragma unroll
          for (int c = 0; c < 32; ++c) tb[c * TSTRIDE + r] = __uint_as_float(v0[c]);
          if (NP > 32) {
#pragma unroll
            for (int c = 0; c < 32; ++c) tb[(32 + c) * TSTRIDE + r] = __uint_as_float(v1[c]);
          }
        }
        asm volatile("bar.arrive %0, %1;" ::"r"(1 + hh), "n"(8 * 32) : "memory");
      }
    }
    // balance the column warps' releases of the last tile (none if this CTA got no tile)
    if (l > 0) {
      asm volatile("bar.sync 3, %0;" ::"n"(8 * 32) : "memory");
      asm volatile("bar.sync 4, %0;" ::"n"(8 * 32) : "memory");
    }
  } else if (warp >= 8) {
    // ======================= column warps: lane = prompt, the per-prompt top-k; warp cw takes
    // prompts 32 (cw & 1) .. + 31 and row chunk cw >> 1 of every half tile (two lists per
    // prompt, folded at the end)
    const int cw = warp - 8, chs = cw >> 1;
    const int p = (cw & 1) * 32 + lane;  // prompt
    const bool active = p < a.N;
    tc::mbar_wait(tc::smem_u32(&sm->bfull), 0);
    const float iq = active ? a.inv_q[p] : 0.f;
    const bool live = (cw & 1) * 32 < NP;  // warp has prompts at all
    const uint32_t scratch = scratch0 + (uint32_t)(cw * 16 * 32 * 4);
    TopList<KMAX> tl;
    tl.clear();
    float thr = active ? -INFINITY : INFINITY;
    uint64_t* gthr_p = a.gthr + (active ? p : 0);
    uint64_t published = 0;
    uint64_t gk = active ? __ldcg(reinterpret_cast<const unsigned long long*>(gthr_p)) : 0;
    for (int64_t l = 0;; ++l) {
      const int li = (int)(l & (INV_SLOTS - 1));
      tc::mbar_wait(tc::smem_u32(&sm->invfull[li]), (uint32_t)((l >> 3) & 1));
      const int64_t t = sm->tile_id[li];
      if (t < 0) break;
      if (gk != 0) thr = fmaxf(thr, key_score(gk));
      for (int hh = 0; hh < 2; ++hh) {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + hh), "n"(8 * 32) : "memory");  // half hh stored
        const float* tb = ttile + (size_t)hh * NP_MAX * TSTRIDE;
        if (live && ARGUS_SCANT_EXP == 0) {
          {
            const int ch = chs;
            const int r0 = ch * 32;                          // rows r0 .. r0+31 of the half
            const int64_t j0 = t * TR + hh * 64 + r0;       // local cache row of the chunk
            uint32_t v[32];
            const float* col = tb + (p < NP ? p : 0) * TSTRIDE + r0;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 f = *reinterpret_cast<const float4*>(col + j);
              v[j] = __float_as_uint(f.x);
              v[j + 1] = __float_as_uint(f.y);
              v[j + 2] = __float_as_uint(f.z);
              v[j + 3] = __float_as_uint(f.w);
            }
            const uint32_t icp = tc::smem_u32(&sm->invc[li][hh * 64 + r0]);
            const int64_t rem_rows = a.m_local - j0;
            const int cmax = rem_rows < 32 ? (rem_rows < 0 ? 0 : (int)rem_rows) : 32;
            if (a.dbg != nullptr && active) epi_dump(v, icp, iq, cmax, a.dbg + (int64_t)p * a.dbg_ld + j0);
            epi_chunk<KMAX>(v, icp, iq, cmax, (uint32_t)(j0 * a.world + a.rank), (uint32_t)a.world, a.head, a.capg,
                            tl, thr, scratch);
          }
          if (active && tl.v[KMAX - 1] > published && tl.v[KMAX - 1] > gk) {
            published = tl.v[KMAX - 1];
            atomicMax(reinterpret_cast<unsigned long long*>(gthr_p), (unsigned long long)published);
          }
        }
        asm volatile("bar.arrive %0, %1;" ::"r"(3 + hh), "n"(8 * 32) : "memory");  // half hh read
      }
      if (active && (l & 3) == 3) gk = __ldcg(reinterpret_cast<const unsigned long long*>(gthr_p));
      tc::mbar_arrive(tc::smem_u32(&sm->invempty[li]));  // inv_c slot l % 8 free
    }
    // fold the two chunk lists of each prompt (the transposed tile is idle now)
    uint64_t* xchg = reinterpret_cast<uint64_t*>(ttile) + (size_t)((cw & 1) * 32 + lane) * KMAX;
    if (chs == 1) {
#pragma unroll
      for (int t2 = 0; t2 < KMAX; ++t2) xchg[t2] = tl.v[t2];
    }
    asm volatile("bar.sync 5, %0;" ::"n"(COLW * 32) : "memory");
    if (chs == 0 && active) {
#pragma unroll
      for (int t2 = 0; t2 < KMAX; ++t2) tl.insert(xchg[t2]);
      uint64_t* out = a.partial + ((int64_t)range * a.N + p) * a.k;
#pragma unroll
      for (int t2 = 0; t2 < KMAX; ++t2)
        if (t2 < a.k) out[t2] = tl.v[t2];
    }
  }

  tc::fence_before();
  __syncthreads();
  if (a.stamp != nullptr && threadIdx.x == 0) a.stamp[4 * blockIdx.x + 3] = gtimer();
  pdl_launch();
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, TMEM_COLS);
  }
}

// Shared memory of a launch with np prompts (B) and nsl ring slots.
static size_t smem_bytes(int np, int nsl) {
  return 1024 + (size_t)KB * np * 128 + (size_t)nsl * SLOT_BYTES + 2 * sizeof(float) * NP_MAX * TSTRIDE +
         COLW * 16 * 32 * 4 + sizeof(TSmem);
}

bool scan_t_supported(int d, int32_t N, int k) { return d == KB * KBLK && N >= 1 && N <= NP_MAX && k >= 1 && k <= 8; }

int scan_t_plan_ranges(int64_t m_local, int num_sms) {
  const int64_t n_chunks = ((m_local + TR - 1) / TR + CHUNK - 1) / CHUNK;
  int64_t r = num_sms < n_chunks ? num_sms : n_chunks;
  return (int)(r > 0 ? r : 1);
}

template <int KMAX>
static cudaError_t launch_t(bool pdl, dim3 grid, size_t smem, cudaStream_t s, const CUtensorMap& tc_,
                            const CUtensorMap& tq16, const ScanArgs& a, int np, int nsl, int64_t n_tiles) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_scan_t<KMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_CAP);
    attr = true;
  }
  return launch_pdl_opt(pdl, k_scan_t<KMAX>, grid, dim3(THREADS), smem, s, tc_, tq16, a, np, nsl, n_tiles);
}

cudaError_t launch_scan_t(const ScanArgs& a, const CUtensorMap* tmap_c, const CUtensorMap* tmap_q16, cudaStream_t s,
                          bool pdl) {
  const int np = (a.N + 15) / 16 * 16;
  int nsl = 16;
  while (nsl > 2 && smem_bytes(np, nsl) > SMEM_CAP) --nsl;
  const int64_t n_tiles = (a.m_local + TR - 1) / TR;
  const dim3 grid(a.P);
  const size_t smem = smem_bytes(np, nsl);
  if (a.k <= 4) return launch_t<4>(pdl, grid, smem, s, *tmap_c, *tmap_q16, a, np, nsl, n_tiles);
  return launch_t<8>(pdl, grid, smem, s, *tmap_c, *tmap_q16, a, np, nsl, n_tiles);
}

}  // namespace argus
