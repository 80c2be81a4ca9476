// k_scan_tc.cu -- K1+K2: the cosine cache scan with the fused per-prompt top-k
// (SURVEY §8(a) rows A2 + A3; §2.1 "Using similarity search, the most
// similar cached prompt is retrieved", §4.5, §4.7).
//
//   S[i, j] = (<Xb_i, Cb_j> * inv_c[j]) * inv_q[i]   bf16 x bf16 -> fp32 accumulate
//   top-k per prompt i over (S desc, global id asc); S never reaches HBM.
//
// B200 design (DESIGN.md §7 "K1"):
//   * one CTA per SM; CTA = one 128-prompt slice; the cache tiles of a slice are
//     handed out dynamically in chunks of CHUNK tiles (one atomic per chunk, fetched
//     a chunk ahead), so CTAs that start late (SMs still busy with the previous
//     batch's tail kernel) just take fewer chunks; CTAs of all slices sweep the
//     cache in the same order, so slices > 1 re-hit each tile in L2 (a lockstep
//     window that forced this at 64 slices cost more in waiting than the HBM
//     re-reads it saved: DESIGN.md §12);
//   * the prompt slice is the UMMA A operand and lives in TMEM for the whole
//     kernel (128 lanes x up to 384 columns, loaded once with tcgen05.st); for
//     d > 768 k-blocks 12.. stay in shared memory (SS-mode MMAs);
//   * cache tiles of 64 rows are the B operand: TMA (128-byte swizzle, L2
//     evict-first for one slice) streams 64x64 bf16 boxes through a ring of 4
//     slots (half tiles, or quarter tiles for d > 768);
//   * tcgen05.mma.cta_group::1.kind::f16, M=128 (prompts) x N=64 (cache rows) x
//     K=16, issued warp-uniformly (elect.sync inside the asm) by two warps (even /
//     odd tiles) into two TMEM accumulators, one tcgen05.commit per slot (a commit
//     costs ~250 issue cycles, an N=64 MMA 32 pipe cycles);
//   * epilogue: 8 warps, TMEM lane = prompt, each thread owns one prompt and one
//     32-column half of every tile and keeps its top-k in registers behind a float
//     threshold shared (monotonically) with the other lists of the same prompt.
// Warp roles: 0 = TMA producer, 1 / 3 = MMA issuers, 2 = TMEM allocator,
// 4..11 = Q loader + epilogue.
#include <cstddef>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"
#include "scan_epi.cuh"

#ifndef ARGUS_SCAN_EXP
#define ARGUS_SCAN_EXP 0  // diagnostics only: 1 = skip epilogue math, 2 = skip MMAs (tools/scan_experiments.sh),
                          // 3 = M = 64 MMAs, 4 = half the k-steps (scripts/r02_power_exp2.sh)
#endif

namespace argus {

namespace {
constexpr int TN = 64;                      // cache rows per tile (UMMA N)
constexpr int TM = 128;                     // prompts per CTA (UMMA M)
constexpr int KBLK = 64;                    // bf16 per 128-byte swizzle row
constexpr int KB_TMEM = 12;                 // k-blocks of the prompt slice resident in TMEM (d <= 768)
constexpr int KB_MAX = 16;                  // d <= 1024: k-blocks 12..15 of A stay in shared memory
constexpr int BOX_BYTES = TN * KBLK * 2;    // 8 KB cache box
constexpr int QBOX_BYTES = TM * KBLK * 2;   // 16 KB prompt box
constexpr int NSLOT = 4;                    // ring of tile-part slots
constexpr int REGION_BYTES = 192 * 1024;    // ring (+ A tail); also holds 12 prompt boxes at start
constexpr int THREADS = 384;               // 4 control warps + 8 epilogue warps
constexpr int EPI_WARPS = 8;
constexpr int ACC_COL0 = 384;               // accumulators after the resident Q (12 k-blocks)
constexpr uint32_t TMEM_COLS = 512;
constexpr int INV_SLOTS = 8;
constexpr int CHUNK = 4;                    // tiles per dynamically scheduled work unit
constexpr size_t SCRATCH_OFF = 4096;        // after the barriers: 8 warps x 16 x 32 fp32 slow-path scratch
constexpr size_t SMEM_BYTES = (size_t)REGION_BYTES + 1024 /*align*/ + SCRATCH_OFF + EPI_WARPS * 16 * 32 * 4;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");

// Shape of one variant.  KBV = 12 (d <= 768): a tile streams through SPT = 2
// half-tile slots of 6 boxes (48 KB), the whole prompt slice is in TMEM.  KBV = 16
// (768 < d <= 1024): k-blocks 12..15 of the prompt slice (the "A tail", 64 KB) stay
// in shared memory at the start of the region and are read by the MMA through a
// descriptor; a tile streams through SPT = 4 quarter-tile slots of 4 boxes (32 KB)
// behind it.  Either way TMEM = 384 columns of A + 2 x 64 accumulator columns.
template <int KBV>
struct Shape {
  static constexpr int SPT = KBV == 12 ? 2 : 4;                 // slots per tile
  static constexpr int SLOT_BOXES = KBV / SPT;                  // 6 or 4
  static constexpr int SLOT_BYTES = SLOT_BOXES * BOX_BYTES;     // 48 or 32 KB
  static constexpr int ATAIL_BYTES = (KBV - KB_TMEM) * QBOX_BYTES;  // 0 or 64 KB
  static constexpr int RING0 = ATAIL_BYTES;                     // ring offset in the region
  static_assert(RING0 + NSLOT * SLOT_BYTES <= REGION_BYTES, "region");
  static_assert(KB_TMEM * QBOX_BYTES <= REGION_BYTES, "prompt staging");
};
}  // namespace

struct ScanSmem {  // placed after the region
  uint64_t full[NSLOT];         // TMA boxes of slot s landed
  uint64_t empty[NSLOT];        // MMAs reading slot s complete (one commit per slot); with SPT = 2
                                // the tile's last slot completing also means the accumulator is final
  uint64_t tempty[2];           // epilogue has read accumulator b
  uint64_t afull[2];            // SPT = 4: accumulator b final (extra commit after the tile's last slot)
  uint64_t qfull;               // prompt slice (TMEM part) landed in shared memory
  uint64_t qready;              // prompt slice is in TMEM; buffers may be reused
  uint64_t atail;               // KBV = 16: A tail landed in shared memory
  uint64_t invfull[INV_SLOTS];  // inv_c slot l % 8 landed (cannot lap, see the epilogue); also
                                // publishes tile_id[l % 8] (-1 = no more tiles)
  int64_t tile_id[INV_SLOTS];   // cache tile of the CTA's l-th tile
  uint32_t tmem_base;
  uint32_t pad_[3];
  alignas(16) float invc[INV_SLOTS][TN];  // inverse cache-row norms of tile l in slot l % 8 (bulk copy)
};
static_assert(offsetof(ScanSmem, invc) % 16 == 0, "bulk-copy / float4 destination");
static_assert(sizeof(ScanSmem) <= SCRATCH_OFF, "barriers fit before the scratch");

// KBF: k-blocks fixed at compile time (12 for d = 768, 16 for d = 1024) so the MMA
// issue loops unroll into constant descriptor offsets; 0 = d / 64 at run time.
template <int KMAX, int KBV, int KBF = 0>
__global__ void __launch_bounds__(THREADS, 1)
    k_scan_tc(const __grid_constant__ CUtensorMap tmap_c, const __grid_constant__ CUtensorMap tmap_q, ScanArgs a,
              int slices, int64_t n_tiles, int l2mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  using SH = Shape<KBV>;
  constexpr int SPT = SH::SPT;
  ScanSmem* sm = reinterpret_cast<ScanSmem*>(ring + (size_t)REGION_BYTES);
  const uint32_t region_s = tc::smem_u32(ring);           // prompt staging, then [A tail | ring]
  const uint32_t ring_s = region_s + (uint32_t)SH::RING0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slice = blockIdx.x % slices;
  const int range = blockIdx.x / slices;  // index of this CTA's candidate list
  const int KB = KBF ? KBF : a.d / KBLK;
  if (a.stamp != nullptr && threadIdx.x == 0) a.stamp[4 * blockIdx.x] = gtimer();

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmap_c);
    tc::prefetch_tmap(&tmap_q);
    for (int s = 0; s < NSLOT; ++s) {
      tc::mbar_init(tc::smem_u32(&sm->full[s]), 1);
      tc::mbar_init(tc::smem_u32(&sm->empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) tc::mbar_init(tc::smem_u32(&sm->tempty[b]), 32 * EPI_WARPS);
    for (int b = 0; b < 2; ++b) tc::mbar_init(tc::smem_u32(&sm->afull[b]), 1);
    tc::mbar_init(tc::smem_u32(&sm->qfull), 1);
    tc::mbar_init(tc::smem_u32(&sm->atail), 1);
    for (int s = 0; s < INV_SLOTS; ++s) tc::mbar_init(tc::smem_u32(&sm->invfull[s]), 1);
    tc::mbar_init(tc::smem_u32(&sm->qready), 32 * EPI_WARPS);
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
  if (a.ready != nullptr) {
    // pipelined one-GPU mode: nothing this scan touches is written by the previous scan
    // (per-parity buffers); its inputs come from K6 on the prep stream, whose completion
    // the prep stream publishes.  Waiting for that flag instead of a stream event keeps
    // the scan stream a pure chain of scans, so this grid launches (programmatically)
    // while the previous scan drains and each CTA starts on the SM its predecessor frees.
    if (threadIdx.x == 0) {
      uint32_t v;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.ready) : "memory");
        if ((int32_t)(v - a.ready_seq) >= 0) break;
        __nanosleep(128);
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");  // K6's stores before this CTA's TMA reads
    }
    __syncthreads();
  } else {
    pdl_wait();  // setup above overlapped the previous kernel; Xb / inv_q / partial are shared
  }
  if (a.stamp != nullptr && threadIdx.x == 0) a.stamp[4 * blockIdx.x + 1] = gtimer();

  if (warp == 0) {
    // ======================= TMA producer
    if (lane == 0) {
      // prompt slice: its first min(KB, 12) boxes of 128 rows x 64 bf16 (16 KB, 128-byte
      // swizzle) into the region, to be moved into TMEM by the epilogue warps
      const int KBT = KB < KB_TMEM ? KB : KB_TMEM;
      const uint32_t qb = tc::smem_u32(&sm->qfull);
      tc::mbar_arrive_expect_tx(qb, (uint32_t)(KBT * QBOX_BYTES));
      for (int kb = 0; kb < KBT; ++kb)
        tc::tma_load_2d(region_s + (uint32_t)(kb * QBOX_BYTES), &tmap_q, qb, kb * KBLK, slice * TM);
      tc::mbar_wait(tc::smem_u32(&sm->qready), 0);  // region free again
      if (KBV > KB_TMEM) {  // the A tail (k-blocks 12..KB-1) stays in shared memory for the whole kernel
        const uint32_t ab = tc::smem_u32(&sm->atail);
        tc::mbar_arrive_expect_tx(ab, (uint32_t)((KB - KB_TMEM) * QBOX_BYTES));
        for (int kb = KB_TMEM; kb < KB; ++kb)
          tc::tma_load_2d(region_s + (uint32_t)((kb - KB_TMEM) * QBOX_BYTES), &tmap_q, ab, kb * KBLK, slice * TM);
      }
      // one slice streams the cache exactly once: evict-first; with several slices the
      // other slices re-read each tile from L2 shortly after the first reader
      const int l2m = l2mode & 15;
      const uint64_t pol = l2m == 0 ? tc::policy_evict_first()
                                    : (l2m == 1 ? tc::policy_evict_normal() : tc::policy_evict_last());
      int* ctr = a.ctr + slice;
      int64_t l = 0;
      // Tiles are handed out by a per-slice counter (in tiles): CHUNK at a time, then
      // one at a time for the last two chunks per CTA of the slice, so the CTAs of a
      // slice finish within about one tile of each other.  The next grab is fetched a
      // chunk ahead (the atomic's latency overlaps this chunk's loads).
      const int64_t tail_tiles = (int64_t)(gridDim.x / slices) * CHUNK * 2;
      int csz = n_tiles > tail_tiles ? CHUNK : 1;
      int64_t c = atomicAdd(ctr, csz);
      for (;;) {
        const int64_t t0 = c;
        if (t0 >= n_tiles) break;
        const int64_t t1 = t0 + csz < n_tiles ? t0 + csz : n_tiles;
        csz = n_tiles - t1 > tail_tiles ? CHUNK : 1;
        c = atomicAdd(ctr, csz);
        for (int64_t t = t0; t < t1; ++t, ++l) {
#pragma unroll
          for (int hh = 0; hh < SPT; ++hh) {
            const int64_t u = SPT * l + hh;  // slot sequence number
            const int sl = (int)(u & (NSLOT - 1));
            tc::mbar_wait(tc::smem_u32(&sm->empty[sl]), (uint32_t)(((u >> 2) & 1) ^ 1));
            const uint32_t fb = tc::smem_u32(&sm->full[sl]);
            const int kb0 = KB * hh / SPT, kb1 = KB * (hh + 1) / SPT;
            tc::mbar_arrive_expect_tx(fb, (uint32_t)((kb1 - kb0) * BOX_BYTES));
            if (hh == 0) {  // the tile's id and inverse norms (rows past capacity read zeros)
              sm->tile_id[l & (INV_SLOTS - 1)] = t;
              const uint32_t ib = tc::smem_u32(&sm->invfull[l & (INV_SLOTS - 1)]);
              tc::mbar_arrive_expect_tx(ib, TN * 4);
              tc::bulk_load_hint(tc::smem_u32(&sm->invc[l & (INV_SLOTS - 1)][0]), a.inv_c + t * TN, TN * 4, ib, pol);
            }
            for (int j = 0; j < kb1 - kb0; ++j)
              tc::tma_load_2d_hint(ring_s + (uint32_t)(sl * SH::SLOT_BYTES + j * BOX_BYTES), &tmap_c, fb,
                                   (kb0 + j) * KBLK, (int32_t)(t * TN), pol);
          }
        }
      }
      // end markers in the next two tile slots (one per MMA issuer).  Before reusing
      // tile-ring entry l % 8 the consumers of tile l - 8 must be done, which the release
      // of an earlier real tile's first slot guarantees (that MMA needed the epilogue's
      // release of a later tile).  SPT = 2: the slot a real tile l would use was last
      // used by tile l - 2.  SPT = 4: every tile uses slot 0, and the marker tiles never
      // fill it, so both markers wait for the last real tile's release of slot 0.
      const int64_t l_end = l;
      for (int e = 0; e < 2; ++e, ++l) {
        if (SPT == 2) {
          const int64_t u = SPT * l;
          tc::mbar_wait(tc::smem_u32(&sm->empty[u & (NSLOT - 1)]), (uint32_t)(((u >> 2) & 1) ^ 1));
        } else if (l_end > 0) {
          const int64_t u = SPT * (l_end - 1);
          tc::mbar_wait(tc::smem_u32(&sm->empty[u & (NSLOT - 1)]), (uint32_t)((u >> 2) & 1));
        }
        sm->tile_id[l & (INV_SLOTS - 1)] = -1;
        tc::mbar_arrive(tc::smem_u32(&sm->invfull[l & (INV_SLOTS - 1)]));
      }
    }
  } else if (warp == 1 || (warp == 3 && !(l2mode & 32))) {
    // ======================= MMA issuers: warp 1 takes the even tiles (half-slots 0,1,
    // accumulator 0), warp 3 the odd ones (half-slots 2,3, accumulator 1).  One warp's
    // issue loop (~14 instructions and a dependent R2UR chain per MMA, plus the
    // commits) is slower than the 32 cycles an M=128 N=64 K=16 MMA executes in; two
    // interleaved issuers keep the tensor pipe fed.  tcgen05.commit tracks the MMAs
    // of the committing thread only, so the two barrier sets stay independent.
    // diagnostics (scores wrong): ARGUS_SCAN_EXP = 3 issues M = 64 MMAs, = 4 half of the k-steps
    constexpr uint32_t IDESC = tc::idesc_bf16_f32(ARGUS_SCAN_EXP == 3 ? 64 : TM, TN);
    tc::mbar_wait(tc::smem_u32(&sm->qready), 0);
    if (KBV > KB_TMEM) tc::mbar_wait(tc::smem_u32(&sm->atail), 0);
    tc::fence_after();
    const uint64_t dbase = tc::desc_kmajor_sw128(ring_s);
    const uint64_t abase = tc::desc_kmajor_sw128(region_s);  // A tail (KBV = 16)
    const int lstep = (l2mode & 32) ? 1 : 2;
    for (int64_t l = warp == 1 ? 0 : 1;; l += lstep) {
      tc::mbar_wait(tc::smem_u32(&sm->invfull[l & (INV_SLOTS - 1)]), (uint32_t)((l >> 3) & 1));
      if (sm->tile_id[l & (INV_SLOTS - 1)] < 0) break;
      const int b = (int)(l & 1);
      tc::mbar_wait(tc::smem_u32(&sm->tempty[b]), (uint32_t)(((l >> 1) & 1) ^ 1));
      tc::fence_after();
      const uint32_t d_tmem = tmem + ACC_COL0 + b * TN;
#pragma unroll
      for (int hh = 0; hh < SPT; ++hh) {
        const int64_t u = SPT * l + hh;
        const int sl = (int)(u & (NSLOT - 1));
        tc::mbar_wait(tc::smem_u32(&sm->full[sl]), (uint32_t)((u >> 2) & 1));
        tc::fence_after();
        const int kb0 = KB * hh / SPT, kb1 = KB * (hh + 1) / SPT;
        const uint64_t dslot = dbase + (uint64_t)((sl * SH::SLOT_BYTES) >> 4);
#pragma unroll
        for (int j = 0; j < kb1 - kb0; ++j) {
          const int kb = kb0 + j;
          if (KBV == KB_TMEM || kb < KB_TMEM) {
#pragma unroll
            for (int kk = 0; kk < KBLK / 16; ++kk)
              if ((ARGUS_SCAN_EXP != 2 || (kb | kk) == 0) && (ARGUS_SCAN_EXP != 4 || (kk & 1) == 0))
                tc::mma_ts_warp(d_tmem, tmem + (uint32_t)((kb * (KBLK / 16) + kk) * 8),
                                dslot + (uint64_t)((j * BOX_BYTES + kk * 32) >> 4), IDESC, (kb | kk) != 0);
          } else {  // A tail from shared memory (same SW128 K-major layout as the TMA box)
#pragma unroll
            for (int kk = 0; kk < KBLK / 16; ++kk)
              tc::mma_ss_warp(d_tmem, abase + (uint64_t)(((kb - KB_TMEM) * QBOX_BYTES + kk * 32) >> 4),
                              dslot + (uint64_t)((j * BOX_BYTES + kk * 32) >> 4), IDESC, 1u);
          }
        }
        // frees slot sl; with SPT = 2 the tile's last slot also marks accumulator b final
        tc::mma_commit_warp(tc::smem_u32(&sm->empty[sl]));
      }
      if (SPT != 2) tc::mma_commit_warp(tc::smem_u32(&sm->afull[b]));
    }
    // every MMA of this CTA is issued: the next grid may be scheduled (its CTAs take the SMs
    // this grid's CTAs free; only the drain of the last tiles and the list write remain)
    if (a.ready != nullptr) pdl_launch();
  } else if (warp >= 4) {
    // ======================= Q into TMEM (A operand), then the epilogue
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int h = (warp - 4) >> 2;          // column half of every tile (32 of the 64 cache rows)
    const int p_local = q * 32 + lane;      // prompt within the slice
    const int p = slice * TM + p_local;     // prompt within the batch
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    {
      tc::mbar_wait(tc::smem_u32(&sm->qfull), 0);
      const int sw = p_local & 7;  // 128-byte swizzle: 16-byte chunk j of row r sits at chunk j ^ (r % 8)
      const int KBT = KB < KB_TMEM ? KB : KB_TMEM;
      for (int c = h; c < KBT; c += 2) {   // 64 bf16 = 32 TMEM columns per box; halves split the boxes
        const uint32_t row = region_s + (uint32_t)(c * QBOX_BYTES + p_local * 128);
        uint32_t r[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 u = tc::lds_u32x4(row + (uint32_t)((j ^ sw) << 4));
          r[4 * j + 0] = u.x;
          r[4 * j + 1] = u.y;
          r[4 * j + 2] = u.z;
          r[4 * j + 3] = u.w;
        }
        tc::tmem_st32(tmem + lane_base + (uint32_t)(c * 32), r);
      }
      tc::tmem_wait_st();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc::fence_before();
      tc::mbar_arrive(tc::smem_u32(&sm->qready));
    }
    const bool active = p < a.N;
    const float iq = a.inv_q[p];
    const uint32_t scratch = region_s + (uint32_t)(REGION_BYTES + SCRATCH_OFF + (warp - 4) * 512 * 4);
    TopList<KMAX> tl;
    tl.clear();
    float thr = active ? -INFINITY : INFINITY;  // padded prompts never take the slow path
    // Shared threshold: gthr[p] is the largest "KMAX-th best key" any list of this
    // prompt has published (all ranges, both column halves).  A row below it cannot
    // be in the prompt's global top-k (KMAX >= k keys beat it), so every epilogue
    // filters with max(own, shared); lists only grow, the shared key only rises, and
    // a stale read is merely conservative.  Exactness is unaffected.
    uint64_t* gthr_p = a.gthr + p;
    uint64_t published = 0;
    uint64_t gk = active ? __ldcg(reinterpret_cast<const unsigned long long*>(gthr_p)) : 0;
    for (int64_t l = 0;; ++l) {
      __syncwarp();
      tc::mbar_wait(tc::smem_u32(&sm->invfull[l & (INV_SLOTS - 1)]), (uint32_t)((l >> 3) & 1));
      const int64_t t = sm->tile_id[l & (INV_SLOTS - 1)];
      if (t < 0) break;
      if (gk != 0) thr = fmaxf(thr, key_score(gk));
      const int b = (int)(l & 1);
      const int64_t j0 = t * TN + h * 32;
      // SPT = 2: the tile's second half-slot (2l+1) % 4 completing means all its MMAs are
      // done; it cannot lap: reuse by tile l+2 needs this warp's release of tile l.
      // SPT = 4: every tile uses all four slots, so a dedicated per-accumulator barrier
      // (completes once per 2 tiles, same no-lap argument).
      if (SPT == 2)
        tc::mbar_wait(tc::smem_u32(&sm->empty[(2 * l + 1) & (NSLOT - 1)]), (uint32_t)((l >> 1) & 1));
      else
        tc::mbar_wait(tc::smem_u32(&sm->afull[b]), (uint32_t)((l >> 1) & 1));
      tc::fence_after();
      uint32_t v[32];
      tc::tmem_ld32(tmem + lane_base + ACC_COL0 + b * TN + h * 32, v);
      tc::tmem_wait_ld();
      if (a.stamp != nullptr && l == 0 && warp == 4 && lane == 0) a.stamp[4 * blockIdx.x + 2] = gtimer();
      // Release accumulator b right away so MMA(l+2) never waits for this tile's
      // processing.  inv_c slot l % 8 stays valid: the producer refills it for tile
      // l+8 only after done(l+6), which needs every epilogue warp's release of tile
      // l+4, which each warp gives only after finishing tile l (program order).
      tc::fence_before();
      tc::mbar_arrive(tc::smem_u32(&sm->tempty[b]));
      if (ARGUS_SCAN_EXP != 1 && __any_sync(0xffffffffu, active)) {
        const uint32_t icp = tc::smem_u32(&sm->invc[l & (INV_SLOTS - 1)][h * 32]);
        const int64_t rem_rows = a.m_local - j0;
        const int cmax = rem_rows < 32 ? (rem_rows < 0 ? 0 : (int)rem_rows) : 32;
        if (a.dbg != nullptr && active) epi_dump(v, icp, iq, cmax, a.dbg + (int64_t)p * a.dbg_ld + j0);
        epi_chunk<KMAX>(v, icp, iq, cmax, (uint32_t)(j0 * a.world + a.rank), (uint32_t)a.world, a.head, a.capg, tl,
                        thr, scratch);
        // publish only a local bound that beats everything seen so far (rare after warm-up)
        if (active && tl.v[KMAX - 1] > published && tl.v[KMAX - 1] > gk) {
          published = tl.v[KMAX - 1];
          atomicMax(reinterpret_cast<unsigned long long*>(gthr_p), (unsigned long long)published);
        }
        // refresh the shared bound every 4th tile (latency overlaps the next barrier waits)
        if (active && (l & 3) == 3) gk = __ldcg(reinterpret_cast<const unsigned long long*>(gthr_p));
      }
    }
    // fold the two column halves of each prompt inside the CTA: half 1 parks its list
    // in the (now idle) tile buffers, half 0 merges and writes one list per range
    const uint32_t xchg = ring_s + (uint32_t)((q * 32 + lane) * KMAX * 8);  // ring idle (MMAs done)
    if (h == 1) {
#pragma unroll
      for (int t2 = 0; t2 < KMAX; ++t2) tc::sts_u64(xchg + t2 * 8, tl.v[t2]);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
    if (h == 0 && active) {
#pragma unroll
      for (int t2 = 0; t2 < KMAX; ++t2) tl.insert(tc::lds_u64(xchg + t2 * 8));
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

int scan_plan_ranges(int64_t m_local, int32_t N, int num_sms) {
  const int slices = (N + TM - 1) / TM;
  int ranges = num_sms / slices;
  if (ranges < 1) ranges = 1;
  const int64_t n_chunks = ((m_local + TN - 1) / TN + CHUNK - 1) / CHUNK;
  if (ranges > n_chunks) ranges = (int)(n_chunks > 0 ? n_chunks : 1);
  return ranges;  // CTAs per slice = candidate lists per prompt
}

bool scan_supported(int d) { return d % KBLK == 0 && d >= KBLK && d / KBLK <= KB_MAX; }

template <int KMAX, int KBV, int KBF = 0>
static void launch_variant(bool pdl, dim3 grid, cudaStream_t s, const CUtensorMap& tc_, const CUtensorMap& tq,
                           const ScanArgs& a, int slices, int64_t n_tiles, int l2mode) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_scan_tc<KMAX, KBV, KBF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
    attr = true;
  }
  launch_pdl_opt(pdl, k_scan_tc<KMAX, KBV, KBF>, grid, dim3(THREADS), SMEM_BYTES, s, tc_, tq, a, slices, n_tiles, l2mode);
}

void launch_scan(const ScanArgs& a, const CUtensorMap* tmap, const CUtensorMap* tmap_q, cudaStream_t s, bool pdl) {
  const int slices = (a.N + TM - 1) / TM;
  const int64_t n_tiles = (a.m_local + TN - 1) / TN;
  const dim3 grid(slices * a.P);
  // L2 policy of the cache stream: evict-first (measured no worse than normal LRU
  // with several slices either, profiles/r02/l2_policy.md; ARGUS_SCAN_L2=1/2
  // overrides for multi-slice experiments)
  static int l2env = -2;
  if (l2env == -2) {
    const char* e = getenv("ARGUS_SCAN_L2");
    l2env = e ? atoi(e) : -1;
  }
  static int stat = getenv("ARGUS_SCAN_1MMA") ? 32 : 0;
  const int l2mode = (l2env >= 0 && slices > 1 ? l2env : 0) | stat;
  const bool wide = a.d / KBLK > KB_TMEM;
  const bool clip = a.d == KB_TMEM * KBLK, clip_h = a.d == KB_MAX * KBLK;  // d = 768 / 1024
  if (a.k <= 4) {
    if (clip) launch_variant<4, 12, 12>(pdl, grid, s, *tmap, *tmap_q, a, slices, n_tiles, l2mode);
    else if (clip_h) launch_variant<4, 16, 16>(pdl, grid, s, *tmap, *tmap_q, a, slices, n_tiles, l2mode);
    else if (wide) launch_variant<4, 16>(pdl, grid, s, *tmap, *tmap_q, a, slices, n_tiles, l2mode);
    else launch_variant<4, 12>(pdl, grid, s, *tmap, *tmap_q, a, slices, n_tiles, l2mode);
  } else {
    if (clip) launch_variant<8, 12, 12>(pdl, grid, s, *tmap, *tmap_q, a, slices, n_tiles, l2mode);
    else if (clip_h) launch_variant<8, 16, 16>(pdl, grid, s, *tmap, *tmap_q, a, slices, n_tiles, l2mode);
    else if (wide) launch_variant<8, 16>(pdl, grid, s, *tmap, *tmap_q, a, slices, n_tiles, l2mode);
    else launch_variant<8, 12>(pdl, grid, s, *tmap, *tmap_q, a, slices, n_tiles, l2mode);
  }
}

}  // namespace argus
