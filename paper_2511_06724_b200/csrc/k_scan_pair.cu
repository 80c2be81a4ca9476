// k_scan_pair.cu -- K1+K2 for batches of more than 128 prompts on CTA pairs
// (SURVEY §8(a) rows A2 + A3; §2.1, §4.5, §4.7).
//
// Same arithmetic, keys and epilogue as k_scan_tc.cu (the score of prompt i and
// cache row j is fl(fl(<Xb_i, Cb_j> * inv_c[j]) * inv_q[i]); top-k by (score desc,
// age asc)), but the MMA is tcgen05.mma.cta_group::2: a cluster of two CTAs on one
// TPC holds a 256-prompt "pair slice" (128 prompts in each CTA's TMEM, the UMMA A
// operand) and every 64-row cache tile is split between the two CTAs' shared
// memories (32 rows each, the B operand).  Per unit of tensor work each SM
// therefore pulls half the cache bytes through TMA; with one slice per CTA the
// multi-slice scans were capped by the chip's TMA/L2->SM throughput (~10 TB/s of
// tile traffic at N = 256..512), and a 256-prompt batch now reads each tile once.
// For d > 768 (KBV = 16) k-blocks 12.. of each CTA's prompts stay in its shared
// memory and those MMAs take A by descriptor, as in k_scan_tc.cu.
//
// Roles (both CTAs unless noted): warp 0 = TMA producer (the leader also fetches
// the pair's tile schedule and publishes every tile id into the peer's ring through
// distributed shared memory); warps 1 / 3 = MMA issuers, leader only (even / odd
// tiles, two TMEM accumulators); warp 2 = TMEM allocator (cta_group::2, both CTAs);
// warps 4..11 = prompt staging into TMEM, then the epilogue of this CTA's 128 prompts
// (which sees all 64 columns of each tile).  Barriers that cross the pair: the
// leader's full[] (both halves of a slot landed: TMA .cta_group::2 signals it from
// the peer), empty[] / afull[] in both CTAs (multicast commits from the leader's MMA
// warps), the leader's tempty[] / qpair (one arrival per epilogue warp of either CTA).
#include <cstddef>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "scan_epi.cuh"
#include "tc.cuh"

namespace argus {

namespace {
constexpr int TN = 64;                       // cache rows per tile (MMA N)
constexpr int HR = 32;                       // rows of each tile held by each CTA
constexpr int TM = 128;                      // prompts per CTA (M = 256 per pair)
constexpr int KBLK = 64;
constexpr int KB_TMEM = 12;                  // k-blocks of A in TMEM (d <= 768)
constexpr int KB_MAX = 16;                   // d <= 1024: k-blocks 12.. of A stay in shared memory
constexpr int BOX_BYTES = HR * KBLK * 2;     // 4 KB: 32 rows x 64 bf16
constexpr int QBOX_BYTES = TM * KBLK * 2;    // 16 KB prompt box
constexpr int NSLOT = 8;                     // tile-part slots
constexpr int REGION_BYTES = 192 * 1024;
static_assert(KB_TMEM * QBOX_BYTES <= REGION_BYTES, "prompt staging");
// KBV = 12: half-tile slots of 6 boxes (24 KB), 4 tiles in flight.  KBV = 16: the A
// tail (64 KB) first, then quarter-tile slots of 4 boxes (16 KB), 2 tiles in flight.
template <int KBV>
struct PShape {
  static constexpr int SPT = KBV == 12 ? 2 : 4;
  static constexpr int SLOT_BYTES = (KBV / SPT) * BOX_BYTES;
  static constexpr int RING0 = (KBV - KB_TMEM) * QBOX_BYTES;
  static_assert(RING0 + NSLOT * SLOT_BYTES <= REGION_BYTES, "ring");
};
constexpr int THREADS = 384;
constexpr int EPI_WARPS = 8;
constexpr int ACC_COL0 = 384;
constexpr uint32_t TMEM_COLS = 512;
constexpr int INV_SLOTS = 8;
constexpr int CHUNK = 4;
constexpr size_t SCRATCH_OFF = 4096;
constexpr size_t SMEM_BYTES = (size_t)REGION_BYTES + 1024 + SCRATCH_OFF + EPI_WARPS * 16 * 32 * 4;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
}  // namespace

struct PairSmem {
  uint64_t full[NSLOT];         // leader: both halves of slot s landed (1 arrival + tx of both CTAs)
  uint64_t empty[NSLOT];        // slot s free again (multicast commit of the leader's MMA warp)
  uint64_t tempty[2];           // leader: accumulator b read by all 16 epilogue warps of the pair
  uint64_t afull[2];            // accumulator b final (multicast commit)
  uint64_t qfull;               // this CTA's prompt boxes landed in shared memory
  uint64_t qlocal;              // this CTA's prompt slice is in TMEM: the region is free
  uint64_t qpair;               // leader: both slices are in TMEM (16 warp arrivals)
  uint64_t atail;               // leader, KBV = 16: both CTAs' A tails landed (tx of both)
  uint64_t tsched[INV_SLOTS];   // peer: the leader published tile_id[l % 8]
  uint64_t invfull[INV_SLOTS];  // inv_c of tile l landed (publishes tile_id[l % 8] locally)
  int64_t tile_id[INV_SLOTS];
  uint32_t tmem_base;
  uint32_t pad_[3];
  alignas(16) float invc[INV_SLOTS][TN];
};
static_assert(offsetof(PairSmem, invc) % 16 == 0, "bulk-copy / float4 destination");
static_assert(sizeof(PairSmem) <= SCRATCH_OFF, "barriers fit before the scratch");

// tile entry: tile (36 bits) | pair slice (8) | list slot (8) | epoch (11); -1 = end
__device__ __forceinline__ int64_t pack_tile(int64_t t, int ps, int slot, int ep) {
  return t | ((int64_t)ps << 36) | ((int64_t)slot << 44) | ((int64_t)ep << 52);
}
__device__ __forceinline__ int64_t tile_of(int64_t pk) { return pk & ((int64_t(1) << 36) - 1); }
__device__ __forceinline__ int pslice_of(int64_t pk) { return (int)((pk >> 36) & 0xFF); }
__device__ __forceinline__ int slot_of(int64_t pk) { return (int)((pk >> 44) & 0xFF); }
__device__ __forceinline__ int epoch_of(int64_t pk) { return (int)(pk >> 52); }

// KBF: the number of k-blocks fixed at compile time (12 for d = 768, the CLIP width),
// so the MMA issue loops unroll into constant descriptor offsets; 0 = d / 64 at run time.
template <int KMAX, int KBV, int KBF = 0>
__global__ void __launch_bounds__(THREADS, 1)
    k_scan_pair(const __grid_constant__ CUtensorMap tmap_c32, const __grid_constant__ CUtensorMap tmap_q, ScanArgs a,
                int pslices, int64_t n_tiles, int l2mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  using SH = PShape<KBV>;
  constexpr int SPT = SH::SPT;
  PairSmem* sm = reinterpret_cast<PairSmem*>(ring + (size_t)REGION_BYTES);
  const uint32_t region_s = tc::smem_u32(ring);  // prompt staging, then [A tail | ring]
  const uint32_t ring_s = region_s + (uint32_t)SH::RING0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = tc::cluster_ctarank();  // 0 = leader (issues the MMAs)
  const bool leader = crank == 0;
  const int pair = blockIdx.x >> 1;
  // With migration the first home_max * pslices pairs are homed round-robin on the pair
  // slices and the rest "float": they keep moving to the slice that is furthest behind,
  // so all slices sweep the cache at about the same pace (L2 reuse) on every TPC.
  const int n_home = a.migrate ? a.home_max * pslices : 1 << 30;
  const bool floater = pair >= n_home;
  const int pslice = floater ? (pair - n_home) % pslices : pair % pslices;
  const int range = floater ? a.home_max + (pair - n_home) : pair / pslices;  // this pair's list slot
  const int KB = KBF ? KBF : a.d / KBLK;
  const int pbase = pslice * 2 * TM + (int)crank * TM;  // this CTA's first prompt

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmap_c32);
    tc::prefetch_tmap(&tmap_q);
    for (int s = 0; s < NSLOT; ++s) {
      tc::mbar_init(tc::smem_u32(&sm->full[s]), 1);
      tc::mbar_init(tc::smem_u32(&sm->empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(tc::smem_u32(&sm->tempty[b]), 2 * EPI_WARPS);
      tc::mbar_init(tc::smem_u32(&sm->afull[b]), 1);
    }
    tc::mbar_init(tc::smem_u32(&sm->qfull), 1);
    tc::mbar_init(tc::smem_u32(&sm->qlocal), EPI_WARPS);
    tc::mbar_init(tc::smem_u32(&sm->qpair), 2 * EPI_WARPS);
    tc::mbar_init(tc::smem_u32(&sm->atail), 1);
    for (int s = 0; s < INV_SLOTS; ++s) {
      tc::mbar_init(tc::smem_u32(&sm->tsched[s]), 1);
      tc::mbar_init(tc::smem_u32(&sm->invfull[s]), 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) {
    tc::tmem_alloc2(tc::smem_u32(&sm->tmem_base), TMEM_COLS);
    tc::tmem_relinquish2();
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();  // the peer's barriers exist before any remote arrive / TMA signal
  tc::fence_after();
  const uint32_t tmem = sm->tmem_base;
  pdl_wait();

  if (warp == 0) {
    // ======================= TMA producers
    if (lane == 0) {
      const int KBT = KB < KB_TMEM ? KB : KB_TMEM;
      const uint32_t qb = tc::smem_u32(&sm->qfull);
      tc::mbar_arrive_expect_tx(qb, (uint32_t)(KBT * QBOX_BYTES));
      for (int kb = 0; kb < KBT; ++kb)
        tc::tma_load_2d(region_s + (uint32_t)(kb * QBOX_BYTES), &tmap_q, qb, kb * KBLK, pbase);
      tc::mbar_wait(tc::smem_u32(&sm->qlocal), 0);  // region free again
      if (KBV > KB_TMEM) {  // A tail: k-blocks 12.. of this CTA's prompts, counted on the leader's atail
        const uint32_t ab_local = tc::smem_u32(&sm->atail);
        if (leader) tc::mbar_arrive_expect_tx(ab_local, (uint32_t)(2 * (KB - KB_TMEM) * QBOX_BYTES));
        const uint32_t ab = tc::mapa(ab_local, 0);
        for (int kb = KB_TMEM; kb < KB; ++kb)
          tc::tma_load_2d_pair(region_s + (uint32_t)((kb - KB_TMEM) * QBOX_BYTES), &tmap_q, ab, kb * KBLK, pbase,
                               tc::policy_evict_normal());
      }
      const int l2m = l2mode & 15;
      const uint64_t pol = l2m == 0 ? tc::policy_evict_first()
                                    : (l2m == 1 ? tc::policy_evict_normal() : tc::policy_evict_last());
      auto issue = [&](int64_t l, int64_t t) {
#pragma unroll
        for (int hh = 0; hh < SPT; ++hh) {
          const int64_t u = SPT * l + hh;
          const int sl = (int)(u & (NSLOT - 1));
          tc::mbar_wait(tc::smem_u32(&sm->empty[sl]), (uint32_t)(((u >> 3) & 1) ^ 1));
          const int kb0 = KB * hh / SPT, kb1 = KB * (hh + 1) / SPT;
          const uint32_t fb_local = tc::smem_u32(&sm->full[sl]);
          if (leader) tc::mbar_arrive_expect_tx(fb_local, (uint32_t)(2 * (kb1 - kb0) * BOX_BYTES));
          if (hh == 0) {  // the tile's inverse norms, for this CTA's epilogue (all 64 rows)
            const uint32_t ib = tc::smem_u32(&sm->invfull[l & (INV_SLOTS - 1)]);
            tc::mbar_arrive_expect_tx(ib, TN * 4);
            tc::bulk_load_hint(tc::smem_u32(&sm->invc[l & (INV_SLOTS - 1)][0]), a.inv_c + t * TN, TN * 4, ib, pol);
          }
          const uint32_t fb = tc::mapa(fb_local, 0);  // the leader's full barrier counts both halves
          for (int j = 0; j < kb1 - kb0; ++j)
            tc::tma_load_2d_pair(ring_s + (uint32_t)(sl * SH::SLOT_BYTES + j * BOX_BYTES), &tmap_c32, fb,
                                 (kb0 + j) * KBLK, (int32_t)(t * TN + (int64_t)crank * HR), pol);
        }
      };
      if (leader) {
        // A tile entry carries the tile, the pair slice, the list slot and the epoch
        // (pack_tile); consumers reload the prompt slice when the epoch changes.
        int cur = pslice, slot = range, ep = 0, since = 0;
        int64_t l = 0;
        // tile-granular counter: CHUNK tiles per grab, single tiles for the last two
        // chunks per pair of the pair slice (see k_scan_tc.cu)
        const int64_t tail_tiles = (int64_t)(gridDim.x / (2 * pslices)) * CHUNK * 2;
        // the pair slice furthest behind that still has some chunks to go (or `keep`)
        auto laggard = [&](int keep) {
          int64_t lo = *reinterpret_cast<volatile int*>(a.ctr + keep);
          int best = keep;
          for (int ps = 0; ps < pslices; ++ps) {
            const int64_t cs = *reinterpret_cast<volatile int*>(a.ctr + ps);
            if (cs + 8 * CHUNK < n_tiles && cs < lo) {
              lo = cs;
              best = ps;
            }
          }
          return best;
        };
        int csz = n_tiles > tail_tiles ? CHUNK : 1;
        int64_t c = atomicAdd(a.ctr + cur, csz);
        int c_ps = cur;  // the pair slice `c` was taken from
        for (;;) {
          int64_t t0 = c;
          if (c_ps != cur) {  // a floater's move takes effect with the chunk it prefetched
            cur = c_ps;
            ++ep;
          }
          if (t0 >= n_tiles) {
            // Migration: this pair slice ran dry; continue the slice with the most tiles
            // left (worth a prompt-slice reload only if it has a few chunks to go).  Home
            // pairs take one of its MAX_VISITS migrant list slots; floaters keep theirs.
            if (!a.migrate) break;
            int next = -1;
            for (int tries = 0; tries < 3 && next < 0; ++tries) {
              int64_t best_rem = 8 * CHUNK - 1;
              int cand = -1;
              for (int ps = 0; ps < pslices; ++ps) {
                const int64_t rem = n_tiles - *reinterpret_cast<volatile int*>(a.ctr + ps);
                if (rem > best_rem) {
                  best_rem = rem;
                  cand = ps;
                }
              }
              if (cand < 0) break;
              int v = 0;
              if (!floater) {
                v = atomicAdd(a.ctr + 2 * MAX_SLICES + cand, 1);
                if (v >= MAX_VISITS) continue;
              }
              const int64_t cc = atomicAdd(a.ctr + cand, CHUNK);
              if (cc < n_tiles) {
                next = cand;
                if (!floater) slot = a.home_max + a.floaters + v;
                c = cc;
                csz = CHUNK;
              }
            }
            if (next < 0) break;
            cur = c_ps = next;
            ++ep;
            t0 = c;
          }
          const int64_t t1 = t0 + csz < n_tiles ? t0 + csz : n_tiles;
          csz = n_tiles - t1 > tail_tiles ? CHUNK : 1;
          // next grab: a floater re-balances every 8 chunks
          int nps = cur;
          if (floater && ++since >= 8) {
            since = 0;
            nps = laggard(cur);
            if (nps != cur) csz = CHUNK;
          }
          c = atomicAdd(a.ctr + nps, csz);
          c_ps = nps;
          for (int64_t t = t0; t < t1; ++t, ++l) {
            // ring entry l % 8 is free in both CTAs once the first slot of tile l was
            // released by its previous tile (4 or 2 tiles back): wait for that first
            const int64_t u = SPT * l;
            tc::mbar_wait(tc::smem_u32(&sm->empty[u & (NSLOT - 1)]), (uint32_t)(((u >> 3) & 1) ^ 1));
            const int64_t pk = pack_tile(t, cur, slot, ep);
            sm->tile_id[l & (INV_SLOTS - 1)] = pk;
            tc::st_async_s64(tc::mapa(tc::smem_u32(&sm->tile_id[l & (INV_SLOTS - 1)]), 1), pk,
                             tc::mapa(tc::smem_u32(&sm->tsched[l & (INV_SLOTS - 1)]), 1));
            issue(l, t);
          }
        }
        // two end markers (one per MMA issuer); the first slot a tile l would use was
        // last used by tile l - 8 / SPT (4 or 2 tiles back): a real tile or none
        for (int e = 0; e < 2; ++e, ++l) {
          const int64_t u = SPT * l;
          tc::mbar_wait(tc::smem_u32(&sm->empty[u & (NSLOT - 1)]), (uint32_t)(((u >> 3) & 1) ^ 1));
          sm->tile_id[l & (INV_SLOTS - 1)] = -1;
          tc::st_async_s64(tc::mapa(tc::smem_u32(&sm->tile_id[l & (INV_SLOTS - 1)]), 1), -1,
                           tc::mapa(tc::smem_u32(&sm->tsched[l & (INV_SLOTS - 1)]), 1));
          tc::mbar_arrive(tc::smem_u32(&sm->invfull[l & (INV_SLOTS - 1)]));
        }
      } else {
        // peer: follow the leader's schedule
        int markers = 0;
        for (int64_t l = 0; markers < 2; ++l) {
          // the leader's st.async delivers tile_id[l % 8] as 8 tx bytes on tsched[l % 8]
          const uint32_t tb = tc::smem_u32(&sm->tsched[l & (INV_SLOTS - 1)]);
          tc::mbar_arrive_expect_tx(tb, 8);
          tc::mbar_wait(tb, (uint32_t)((l >> 3) & 1));
          const int64_t pk = *reinterpret_cast<volatile int64_t*>(&sm->tile_id[l & (INV_SLOTS - 1)]);
          if (pk < 0) {
            tc::mbar_arrive(tc::smem_u32(&sm->invfull[l & (INV_SLOTS - 1)]));
            ++markers;
            continue;
          }
          issue(l, tile_of(pk));
        }
      }
    }
  } else if (leader && (warp == 1 || warp == 3)) {
    // ======================= MMA issuers (leader): M = 256 (both CTAs' prompts) x N = 64
    constexpr uint32_t IDESC = tc::idesc_bf16_f32(2 * TM, TN);
    tc::mbar_wait_warp(tc::smem_u32(&sm->qpair), 0);
    if (KBV > KB_TMEM) tc::mbar_wait_warp(tc::smem_u32(&sm->atail), 0);
    tc::fence_after();
    const uint64_t dbase = tc::desc_kmajor_sw128(ring_s);
    const uint64_t abase = tc::desc_kmajor_sw128(region_s);  // A tail (KBV = 16)
    int my_ep = 0;
    for (int64_t l = warp == 1 ? 0 : 1;; l += 2) {
      tc::mbar_wait_warp(tc::smem_u32(&sm->invfull[l & (INV_SLOTS - 1)]), (uint32_t)((l >> 3) & 1));
      const int64_t pk = __shfl_sync(0xffffffffu, (long long)sm->tile_id[l & (INV_SLOTS - 1)], 0);  // uniform
      if (pk < 0) break;
      if (epoch_of(pk) != my_ep) {  // both CTAs reloaded their prompt halves of the new pair slice
        my_ep = epoch_of(pk);
        tc::mbar_wait_warp(tc::smem_u32(&sm->qpair), (uint32_t)(my_ep & 1));
        tc::fence_after();
      }
      const int b = (int)(l & 1);
      tc::mbar_wait_warp(tc::smem_u32(&sm->tempty[b]), (uint32_t)(((l >> 1) & 1) ^ 1));
      tc::fence_after();
      const uint32_t d_tmem = tmem + ACC_COL0 + b * TN;
#pragma unroll
      for (int hh = 0; hh < SPT; ++hh) {
        const int64_t u = SPT * l + hh;
        const int sl = (int)(u & (NSLOT - 1));
        tc::mbar_wait_warp(tc::smem_u32(&sm->full[sl]), (uint32_t)((u >> 3) & 1));
        tc::fence_after();
        const int kb0 = KB * hh / SPT, kb1 = KB * (hh + 1) / SPT;
        const uint64_t dslot = dbase + (uint64_t)((sl * SH::SLOT_BYTES) >> 4);
#pragma unroll
        for (int j = 0; j < kb1 - kb0; ++j) {
          const int kb = kb0 + j;
          if (KBV == KB_TMEM || kb < KB_TMEM) {
#pragma unroll
            for (int kk = 0; kk < KBLK / 16; ++kk)
              tc::mma_ts_pair_warp(d_tmem, tmem + (uint32_t)((kb * (KBLK / 16) + kk) * 8),
                                   dslot + (uint64_t)((j * BOX_BYTES + kk * 32) >> 4), IDESC, (kb | kk) != 0);
          } else {  // A tail from shared memory (each CTA holds its 128 rows at this offset)
#pragma unroll
            for (int kk = 0; kk < KBLK / 16; ++kk)
              tc::mma_ss_pair_warp(d_tmem, abase + (uint64_t)(((kb - KB_TMEM) * QBOX_BYTES + kk * 32) >> 4),
                                   dslot + (uint64_t)((j * BOX_BYTES + kk * 32) >> 4), IDESC, 1u);
          }
        }
        tc::mma_commit_pair_warp(tc::smem_u32(&sm->empty[sl]), (uint16_t)0x3);  // slot free in both CTAs
      }
      tc::mma_commit_pair_warp(tc::smem_u32(&sm->afull[b]), (uint16_t)0x3);    // accumulator b final in both
    }
  } else if (warp >= 4) {
    // ======================= this CTA's prompt slice into TMEM, then the epilogue
    const int q = warp & 3;
    const int h = (warp - 4) >> 2;          // column half of every tile (32 of the 64 rows)
    const int p_local = q * 32 + lane;
    const int p0 = pbase + p_local;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t tempty_c[2] = {tc::mapa(tc::smem_u32(&sm->tempty[0]), 0), tc::mapa(tc::smem_u32(&sm->tempty[1]), 0)};
    {
      tc::mbar_wait(tc::smem_u32(&sm->qfull), 0);
      const int sw = p_local & 7;
      const int KBT = KB < KB_TMEM ? KB : KB_TMEM;
      for (int c = h; c < KBT; c += 2) {
        const uint32_t row = region_s + (uint32_t)(c * QBOX_BYTES + p_local * 128);
        uint32_t r[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 u4 = tc::lds_u32x4(row + (uint32_t)((j ^ sw) << 4));
          r[4 * j + 0] = u4.x;
          r[4 * j + 1] = u4.y;
          r[4 * j + 2] = u4.z;
          r[4 * j + 3] = u4.w;
        }
        tc::tmem_st32(tmem + lane_base + (uint32_t)(c * 32), r);
      }
      tc::tmem_wait_st();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc::fence_before();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(tc::smem_u32(&sm->qlocal));
        tc::mbar_arrive_cluster_relaxed(tc::mapa(tc::smem_u32(&sm->qpair), 0));
      }
    }
    const uint32_t scratch = region_s + (uint32_t)(REGION_BYTES + SCRATCH_OFF + (warp - 4) * 512 * 4);
    // per-epoch state: the prompt this thread scores, its list, the shared threshold
    int p = p0;
    int slot = range;
    int my_ep = 0;
    bool active = p < a.N;
    float iq = a.inv_q[p];
    TopList<KMAX> tl;
    tl.clear();
    float thr = active ? -INFINITY : INFINITY;
    uint64_t* gthr_p = a.gthr + p;
    uint64_t published = 0;
    uint64_t gk = active ? __ldcg(reinterpret_cast<const unsigned long long*>(gthr_p)) : 0;
    // fold the two column halves of each prompt through the warps' slow-path scratch
    // (half 1 parks its list in its own scratch, half 0 of the same lane quarter merges)
    // and write one candidate list per (epoch, prompt) into list slot `slot`
    auto flush = [&]() {
      const uint32_t mine = scratch + (uint32_t)(lane * KMAX * 8);
      const uint32_t partner = mine + (uint32_t)(4 * 512 * 4);  // warp q + 8's scratch, same lane
      if (h == 1) {
#pragma unroll
        for (int t2 = 0; t2 < KMAX; ++t2) tc::sts_u64(mine + t2 * 8, tl.v[t2]);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
      if (h == 0 && active) {
#pragma unroll
        for (int t2 = 0; t2 < KMAX; ++t2) tl.insert(tc::lds_u64(partner + t2 * 8));
        uint64_t* out = a.partial + ((int64_t)slot * a.N + p) * a.k;
        if (a.migrate)  // a floater's slot may already hold its list from an earlier visit
#pragma unroll
          for (int t2 = 0; t2 < KMAX; ++t2)
            if (t2 < a.k) tl.insert(out[t2]);
#pragma unroll
        for (int t2 = 0; t2 < KMAX; ++t2)
          if (t2 < a.k) out[t2] = tl.v[t2];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");  // scratch free again
    };
    for (int64_t l = 0;; ++l) {
      __syncwarp();
      tc::mbar_wait(tc::smem_u32(&sm->invfull[l & (INV_SLOTS - 1)]), (uint32_t)((l >> 3) & 1));
      const int64_t pk = sm->tile_id[l & (INV_SLOTS - 1)];
      if (pk < 0) break;
      if (epoch_of(pk) != my_ep) {
        // Migration: every tile of the previous epoch is done (tiles are processed in
        // order and each one's accumulator was read after its MMAs, which read both
        // CTAs' A), so the old list is final and the A operand may be replaced by this
        // CTA's half of the new pair slice, loaded straight from global memory.
        flush();
        my_ep = epoch_of(pk);
        slot = slot_of(pk);
        p = pslice_of(pk) * 2 * TM + (int)crank * TM + p_local;
        const uint4* src = reinterpret_cast<const uint4*>(a.Xb + (int64_t)p * a.d);
        const int KBT = KB < KB_TMEM ? KB : KB_TMEM;
        for (int c = h; c < KBT; c += 2) {
          uint32_t r[32];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 u4 = __ldcg(src + c * 8 + j);
            r[4 * j + 0] = u4.x;
            r[4 * j + 1] = u4.y;
            r[4 * j + 2] = u4.z;
            r[4 * j + 3] = u4.w;
          }
          tc::tmem_st32(tmem + lane_base + (uint32_t)(c * 32), r);
        }
        if (KBV > KB_TMEM) {  // the A tail in shared memory, in the TMA's 128-byte swizzle
          const int sw = p_local & 7;
          for (int c = KB_TMEM + h; c < KB; c += 2)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint4 u4 = __ldcg(src + c * 8 + j);
              const uint32_t dst = region_s + (uint32_t)((c - KB_TMEM) * QBOX_BYTES + p_local * 128 + ((j ^ sw) << 4));
              asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(u4.x), "r"(u4.y), "r"(u4.z),
                           "r"(u4.w)
                           : "memory");
            }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        tc::tmem_wait_st();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(tc::mapa(tc::smem_u32(&sm->qpair), 0));  // release: smem A tail
        active = p < a.N;
        iq = a.inv_q[p];
        tl.clear();
        thr = active ? -INFINITY : INFINITY;
        gthr_p = a.gthr + p;
        published = 0;
        gk = active ? __ldcg(reinterpret_cast<const unsigned long long*>(gthr_p)) : 0;
      }
      const int64_t t = tile_of(pk);
      if (gk != 0) thr = fmaxf(thr, key_score(gk));
      const int b = (int)(l & 1);
      const int64_t j0 = t * TN + h * 32;
      tc::mbar_wait(tc::smem_u32(&sm->afull[b]), (uint32_t)((l >> 1) & 1));
      tc::fence_after();
      uint32_t v[32];
      tc::tmem_ld32(tmem + lane_base + ACC_COL0 + b * TN + h * 32, v);
      tc::tmem_wait_ld();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster_relaxed(tempty_c[b]);  // one arrival per warp, on the leader
      if (__any_sync(0xffffffffu, active)) {
        const uint32_t icp = tc::smem_u32(&sm->invc[l & (INV_SLOTS - 1)][h * 32]);
        const int64_t rem_rows = a.m_local - j0;
        const int cmax = rem_rows < 32 ? (rem_rows < 0 ? 0 : (int)rem_rows) : 32;
        if (a.dbg != nullptr && active) epi_dump(v, icp, iq, cmax, a.dbg + (int64_t)p * a.dbg_ld + j0);
        epi_chunk<KMAX>(v, icp, iq, cmax, (uint32_t)(j0 * a.world + a.rank), (uint32_t)a.world, a.head, a.capg, tl,
                        thr, scratch);
        if (active && tl.v[KMAX - 1] > published && tl.v[KMAX - 1] > gk) {
          published = tl.v[KMAX - 1];
          atomicMax(reinterpret_cast<unsigned long long*>(gthr_p), (unsigned long long)published);
        }
        if (active && (l & 3) == 3) gk = __ldcg(reinterpret_cast<const unsigned long long*>(gthr_p));
      }
    }
    flush();
  }

  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();  // no remote arrive / TMA signal may target a CTA that has left
  pdl_launch();
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc2(tmem, TMEM_COLS);
  }
}

// pair slices of 256 prompts; pairs per pair slice = candidate lists per prompt
int scan_pair_plan(int64_t m_local, int32_t N, int num_sms) {
  const int pslices = (N + 2 * TM - 1) / (2 * TM);
  int ranges = (num_sms / 2) / pslices;
  if (ranges < 1) ranges = 1;
  const int64_t n_chunks = ((m_local + TN - 1) / TN + CHUNK - 1) / CHUNK;
  if (ranges > n_chunks) ranges = (int)(n_chunks > 0 ? n_chunks : 1);
  return ranges;
}

// An even number of 128-prompt slices (N in (128, 256], (384, 512], ...): pairing
// them costs no extra tensor work.  With an odd number the last pair would compute a
// whole 128-row half for padding (33 % more MMA work at N = 257..384), which the
// halved TMA traffic does not pay for; those batches keep one slice per CTA.
bool scan_pair_supported(int d, int32_t N) {
  const int slices = (N + TM - 1) / TM;
  return d % KBLK == 0 && d / KBLK <= KB_MAX && slices >= 2 && slices % 2 == 0;
}

template <int KMAX, int KBV, int KBF = 0>
static cudaError_t launch_pair_variant(bool pdl, dim3 grid, cudaStream_t s, const CUtensorMap& tc32,
                                       const CUtensorMap& tq, const ScanArgs& a, int pslices, int64_t n_tiles,
                                       int l2mode) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_scan_pair<KMAX, KBV, KBF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  static bool told = false;
  if (!told && getenv("ARGUS_DEBUG")) {
    int nc = -1;
    cudaOccupancyMaxActiveClusters(&nc, (const void*)k_scan_pair<KMAX, KBV, KBF>, &cfg);
    fprintf(stderr, "argus: pair scan grid %u CTAs, max co-resident 2-CTA clusters %d\n", grid.x, nc);
    told = true;
  }
  return cudaLaunchKernelEx(&cfg, k_scan_pair<KMAX, KBV, KBF>, tc32, tq, a, pslices, n_tiles, l2mode);
}

cudaError_t launch_scan_pair(const ScanArgs& a, const CUtensorMap* tmap_c32, const CUtensorMap* tmap_q,
                             cudaStream_t s, bool pdl) {
  const int pslices = (a.N + 2 * TM - 1) / (2 * TM);
  const int64_t n_tiles = (a.m_local + TN - 1) / TN;
  const dim3 grid(a.migrate ? a.grid_ctas : 2 * pslices * a.P);
  // L2 policy of the cache stream: evict-first at every slice count.  Even when
  // several pair slices re-read a tile, evict-first is the lower-DRAM choice:
  // the slices run a few tiles apart, so a tile is re-read while it is still the
  // newest line in its set, and marking it evict-first keeps the older ring
  // traffic from pushing it out (C4 N = 8192: 9.71 GB normal, 8.24 GB evict-first
  // against 8.21 GB algorithmic; profiles/r02/l2_policy.md).  ARGUS_SCAN_L2 overrides.
  static int l2env = -2;
  if (l2env == -2) {
    const char* e = getenv("ARGUS_SCAN_L2");
    l2env = e ? atoi(e) : -1;
  }
  const int l2mode = l2env >= 0 ? l2env : 0;
  const bool wide = a.d / KBLK > KB_TMEM;
  const bool clip = a.d == KB_TMEM * KBLK;  // d = 768 (CLIP): compile-time k-block count
  const bool clip_h = a.d == KB_MAX * KBLK;  // d = 1024 (OpenCLIP-H)
  if (a.k <= 4) {
    if (clip) return launch_pair_variant<4, 12, 12>(pdl, grid, s, *tmap_c32, *tmap_q, a, pslices, n_tiles, l2mode);
    if (clip_h) return launch_pair_variant<4, 16, 16>(pdl, grid, s, *tmap_c32, *tmap_q, a, pslices, n_tiles, l2mode);
    return wide ? launch_pair_variant<4, 16>(pdl, grid, s, *tmap_c32, *tmap_q, a, pslices, n_tiles, l2mode)
                : launch_pair_variant<4, 12>(pdl, grid, s, *tmap_c32, *tmap_q, a, pslices, n_tiles, l2mode);
  }
  if (clip) return launch_pair_variant<8, 12, 12>(pdl, grid, s, *tmap_c32, *tmap_q, a, pslices, n_tiles, l2mode);
  if (clip_h) return launch_pair_variant<8, 16, 16>(pdl, grid, s, *tmap_c32, *tmap_q, a, pslices, n_tiles, l2mode);
  return wide ? launch_pair_variant<8, 16>(pdl, grid, s, *tmap_c32, *tmap_q, a, pslices, n_tiles, l2mode)
              : launch_pair_variant<8, 12>(pdl, grid, s, *tmap_c32, *tmap_q, a, pslices, n_tiles, l2mode);
}

}  // namespace argus
