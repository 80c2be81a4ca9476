// k_tail.cu -- everything after the scan, in ONE launch:
//
//   phase M  (every CTA)     merge the P candidate lists of its 16 prompts into the
//                            final top-k (K5 semantics; CTAs of a prompt block merge
//                            redundantly, blockIdx.y == 0 writes topk_idx / topk_score)
//   phase 1  (every CTA)     predictor layer 1 for 16 prompts x 32 hidden units:
//                            h = relu(W1x . bf16(x) + W1s . s + b1)
//   phase 2  (last CTA of a  layer 2 r_v = 1/(1+exp(-(W2 . h + b2)_v)), r_0 := 1 and A5:
//            prompt block)     A_i = {v : v = 0 or k_skip_v = 0 or s_i1 >= tau_v}
//                              C_i = {v in A_i : r_v >= delta}
//                              pi_i = A_i by (r desc, p_th desc, v asc)
//   phase 3  (last CTA of    priority (|C_i| asc, i asc) counting sort + serial dictatorship
//            the launch)       under the quotas c_v
//
// The "last CTA" elections are atomic tickets (reset by the winner for the next
// launch).  Fusing the four steps removes three kernel boundaries per batch; the
// only redundant work is the 8-fold merge of each prompt block's candidates.
//
// Layer 1 runs on mma.sync m16n8k16 (bf16, fp32 accumulate): the whole predictor is
// < 0.03 % of the scan's flops and this product (16 x d x 32 per CTA) is far below a
// tcgen05 tile.  W1x is pre-arranged at init in per-lane fragment order so each B
// fragment is one coalesced 8-byte load.  In phase 2 one warp owns two prompts and
// lane v owns option v (L <= 32): masks are ballots, the preference rank is a
// branch-free compare-count against the static (p_th, index) order, o_i three warp
// reductions, and pi_i goes to phase 3 in inverse form (rank of each option, one
// 32-byte row per prompt).  Phase 3 runs the serial dictatorship in one warp, one
// prompt per redux.sync step (lane = option) or, for large batches, 32 prompts per
// window step (lane = prompt; see assign_all).
#include <cstdio>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

#ifndef ARGUS_TAIL_TIMING
#define ARGUS_TAIL_TIMING 0  // diagnostics build only: device printf of phase timestamps
#endif

namespace argus {

// diagnostics build: thread 0 stamps %globaltimer into shared memory at phase boundaries
// (no registers held across the phases, so the instrumented kernel keeps the product's
// register allocation); the launch's last CTA prints them
__shared__ unsigned long long tail_ts[24];  // 20: clock64 at entry
#define TS(i)                                                   \
  do {                                                          \
    if (ARGUS_TAIL_TIMING && threadIdx.x == 0) tail_ts[i] = gtimer(); \
  } while (0)

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}


constexpr int PB = 16;  // prompts per block (the MMA M dimension)
constexpr int TT = 256;  // threads per CTA
constexpr int TW = TT / 32;
constexpr int NB = 33;   // |C_i| in [1, 32]
constexpr int CH = 1024; // prompts per staged assignment chunk

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint2 b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

__device__ __forceinline__ uint64_t half_max_u64(uint64_t x) {  // max over the 16 lanes of a half-warp
#pragma unroll
  for (int m = 8; m > 0; m >>= 1) {
    const uint64_t y = shfl_xor_u64(x, m);
    x = y > x ? y : x;
  }
  return x;
}

// Shared-memory layout of phases M / 1: [xs: PB x (d + 8) bf16][red: TW x PB x 32 f32][ss: PB x 8 f32]
// [kst: P x PB x k u64].  Phase 2: [hs: PB x H f32] at 0 and W2 (rows padded to H + 4) at
// w2_off = max(kst offset, PB H 4): the kst area is dead once the lists are merged, so W2 is
// prefetched there during phase 1 and never collides with hs.
__host__ __device__ __forceinline__ size_t kst_offset(int d) {
  return (size_t)PB * (d + 8) * 2 + sizeof(float) * ((size_t)TW * PB * 32 + (size_t)PB * 8);
}
__host__ __device__ __forceinline__ size_t w2_offset(int d, int H) {
  const size_t a = kst_offset(d), b = sizeof(float) * (size_t)PB * H;
  return a > b ? a : b;
}
// Staged candidate lists are list-major with a padded list stride of S(k) keys: a list's
// 16 prompts x k keys plus k pad keys (17 k, rounded up to even so every list starts on a
// 16-byte boundary for the bulk copies).  With k | 16 the 16 / k lists a half-warp reads
// at once then start k keys apart modulo 16 keys (32 banks): conflict-free.
__host__ __device__ __forceinline__ int list_stride(int k) { return 17 * k + (k & 1); }
static size_t phase1_bytes(int d, int k, int P_max) {
  return kst_offset(d) + sizeof(uint64_t) * (size_t)P_max * list_stride(k);
}
static size_t phase2_bytes(int d, int H, int L) {
  return w2_offset(d, H) + sizeof(float) * ((size_t)L * (H + 4) + (size_t)TW * (PB / TW) * 32 + 32);  // W2 | r | p_th
}
// Phase 3 layout: [order: N i32][cc: N u8, padded to 16][rk: CH x 32 u8][cm: CH u32][st: CH u8]
// [opt: CH u8][lst: 32 x 32 u8, the window warp's per-lane pi as a list].
// rk rows are pi_i in inverse form (rank of option v in pi_i, 0xFF if v is not admissible),
// as phase 2 writes them.  With N <= CH ("by index") rk / cm / st hold every prompt's row
// at its index, staged in the same round trip as |C_i|; larger batches stage rows chunk by
// chunk in priority order.
__host__ __device__ __forceinline__ size_t p3_rk_offset(int N) {  // 16-byte aligned
  return ((sizeof(int32_t) * (size_t)N + 15) & ~(size_t)15) + (((size_t)N + 15) & ~(size_t)15);
}
static size_t phase3_bytes(int N) {
  return p3_rk_offset(N) + (size_t)CH * 32 + sizeof(uint32_t) * CH + 2 * (size_t)CH + 32 * 32;
}

size_t tail_smem_bytes(int d, int k, int H, int L, int max_batch, int P_max) {
  size_t b = phase1_bytes(d, k, P_max);
  b = b > phase2_bytes(d, H, L) ? b : phase2_bytes(d, H, L);
  b = b > phase3_bytes(max_batch) ? b : phase3_bytes(max_batch);
  return b;
}

// ------------------------------------------------------------------ phase 3
// Serial dictatorship: prompts in priority order, each takes the first option of
// its pi_i whose quota is not used up.  Two exact schedules of the same sequential result:
//  * one prompt per step (small batches): lane v = option v offers its rank in pi_i while
//    rem_v > 0; the prompt's choice is the lane of the minimum offer (one redux.sync), and
//    that lane decrements rem_v -- select, redux, compare, decrement per prompt (67 cycles
//    on one warp, tools/sd_bench.cu);
//  * windows of 32 prompts (large batches), lane = prompt: every pending lane takes the
//    first option of its pi with quota left; the choices equal the sequential ones up to the
//    first lane whose option earlier pending lanes used up (their count >= rem), so those
//    lanes commit and the rest retry.  An option runs out at most once, so a window takes at
//    most 1 + L steps (about 615 cycles each).
// On one warp (tools/sd_bench.cu) the per-prompt schedule takes 67 N cycles and the windows
// about 615 (N / 32 + L); inside the tail (cold code, the timing build's phase stamps) 85-90
// cycles per prompt against 1300 per window step, so prompts go one per step up to
// TailArgs::sd_pp_max = 512 (equal times there), windows beyond.
__device__ void assign_all(const TailArgs& a, uint8_t* smraw) {
  const int N = a.N, L = a.L;
  const bool byidx = N <= CH;
  const bool small = N <= TT;  // priority order by a compare-count instead of the counting sort
  const bool pp = byidx && N <= a.sd_pp_max;
  int32_t* order_s = reinterpret_cast<int32_t*>(smraw);                   // [N]
  uint8_t* cc_s = smraw + sizeof(int32_t) * (size_t)N;                    // [N]
  uint8_t* rk_s = smraw + p3_rk_offset(N);                                 // [CH][32]
  uint32_t* cm_s = reinterpret_cast<uint32_t*>(rk_s + (size_t)CH * 32);   // [CH]
  uint8_t* st_s = reinterpret_cast<uint8_t*>(cm_s + CH);                   // [CH]
  uint8_t* opt_s = st_s + CH;                                              // [CH] (option | 0x80 overflow)
  __shared__ int32_t base[NB];
  __shared__ int32_t tot[NB];
  __shared__ int32_t wcnt[TW][NB];
  __shared__ int32_t rem_s[32];
  __shared__ __align__(16) uint16_t key_s[TT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint4* rk16 = reinterpret_cast<const uint4*>(a.prefl);
  TS(12);

  // one round trip: |C_i| of every prompt (and, by index, its mask, pi_i and status)
  if (tid < NB) base[tid] = 0;
  if (tid < 32) {
    int c = tid < L ? (a.quota_dev ? a.quota_dev[tid] : a.quota[tid]) : 0;
    if (c < 0) {  // only reachable through the broadcast (the host API checks its own argument)
      atomicOr(a.flags, FLAG_INVALID_INPUT);
      c = 0;
    }
    rem_s[tid] = c;
  }
  if (small) {
    // priority position of prompt i = #{j : (|C_j|, j) < (|C_i|, i)}: 16-bit keys |C| << 10 | i
    const int i = tid;
    uint32_t key = 0xFFFFu;
    if (i < N) {
      const int b = (int)__ldcg(a.ccount + i);
      cm_s[i] = __ldcg(a.cmask + i);
      st_s[i] = __ldcg(a.status + i);
      const uint4 w0 = __ldcg(rk16 + 2 * i), w1 = __ldcg(rk16 + 2 * i + 1);
      reinterpret_cast<uint4*>(rk_s)[2 * i] = w0;
      reinterpret_cast<uint4*>(rk_s)[2 * i + 1] = w1;
      key = (uint32_t)b << 10 | (uint32_t)i;
    }
    key_s[tid] = (uint16_t)key;
    __syncthreads();
    TS(13);
    if (i < N) {
      int pos = 0;
      const uint4* k4 = reinterpret_cast<const uint4*>(key_s);
#pragma unroll 2
      for (int j8 = 0; j8 < (N + 7) / 8; ++j8) {  // 8 keys per 16-byte broadcast read
        const uint4 w = k4[j8];
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) pos += (int)((ws[h] & 0xFFFFu) < key) + (int)((ws[h] >> 16) < key);
      }
      order_s[pos] = i;
    }
    __syncthreads();
  } else {
    // counting sort by |C_i| (stable): warp-aggregated histogram, scan, ordered scatter
    __syncthreads();
    for (int i0 = 0; i0 < N; i0 += TT) {
      const int i = i0 + tid;
      const int b = i < N ? (int)__ldcg(a.ccount + i) : -1;
      if (byidx && i < N) {
        cm_s[i] = __ldcg(a.cmask + i);
        st_s[i] = __ldcg(a.status + i);
        const uint4 w0 = __ldcg(rk16 + 2 * i), w1 = __ldcg(rk16 + 2 * i + 1);
        reinterpret_cast<uint4*>(rk_s)[2 * i] = w0;
        reinterpret_cast<uint4*>(rk_s)[2 * i + 1] = w1;
      }
      if (i < N) cc_s[i] = (uint8_t)b;
      const uint32_t peers = __match_any_sync(0xffffffffu, b);
      if (b >= 0 && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&base[b], __popc(peers));
    }
    __syncthreads();
    TS(13);
    if (warp == 0) {  // exclusive scan of the 33 bucket counts
      const int c0 = base[lane];
      int x = c0;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, m);
        if (lane >= m) x += y;
      }
      const int tot31 = __shfl_sync(0xffffffffu, x, 31);
      base[lane] = x - c0;
      if (lane == 0) base[32] = tot31;
    }
    __syncthreads();
    for (int c0 = 0; c0 < N; c0 += TT) {  // stable scatter into priority order
      const int i = c0 + tid;
      const int b = i < N ? (int)cc_s[i] : -1;
      for (int x = tid; x < TW * NB; x += TT) (&wcnt[0][0])[x] = 0;
      __syncthreads();
      const uint32_t peers = __match_any_sync(0xffffffffu, b);
      const int wrank = __popc(peers & ((1u << lane) - 1u));
      if (b >= 0 && wrank == 0) wcnt[warp][b] = __popc(peers);
      __syncthreads();
      if (tid < NB) {
        int run = 0;
#pragma unroll
        for (int w = 0; w < TW; ++w) { const int c = wcnt[w][tid]; wcnt[w][tid] = run; run += c; }
        tot[tid] = run;
      }
      __syncthreads();
      if (b >= 0) order_s[base[b] + wcnt[warp][b] + wrank] = i;
      __syncthreads();
      if (tid < NB) base[tid] += tot[tid];
    }
    __syncthreads();
  }

  TS(14);
  bool any_overflow = false;
  int rem_r = rem_s[lane];  // warp 0: lane v holds rem_v
  if (ARGUS_TAIL_TIMING && tid == 0) tail_ts[22] = 0;
  if (pp) {
    if (warp == 0) {
      // the rows of the next 4 prompts are read while the current 4 are decided, so the
      // chain per prompt is only select -> redux -> compare -> decrement
      auto rows4 = [&](int t0, uint32_t (&rk)[4]) {
#pragma unroll
        for (int u = 0; u < 4; ++u) rk[u] = t0 + u < N ? rk_s[(size_t)order_s[t0 + u] * 32 + lane] : 0xFFu;
      };
      uint32_t cur[4], nxt[4];
      rows4(0, cur);
#pragma unroll 1
      for (int t0 = 0; t0 < N; t0 += 4) {
        rows4(t0 + 4, nxt);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t mine = cur[u] << 5 | (uint32_t)lane;
          const uint32_t offer = (rem_r > 0 && cur[u] != 0xFFu) ? mine : 0xFFFFu;
          const uint32_t m = __reduce_min_sync(0xffffffffu, offer);
          rem_r -= (m == mine) ? 1 : 0;  // only the chosen lane's offer equals m
          const bool live = t0 + u < N;
          if (lane == 0 && live) opt_s[t0 + u] = m == 0xFFFFu ? (uint8_t)0x80 : (uint8_t)(m & 31u);
          any_overflow |= live && m == 0xFFFFu;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
      }
      if (ARGUS_TAIL_TIMING && lane == 0) tail_ts[22] = N;
    }
    __syncthreads();
    TS(15);
    for (int t = tid; t < N; t += TT) {
      const int i = order_s[t];
      const int o = opt_s[t] & 0x7F;
      uint8_t st = st_s[i];
      if (opt_s[t] & 0x80) st |= 1u;              // ARGUS_ST_OVERFLOW (option 0)
      if (!((cm_s[i] >> o) & 1u)) st |= 2u;       // ARGUS_ST_NONCOMPLIANT
      a.status[i] = st;
      a.option_out[i] = o;
    }
  } else {
    uint32_t avail_r = __ballot_sync(0xffffffffu, lane < L && rem_r > 0);
    for (int c0 = 0; c0 < N; c0 += CH) {
      const int n = min(CH, N - c0);
      if (!byidx) {
        for (int t0 = tid; t0 < n; t0 += 4 * TT) {  // gather rows in priority order, 4 rows in flight
          int ii[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int t = t0 + u * TT;
            ii[u] = t < n ? order_s[c0 + t] : -1;
          }
          uint32_t cm[4];
          uint8_t st[4];
          uint4 wd[4][2];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            cm[u] = ii[u] >= 0 ? __ldcg(a.cmask + ii[u]) : 0u;
            st[u] = ii[u] >= 0 ? __ldcg(a.status + ii[u]) : (uint8_t)0;
            wd[u][0] = ii[u] >= 0 ? __ldcg(rk16 + 2 * ii[u]) : make_uint4(0, 0, 0, 0);
            wd[u][1] = ii[u] >= 0 ? __ldcg(rk16 + 2 * ii[u] + 1) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int t = t0 + u * TT;
            if (t < n) {
              cm_s[t] = cm[u];
              st_s[t] = st[u];
              reinterpret_cast<uint4*>(rk_s)[2 * t] = wd[u][0];
              reinterpret_cast<uint4*>(rk_s)[2 * t + 1] = wd[u][1];
            }
          }
        }
        __syncthreads();
      }
      if (warp == 0) {
        // lane = rank in the window; each lane keeps the ranks (positions in its pi) still
        // available as a bit mask A, clears the rank of each option that ran out (its row of
        // rk_s is the inverse of pi) and reads its choice at the lowest remaining rank from
        // its pi as a list (lst, built from the inverse row)
        uint8_t* lst = opt_s + CH + lane * 32;
#pragma unroll 1
        for (int t0 = 0; t0 < n; t0 += 32) {
          const int jj = t0 + lane;
          const bool act = jj < n;
          const uint8_t* inv = rk_s + (size_t)(act ? (byidx ? order_s[c0 + jj] : jj) : 0) * 32;
          uint32_t A = 0;  // ranks whose option has quota left
          if (act) {  // branch-free: predicated stores, masks by select
            const uint32_t* inv32 = reinterpret_cast<const uint32_t*>(inv);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (4 * q < L) {  // uniform
                const uint32_t w = inv32[q];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                  const int v = 4 * q + b;
                  const uint32_t r = (w >> (8 * b)) & 0xFFu;  // 0xFF for v >= L too
                  const bool ok = r != 0xFFu;
                  if (ok) lst[r] = (uint8_t)v;
                  A |= (ok && ((avail_r >> v) & 1u)) ? (1u << (r & 31u)) : 0u;
                }
              }
            }
          }
          __syncwarp();
          uint32_t pending = __ballot_sync(0xffffffffu, act);
          const uint32_t lt = (1u << lane) - 1u;
          uint32_t seen = avail_r;  // options whose exhaustion A already reflects
#pragma unroll 1
          while (pending) {
            for (uint32_t ex = seen & ~avail_r; ex; ex &= ex - 1) {  // options that ran out
              const uint32_t r = inv[__ffs(ex) - 1];
              if (r != 0xFFu) A &= ~(1u << r);
            }
            seen = avail_r;
            const bool mine = (pending >> lane) & 1u;
            const int choice = A ? (int)lst[__ffs(A) - 1] : 0xFF;  // 0xFF: no quota left, overflow
            // lanes with the same choice from five bit-ballots
            const bool real = mine && choice != 0xFF;
            const uint32_t V = __ballot_sync(0xffffffffu, real);
            uint32_t same = V, mv = V;  // lanes choosing my option / choosing option `lane`
#pragma unroll
            for (int b = 0; b < 5; ++b) {
              const uint32_t B = __ballot_sync(0xffffffffu, real && ((choice >> b) & 1));
              same &= ((choice >> b) & 1) ? B : ~B;
              mv &= ((lane >> b) & 1) ? B : ~B;
            }
            const int before = __popc(same & lt);
            const int remc = __shfl_sync(0xffffffffu, rem_r, choice & 31);
            const bool ok = !real || before < remc;
            const uint32_t bad = __ballot_sync(0xffffffffu, !ok);
            const uint32_t commit = bad ? (pending & ((1u << (__ffs(bad) - 1)) - 1u)) : pending;
            if ((commit >> lane) & 1u) {
              opt_s[jj] = choice == 0xFF ? (uint8_t)0x80 : (uint8_t)choice;
              any_overflow |= choice == 0xFF;
            }
            rem_r -= __popc(mv & commit);  // lane v: committed lanes that chose v
            avail_r = __ballot_sync(0xffffffffu, lane < L && rem_r > 0);
            pending &= ~commit;
            if (ARGUS_TAIL_TIMING && lane == 0) tail_ts[22]++;
          }
        }
      }
      __syncthreads();
      TS(15);
      for (int t = tid; t < n; t += TT) {
        const int i = order_s[c0 + t];
        const int row = byidx ? i : t;
        const int o = opt_s[t] & 0x7F;
        uint8_t st = st_s[row];
        if (opt_s[t] & 0x80) st |= 1u;              // ARGUS_ST_OVERFLOW (option 0)
        if (!((cm_s[row] >> o) & 1u)) st |= 2u;     // ARGUS_ST_NONCOMPLIANT
        a.status[i] = st;
        a.option_out[i] = o;
      }
      __syncthreads();
    }
  }
  if (warp == 0 && __any_sync(0xffffffffu, any_overflow) && lane == 0) atomicOr(a.flags, FLAG_OVERFLOW);
  TS(16);
}

// ------------------------------------------------------------------ F1: PASM sampling
// Philox4x32-10 (Salmon et al., SC'11), first output word only is used.
__device__ __forceinline__ uint32_t philox_x0(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                              uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c0;
}

// ------------------------------------------------------------------ F3: Eq. 3
// One warp per option v: lanes hold the workers serving v (<= 32, ascending id) and
// their queue lengths; the warp walks the batch in index order (ballots over 32
// prompts), and each prompt assigned v takes argmin (fl(float(R_w) * t_w), w), which
// then increments.  Options are independent, so warps run them concurrently.
__device__ void select_workers(const TailArgs& a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int v = warp; v < a.L; v += TW) {
    const int nw = a.wcount[v];
    const int w = lane < nw ? (int)a.wlist[v * 32 + lane] : 0x7fffffff;
    int q = lane < nw ? a.queue[w] : 0;
    const float t = lane < nw ? a.wtime[w] : 0.f;
    for (int c0 = 0; c0 < a.N; c0 += 32) {
      const int i = c0 + lane;
      const int o = i < a.N ? __ldcg(a.option_out + i) : -1;
      uint32_t m = __ballot_sync(0xffffffffu, o == v);
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        float cost = lane < nw ? __fmul_rn((float)q, t) : INFINITY;
        int who = w;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
          const float oc = __shfl_xor_sync(0xffffffffu, cost, s);
          const int ow = __shfl_xor_sync(0xffffffffu, who, s);
          if (oc < cost || (oc == cost && ow < who)) {
            cost = oc;
            who = ow;
          }
        }
        if (lane < nw && w == who) ++q;
        if (lane == 0 && a.worker_out) a.worker_out[c0 + b] = nw > 0 ? who : -1;
      }
    }
    if (lane < nw) a.queue[w] = q;
  }
}

// ------------------------------------------------------------------ the fused tail
// Phase M for one prompt, by the 16 lanes of a half-warp (lane hl): its P candidate lists
// of k keys are at kp[p * S + t] (list-major, padded stride S).  Every key goes through a
// branch-free insertion network (KM compare-exchanges into the lane's sorted register
// list).  Keys are unique, so the order of the inputs does not matter.
// merge_net<K>: k = K divides 16; the half-warp reads 16 / K whole lists per step (lane =
// list offset, key), conflict-free thanks to the padded stride, with every index a
// compile-time shift.  Measured on one SM (tools/merge_bench.cu), 148 lists of 4 keys:
// 2.6k cycles, against 12k for the same network with a runtime k, and 7-8k for an
// early-exit insert behind a data-dependent branch.
template <int KM>
__device__ __forceinline__ void net_insert(uint64_t (&v)[KM], uint64_t y) {
#pragma unroll
  for (int i = 0; i < KM; ++i) {  // v stays sorted descending; y carries the smaller
    const uint64_t hi = v[i] > y ? v[i] : y, lo = v[i] > y ? y : v[i];
    v[i] = hi;
    y = lo;
  }
}

template <int KM>
__device__ __forceinline__ void extract_topk(uint64_t (&v)[KM], int k, int hl, uint64_t* out) {
  for (int t = 0; t < k; ++t) {  // half-warp extraction (keys unique apart from 0)
    const uint64_t m = half_max_u64(v[0]);
    if (hl == 0) out[t] = m;
    if (m != 0 && v[0] == m) {
#pragma unroll
      for (int q = 0; q < KM - 1; ++q) v[q] = v[q + 1];
      v[KM - 1] = 0;
    }
  }
}

template <int K>
__device__ __forceinline__ void merge_net(const uint64_t* kp, int P, int hl, bool valid, uint64_t* out) {
  constexpr int S = 17 * K + (K & 1), G = 16 / K;
  const int po = hl / K, to = hl % K;
  uint64_t v[K];
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = 0;
  if (valid) {
    const uint64_t* q = kp + po * S + to;
#pragma unroll 4
    for (int p0 = 0; p0 < P; p0 += G) net_insert<K>(v, p0 + po < P ? q[p0 * S] : 0ull);
  }
  extract_topk<K>(v, K, hl, out);
}

// any k <= 8: every lane takes whole lists (k = 3, 5, 6, 7)
__device__ __forceinline__ void merge_any(const uint64_t* kp, int P, int k, int hl, bool valid, uint64_t* out) {
  const int S = list_stride(k);
  uint64_t v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = 0;
  if (valid) {
#pragma unroll 1
    for (int p = hl; p < P; p += 16)
      for (int t = 0; t < k; ++t) net_insert<8>(v, kp[(size_t)p * S + t]);
  }
  extract_topk<8>(v, k, hl, out);
}

__global__ void __launch_bounds__(TT, 1) k_tail(TailArgs a) {
  extern __shared__ __align__(16) uint8_t smraw[];
  __shared__ int is_last;
  __shared__ uint64_t mk[PB][8];  // merged top-k keys of the block (k <= 8)
  const int d = a.d, H = a.H, L = a.L, k = a.k;
  const int RS = d + 8;                                               // padded bf16 row stride
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(smraw);        // [PB][RS]
  float* red = reinterpret_cast<float*>(smraw + (size_t)PB * RS * 2);  // [TW][PB*32]
  float* ss = red + TW * PB * 32;                                     // [PB][k]
  const int pb = blockIdx.x;
  const int i0 = pb * PB;
  const int nP = min(PB, a.N - i0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  TS(0);
  if (ARGUS_TAIL_TIMING && tid == 0) tail_ts[20] = clock64();
  // phase-2 option constants of lane v (init-time data, nothing upstream writes them), read
  // before the predecessor finishes so phase 2 of the last CTA has no global round trip
  const bool act = lane < L;
  const float b2_v = act ? __ldg(a.b2 + lane) : 0.f;
  const int ks_v = act ? __ldg(a.kskip + lane) : 0;
  const float gate_v = act ? __ldg(a.gate + lane) : 0.f;
  const float pth_v = act ? __ldg(a.pth + lane) : 0.f;
  // the options' static order (init-time data): po_s[v] = position of v by (p_th desc, v asc),
  // pg_s[v] = #{u : p_th_u > p_th_v} (equal thresholds, equal value), for A5's rank and o_i
  __shared__ int po_s[32], pg_s[32];
  if (warp == 0) {
    int po = 0, pg = 0;
#pragma unroll 8
    for (int u = 0; u < 32; ++u) {
      const float pu = __shfl_sync(0xffffffffu, pth_v, u);
      const int in = u < L;
      pg += in & (int)(pu > pth_v);
      po += in & ((int)(pu > pth_v) | ((int)(pu == pth_v) & (int)(u < lane)));
    }
    po_s[lane] = po;
    pg_s[lane] = pg;
  }
  // layer-1 weights of this CTA's first hidden chunk (init-time data), also before the
  // predecessor finishes: B fragments of W1x, W1s and b1 columns
  constexpr int KSW = 8;  // k-steps per warp for d <= 1024: all B fragments in one round trip
  const int KS = d / 16;
  const int ks0 = KS * warp / TW, ks1 = KS * (warp + 1) / TW;
  const uint2* wf = reinterpret_cast<const uint2*>(a.W1xF);
  uint2 bf[KSW][4];
  float w1s_r[2][8], b1_r[2];
  auto load_w1 = [&](int cc) {
#pragma unroll
    for (int q = 0; q < KSW; ++q)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
        bf[q][nt] = (ks0 + q < ks1) ? __ldg(wf + ((int64_t)(cc * 4 + nt) * KS + ks0 + q) * 32 + lane) : make_uint2(0, 0);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = cc * 32 + ((tid + u * TT) & 31);
      b1_r[u] = __ldg(a.b1 + j);
#pragma unroll
      for (int q = 0; q < 8; ++q) w1s_r[u][q] = q < k ? __ldg(a.W1sT + q * H + j) : 0.f;
    }
  };
  load_w1(blockIdx.y);
  pdl_wait();
  if (a.p2p_flags != nullptr) {
    // fused exchange (k_merge_send): the P ranks' keys are in this rank's inbox once their
    // flags carry this batch's sequence number (acquire; the senders fenced at sys scope)
    if (tid < a.P) {
      const uint64_t t0 = gtimer();
      while (ld_acquire_sys(a.p2p_flags + tid) < a.p2p_seq) {
        __nanosleep(100);
        if (gtimer() - t0 > P2P_TIMEOUT_NS) {
          atomicOr(a.flags, FLAG_PEER_TIMEOUT);
          break;
        }
      }
    }
    __syncthreads();
  }
  TS(1);
  // inverse norm of prompt tid of the block (0 marks an invalid prompt): K6 flags such a
  // prompt only where it runs (the root); every rank sees the broadcast inv_q = 0, so every
  // rank fails the call.  Loaded here, tested once the staging copies have landed.
  const float iq = (blockIdx.y == 0 && tid < nP) ? __ldcg(a.inv_q + i0 + tid) : 1.f;

  // ---- stage the prompt block (16 rows of Xb; rows past N are zero padding) and the
  // block's candidate keys: list p's keys of prompts i0 .. i0 + nP - 1 are one contiguous
  // run at (p N + i0) k, copied by one warp (16-byte cp.async when the runs are 16-byte
  // aligned, i.e. k even, else 8-byte).  Measured: 2.4k cycles for 148 runs of 512 B,
  // against 9k for one TMA bulk copy per run (tools/merge_bench.cu).
  for (int idx = tid; idx < PB * (d / 8); idx += TT) {
    const int p = idx / (d / 8), c = idx - p * (d / 8);
    cp_async16(xs + p * RS + c * 8, reinterpret_cast<const uint4*>(a.Xb + (int64_t)(i0 + p) * d) + c);
  }
  uint64_t* kst = reinterpret_cast<uint64_t*>(ss + PB * 8);  // [P][S(k)]
  const int S = list_stride(k);
  if (((k & 1) | (int)(reinterpret_cast<uintptr_t>(a.keys_in) & 15)) == 0) {
    const int nc = nP * k / 2;  // 16-byte chunks of a run
    for (int p = warp; p < a.P; p += TW) {
      const uint64_t* src = a.keys_in + ((int64_t)p * a.N + i0) * k;
      for (int c = lane; c < nc; c += 32) cp_async16(kst + (size_t)p * S + 2 * c, src + 2 * c);
    }
  } else {
    const int nk = nP * k;
    for (int p = warp; p < a.P; p += TW) {
      const uint64_t* src = a.keys_in + ((int64_t)p * a.N + i0) * k;
      for (int e = lane; e < nk; e += 32) cp_async8(kst + (size_t)p * S + e, src + e);
    }
  }
  if (iq == 0.f) atomicOr(a.flags, FLAG_INVALID_INPUT);
  cp_async_wait_all();
  __syncthreads();
  TS(2);
  {
    const int hl = lane & 15, pl = 2 * warp + (lane >> 4);
    const int i = i0 + pl;
    const uint64_t* kp = kst + (size_t)pl * k;
    const bool valid = pl < nP;
    switch (k) {  // k = 0: SM mode, no candidate lists
      case 0: break;
      case 1: merge_net<1>(kp, a.P, hl, valid, mk[pl]); break;
      case 2: merge_net<2>(kp, a.P, hl, valid, mk[pl]); break;
      case 4: merge_net<4>(kp, a.P, hl, valid, mk[pl]); break;
      case 8: merge_net<8>(kp, a.P, hl, valid, mk[pl]); break;
      default: merge_any(kp, a.P, k, hl, valid, mk[pl]); break;
    }
    TS(3);
    __syncwarp();
    if (pl < nP && hl < k) {
      const uint64_t key = mk[pl][hl];
      ss[pl * k + hl] = key_score(key);
      if (blockIdx.y == 0) {
        const uint32_t age = key_id(key);  // 0xFFFFFFFF for an empty slot (M < k)
        a.topk_idx[(int64_t)i * k + hl] = key == 0 ? 0xFFFFFFFFu : a.id_base + age;
        a.topk_score[(int64_t)i * k + hl] = key_score(key);
        if (a.topk_handle) {
          uint32_t pos = a.head + age;
          if (a.capg && pos >= a.capg) pos -= a.capg;
          a.topk_handle[(int64_t)i * k + hl] = key == 0 ? 0ull : a.handle[pos];
        }
      }
    } else if (pl >= nP && hl < k) {
      ss[pl * k + hl] = 0.f;
    }
  }
  TS(4);
  __syncthreads();
  // the key staging area is free: prefetch W2 (rows padded to H + 4 so lane v's float4
  // reads fall in different banks) for phase 2, in case this CTA is the block's last
  float* w2s = reinterpret_cast<float*>(smraw + w2_offset(d, H));  // [L][H + 4]
  const int H4 = H + 4;
  for (int e = tid; e < L * H / 4; e += TT) {
    const int v = e / (H / 4), j4 = e - v * (H / 4);
    cp_async16(w2s + v * H4 + 4 * j4, a.W2 + 4 * e);
  }
  TS(5);

  // ---- phase 1: hidden units [32 cc, 32 cc + 32) for cc = blockIdx.y, blockIdx.y +
  // gridDim.y, ...; warp w takes a 1/8 slice of d.  gridDim.y = H / 32 spreads a block
  // over H / 32 CTAs (lowest latency); gridDim.y = 1 keeps the block in one CTA, so the
  // candidate lists are merged once, not H / 32 times, and a pipelined tail occupies
  // few SMs while the next batch's scan starts.
  for (int cc = blockIdx.y; cc < H / 32; cc += gridDim.y) {
    if (cc != (int)blockIdx.y) load_w1(cc);
    const int g = lane >> 2, t = lane & 3;
    const uint32_t* x32 = reinterpret_cast<const uint32_t*>(xs);
    const int RSW = RS / 2;
    float acc[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
#pragma unroll
    for (int q = 0; q < KSW; ++q) {
      if (ks0 + q < ks1) {
        const int ks = ks0 + q;
        uint32_t af[4];
        af[0] = x32[g * RSW + ks * 8 + t];
        af[1] = x32[(g + 8) * RSW + ks * 8 + t];
        af[2] = x32[g * RSW + ks * 8 + 4 + t];
        af[3] = x32[(g + 8) * RSW + ks * 8 + 4 + t];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) mma_bf16_16816(acc[nt], af, bf[q][nt]);
      }
    }
    float* rw = red + warp * PB * 32;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) rw[(g + (e >> 1) * 8) * 32 + nt * 8 + 2 * t + (e & 1)] = acc[nt][e];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {  // PB * 32 = 2 * TT: reduce split-K partials in a fixed order
      const int e = tid + u * TT;
      const int row = e >> 5, j = cc * 32 + (e & 31);
      float z = 0.f;
#pragma unroll
      for (int w = 0; w < TW; ++w) z = __fadd_rn(z, red[w * PB * 32 + e]);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < k) z = __fmaf_rn(w1s_r[u][q], ss[row * k + q], z);
      a.hbuf[(int64_t)(i0 + row) * H + j] = fmaxf(__fadd_rn(z, b1_r[u]), 0.f);
    }
    __syncthreads();  // red is reused by the next chunk
  }
  TS(6);
  __threadfence();
  __syncthreads();
  if (tid == 0) is_last = atomicAdd(&a.block_cnt[pb], 1) == (int)gridDim.y - 1;
  __syncthreads();
  pdl_launch();
  if (!is_last) {
    cp_async_wait_all();  // the W2 prefetch lands before the CTA retires
    return;
  }

  // ---- phase 2: layer 2 + A5 for the 16 prompts of this block
  __threadfence();
  if (tid == 0) a.block_cnt[pb] = 0;  // ready for the next launch
  float s1_r[PB / TW];
#pragma unroll
  for (int r = 0; r < PB / TW; ++r) {
    const int p = warp + r * TW;
    s1_r[r] = p < nP ? ss[p * k] : 0.f;
  }
  __syncthreads();  // ss (inside the staging area) is overwritten below
  float* hs = reinterpret_cast<float*>(smraw);  // [PB][H]
  for (int e = tid; e < PB * H / 4; e += TT) cp_async16(hs + 4 * e, a.hbuf + (int64_t)i0 * H + 4 * e);
  cp_async_wait_all();
  __syncthreads();
  TS(7);
  // layer 2 for both of this warp's prompts at once: lane v owns option v, z_v = b2_v +
  // sum_j W2[v][j] h_j as four interleaved partial sums per prompt.  With L <= 16 lanes v
  // and v + 16 each take half of the hidden units of option v and add their halves with
  // one shuffle (fadd is commutative: both lanes get the same bits).
  const bool split = L <= 16;
  const int ov = split ? (lane & 15) : lane;
  float zr[PB / TW];
  {
    float z[PB / TW][4];
#pragma unroll
    for (int r = 0; r < PB / TW; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) z[r][c] = 0.f;
    if (ov < L) {
      const float* w2r = w2s + ov * H4;
      const int jb = split ? (lane >> 4) * (H / 2) : 0, je = split ? jb + H / 2 : H;
#pragma unroll 2
      for (int j = jb; j < je; j += 4) {
        const float4 w4 = *reinterpret_cast<const float4*>(w2r + j);
#pragma unroll
        for (int r = 0; r < PB / TW; ++r) {
          const float4 h4 = *reinterpret_cast<const float4*>(hs + (warp + r * TW) * H + j);
          z[r][0] = __fmaf_rn(w4.x, h4.x, z[r][0]);
          z[r][1] = __fmaf_rn(w4.y, h4.y, z[r][1]);
          z[r][2] = __fmaf_rn(w4.z, h4.z, z[r][2]);
          z[r][3] = __fmaf_rn(w4.w, h4.w, z[r][3]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < PB / TW; ++r) {
      float zz = (ov < L) ? __fadd_rn(__fadd_rn(z[r][0], z[r][1]), __fadd_rn(z[r][2], z[r][3])) : 0.f;
      if (split) zz = __fadd_rn(zz, __shfl_xor_sync(0xffffffffu, zz, 16));
      zr[r] = zz;
    }
  }
  TS(8);
  // A5 for both prompts of the warp together (independent chains interleave): r_v, masks,
  // the preference rank of v from a per-warp shared table of r and the static option order
  // (po_s), o_i by three warp reductions; no data-dependent branches
  constexpr int R = PB / TW;
  float* rr_s = reinterpret_cast<float*>(smraw + w2_offset(d, H) + sizeof(float) * (size_t)L * H4) + warp * R * 32;
  float rr[R];
  uint32_t amask[R], cmask[R];
  bool adm[R], cmp[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    rr[r] = 0.f;
    if (act) {
      const float z = __fadd_rn(zr[r], b2_v);
      rr[r] = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z)));
      if (lane == 0) rr[r] = 1.0f;
    }
    rr_s[r * 32 + lane] = rr[r];
    const float s1 = s1_r[r];
    adm[r] = act && (lane == 0 || ks_v == 0 || s1 >= gate_v);
    cmp[r] = adm[r] && rr[r] >= a.delta;
    amask[r] = __ballot_sync(0xffffffffu, adm[r]);
    cmask[r] = __ballot_sync(0xffffffffu, cmp[r]);
  }
  const uint32_t gmask = __ballot_sync(0xffffffffu, act && ks_v != 0);
  uint32_t pmask[R];
#pragma unroll
  for (int r = 0; r < R; ++r) pmask[r] = __ballot_sync(0xffffffffu, act && ks_v != 0 && s1_r[r] >= gate_v);
  __syncwarp();  // rr_s of this warp
  TS(21);
  // rank of v in pi_i: admissible options before v by r desc, then p_th desc,
  // then index asc -- the last two are the static order po_s
  const int po_v = po_s[lane], pg_v = pg_s[lane];
  int rank[R], oi[R];
#pragma unroll
  for (int r = 0; r < R; ++r) rank[r] = 0;
#pragma unroll 4
  for (int u = 0; u < L; ++u) {
    const uint32_t pb = (uint32_t)(po_s[u] < po_v);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float ru = rr_s[r * 32 + u];
      rank[r] += (int)((amask[r] >> u) & ((uint32_t)(ru > rr[r]) | ((uint32_t)(ru == rr[r]) & pb)) & 1u);
    }
  }
  // o_i (DESIGN R18): the compliant option with the largest p_th, then the larger
  // r, then the lower index (r >= 0, so its bits order like the value)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool c = (cmask[r] >> lane) & 1u;
    const uint32_t m1 = __reduce_min_sync(0xffffffffu, c ? (uint32_t)pg_v : 0xFFu);
    const bool t1 = c && (uint32_t)pg_v == m1;
    const uint32_t rb = __float_as_uint(rr[r]) + 1u;
    const uint32_t m2 = __reduce_max_sync(0xffffffffu, t1 ? rb : 0u);
    const uint32_t w = __ballot_sync(0xffffffffu, t1 && rb == m2);
    oi[r] = w ? __ffs(w) - 1 : 0;
  }
  TS(18);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int p = warp + r * TW;
    if (p >= nP) break;
    const int i = i0 + p;
    if (act) a.rhat[(int64_t)i * L + lane] = rr[r];
    // pi_i in inverse form: rank of option v, 0xFF if v is not admissible
    a.prefl[(int64_t)i * 32 + lane] = adm[r] ? (uint8_t)rank[r] : (uint8_t)0xFF;
    uint8_t st = (gmask != 0 && pmask[r] == 0) ? 4u /*ARGUS_ST_GATED_ALL*/ : 0u;
    if (a.policy == 1) {
      // PASM sample: u = Philox word >> 8 scaled by 2^-24 (exact), the
      // first option whose float32 running sum exceeds u, then the gate fallback
      const uint32_t x0 = philox_x0((uint32_t)i, a.seq_lo, a.seq_hi, 0u, a.seed_lo, a.seed_hi);
      const float u = (float)(x0 >> 8) * 5.9604644775390625e-8f;
      const bool hit = act && u < a.pasm_cdf[oi[r] * 32 + lane];
      const uint32_t hm = __ballot_sync(0xffffffffu, hit);
      const int as = hm ? __ffs(hm) - 1 : (int)a.pasm_last[oi[r]];
      const uint32_t below = amask[r] & (as >= 31 ? 0xffffffffu : ((2u << as) - 1u));
      const int af = 31 - __clz(below);  // bit 0 is always admissible
      if (lane == 0) {
        a.option_out[i] = af;
        if (!((cmask[r] >> af) & 1u)) st |= 2u;  // ARGUS_ST_NONCOMPLIANT
      }
    }
    if (lane == 0) {
      a.ccount[i] = (uint8_t)__popc(cmask[r]);
      a.cmask[i] = cmask[r];
      a.status[i] = st;
      if (a.optimal_out) a.optimal_out[i] = oi[r];
      if (a.aff_win > 0 && i >= a.N - a.aff_win) a.aff_ring[(a.aff_pos0 + i) % a.aff_win] = (uint8_t)oi[r];
    }
  }
  TS(19);

  // ---- phase 3: the last block to finish phase 2 runs the assignment for all N
  TS(9);
  __threadfence();
  __syncthreads();
  if (tid == 0) is_last = atomicAdd(a.launch_cnt, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (tid == 0) *a.launch_cnt = 0;
  // every CTA of the launch has staged its inbox keys: the senders may reuse the slot
  if (a.p2p_consumed != nullptr && tid == 0) st_release_sys(a.p2p_consumed, a.p2p_seq);
  TS(10);
  if (a.policy == 0) assign_all(a, smraw);
  if (a.n_workers > 0) {
    __syncthreads();  // option_out of this CTA's own phase 3 is visible to the block
    select_workers(a);
  }
  if (ARGUS_TAIL_TIMING) {
    __syncthreads();
    TS(11);
    if (tid == 0) {
      const unsigned long long c1 = clock64();
      const unsigned long long* t = tail_ts;
      printf("[tail] N=%d MHz %.0f | pdl %llu stage %llu merge %llu out %llu w2 %llu layer1 %llu | ticket+h %llu l2dot %llu A5 %llu "
             "| ticket %llu | assign: load %llu sort %llu sd %llu write %llu | total %llu ns | P %d | A5[0]: sigm %llu rank %llu omax %llu | sd steps %llu\n",
             a.N, 1e3 * (double)(c1 - t[20]) / (double)(t[11] - t[0]), t[1] - t[0], t[2] - t[1], t[3] - t[2],
             t[4] - t[3], t[5] - t[4], t[6] - t[5], t[7] - t[6], t[8] - t[7], t[9] - t[8], t[10] - t[9],
             t[13] - t[12], t[14] - t[13], t[15] - t[14], t[16] - t[15], t[11] - t[0], a.P, t[21] - t[8], t[18] - t[21], t[19] - t[18], t[22]);
    }
  }
}

// W1x [H][d] (fp32 rows of w1 [H][d+k]) -> bf16 (RNE) in mma.sync B-fragment order:
// Wf[(nb * KS + ks) * 32 + lane] = {W[n][k0..k0+1], W[n][k0+8..k0+9]},
// n = nb * 8 + lane / 4, k0 = ks * 16 + (lane % 4) * 2.
__global__ void k_prep_w1_frag(const float* __restrict__ w1, int d, int k, int H, uint2* __restrict__ Wf) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int KS = d / 16;
  const int64_t total = (int64_t)(H / 8) * KS * 32;
  if (idx >= total) return;
  const int lane = (int)(idx & 31);
  const int64_t q = idx >> 5;
  const int ks = (int)(q % KS), nb = (int)(q / KS);
  const int n = nb * 8 + lane / 4, k0 = ks * 16 + (lane % 4) * 2;
  const float* row = w1 + (int64_t)n * (d + k);
  __nv_bfloat162 lo = __floats2bfloat162_rn(row[k0], row[k0 + 1]);
  __nv_bfloat162 hi = __floats2bfloat162_rn(row[k0 + 8], row[k0 + 9]);
  Wf[idx] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}

void launch_prep_w1_frag(const float* w1, int d, int k, int H, void* Wf, cudaStream_t s) {
  const int64_t total = (int64_t)(H / 8) * (d / 16) * 32;
  k_prep_w1_frag<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(w1, d, k, H, reinterpret_cast<uint2*>(Wf));
}

void launch_tail(const TailArgs& a, size_t smem, cudaStream_t s, bool pdl, int ysplit) {
  static size_t attr_set = 0;
  if (smem > attr_set) {
    cudaFuncSetAttribute(k_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = smem;
  }
  const int ys = ysplit < 1 ? 1 : (ysplit > a.H / 32 ? a.H / 32 : ysplit);
  const dim3 grid((a.N + PB - 1) / PB, ys);
  launch_pdl_opt(pdl, k_tail, grid, dim3(TT), smem, s, a);
}

}  // namespace argus
