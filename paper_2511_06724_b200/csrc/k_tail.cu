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
// fragment is one coalesced 8-byte load.  In phase 2 one warp owns one prompt and
// lane v owns option v (L <= 32): masks are ballots, the preference rank is a
// 32-lane compare-count, scattered into the list pi_i that phase 3 consumes.  Phase 3
// runs the serial dictatorship 32 prompts at a time in one warp: each lane takes the
// first option of its pi_i with quota left, and the group commits up to the first
// lane whose option the earlier lanes used up (at most N/32 + L group steps).
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

#ifndef ARGUS_TAIL_TIMING
#define ARGUS_TAIL_TIMING 0  // diagnostics build only: device printf of phase timestamps
#endif

namespace argus {

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
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

static size_t phase1_bytes(int d, int k, int P_max) {
  return (size_t)PB * (d + 8) * 2 + sizeof(float) * ((size_t)TW * PB * 32 + (size_t)PB * 8) +
         sizeof(uint64_t) * (size_t)P_max * PB * k;
}
static size_t phase2_bytes(int H, int L) { return sizeof(float) * ((size_t)PB * H + (size_t)L * (H + 4)); }
static size_t phase3_bytes(int N, int L) {
  const int Lw = (L + 3) / 4 * 4;
  return sizeof(int32_t) * (size_t)N + (size_t)CH * Lw + sizeof(uint32_t) * CH + CH;
}

size_t tail_smem_bytes(int d, int k, int H, int L, int max_batch, int P_max) {
  size_t b = phase1_bytes(d, k, P_max);
  b = b > phase2_bytes(H, L) ? b : phase2_bytes(H, L);
  b = b > phase3_bytes(max_batch, L) ? b : phase3_bytes(max_batch, L);
  return b;
}

// ------------------------------------------------------------------ phase 3
__device__ void assign_all(const TailArgs& a, uint8_t* smraw) {
  const int N = a.N, L = a.L, Lw = a.Lw;
  int32_t* order_s = reinterpret_cast<int32_t*>(smraw);                  // [N]
  uint8_t* rk_s = smraw + sizeof(int32_t) * (size_t)N;                   // [CH][Lw]
  uint32_t* cm_s = reinterpret_cast<uint32_t*>(rk_s + (size_t)CH * Lw);  // [CH]
  uint8_t* opt_s = reinterpret_cast<uint8_t*>(cm_s + CH);                 // [CH] (option | 0x80 overflow)
  __shared__ int32_t base[NB];
  __shared__ int32_t tot[NB];
  __shared__ int32_t wcnt[TW][NB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // stable counting sort of prompts by |C_i|
  if (tid < NB) base[tid] = 0;
  __syncthreads();
  for (int i0 = 0; i0 < N; i0 += TT) {  // warp-aggregated histogram
    const int i = i0 + tid;
    const int b = i < N ? (int)__ldcg(a.ccount + i) : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, b);
    if (b >= 0 && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&base[b], __popc(peers));
  }
  __syncthreads();
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
  for (int c0 = 0; c0 < N; c0 += TT) {
    const int i = c0 + tid;
    const int b = i < N ? (int)__ldcg(a.ccount + i) : -1;
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

  // serial dictatorship over staged chunks
  __shared__ int32_t rem_s[32];
  if (tid < 32) {
    int c = tid < L ? (a.quota_dev ? a.quota_dev[tid] : a.quota[tid]) : 0;
    if (c < 0) {  // only reachable through the broadcast (the host API checks its own argument)
      atomicOr(a.flags, FLAG_INVALID_INPUT);
      c = 0;
    }
    rem_s[tid] = c;
  }
  bool any_overflow = false;
  const int W = Lw / 4;
  const uint32_t* rk32 = reinterpret_cast<const uint32_t*>(a.prefl);
  for (int c0 = 0; c0 < N; c0 += CH) {
    const int n = min(CH, N - c0);
    for (int t0 = tid; t0 < n; t0 += 4 * TT) {  // gather rows in priority order, 4 rows in flight
      int ii[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u * TT;
        ii[u] = t < n ? order_s[c0 + t] : -1;
      }
      uint32_t cm[4];
      uint32_t wd[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        cm[u] = ii[u] >= 0 ? __ldcg(a.cmask + ii[u]) : 0u;
#pragma unroll
        for (int w = 0; w < 8; ++w) wd[u][w] = (ii[u] >= 0 && w < W) ? __ldcg(rk32 + (int64_t)ii[u] * W + w) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u * TT;
        if (t < n) {
          cm_s[t] = cm[u];
#pragma unroll
          for (int w = 0; w < 8; ++w)
            if (w < W) reinterpret_cast<uint32_t*>(rk_s + (size_t)t * Lw)[w] = wd[u][w];
        }
      }
    }
    __syncthreads();
    if (warp == 0) {
      // Serial dictatorship, 32 prompts at a time.  Each lane takes the first option of
      // its pi_i that had quota left when the group started; the group's choices are
      // exactly the sequential ones up to the first lane whose option was used up by
      // earlier lanes of the group (running count >= remaining quota).  Those lanes
      // commit, the rest restart with the new quotas.  An option runs out at most once,
      // so a batch takes at most N/32 + L group steps.
      uint32_t avail = __ballot_sync(0xffffffffu, lane < L && rem_s[lane] > 0);
#pragma unroll 1
      for (int t = 0; t < n;) {
        const int j = t + lane;
        int choice = 0xFF;  // no admissible option with quota left: overflow
        if (j < n) {
          const uint8_t* row = rk_s + (size_t)j * Lw;
#pragma unroll 1
          for (int r = 0; r < Lw; ++r) {
            const int o = row[r];
            if (o == 0xFF) break;
            if ((avail >> o) & 1u) {
              choice = o;
              break;
            }
          }
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, choice);
        const int before = __popc(peers & ((1u << lane) - 1u));
        const bool ok = j >= n || choice == 0xFF || before < rem_s[choice];
        const uint32_t bad = __ballot_sync(0xffffffffu, !ok);
        const int take = min(bad ? __ffs(bad) - 1 : 32, n - t);  // >= 1: lane 0 is always ok
        __syncwarp();
        if (lane < take) {
          opt_s[j] = choice == 0xFF ? (uint8_t)0x80 : (uint8_t)choice;
          if (choice != 0xFF) atomicSub(&rem_s[choice], 1);
          any_overflow |= choice == 0xFF;
        }
        __syncwarp();
        avail = __ballot_sync(0xffffffffu, lane < L && rem_s[lane] > 0);
        t += take;
      }
    }
    __syncthreads();
    for (int t = tid; t < n; t += TT) {
      const int i = order_s[c0 + t];
      const int o = opt_s[t] & 0x7F;
      uint8_t st = __ldcg(a.status + i);
      if (opt_s[t] & 0x80) st |= 1u;         // ARGUS_ST_OVERFLOW (option 0)
      if (!((cm_s[t] >> o) & 1u)) st |= 2u;  // ARGUS_ST_NONCOMPLIANT
      a.status[i] = st;
      a.option_out[i] = o;
    }
    __syncthreads();
  }
  if (warp == 0 && __any_sync(0xffffffffu, any_overflow) && lane == 0) atomicOr(a.flags, FLAG_OVERFLOW);
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
__global__ void __launch_bounds__(TT) k_tail(TailArgs a) {
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
  uint64_t T[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint64_t U[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (ARGUS_TAIL_TIMING) T[0] = gtimer();
  pdl_wait();
  if (ARGUS_TAIL_TIMING) T[1] = gtimer();

  // stage the prompt block (rows past N in Xb are zero padding) with async copies
  for (int idx = tid; idx < PB * (d / 8); idx += TT) {
    const int p = idx / (d / 8), c = idx - p * (d / 8);
    cp_async16(xs + p * RS + c * 8, reinterpret_cast<const uint4*>(a.Xb + (int64_t)(i0 + p) * d) + c);
  }
  if (ARGUS_TAIL_TIMING) U[0] = gtimer();
  // ---- phase M: merge the P lists of k keys of each prompt of the block.  All of the
  // block's keys (P slabs of 16 prompts x k, contiguous per list) arrive with one burst of
  // async copies; then one half-warp per prompt folds them from shared memory.
  uint64_t* kst = reinterpret_cast<uint64_t*>(ss + PB * 8);  // [P][PB][k]
  // A list starts at (p * N + i0) * k keys: 16-byte aligned for every p only when N * k
  // is even (and the buffer itself is); otherwise the keys move 8 bytes at a time.
  if ((((a.N * k) & 1) | (int)(reinterpret_cast<uintptr_t>(a.keys_in) & 15)) == 0) {
    const int slab = PB * k / 2;  // 16-byte chunks per list
    for (int x = tid; x < a.P * slab; x += TT) {
      const int p = x / slab, c = x - p * slab;
      if (i0 * k + 2 * c < a.N * k)  // prompts past N: left unfilled, never read
        cp_async16(kst + (size_t)p * PB * k + 2 * c,
                   reinterpret_cast<const uint4*>(a.keys_in + ((int64_t)p * a.N + i0) * k) + c);
    }
  } else {
    const int slab = PB * k;  // keys per list
    for (int x = tid; x < a.P * slab; x += TT) {
      const int p = x / slab, e = x - p * slab;
      if (i0 * k + e < a.N * k)  // exactly the keys of prompts < N: nothing past the buffer
        cp_async8(kst + (size_t)p * PB * k + e, a.keys_in + ((int64_t)p * a.N + i0) * k + e);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if (ARGUS_TAIL_TIMING) U[0] = gtimer();
  {
    const int hl = lane & 15, pl = 2 * warp + (lane >> 4);
    const int i = i0 + pl;
    TopList<8> tl;
    tl.clear();
    if (pl < nP) {
      const int total = a.P * k;
#pragma unroll 1
      for (int e = hl; e < total; e += 16) {
        const int p = e / k, t = e - p * k;
        tl.insert(kst[((size_t)p * PB + pl) * k + t]);
      }
    }
    if (ARGUS_TAIL_TIMING) U[1] = gtimer();
    for (int t = 0; t < k; ++t) {  // half-warp extraction (keys unique apart from 0)
      const uint64_t m = half_max_u64(tl.v[0]);
      if (hl == 0) mk[pl][t] = m;
      if (m != 0 && tl.v[0] == m) {
#pragma unroll
        for (int q = 0; q < 7; ++q) tl.v[q] = tl.v[q + 1];
        tl.v[7] = 0;
      }
    }
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
  if (ARGUS_TAIL_TIMING) U[2] = gtimer();
  __syncthreads();
  if (ARGUS_TAIL_TIMING) T[2] = gtimer();

  // ---- phase 1: hidden units [32 cc, 32 cc + 32) for cc = blockIdx.y, blockIdx.y +
  // gridDim.y, ...; warp w takes a 1/8 slice of d.  gridDim.y = H / 32 spreads a block
  // over H / 32 CTAs (lowest latency); gridDim.y = 1 keeps the block in one CTA, so the
  // candidate lists are merged once, not H / 32 times, and a pipelined tail occupies
  // few SMs while the next batch's scan starts.
  for (int cc = blockIdx.y; cc < H / 32; cc += gridDim.y) {
    float w1s_r[2][8], b1_r[2];  // per-thread epilogue constants of this chunk
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = cc * 32 + ((tid + u * TT) & 31);
      b1_r[u] = __ldg(a.b1 + j);
#pragma unroll
      for (int q = 0; q < 8; ++q) w1s_r[u][q] = q < k ? __ldg(a.W1sT + q * H + j) : 0.f;
    }
    const int g = lane >> 2, t = lane & 3;
    const uint32_t* x32 = reinterpret_cast<const uint32_t*>(xs);
    const int RSW = RS / 2;
    const int KS = d / 16;
    const int ks0 = KS * warp / TW, ks1 = KS * (warp + 1) / TW;
    const uint2* wf = reinterpret_cast<const uint2*>(a.W1xF);
    float acc[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
    constexpr int KSW = 8;  // k-steps per warp for d <= 1024: all B fragments in one round trip
    uint2 bf[KSW][4];
#pragma unroll
    for (int q = 0; q < KSW; ++q)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
        bf[q][nt] = (ks0 + q < ks1) ? __ldg(wf + ((int64_t)(cc * 4 + nt) * KS + ks0 + q) * 32 + lane) : make_uint2(0, 0);
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
  if (ARGUS_TAIL_TIMING) T[3] = gtimer();
  __threadfence();
  __syncthreads();
  if (tid == 0) is_last = atomicAdd(&a.block_cnt[pb], 1) == (int)gridDim.y - 1;
  __syncthreads();
  pdl_launch();
  if (!is_last) return;

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
  float* w2s = hs + PB * H;                     // [L][H]
  for (int e = tid; e < PB * H / 4; e += TT) cp_async16(hs + 4 * e, a.hbuf + (int64_t)i0 * H + 4 * e);
  const int H4 = H + 4;  // padded W2 rows: lane v's float4 reads fall in different banks
  for (int e = tid; e < L * H / 4; e += TT) {
    const int v = e / (H / 4), j4 = e - v * (H / 4);
    cp_async16(w2s + v * H4 + 4 * j4, a.W2 + 4 * e);
  }
  cp_async_wait_all();
  __syncthreads();
  if (ARGUS_TAIL_TIMING) U[3] = gtimer();
#pragma unroll
  for (int r = 0; r < PB / TW; ++r) {
    const int p = warp + r * TW;
    if (p >= nP) break;
    const int i = i0 + p;
    const bool act = lane < L;
    // lane v owns option v: z_v = b2_v + sum_j W2[v][j] h_j, four interleaved partial
    // sums in a compact (not unrolled) loop -- this phase runs once per CTA from a cold
    // instruction cache, so code size, not arithmetic, is what costs here
    // With L <= 16 lanes v and v + 16 each take half of the hidden units of option v
    // and add their halves with one shuffle (fadd is commutative: both lanes get the
    // same bits), halving the loop on the tail's critical path.
    float z = 0.f;
    const bool split = L <= 16;
    const int ov = split ? (lane & 15) : lane;
    if (ov < L) {
      float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
      const float* w2r = w2s + ov * H4;
      const float* hp = hs + p * H;
      const int jb = split ? (lane >> 4) * (H / 2) : 0, je = split ? jb + H / 2 : H;
#pragma unroll 1
      for (int j = jb; j < je; j += 4) {
        const float4 w4 = *reinterpret_cast<const float4*>(w2r + j);
        const float4 h4 = *reinterpret_cast<const float4*>(hp + j);
        z0 = __fmaf_rn(w4.x, h4.x, z0);
        z1 = __fmaf_rn(w4.y, h4.y, z1);
        z2 = __fmaf_rn(w4.z, h4.z, z2);
        z3 = __fmaf_rn(w4.w, h4.w, z3);
      }
      z = __fadd_rn(__fadd_rn(z0, z1), __fadd_rn(z2, z3));
    }
    if (split) z = __fadd_rn(z, __shfl_xor_sync(0xffffffffu, z, 16));
    float rr = 0.f;
    if (act) {
      z = __fadd_rn(z, a.b2[lane]);
      rr = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z)));
      if (lane == 0) rr = 1.0f;
    }
    const float s1 = s1_r[r];
    const int ks_ = act ? a.kskip[lane] : 0;
    const float gate = act ? a.gate[lane] : 0.f;
    const bool gated_pass = act && ks_ != 0 && s1 >= gate;
    const bool adm = act && (lane == 0 || ks_ == 0 || s1 >= gate);
    const bool cmp = adm && rr >= a.delta;
    const uint32_t amask = __ballot_sync(0xffffffffu, adm);
    const uint32_t cmask = __ballot_sync(0xffffffffu, cmp);
    const uint32_t gmask = __ballot_sync(0xffffffffu, act && ks_ != 0);
    const uint32_t pmask = __ballot_sync(0xffffffffu, gated_pass);
    const float pth = act ? a.pth[lane] : 0.f;
    int rank = 0;
    for (int u = 0; u < L; ++u) {
      const float ru = __shfl_sync(0xffffffffu, rr, u);
      const float pu = __shfl_sync(0xffffffffu, pth, u);
      const bool before = ((amask >> u) & 1u) &&
                          (ru > rr || (ru == rr && (pu > pth || (pu == pth && u < lane))));
      rank += before ? 1 : 0;
    }
    if (act) a.rhat[(int64_t)i * L + lane] = rr;
    // pi_i as a list: admissible option v at its position, 0xFF after the last
    if (adm) a.prefl[(int64_t)i * a.Lw + rank] = (uint8_t)lane;
    if (lane < a.Lw && lane >= __popc(amask)) a.prefl[(int64_t)i * a.Lw + lane] = 0xFF;
    // optimal option o_i: the compliant option with the largest p_th, then
    // the larger r, then the lower index (DESIGN R18); option 0 is always compliant
    float kp = cmp ? pth : -INFINITY, kr = cmp ? rr : -INFINITY;
    int kv = lane;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const float op = __shfl_xor_sync(0xffffffffu, kp, s), orr = __shfl_xor_sync(0xffffffffu, kr, s);
      const int ov = __shfl_xor_sync(0xffffffffu, kv, s);
      if (op > kp || (op == kp && (orr > kr || (orr == kr && ov < kv)))) {
        kp = op;
        kr = orr;
        kv = ov;
      }
    }
    const int oi = kp == -INFINITY ? 0 : kv;
    uint8_t st = (gmask != 0 && pmask == 0) ? 4u /*ARGUS_ST_GATED_ALL*/ : 0u;
    if (a.policy == 1) {
      // PASM sample: u = Philox word >> 8 scaled by 2^-24 (exact), the
      // first option whose float32 running sum exceeds u, then the gate fallback
      const uint32_t x0 = philox_x0((uint32_t)i, a.seq_lo, a.seq_hi, 0u, a.seed_lo, a.seed_hi);
      const float u = (float)(x0 >> 8) * 5.9604644775390625e-8f;
      const bool hit = act && u < a.pasm_cdf[oi * 32 + lane];
      const uint32_t hm = __ballot_sync(0xffffffffu, hit);
      const int as = hm ? __ffs(hm) - 1 : (int)a.pasm_last[oi];
      const uint32_t below = amask & (as >= 31 ? 0xffffffffu : ((2u << as) - 1u));
      const int af = 31 - __clz(below);  // bit 0 is always admissible
      if (lane == 0) {
        a.option_out[i] = af;
        if (!((cmask >> af) & 1u)) st |= 2u;  // ARGUS_ST_NONCOMPLIANT
      }
    }
    if (lane == 0) {
      // K6 flags a non-finite / zero-norm prompt only where it runs (the root); every
      // rank sees the broadcast inv_q = 0 of that prompt, so every rank fails the call
      if (__ldg(a.inv_q + i) == 0.f) atomicOr(a.flags, FLAG_INVALID_INPUT);
      a.ccount[i] = (uint8_t)__popc(cmask);
      a.cmask[i] = cmask;
      a.status[i] = st;
      if (a.optimal_out) a.optimal_out[i] = oi;
      if (a.aff_win > 0 && i >= a.N - a.aff_win) a.aff_ring[(a.aff_pos0 + i) % a.aff_win] = (uint8_t)oi;
    }
  }

  // ---- phase 3: the last block to finish phase 2 runs the assignment for all N
  if (ARGUS_TAIL_TIMING) T[4] = gtimer();
  __threadfence();
  __syncthreads();
  if (tid == 0) is_last = atomicAdd(a.launch_cnt, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (tid == 0) *a.launch_cnt = 0;
  if (ARGUS_TAIL_TIMING) T[5] = gtimer();
  if (a.policy == 0) assign_all(a, smraw);
  if (a.n_workers > 0) {
    __syncthreads();  // option_out of this CTA's own phase 3 is visible to the block
    select_workers(a);
  }
  if (ARGUS_TAIL_TIMING) {
    T[6] = gtimer();
    if (tid == 0)
      printf("[tail] N=%d pdl %llu | pre-merge %llu loads %llu extract %llu cpwait %llu | layer1 %llu | ticket+stage2 %llu l2+A5 %llu | ticket %llu | assign %llu ns\n",
             a.N, (unsigned long long)(T[1] - T[0]), (unsigned long long)(U[0] - T[1]),
             (unsigned long long)(U[1] - U[0]), (unsigned long long)(U[2] - U[1]), (unsigned long long)(T[2] - U[2]),
             (unsigned long long)(T[3] - T[2]), (unsigned long long)(U[3] - T[3]), (unsigned long long)(T[4] - U[3]),
             (unsigned long long)(T[5] - T[4]), (unsigned long long)(T[6] - T[5]));
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
