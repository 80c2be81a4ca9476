// k_merge.cu -- K5: merge per-range / per-shard top-k candidate lists
// (SURVEY §8(a) row A3, steps 5-6).  Keys are unique (the global id is in the
// low word), so the merged result is independent of the order of the inputs:
// the same keys come out whether the cache was scanned by 1 CTA range or 296,
// on 1 GPU or 8 (G-invariance).
//
// One CTA of 4 warps per prompt: each warp folds a quarter of the P*k candidate
// keys into per-lane register lists (loads batched 8 deep so the L2 latency
// overlaps), reduces them to its top-k, and warp 0 merges the 4 warp lists.
#include "common.cuh"
#include "kernels.h"

namespace argus {

constexpr int MERGE_WARPS = 4;

template <int KMAX>
__global__ void __launch_bounds__(MERGE_WARPS * 32) k_merge_topk(const uint64_t* __restrict__ in, int P, int N, int k,
                                                               uint64_t* __restrict__ keys_out,
                                                               uint32_t* __restrict__ idx_out,
                                                               float* __restrict__ score_out) {
  const int i = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ uint64_t wl[MERGE_WARPS][KMAX];
  pdl_wait();
  TopList<KMAX> l;
  l.clear();
  const int total = P * k;
  const int per = (total + MERGE_WARPS - 1) / MERGE_WARPS;
  const int e0 = warp * per, e1 = min(total, e0 + per);
  constexpr int B = 8;
  for (int e = e0 + lane; e < e1; e += 32 * B) {
    uint64_t buf[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int ee = e + u * 32;
      uint64_t key = 0;
      if (ee < e1) {
        const int p = ee / k, t = ee - p * k;
        key = __ldg(reinterpret_cast<const unsigned long long*>(in) + ((int64_t)p * N + i) * k + t);
      }
      buf[u] = key;
    }
#pragma unroll
    for (int u = 0; u < B; ++u) l.insert_nb(buf[u]);
  }
  warp_merge_topk<KMAX>(l, k, wl[warp]);
  __syncthreads();
  pdl_launch();
  if (warp == 0) {
    TopList<KMAX> m;
    m.clear();
    if (lane < MERGE_WARPS * k) m.insert(wl[lane / k][lane % k]);
    __shared__ uint64_t out_s[KMAX];
    warp_merge_topk<KMAX>(m, k, out_s);
    __syncwarp();
    if (lane < k) {
      const uint64_t key = out_s[lane];
      if (keys_out) keys_out[(int64_t)i * k + lane] = key;
      if (idx_out) idx_out[(int64_t)i * k + lane] = key_id(key);
      if (score_out) score_out[(int64_t)i * k + lane] = key_score(key);
    }
  }
}

void launch_merge_topk(const uint64_t* in, int32_t P, int32_t N, int32_t k, uint64_t* keys_out,
                       uint32_t* idx_out, float* score_out, cudaStream_t s) {
  if (k <= 4)
    launch_pdl(k_merge_topk<4>, dim3(N), dim3(MERGE_WARPS * 32), 0, s, in, P, N, k, keys_out, idx_out, score_out);
  else
    launch_pdl(k_merge_topk<8>, dim3(N), dim3(MERGE_WARPS * 32), 0, s, in, P, N, k, keys_out, idx_out, score_out);
}


// ------------------------------------------------------------------ K5 + C-2 fused over peer memory
// The shard's merge of its P per-range lists, with the exchange step folded in: each
// prompt's k merged keys are stored straight into slot [rank] of every rank's inbox
// (NVLink peer stores through CUDA IPC mappings; the own inbox is local memory), and
// the launch's last CTA, after a system-scope fence, publishes the batch sequence
// number in every inbox's flag word [rank] with a release store.  The receivers' tails
// acquire the G flags before reading their inbox (one exchange of N*k
// keys per batch, here without an NCCL call or a separate kernel).  Inbox slots are
// double-buffered by batch parity; before storing into a peer's slot, each CTA waits
// (one acquire load per peer, normally already satisfied) until that peer's tail has
// consumed the batch that used the slot two batches ago, so no rank can overwrite keys
// a slower rank has not read yet, whatever the collectives' buffering lets run ahead.
namespace {
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
}  // namespace

template <int KMAX>
__global__ void __launch_bounds__(MERGE_WARPS * 32) k_merge_send(const uint64_t* __restrict__ in, int P, int N, int k,
                                                                P2PSend dst, int* ticket) {
  // a capped grid (at most one CTA per SM) loops over the prompts: CTAs spinning on a
  // credit can never fill the SMs a receiving tail needs to make that credit arrive
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ uint64_t wl[MERGE_WARPS][KMAX];
  __shared__ uint64_t out_s[KMAX];
  __shared__ int is_last;
  pdl_wait();
  if (threadIdx.x < dst.G && dst.seq > 2) {  // credit: peer's slot of this parity is free again
    const uint64_t t0 = gtime();
    while (ld_acquire_sys(dst.consumed[threadIdx.x]) + 2 < dst.seq) {
      __nanosleep(200);
      if (gtime() - t0 > P2P_TIMEOUT_NS) {
        atomicOr(dst.err, FLAG_PEER_TIMEOUT);
        break;
      }
    }
  }
  __syncthreads();
  const int total = P * k;
  const int per = (total + MERGE_WARPS - 1) / MERGE_WARPS;
  const int e0 = warp * per, e1 = min(total, e0 + per);
  constexpr int B = 8;
  for (int i = blockIdx.x; i < N; i += gridDim.x) {
    TopList<KMAX> l;
    l.clear();
    for (int e = e0 + lane; e < e1; e += 32 * B) {
      uint64_t buf[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int ee = e + u * 32;
        uint64_t key = 0;
        if (ee < e1) {
          const int p = ee / k, t = ee - p * k;
          key = __ldg(reinterpret_cast<const unsigned long long*>(in) + ((int64_t)p * N + i) * k + t);
        }
        buf[u] = key;
      }
#pragma unroll
      for (int u = 0; u < B; ++u) l.insert_nb(buf[u]);
    }
    warp_merge_topk<KMAX>(l, k, wl[warp]);
    __syncthreads();
    if (warp == 0) {
      TopList<KMAX> m;
      m.clear();
      if (lane < MERGE_WARPS * k) m.insert(wl[lane / k][lane % k]);
      warp_merge_topk<KMAX>(m, k, out_s);
      __syncwarp();
      // lane (g, t): key t of this prompt into inbox g, slot [rank][i]
      for (int x = lane; x < dst.G * k; x += 32) {
        const int g = x / k, t = x - g * k;
        dst.keys[g][((int64_t)dst.rank * N + i) * k + t] = out_s[t];
      }
    }
    __syncthreads();  // wl / out_s are reused by the next prompt
  }
  // The CTA's peer stores are released by its ticket increment (acq_rel, system scope,
  // after the CTA barrier, which makes every thread's stores part of thread 0's release);
  // the last CTA's increment acquires all of them and its release store of each flag
  // publishes them (cumulativity) -- no sequentially consistent system fence needed.
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t old;
    asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ticket) : "memory");
    is_last = old == gridDim.x - 1;
  }
  __syncthreads();
  pdl_launch();
  if (is_last && threadIdx.x < dst.G) {
    st_release_sys(dst.flag[threadIdx.x], dst.seq);
    if (threadIdx.x == 0) *ticket = 0;  // ready for the next launch (stream-ordered)
  }
}

void launch_merge_send(const uint64_t* in, int32_t P, int32_t N, int32_t k, const P2PSend& dst, int* ticket,
                       cudaStream_t s, bool pdl, int max_ctas) {
  const dim3 grid(N < max_ctas ? N : max_ctas);
  if (k <= 4)
    launch_pdl_opt(pdl, k_merge_send<4>, grid, dim3(MERGE_WARPS * 32), 0, s, in, P, N, k, dst, ticket);
  else
    launch_pdl_opt(pdl, k_merge_send<8>, grid, dim3(MERGE_WARPS * 32), 0, s, in, P, N, k, dst, ticket);
}

}  // namespace argus
