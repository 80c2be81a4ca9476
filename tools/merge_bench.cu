// Microbenchmark: cycles of the tail's list-merge loop shapes on one CTA (diagnostics).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_06724_b200/csrc tools/merge_bench.cu -o tools/merge_bench
#include <cstdio>
#include <cstdint>
#include "common.cuh"
#include "tc.cuh"
using namespace argus;

__device__ __forceinline__ uint64_t half_max(uint64_t x) {
  for (int m = 8; m > 0; m >>= 1) { uint64_t y = shfl_xor_u64(x, m); x = y > x ? y : x; }
  return x;
}

constexpr int PB = 16;
__device__ __forceinline__ uint64_t half_max_u64(uint64_t x) { return half_max(x); }
__host__ __device__ __forceinline__ int list_stride(int k) { return 17 * k + (k & 1); }
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

__global__ void kmerge(const uint64_t* g, int P, int k, unsigned long long* out) {
  extern __shared__ uint64_t kst[];
  __shared__ uint64_t mk[16][8];
  for (int i = threadIdx.x; i < P * 68; i += blockDim.x) kst[i] = g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, hl = lane & 15, pl = (threadIdx.x >> 5) * 2 + (lane >> 4);
  unsigned long long t0 = clock64();
  merge_net<4>(kst + pl * k, P, hl, true, mk[pl]);
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = mk[0][0]; }
}

template <int MODE>
__global__ void kbench(const uint64_t* g, int P, int k, uint64_t lb, unsigned long long* out) {
  extern __shared__ uint64_t kst[];
  for (int i = threadIdx.x; i < P * 68; i += blockDim.x) kst[i] = g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, hl = lane & 15, pl = (threadIdx.x >> 5) * 2 + (lane >> 4);
  const uint64_t* kp = kst + pl * k;
  const int S = 68, gg = 4, po = hl / 4, to = hl & 3;
  unsigned long long t0 = clock64();
  TopList<4> tl;
  tl.clear();
  uint64_t acc = 0;
#pragma unroll 1
  for (int p0 = 0; p0 < (MODE == 4 ? 0 : P); p0 += gg) {
    const int p = p0 + po;
    const uint64_t x = p < P ? kp[p * S + to] : 0ull;
    if (MODE == 0) {
      acc ^= x;
    } else if (MODE == 1) {
      const bool cand = x != 0 && x >= lb;
      if (__any_sync(0xffffffffu, cand)) { if (cand) tl.insert(x); }
    } else if (MODE == 2) {
      if (x >= lb) tl.insert(x);
    } else if (MODE == 3) {  // branch-free insertion network
      uint64_t y = x;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t hi = tl.v[i] > y ? tl.v[i] : y, lo = tl.v[i] > y ? y : tl.v[i];
        tl.v[i] = hi;
        y = lo;
      }
    }
  }
  if (MODE == 4) {  // chunks of 8 keys: loads + candidate mask, then inserts of candidates only
#pragma unroll 1
    for (int p0 = 0; p0 < P; p0 += 8 * gg) {
      uint64_t xs[8];
      uint32_t mask = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int p = p0 + u * gg + po;
        xs[u] = p < P ? kp[p * S + to] : 0ull;
        mask |= (xs[u] >= lb && xs[u] > tl.v[3]) ? (1u << u) : 0u;
      }
      while (mask) {
        const int u = __ffs(mask) - 1;
        mask &= mask - 1;
        uint64_t y = xs[u];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint64_t hi = tl.v[i] > y ? tl.v[i] : y, lo = tl.v[i] > y ? y : tl.v[i];
          tl.v[i] = hi;
          y = lo;
        }
      }
    }
  }
  uint64_t m = half_max(tl.v[0]) ^ acc;
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = m; }
}

// staging of P lists x 512 B (16 prompts x 4 keys) from a [P][N][4] buffer
template <int MODE>
__global__ void kstage(const uint64_t* keys, int P, int N, unsigned long long* out) {
  extern __shared__ uint64_t kst[];
  __shared__ __align__(8) uint64_t bar_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t bar = tc::smem_u32(&bar_s);
  if (tid == 0) { tc::mbar_init(bar, 1); tc::fence_barrier_init(); }
  __syncthreads();
  unsigned long long t0 = clock64();
  if (MODE == 0) {  // bulk per list
    if (warp == 0) {
      if (lane == 0) tc::mbar_arrive_expect_tx(bar, P * 512);
      __syncwarp();
      for (int p = lane; p < P; p += 32) tc::bulk_load(tc::smem_u32(kst + p * 68), keys + (size_t)p * N * 4, 512, bar);
    }
    tc::mbar_wait(bar, 0);
  } else if (MODE == 1) {  // cp.async 16 B, thread per chunk (original layout)
    for (int x = tid; x < P * 32; x += 256) {
      const int p = x >> 5, c = x & 31;
      cp_async16(kst + p * 64 + 2 * c, keys + (size_t)p * N * 4 + 2 * c);
    }
    cp_async_wait_all();
  } else {  // plain 16 B loads into registers then st.shared
    for (int x = tid; x < P * 32; x += 256) {
      const int p = x >> 5, c = x & 31;
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(keys + (size_t)p * N * 4) + c);
      *reinterpret_cast<uint4*>(kst + p * 64 + 2 * c) = v;
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (tid == 0) { out[0] = t1 - t0; out[1] = kst[5]; }
}

__global__ void kwrite(uint64_t* keys, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) keys[i] = i * 0x9E3779B97F4A7C15ull;
}

int main() {
  const int P = 148, k = 4;
  uint64_t* h = new uint64_t[P * 68];
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < P * 68; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s; }
  uint64_t* d; unsigned long long* o;
  cudaMalloc(&d, P * 68 * 8); cudaMalloc(&o, 16);
  cudaMemcpy(d, h, P * 68 * 8, cudaMemcpyHostToDevice);
  unsigned long long r[2];
  cudaFuncSetAttribute(kbench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 148 * 68 * 8);
  cudaFuncSetAttribute(kbench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 148 * 68 * 8);
  cudaFuncSetAttribute(kbench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 148 * 68 * 8);
  cudaFuncSetAttribute(kbench<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 148 * 68 * 8);
  cudaFuncSetAttribute(kbench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 148 * 68 * 8);
  const uint64_t lbs[3] = {0ull, 0x8000000000000000ull, 0xF000000000000000ull};
  for (int rep = 0; rep < 2; ++rep) {
    kbench<0><<<1, 256, 148 * 68 * 8>>>(d, P, k, 0, o); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
    printf("mode0 (load only): %llu cycles\n", r[0]);
    for (uint64_t lb : lbs) {
      kbench<1><<<1, 256, 148 * 68 * 8>>>(d, P, k, lb, o); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
      printf("mode1 (vote-guarded insert) lb=%016llx: %llu cycles\n", (unsigned long long)lb, r[0]);
      kbench<2><<<1, 256, 148 * 68 * 8>>>(d, P, k, lb, o); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
      printf("mode2 (plain insert)        lb=%016llx: %llu cycles\n", (unsigned long long)lb, r[0]);
      kbench<3><<<1, 256, 148 * 68 * 8>>>(d, P, k, lb, o); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
      printf("mode3 (branch-free network) lb=%016llx: %llu cycles\n", (unsigned long long)lb, r[0]);
      kbench<4><<<1, 256, 148 * 68 * 8>>>(d, P, k, lb, o); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
      printf("mode4 (chunk mask + insert) lb=%016llx: %llu cycles\n", (unsigned long long)lb, r[0]);
    }
  }
  cudaFuncSetAttribute(kmerge, cudaFuncAttributeMaxDynamicSharedMemorySize, 148 * 68 * 8);
  for (int rep = 0; rep < 3; ++rep) {
    kmerge<<<1, 256, 148 * 68 * 8>>>(d, P, k, o); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
    printf("k_tail merge_net<4>: %llu cycles\n", r[0]);
  }
  {
    const int N = 48;
    uint64_t* keys; cudaMalloc(&keys, (size_t)P * N * 4 * 8);
    cudaFuncSetAttribute(kstage<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 148 * 68 * 8);
    cudaFuncSetAttribute(kstage<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 148 * 68 * 8);
    cudaFuncSetAttribute(kstage<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 148 * 68 * 8);
    for (int rep = 0; rep < 3; ++rep) {
      kwrite<<<148, 256>>>(keys, (size_t)P * N * 4);
      kstage<0><<<1, 256, 148 * 68 * 8>>>(keys, P, N, o); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
      printf("stage bulk/list: %llu cycles\n", r[0]);
      kwrite<<<148, 256>>>(keys, (size_t)P * N * 4);
      kstage<1><<<1, 256, 148 * 68 * 8>>>(keys, P, N, o); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
      printf("stage cp.async16: %llu cycles\n", r[0]);
      kwrite<<<148, 256>>>(keys, (size_t)P * N * 4);
      kstage<2><<<1, 256, 148 * 68 * 8>>>(keys, P, N, o); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
      printf("stage ld+st: %llu cycles\n", r[0]);
    }
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock rate attr %d kHz\n", clk);
  }
  return 0;
}
