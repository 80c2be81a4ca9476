// mma_bench.cu -- microbenchmark: cycles per tcgen05.mma.cta_group::1.kind::f16
// for A from TMEM (TS) vs A from shared memory (SS), M in {64,128}, N in {32..256}.
// Used to pick the scan kernel's tile shape.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2511_06724_b200/csrc mma_bench.cu -o mma_bench
#include <cstdio>
#include <cstdint>
#include "tc.cuh"

using namespace argus;

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

// "scan-like" issue: A walks 48 column groups of a 384-column resident operand,
// D double-buffered at 384/448, B walks 6 boxes of a slot, one commit per 24 MMAs.
__global__ void bench_scanlike(int iters, int N, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    tc::tmem_alloc(tc::smem_u32(&tbase), 512);
    tc::tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&bar), 1);
    tc::fence_barrier_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_bf16_f32(128, N);
    const uint32_t sb0 = tc::smem_u32(sm);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int kb = (i >> 2) % 12, kk = i & 3;
      const uint32_t dcol = 384 + ((i / 48) & 1) * 64;
      tc::mma_ts(tmem + dcol, tmem + (uint32_t)((kb * 4 + kk) * 8), tc::desc_kmajor_sw128(sb0 + (kb % 6) * 8192 + kk * 32),
                 idesc, (kb | kk) != 0);
      if ((i % 24) == 23) tc::mma_commit(tc::smem_u32(&bar));
    }
    tc::mma_commit(tc::smem_u32(&bar));
    long long t1 = clock64();
    // drain
    for (int ph = 0; ph < 1; ++ph) {}
    out[0] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

__device__ __forceinline__ void mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.b32 q, %4, 0;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, q;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}

// warp-uniform scan-like issue: whole warp runs the loop (uniform registers),
// elect.sync inside the asm picks the issuing lane; descriptors precomputed.
__global__ void bench_scanlike_warp(int tiles, int N, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    tc::tmem_alloc(tc::smem_u32(&tbase), 512);
    tc::tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&bar), 1);
    tc::fence_barrier_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    const uint32_t idesc = tc::idesc_bf16_f32(128, N);
    const uint64_t dbase = tc::desc_kmajor_sw128(tc::smem_u32(sm));
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t dcol = tmem + 384 + (t & 1) * 64;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
        for (int j = 0; j < 6; ++j)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int kb = hh * 6 + j;
            mma_ts_elect(dcol, tmem + (uint32_t)((kb * 4 + kk) * 8), dbase + (uint64_t)((j * 8192 + kk * 32) >> 4),
                         idesc, (kb | kk) != 0);
          }
        commit_elect(tc::smem_u32(&bar));
      }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

// commit_every: 0 = single commit at the end; c > 0: a tcgen05.commit after every c MMAs.
// warp_issue: the whole warp runs the loop, elect.sync picks the issuing lane.
template <bool TS>
__global__ void bench(int M, int N, int iters, long long* out, int commit_every = 0, int warp_issue = 0) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    tc::tmem_alloc(tc::smem_u32(&tbase), 512);
    tc::tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&bar), 1);
    tc::mbar_init(tc::smem_u32(&bar2), 1);
    tc::fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 60 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t tmem = tbase;
  if (warp_issue && warp == 0) {
    const uint32_t idesc = tc::idesc_bf16_f32(M, N);
    const uint32_t sa = tc::smem_u32(sm);
    const uint32_t sb = sa + 32 * 1024;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 3;
      if (elect_one()) {
        if (TS)
          tc::mma_ts(tmem + 256, tmem + (uint32_t)(kk * 8), tc::desc_kmajor_sw128(sb + kk * 32), idesc, 1);
        else
          mma_ss(tmem + 256, tc::desc_kmajor_sw128(sa + kk * 32), tc::desc_kmajor_sw128(sb + kk * 32), idesc, 1);
        if (commit_every && (i % commit_every) == commit_every - 1) tc::mma_commit(tc::smem_u32(&bar2));
      }
      __syncwarp();
    }
    if (elect_one()) tc::mma_commit(tc::smem_u32(&bar));
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  } else if (!warp_issue && threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_bf16_f32(M, N);
    const uint32_t sa = tc::smem_u32(sm);
    const uint32_t sb = sa + 32 * 1024;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 3;
      if (TS)
        tc::mma_ts(tmem + 256, tmem + (uint32_t)(kk * 8), tc::desc_kmajor_sw128(sb + kk * 32), idesc, 1);
      else
        mma_ss(tmem + 256, tc::desc_kmajor_sw128(sa + kk * 32), tc::desc_kmajor_sw128(sb + kk * 32), idesc, 1);
      if (commit_every && (i % commit_every) == commit_every - 1) tc::mma_commit(tc::smem_u32(&bar2));
    }
    tc::mma_commit(tc::smem_u32(&bar));
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65 * 1024);
  cudaFuncSetAttribute(bench<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65 * 1024);
  const int iters = 4096;
  for (int ts = 0; ts < 2; ++ts)
    for (int M : {64, 128})
      for (int N : {16, 32, 64, 128, 256}) {
        if (M == 128 && N < 16) continue;
        long long c = 0;
        for (int rep = 0; rep < 3; ++rep) {
          if (ts) bench<true><<<1, 128, 64 * 1024 + 1024>>>(M, N, iters, d);
          else bench<false><<<1, 128, 64 * 1024 + 1024>>>(M, N, iters, d);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
          cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        }
        const double cyc = (double)c / iters;
        const double macs = (double)M * N * 16;
        printf("%s M=%3d N=%3d : %7.2f cycles/mma  %7.1f MAC/cycle\n", ts ? "TS" : "SS", M, N, cyc, macs / cyc);
      }
  cudaFuncSetAttribute(bench_scanlike, cudaFuncAttributeMaxDynamicSharedMemorySize, 65 * 1024);
  cudaFuncSetAttribute(bench_scanlike_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 65 * 1024);
  {
    long long c = 0;
    for (int rep = 0; rep < 3; ++rep) {
      bench_scanlike_warp<<<1, 128, 64 * 1024 + 1024>>>(100, 64, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    }
    printf("scan-like WARP-uniform issue N=64: %7.2f cycles/mma (2 commits / 48 mma)\n", (double)c / 4800);
  }
  for (int N : {64}) {
    long long c = 0;
    for (int rep = 0; rep < 3; ++rep) {
      bench_scanlike<<<1, 128, 64 * 1024 + 1024>>>(4800, N, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    }
    printf("scan-like issue N=%d: %7.2f cycles/mma (issue side, 1 commit / 24 mma)\n", N, (double)c / 4800);
  }
  // commit cadence / issue style at M=128 TS
  for (int wi = 0; wi < 2; ++wi)
    for (int ce : {0, 4, 1})
      for (int N : {64, 128, 256}) {
        long long c = 0;
        for (int rep = 0; rep < 3; ++rep) {
          bench<true><<<1, 128, 64 * 1024 + 1024>>>(128, N, iters, d, ce, wi);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
          cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        }
        printf("TS M=128 N=%3d commit_every=%d warp_issue=%d : %7.2f cycles/mma\n", N, ce, wi, (double)c / iters);
      }
  return 0;
}
