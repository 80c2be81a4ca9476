// mma_ss_tail.cu -- microbenchmark for the d = 1024 scan shape (KBV = 16): cycles per
// M=128 N=64 K=16 MMA when k-blocks [12, 16) read A from shared memory (SS form)
// instead of TMEM, issued warp-uniformly like the scan's MMA warps.  Not part of
// the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2511_06724_b200/csrc mma_ss_tail.cu
#include <cstdio>
#include <cstdint>
#include "tc.cuh"

using namespace argus;

// n_ss: how many of the 16 k-blocks take A from shared memory; the rest from TMEM
// (TMEM A would need 512 columns for all 16, so the TS k-blocks reuse columns mod 12).
// B: 16 boxes of 64 rows x 64 cols (8 KB each), A tail: 4 blocks of 128 x 64 (16 KB each).
template <int NSS, int CEVERY = 64>
__global__ void bench_tile(int tiles, int n_cols, long long* out) {
  constexpr int n_ss = NSS;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bar2;
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
  for (int i = threadIdx.x; i < 192 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t tmem = tbase;
  if (warp == 0) {
    const uint32_t idesc = tc::idesc_bf16_f32(128, n_cols);
    const uint32_t sb = tc::smem_u32(sm);
    const uint32_t sa = sb + 128 * 1024;
    const uint64_t bdesc = tc::desc_kmajor_sw128(sb);
    const uint64_t adesc = tc::desc_kmajor_sw128(sa);
    constexpr int kb_ts = 16 - n_ss;
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t dcol = tmem + 384 + (t & 1) * 64;
#pragma unroll
      for (int kb = 0; kb < 16; ++kb) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = bdesc + (uint64_t)((kb * 8192 + kk * 32) >> 4);
          if (kb < kb_ts)
            tc::mma_ts_warp(dcol, tmem + (uint32_t)(((kb % 12) * 4 + kk) * 8), bd, idesc, (kb | kk) != 0);
          else
            tc::mma_ss_warp(dcol, adesc + (uint64_t)((((kb - kb_ts) & 3) * 16384 + kk * 32) >> 4), bd, idesc,
                            (kb | kk) != 0);
          if (CEVERY < 64 && ((kb * 4 + kk) % CEVERY) == CEVERY - 1 && (kb * 4 + kk) != 63)
            tc::mma_commit_warp(tc::smem_u32(&bar2));  // extra per-slot commits (tracked, never waited)
        }
      }
      tc::mma_commit_warp(tc::smem_u32(&bar));
    }
    tc::mbar_wait(tc::smem_u32(&bar), (tiles - 1) & 1);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

template <int NSS, int CEVERY = 64>
static double run(int tiles, int n, int ctas) {
  static long long* d = nullptr;
  if (!d) cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench_tile<NSS, CEVERY>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  long long c = 0;
  for (int rep = 0; rep < 3; ++rep) {
    bench_tile<NSS, CEVERY><<<ctas, 128, 200 * 1024>>>(tiles, n, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  }
  return (double)c / (tiles * 64.0);
}

int main() {
  printf("M=128 N=64,  0 of 16 k-blocks SS: %7.2f cycles/mma\n", run<0>(400, 64, 1));
  printf("M=128 N=64,  4 of 16 k-blocks SS: %7.2f cycles/mma\n", run<4>(400, 64, 1));
  printf("M=128 N=64,  8 of 16 k-blocks SS: %7.2f cycles/mma\n", run<8>(400, 64, 1));
  printf("M=128 N=64, 16 of 16 k-blocks SS: %7.2f cycles/mma\n", run<16>(400, 64, 1));
  printf("M=128 N=32,  0 of 16 k-blocks SS: %7.2f cycles/mma\n", run<0>(400, 32, 1));
  printf("M=128 N=32,  4 of 16 k-blocks SS: %7.2f cycles/mma\n", run<4>(400, 32, 1));
  printf("148 CTAs N=64, 0 SS: %7.2f cycles/mma (CTA 0)\n", run<0>(4000, 64, 148));
  printf("148 CTAs N=64, 4 SS: %7.2f cycles/mma (CTA 0)\n", run<4>(4000, 64, 148));
  printf("M=128 N=64, 0 SS, commit every 32 MMAs: %7.2f cycles/mma\n", run<0, 32>(400, 64, 1));
  printf("M=128 N=64, 0 SS, commit every 16 MMAs: %7.2f cycles/mma\n", run<0, 16>(400, 64, 1));
  printf("M=128 N=64, 4 SS, commit every 16 MMAs: %7.2f cycles/mma\n", run<4, 16>(400, 64, 1));
  return 0;
}
