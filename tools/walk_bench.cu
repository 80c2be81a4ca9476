// walk_bench.cu -- microbenchmark of the serial-dictatorship walk (one warp):
// cycles per prompt for several formulations.  Diagnostics only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 walk_bench.cu -o walk_bench
#include <cstdint>
#include <cstdio>

constexpr int L = 12, LW = 12;

// A: REDUX.MIN over per-option positions (product formulation)
__global__ void walk_redux(const uint8_t* rk, int N, const int* quota, uint8_t* out, long long* cyc) {
  __shared__ uint8_t rk_s[2048 * LW];
  __shared__ uint8_t opt_s[2048];
  const int lane = threadIdx.x;
  for (int i = lane; i < N * LW; i += 32) rk_s[i] = rk[i];
  __syncwarp();
  int rem = lane < L ? quota[lane] : 0;
  long long t0 = clock64();
  uint32_t nxt = lane < L ? rk_s[lane] : 0xFFu;
  for (int t = 0; t < N; ++t) {
    const uint32_t r = nxt;
    if (t + 1 < N) nxt = lane < L ? rk_s[(t + 1) * LW + lane] : 0xFFu;
    const uint32_t cand = (r != 0xFFu && rem > 0) ? r : 0xFFu;
    const uint32_t best = __reduce_min_sync(0xffffffffu, cand);
    const bool mine = best != 0xFFu && cand == best;
    rem -= mine ? 1 : 0;
    const uint32_t who = __ballot_sync(0xffffffffu, mine);
    if (lane == 0) opt_s[t] = who ? (uint8_t)(__ffs(who) - 1) : 0x80;
  }
  long long t1 = clock64();
  __syncwarp();
  for (int i = lane; i < N; i += 32) out[i] = opt_s[i];
  if (lane == 0) cyc[0] = t1 - t0;
}

// B: availability bitmask + preference order pi (lane r holds pi[r]); ballot/ffs/shfl
__global__ void walk_ballot(const uint8_t* pref, int N, const int* quota, uint8_t* out, long long* cyc) {
  __shared__ uint8_t p_s[2048 * LW];
  __shared__ uint8_t opt_s[2048];
  const int lane = threadIdx.x;
  for (int i = lane; i < N * LW; i += 32) p_s[i] = pref[i];
  __syncwarp();
  int rem = lane < L ? quota[lane] : 0;
  uint32_t avail = __ballot_sync(0xffffffffu, rem > 0);
  long long t0 = clock64();
  uint32_t nxt = lane < L ? p_s[lane] : 0xFFu;
  for (int t = 0; t < N; ++t) {
    const uint32_t pv = nxt;
    if (t + 1 < N) nxt = lane < L ? p_s[(t + 1) * LW + lane] : 0xFFu;
    const bool ok = pv != 0xFFu && ((avail >> pv) & 1u);
    const uint32_t b = __ballot_sync(0xffffffffu, ok);
    int opt = 0x80;
    if (b) {
      opt = (int)__shfl_sync(0xffffffffu, pv, __ffs(b) - 1);
      if (lane == opt) --rem;
      avail = __ballot_sync(0xffffffffu, rem > 0);
    }
    if (lane == 0) opt_s[t] = (uint8_t)opt;
  }
  long long t1 = clock64();
  __syncwarp();
  for (int i = lane; i < N; i += 32) out[i] = opt_s[i];
  if (lane == 0) cyc[0] = t1 - t0;
}

// C: single thread, availability mask in a register, preference lists scanned in order
__global__ void walk_scalar(const uint8_t* pref, int N, const int* quota, uint8_t* out, long long* cyc) {
  __shared__ uint8_t p_s[2048 * LW];
  __shared__ int rem_s[32];
  const int lane = threadIdx.x;
  for (int i = lane; i < N * LW; i += 32) p_s[i] = pref[i];
  if (lane < 32) rem_s[lane] = lane < L ? quota[lane] : 0;
  __syncwarp();
  if (lane != 0) return;
  uint32_t avail = 0;
  for (int v = 0; v < L; ++v) avail |= (rem_s[v] > 0 ? 1u : 0u) << v;
  long long t0 = clock64();
  for (int t = 0; t < N; ++t) {
    const uint32_t* row = reinterpret_cast<const uint32_t*>(p_s + t * LW);
    int opt = 0x80;
    for (int w = 0; w < LW / 4 && opt == 0x80; ++w) {
      const uint32_t word = row[w];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t pv = (word >> (8 * e)) & 0xFFu;
        if (opt == 0x80 && pv != 0xFFu && ((avail >> pv) & 1u)) opt = (int)pv;
      }
    }
    if (opt != 0x80) {
      if (--rem_s[opt] == 0) avail &= ~(1u << opt);
    }
    out[t] = (uint8_t)opt;
  }
  long long t1 = clock64();
  cyc[0] = t1 - t0;
}

// dependent-load latency (pointer chase) over an L2-resident 4 MB ring
__global__ void chase(const uint32_t* nxt, int steps, long long* cyc, uint32_t* sink) {
  uint32_t j = 0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) j = __ldcg(nxt + j);
  long long t1 = clock64();
  cyc[0] = t1 - t0;
  sink[0] = j;
}

int main() {
  const int N = 2048;
  uint8_t *rk, *pref, *out;
  int* quota;
  long long* cyc;
  cudaMallocManaged(&rk, N * LW);
  cudaMallocManaged(&pref, N * LW);
  cudaMallocManaged(&out, N);
  cudaMallocManaged(&quota, 32 * 4);
  cudaMallocManaged(&cyc, 8);
  unsigned s = 12345;
  for (int i = 0; i < N; ++i) {
    int perm[L];
    for (int v = 0; v < L; ++v) perm[v] = v;
    for (int v = L - 1; v > 0; --v) {
      s = s * 1103515245u + 12345u;
      int j = (s >> 8) % (v + 1);
      int tmp = perm[v]; perm[v] = perm[j]; perm[j] = tmp;
    }
    for (int r = 0; r < LW; ++r) pref[i * LW + r] = r < L ? (uint8_t)perm[r] : 0xFF;
    for (int r = 0; r < L; ++r) rk[i * LW + perm[r]] = (uint8_t)r;
  }
  for (int v = 0; v < L; ++v) quota[v] = N / L;
  for (int rep = 0; rep < 2; ++rep) {
    walk_redux<<<1, 32>>>(rk, N, quota, out, cyc);
    cudaDeviceSynchronize();
  }
  printf("redux  : %.1f cycles/prompt\n", (double)cyc[0] / N);
  for (int rep = 0; rep < 2; ++rep) {
    walk_ballot<<<1, 32>>>(pref, N, quota, out, cyc);
    cudaDeviceSynchronize();
  }
  printf("ballot : %.1f cycles/prompt\n", (double)cyc[0] / N);
  for (int rep = 0; rep < 2; ++rep) {
    walk_scalar<<<1, 32>>>(pref, N, quota, out, cyc);
    cudaDeviceSynchronize();
  }
  printf("scalar : %.1f cycles/prompt\n", (double)cyc[0] / N);
  {
    const int M = 1 << 20;
    uint32_t* nx;
    cudaMallocManaged(&nx, M * 4);
    for (int i = 0; i < M; ++i) nx[i] = (uint32_t)((i + 4099 * 37) % M);
    cudaMemPrefetchAsync(nx, M * 4, 0);
    cudaDeviceSynchronize();
    for (int rep = 0; rep < 3; ++rep) {
      chase<<<1, 1>>>(nx, 4000, cyc, reinterpret_cast<uint32_t*>(out));
      cudaDeviceSynchronize();
    }
    printf("L2 dependent load: %.1f cycles\n", (double)cyc[0] / 4000);
  }
  return 0;
}
