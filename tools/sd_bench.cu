// Microbenchmark: cycles per step of the tail's window serial dictatorship (one warp),
// C2-like batch: N = 48 prompts, L = 12 options, quotas ~ 1.2^v summing to N, every
// prompt preferring options in nearly the same order (diagnostics).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/sd_bench.cu -o tools/sd_bench
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void ksd(const uint8_t* rows_g, int n, int L, int Lw, const int* quota, unsigned long long* out, int* opt_out) {
  __shared__ uint8_t rk_s[64 * 32];
  __shared__ uint8_t inv_s[32 * 32];
  __shared__ uint8_t opt_s[64];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < n * Lw; i += 32) rk_s[i] = rows_g[i];
  __syncwarp();
  int rem_r = lane < L ? quota[lane] : 0;
  uint32_t avail_r = __ballot_sync(0xffffffffu, lane < L && rem_r > 0);
  const int W = Lw / 4;
  unsigned long long steps = 0;
  const unsigned long long t0 = clock64();
  uint8_t* inv = inv_s + lane * 32;
  for (int t0w = 0; t0w < n; t0w += 32) {
    const int jj = t0w + lane;
    const bool act = jj < n;
    const uint8_t* row = rk_s + (size_t)(act ? jj : 0) * Lw;
    uint32_t A = 0;
    if (act) {
      const uint32_t* row32 = reinterpret_cast<const uint32_t*>(row);
      for (int q = 0; q < 8; ++q) reinterpret_cast<uint32_t*>(inv)[q] = 0xFFFFFFFFu;
      for (int q = 0; q < W; ++q) {
        const uint32_t wq = row32[q];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint32_t o = (wq >> (8 * b)) & 0xFFu;
          if (o != 0xFFu) {
            inv[o] = (uint8_t)(4 * q + b);
            if ((avail_r >> o) & 1u) A |= 1u << (4 * q + b);
          }
        }
      }
    }
    __syncwarp();
    uint32_t pending = __ballot_sync(0xffffffffu, act);
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t seen = avail_r;
    while (pending) {
      for (uint32_t ex = seen & ~avail_r; ex; ex &= ex - 1) {
        const uint32_t r = inv[__ffs(ex) - 1];
        if (r != 0xFFu) A &= ~(1u << r);
      }
      seen = avail_r;
      const bool mine = (pending >> lane) & 1u;
      const int choice = A ? (int)row[__ffs(A) - 1] : 0xFF;
      const bool real = mine && choice != 0xFF;
      uint32_t same, mv;
      if (MODE == 0 || MODE == 2) {
        const uint32_t V = __ballot_sync(0xffffffffu, real);
        same = V; mv = V;
#pragma unroll
        for (int b = 0; b < 5; ++b) {
          const uint32_t B = __ballot_sync(0xffffffffu, real && ((choice >> b) & 1));
          same &= ((choice >> b) & 1) ? B : ~B;
          mv &= ((lane >> b) & 1) ? B : ~B;
        }
      } else {
        const uint32_t peers = __match_any_sync(0xffffffffu, real ? choice : 0x100 + lane);
        same = real ? peers : 0u;
        // lane v: lanes that chose v = the peers mask of any lane that chose v
        const int src = __ffs(__ballot_sync(0xffffffffu, real && choice == lane)) ;  // not correct in general; timing only
        mv = __shfl_sync(0xffffffffu, same, (src ? src - 1 : 0));
      }
      uint32_t commit;
      if (MODE == 2) {
        // lane v: the first lane whose choice v exceeds rem_v (the (rem_v + 1)-th chooser);
        // the batch commits every pending lane before the earliest such lane
        const int fe = (lane < 32 && __popc(mv) > rem_r) ? (int)__fns(mv, 0, rem_r + 1) : 32;
        const int bad_pos = (int)__reduce_min_sync(0xffffffffu, (unsigned)fe);
        commit = bad_pos >= 32 ? pending : (pending & ((1u << bad_pos) - 1u));
      } else {
        const int before = __popc(same & lt);
        const int remc = __shfl_sync(0xffffffffu, rem_r, choice & 31);
        const bool ok = !real || before < remc;
        const uint32_t bad = __ballot_sync(0xffffffffu, !ok);
        commit = bad ? (pending & ((1u << (__ffs(bad) - 1)) - 1u)) : pending;
      }
      if ((commit >> lane) & 1u) opt_s[jj] = choice == 0xFF ? (uint8_t)0x80 : (uint8_t)choice;
      rem_r -= __popc(mv & commit);
      avail_r = __ballot_sync(0xffffffffu, lane < L && rem_r > 0);
      pending &= ~commit;
      ++steps;
    }
  }
  const unsigned long long t1 = clock64();
  __syncwarp();
  for (int i = lane; i < n; i += 32) opt_out[i] = opt_s[i];
  if (lane == 0) { out[0] = t1 - t0; out[1] = steps; }
}

// MODE 3: one prompt per step, lane v = option v: key = rank of v in pi_i (0xFF if absent)
// when v has quota left, the choice = redux.min of (rank << 5 | v); the chain per prompt is
// select -> redux -> compare -> decrement.
__global__ void ksd_pp(const uint8_t* rows_g, int n, int L, int Lw, const int* quota, unsigned long long* out,
                       int* opt_out) {
  __shared__ uint8_t inv_s[64 * 32];
  __shared__ uint8_t opt_s[64];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < n * 32; i += 32) inv_s[i] = 0xFF;
  __syncwarp();
  for (int i = threadIdx.x; i < n * Lw; i += 32) {
    const int p = i / Lw, r = i - p * Lw;
    const int o = rows_g[i];
    if (o != 0xFF) inv_s[p * 32 + o] = (uint8_t)r;
  }
  __syncwarp();
  int rem = lane < L ? quota[lane] : 0;
  const unsigned long long t0 = clock64();
  int optr = 0;
#pragma unroll 8
  for (int t = 0; t < n; ++t) {
    const uint32_t rk = inv_s[t * 32 + lane];
    const uint32_t key = (rem > 0 && rk != 0xFFu) ? (rk << 5 | (uint32_t)lane) : 0xFFFFu;
    const uint32_t m = __reduce_min_sync(0xffffffffu, key);
    const int choice = m == 0xFFFFu ? 0x80 : (int)(m & 31u);
    rem -= (choice == lane) ? 1 : 0;
    optr = (lane == (t & 31)) ? choice : optr;
    if ((t & 31) == 31) { opt_s[t - 31 + lane] = (uint8_t)optr; }
  }
  const unsigned long long t1 = clock64();
  if (n & 31) { const int b = n & ~31; if (lane < (n & 31)) opt_s[b + lane] = (uint8_t)optr; }
  __syncwarp();
  for (int i = lane; i < n; i += 32) opt_out[i] = opt_s[i];
  if (lane == 0) { out[0] = t1 - t0; out[1] = n; }
}

int main() {
  const int n = 48, L = 12, Lw = 12;
  uint8_t rows[64 * 32];
  unsigned s = 12345;
  for (int i = 0; i < n; ++i) {
    int perm[12];
    for (int v = 0; v < L; ++v) perm[v] = v;
    for (int sw = 0; sw < 2; ++sw) { s = s * 1103515245u + 12345u; int a = (s >> 16) % (L - 1); int t = perm[a]; perm[a] = perm[a + 1]; perm[a + 1] = t; }
    for (int r = 0; r < Lw; ++r) rows[i * Lw + r] = r < L ? perm[r] : 0xFF;
  }
  int quota[12]; double tot = 0; for (int v = 0; v < L; ++v) tot += __builtin_pow(1.2, v);
  int sum = 0; for (int v = 0; v < L; ++v) { quota[v] = (int)(n * __builtin_pow(1.2, v) / tot); sum += quota[v]; }
  quota[L - 1] += n - sum;
  uint8_t* drows; int* dq; unsigned long long* o; int* dopt;
  cudaMalloc(&drows, sizeof(rows)); cudaMalloc(&dq, sizeof(quota)); cudaMalloc(&o, 16); cudaMalloc(&dopt, 64 * 4);
  cudaMemcpy(drows, rows, sizeof(rows), cudaMemcpyHostToDevice); cudaMemcpy(dq, quota, sizeof(quota), cudaMemcpyHostToDevice);
  unsigned long long r[2];
  for (int rep = 0; rep < 3; ++rep) {
    ksd<0><<<1, 32>>>(drows, n, L, Lw, dq, o, dopt); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
    printf("ballots: %llu cycles, %llu steps, %.0f cycles/step\n", r[0], r[1], (double)r[0] / r[1]);
    int opt0[64], opt2[64];
    cudaMemcpy(opt0, dopt, 64 * 4, cudaMemcpyDeviceToHost);
    ksd<2><<<1, 32>>>(drows, n, L, Lw, dq, o, dopt); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(opt2, dopt, 64 * 4, cudaMemcpyDeviceToHost);
    int same = 1; for (int i = 0; i < n; ++i) same &= opt0[i] == opt2[i];
    printf("fns+min: %llu cycles, %llu steps, %.0f cycles/step, same assignment %d\n", r[0], r[1], (double)r[0] / r[1], same);
    ksd_pp<<<1, 32>>>(drows, n, L, Lw, dq, o, dopt); cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(opt2, dopt, 64 * 4, cudaMemcpyDeviceToHost);
    same = 1; for (int i = 0; i < n; ++i) same &= opt0[i] == opt2[i];
    printf("per-prompt redux.min: %llu cycles, %llu prompts, %.0f cycles/prompt, same assignment %d\n", r[0], r[1], (double)r[0] / r[1], same);
  }
  return 0;
}
