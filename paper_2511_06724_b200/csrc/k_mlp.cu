// k_mlp.cu -- K3: quality predictor with the A5
// compliance / preference / priority derivation fused into its epilogue.
//
//   h   = relu(W1x . bf16(x) + W1s . s + b1)          fp32 accumulate
//   r_v = 1 / (1 + exp(-(W2 . h + b2)_v)),  r_0 := 1   (
//                                                      reading R7: relative to the full model)
//   A_i = {v : v = 0 or k_skip_v = 0 or s_i1 >= tau_v}
//   C_i = {v in A_i : r_v >= delta}                     (reading R6)
//   pi_i = A_i sorted by (r desc, p_th desc, v asc)     (reading R13)
//
// Grid = (prompt blocks of 16) x (hidden chunks of 32): a small batch still
// spreads over many SMs.  Layer 1 per CTA is a [16 x d] x [d x 32] bf16 product
// on the tensor cores (mma.sync m16n8k16, fp32 accumulate; the whole predictor is
// < 0.03 % of the scan's flops), split over 8 warps along d and reduced in shared
// memory.  W1x is pre-arranged at init in per-lane fragment order so each B
// fragment is one coalesced 8-byte load.  The last CTA of a prompt block (atomic
// ticket) runs layer 2 + A5 for its 16 prompts: one warp per prompt, lanes split
// the hidden units, lane v finally owns option v (L <= 32), so masks are ballots
// and the preference rank is a 32-lane compare-count (stored per option: the
// inverse permutation of pi_i, which is what the assignment walk consumes).
#include "common.cuh"
#include "kernels.h"

namespace argus {

constexpr int PB = 16;  // prompts per block (the MMA M dimension)
constexpr int MLP_THREADS = 256;
constexpr int MLP_WARPS = MLP_THREADS / 32;

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint2 b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

__global__ void __launch_bounds__(MLP_THREADS) k_mlp(MlpArgs a) {
  extern __shared__ __align__(16) uint8_t smraw[];
  __shared__ int is_last;
  const int d = a.d, H = a.H, L = a.L, k = a.k;
  const int RS = d + 8;                                               // padded bf16 row stride
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(smraw);        // [PB][RS]
  float* red = reinterpret_cast<float*>(smraw + (size_t)PB * RS * 2);  // [MLP_WARPS][PB*32]
  float* ss = red + MLP_WARPS * PB * 32;                              // [PB][k]
  const int pb = blockIdx.x, cc = blockIdx.y;
  const int i0 = pb * PB;
  const int nP = min(PB, a.N - i0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_wait();

  // stage the prompt block (rows past N in Xb are zero padding) with async copies
  for (int idx = tid; idx < PB * (d / 8); idx += MLP_THREADS) {
    const int p = idx / (d / 8), c = idx - p * (d / 8);
    cp_async16(xs + p * RS + c * 8, reinterpret_cast<const uint4*>(a.Xb + (int64_t)(i0 + p) * d) + c);
  }
  for (int idx = tid; idx < PB * k; idx += MLP_THREADS) {
    const int p = idx / k;
    ss[idx] = p < nP ? a.topk_score[(int64_t)(i0 + p) * k + (idx - p * k)] : 0.f;
  }
  // per-thread epilogue constants of layer 1 (independent of the staging above)
  float w1s_r[2][8], b1_r[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int j = cc * 32 + ((tid + u * MLP_THREADS) & 31);
    b1_r[u] = __ldg(a.b1 + j);
#pragma unroll
    for (int q = 0; q < 8; ++q) w1s_r[u][q] = q < k ? __ldg(a.W1sT + q * H + j) : 0.f;
  }
  cp_async_wait_all();
  __syncthreads();

  // ---- layer 1, hidden units [32 cc, 32 cc + 32), warp w takes a 1/8 slice of d
  {
    const int g = lane >> 2, t = lane & 3;
    const uint32_t* x32 = reinterpret_cast<const uint32_t*>(xs);
    const int RSW = RS / 2;
    const int KS = d / 16;
    const int ks0 = KS * warp / MLP_WARPS, ks1 = KS * (warp + 1) / MLP_WARPS;
    const uint2* wf = reinterpret_cast<const uint2*>(a.W1xF);
    float acc[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
    // all of this warp's B fragments first (<= 8 k-steps x 4 n-tiles): one memory round trip
    constexpr int KSW = 8;  // k-steps per warp for d <= 1024
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
  }
  __syncthreads();
  // reduce the 8 split-K partials (fixed order), + W1s . s + b1, relu -> h (global)
#pragma unroll
  for (int u = 0; u < 2; ++u) {  // PB * 32 = 2 * MLP_THREADS elements
    const int e = tid + u * MLP_THREADS;
    const int row = e >> 5, j = cc * 32 + (e & 31);
    float z = 0.f;
#pragma unroll
    for (int w = 0; w < MLP_WARPS; ++w) z = __fadd_rn(z, red[w * PB * 32 + e]);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < k) z = __fmaf_rn(w1s_r[u][q], ss[row * k + q], z);
    a.hbuf[(int64_t)(i0 + row) * H + j] = fmaxf(__fadd_rn(z, b1_r[u]), 0.f);
  }
  // ---- the last CTA of this prompt block runs layer 2 + A5
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int ticket = atomicAdd(&a.block_cnt[pb], 1);
    is_last = ticket == (int)gridDim.y - 1;
  }
  __syncthreads();
  pdl_launch();
  if (!is_last) return;
  __threadfence();
  if (tid == 0) a.block_cnt[pb] = 0;  // ready for the next launch
  float* hs = reinterpret_cast<float*>(smraw);  // [PB][H]  (reuses the staging area)
  float* w2s = hs + PB * H;                     // [L][H]
  // cp.async.cg reads through L2 only (hbuf was written by other CTAs of this launch)
  for (int e = tid; e < PB * H / 4; e += MLP_THREADS) cp_async16(hs + 4 * e, a.hbuf + (int64_t)i0 * H + 4 * e);
  for (int e = tid; e < L * H / 4; e += MLP_THREADS) cp_async16(w2s + 4 * e, a.W2 + 4 * e);
  cp_async_wait_all();
  __syncthreads();

  for (int p = warp; p < nP; p += MLP_WARPS) {
    const int i = i0 + p;
    const bool act = lane < L;
    // z_v = b2_v + sum_j W2[v][j] h_j: lanes split j, butterfly-reduce per option
    float part[32];
#pragma unroll
    for (int v = 0; v < 32; ++v) part[v] = 0.f;
    for (int j = lane; j < H; j += 32) {
      const float hj = hs[p * H + j];
#pragma unroll
      for (int v = 0; v < 32; ++v)
        if (v < L) part[v] = __fmaf_rn(w2s[v * H + j], hj, part[v]);
    }
    float z = 0.f;
#pragma unroll
    for (int v = 0; v < 32; ++v) {
      if (v < L) {
        float sv = part[v];
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) sv = __fadd_rn(sv, __shfl_xor_sync(0xffffffffu, sv, m));
        if (lane == v) z = sv;
      }
    }
    float r = 0.f;
    if (act) {
      z = __fadd_rn(z, a.b2[lane]);
      r = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z)));
      if (lane == 0) r = 1.0f;
    }
    const float s1 = __ldcg(a.topk_score + (int64_t)i * k);
    const int ks_ = act ? a.kskip[lane] : 0;
    const float gate = act ? a.gate[lane] : 0.f;
    const bool gated_pass = act && ks_ != 0 && s1 >= gate;
    const bool adm = act && (lane == 0 || ks_ == 0 || s1 >= gate);
    const bool cmp = adm && r >= a.delta;
    const uint32_t amask = __ballot_sync(0xffffffffu, adm);
    const uint32_t cmask = __ballot_sync(0xffffffffu, cmp);
    const uint32_t gmask = __ballot_sync(0xffffffffu, act && ks_ != 0);
    const uint32_t pmask = __ballot_sync(0xffffffffu, gated_pass);
    const float pth = act ? a.pth[lane] : 0.f;
    int rank = 0;
    for (int u = 0; u < L; ++u) {
      const float ru = __shfl_sync(0xffffffffu, r, u);
      const float pu = __shfl_sync(0xffffffffu, pth, u);
      const bool before = ((amask >> u) & 1u) &&
                          (ru > r || (ru == r && (pu > pth || (pu == pth && u < lane))));
      rank += before ? 1 : 0;
    }
    if (act) {
      a.rhat[(int64_t)i * L + lane] = r;
      a.rankof[(int64_t)i * a.Lw + lane] = adm ? (uint8_t)rank : (uint8_t)0xFF;  // position of v in pi_i
    } else if (lane < a.Lw) {
      a.rankof[(int64_t)i * a.Lw + lane] = 0xFF;
    }
    if (lane == 0) {
      a.ccount[i] = (uint8_t)__popc(cmask);
      a.cmask[i] = cmask;
      a.status[i] = (gmask != 0 && pmask == 0) ? 4u /*ARGUS_ST_GATED_ALL*/ : 0u;
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

size_t mlp_smem_bytes(int d, int k, int H, int L) {
  const size_t phase1 = (size_t)PB * (d + 8) * 2 + sizeof(float) * ((size_t)MLP_WARPS * PB * 32 + (size_t)PB * k);
  const size_t phase2 = sizeof(float) * ((size_t)PB * H + (size_t)L * H);
  return phase1 > phase2 ? phase1 : phase2;
}

void launch_mlp(const MlpArgs& a, cudaStream_t s) {
  const size_t smem = mlp_smem_bytes(a.d, a.k, a.H, a.L);
  static size_t attr_set = 0;
  if (smem > attr_set) {
    cudaFuncSetAttribute(k_mlp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = smem;
  }
  const dim3 grid((a.N + PB - 1) / PB, a.H / 32);
  launch_pdl(k_mlp, grid, dim3(MLP_THREADS), smem, s, a);
}

}  // namespace argus
