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
// One CTA = H threads (one per hidden unit) x PB prompts.  W1x is stored
// transposed [d][H] in bf16 so a warp's loads are coalesced; the prompt block
// sits in shared memory as fp32.  Layer 2 + A5 run one warp per prompt with
// lane v owning option v (L <= 32), so masks are ballots and the preference
// rank is a 32-lane compare-count.
#include "common.cuh"
#include "kernels.h"

namespace argus {

constexpr int PB = 8;  // prompts per CTA

__global__ void __launch_bounds__(1024) k_mlp(MlpArgs a) {
  extern __shared__ float sm[];
  const int d = a.d, H = a.H, L = a.L, k = a.k;
  float* xs = sm;                    // [d][PB]
  float* ss = xs + (size_t)d * PB;   // [PB][k]
  float* hs = ss + PB * k;           // [PB][H]
  float* w2 = hs + (size_t)PB * H;   // [H][L]
  const int i0 = blockIdx.x * PB;
  const int nP = min(PB, a.N - i0);
  const int tid = threadIdx.x;

  for (int idx = tid; idx < d * PB; idx += blockDim.x) {
    const int p = idx / d, l = idx - p * d;
    xs[l * PB + p] = p < nP ? __bfloat162float(a.Xb[(int64_t)(i0 + p) * d + l]) : 0.f;
  }
  for (int idx = tid; idx < PB * k; idx += blockDim.x) {
    const int p = idx / k;
    ss[idx] = p < nP ? a.topk_score[(int64_t)(i0 + p) * k + (idx - p * k)] : 0.f;
  }
  for (int idx = tid; idx < H * L; idx += blockDim.x) w2[idx] = a.W2T[idx];
  __syncthreads();

  // ---- layer 1: thread j = hidden unit
  for (int j = tid; j < H; j += blockDim.x) {
    float acc[PB];
#pragma unroll
    for (int p = 0; p < PB; ++p) acc[p] = 0.f;
#pragma unroll 4
    for (int l = 0; l < d; ++l) {
      const float w = __bfloat162float(a.W1xT[(int64_t)l * H + j]);
      const float4 x0 = *reinterpret_cast<const float4*>(xs + l * PB);
      const float4 x1 = *reinterpret_cast<const float4*>(xs + l * PB + 4);
      acc[0] = __fmaf_rn(w, x0.x, acc[0]);
      acc[1] = __fmaf_rn(w, x0.y, acc[1]);
      acc[2] = __fmaf_rn(w, x0.z, acc[2]);
      acc[3] = __fmaf_rn(w, x0.w, acc[3]);
      acc[4] = __fmaf_rn(w, x1.x, acc[4]);
      acc[5] = __fmaf_rn(w, x1.y, acc[5]);
      acc[6] = __fmaf_rn(w, x1.z, acc[6]);
      acc[7] = __fmaf_rn(w, x1.w, acc[7]);
    }
    for (int t = 0; t < k; ++t) {
      const float w = a.W1sT[t * H + j];
#pragma unroll
      for (int p = 0; p < PB; ++p) acc[p] = __fmaf_rn(w, ss[p * k + t], acc[p]);
    }
    const float bj = a.b1[j];
#pragma unroll
    for (int p = 0; p < PB; ++p) hs[p * H + j] = fmaxf(__fadd_rn(acc[p], bj), 0.f);
  }
  __syncthreads();

  // ---- layer 2 + A5: warp per prompt, lane v = option v
  const int warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  for (int p = warp; p < nP; p += nwarps) {
    const int i = i0 + p;
    const bool act = lane < L;
    float r = 0.f;
    if (act) {
      float z = a.b2[lane];
      for (int j = 0; j < H; ++j) z = __fmaf_rn(w2[j * L + lane], hs[p * H + j], z);
      r = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z)));
      if (lane == 0) r = 1.0f;
    }
    const float s1 = ss[p * k];
    const int ks = act ? a.kskip[lane] : 0;
    const float gate = act ? a.gate[lane] : 0.f;
    const bool gated_pass = act && ks != 0 && s1 >= gate;
    const bool adm = act && (lane == 0 || ks == 0 || s1 >= gate);
    const bool cmp = adm && r >= a.delta;
    const uint32_t amask = __ballot_sync(0xffffffffu, adm);
    const uint32_t cmask = __ballot_sync(0xffffffffu, cmp);
    const uint32_t gmask = __ballot_sync(0xffffffffu, act && ks != 0);
    const uint32_t pmask = __ballot_sync(0xffffffffu, gated_pass);
    // preference rank among admissible options
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
      a.pref[(int64_t)i * L + lane] = 0xFF;
    }
    __syncwarp();
    if (adm) a.pref[(int64_t)i * L + rank] = (uint8_t)lane;
    if (lane == 0) {
      a.ccount[i] = (uint8_t)__popc(cmask);
      a.cmask[i] = cmask;
      a.status[i] = (gmask != 0 && pmask == 0) ? 4u /*ARGUS_ST_GATED_ALL*/ : 0u;
    }
  }
}

void launch_mlp(const MlpArgs& a, cudaStream_t s) {
  const int threads = a.H < 1024 ? a.H : 1024;
  const size_t smem = sizeof(float) * ((size_t)a.d * PB + PB * a.k + (size_t)PB * a.H + (size_t)a.H * a.L);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_mlp, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  k_mlp<<<(a.N + PB - 1) / PB, threads, smem, s>>>(a);
}

}  // namespace argus
