// common.cuh -- device helpers shared by the libargus kernels (sm_100a).
// Key packing for the fused top-k: a 64-bit key whose
// unsigned order is (score desc, global id asc), so every top-k step is an
// integer compare and the result does not depend on reduction order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace argus {

// Programmatic dependent launch (PDL): every per-batch kernel is launched with
// programmatic stream serialization, waits for its predecessor's memory with
// griddepcontrol.wait before touching shared buffers, and lets its successor be
// scheduled (griddepcontrol.launch_dependents) once its own main work is issued.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint64_t gtimer() {  // diagnostics stamps (ns)
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// 16-byte asynchronous global -> shared copy (LDGSTS): many in flight per thread,
// no register round trip; cp_async_wait_all() before __syncthreads().
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
// 8-byte variant (LDGSTS.64, L1-allocating .ca: .cg takes 16-byte copies only) for
// sources that are only 8-byte aligned.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Monotone map fp32 -> u32 (a < b  <=>  ord(a) < ord(b) for non-NaN a, b).
__device__ __forceinline__ uint32_t ord_f32(float s) {
  uint32_t u = __float_as_uint(s);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float unord_f32(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(u);
}

// key = ord(score) << 32 | (0xFFFFFFFF - g).  -0 is canonicalised to +0 first so
// the two zeros tie (and break by id).  key 0 is "empty" (below every real key).
__device__ __forceinline__ uint64_t pack_key(float s, uint32_t g) {
  s = __fadd_rn(s, 0.0f);
  return ((uint64_t)ord_f32(s) << 32) | (uint64_t)(0xffffffffu - g);
}

__device__ __forceinline__ uint32_t key_id(uint64_t key) {
  return key == 0 ? 0xffffffffu : 0xffffffffu - (uint32_t)(key & 0xffffffffu);
}

__device__ __forceinline__ float key_score(uint64_t key) {
  return key == 0 ? -1.0f : unord_f32((uint32_t)(key >> 32));
}

// Sorted (descending) top-KMAX list held in registers.  Entries start at 0
// (empty).  insert() keeps the KMAX largest keys; keys are unique except 0.
template <int KMAX>
struct TopList {
  uint64_t v[KMAX];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int i = 0; i < KMAX; ++i) v[i] = 0;
  }
  __device__ __forceinline__ uint64_t min_key() const { return v[KMAX - 1]; }
  // branch-free insert: KMAX compare-exchanges whatever the key (for loops over many
  // keys: a data-dependent early exit there costs more than the network)
  __device__ __forceinline__ void insert_nb(uint64_t y) {
#pragma unroll
    for (int i = 0; i < KMAX; ++i) {
      const uint64_t hi = v[i] > y ? v[i] : y, lo = v[i] > y ? y : v[i];
      v[i] = hi;
      y = lo;
    }
  }
  __device__ __forceinline__ void insert(uint64_t key) {
    if (key <= v[KMAX - 1]) return;
    v[KMAX - 1] = key;
#pragma unroll
    for (int i = KMAX - 1; i > 0; --i) {
      if (v[i] > v[i - 1]) {
        uint64_t t = v[i];
        v[i] = v[i - 1];
        v[i - 1] = t;
      }
    }
  }
};

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t x, int m) {
  uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)x, m);
  uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(x >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t x) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    uint64_t y = shfl_xor_u64(x, m);
    x = y > x ? y : x;
  }
  return x;
}

// Merge the per-lane lists of a warp into the warp's top-k (k <= KMAX), written
// by lane 0 to out[0..k).  Keys are unique apart from 0, so exactly one lane
// owns each extracted non-zero maximum.
template <int KMAX>
__device__ __forceinline__ void warp_merge_topk(TopList<KMAX>& l, int k, uint64_t* out) {
  const int lane = threadIdx.x & 31;
  for (int t = 0; t < k; ++t) {
    uint64_t m = warp_max_u64(l.v[0]);
    if (lane == 0) out[t] = m;
    if (m != 0 && l.v[0] == m) {
#pragma unroll
      for (int i = 0; i < KMAX - 1; ++i) l.v[i] = l.v[i + 1];
      l.v[KMAX - 1] = 0;
    }
  }
}

}  // namespace argus
