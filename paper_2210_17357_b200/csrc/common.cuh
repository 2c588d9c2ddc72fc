// common.cuh -- device helpers shared by the lgreco kernels (product path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lgreco.h"

#define LG_WARP 32
#define LG_FULL 0xffffffffu

namespace lg {

// Per-layer descriptor uploaded once per ctx (plan-independent part) -----------
struct DevLayer {
  int64_t offset;    // element offset in the flat gradient
  int64_t numel;
  int64_t bucket0;   // global index of the layer's first record (bucket)
  int32_t rows, cols;
  int32_t compress;
  int32_t pad;
};

// Per-layer plan descriptor (depends on the chosen parameter) -----------------
struct DevPlan {
  int64_t pay_off;   // byte offset of the layer's records in the payload
  int32_t bits;      // QSGD bits (0 = lossless record stream)
  int32_t rec_bytes; // bytes of a full record
};

// Philox4x32-10 (Salmon et al. SC'11), R3.  Own implementation.
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                       uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;  // IMAD.WIDE.U32: hi and lo at once
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c0 = n0; c1 = (uint32_t)p1; c2 = n2; c3 = (uint32_t)p0;
  }
  return U4{c0, c1, c2, c3};
}

// The ten round keys of Philox4x32-10 (k0 + r W0, k1 + r W1), precomputed on the host and
// passed as a kernel parameter: the rounds then read them straight from the parameter
// bank (a LOP3 operand) instead of re-deriving them in the loop.
struct PhiloxRK { uint32_t k[20]; };
__host__ __device__ inline PhiloxRK philox_rk(uint32_t k0, uint32_t k1) {
  PhiloxRK r;
  for (int i = 0; i < 10; ++i) { r.k[2 * i] = k0 + 0x9E3779B9u * (uint32_t)i; r.k[2 * i + 1] = k1 + 0xBB67AE85u * (uint32_t)i; }
  return r;
}
__device__ __forceinline__ U4 philox10_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const PhiloxRK& rk) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ rk.k[2 * r];
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ rk.k[2 * r + 1];
    c0 = n0; c1 = (uint32_t)p1; c2 = n2; c3 = (uint32_t)p0;
  }
  return U4{c0, c1, c2, c3};
}

// u = (w >> 8) * 2^-24 (exact)
__device__ __forceinline__ float word_u(uint32_t w) {
  return __fmul_rn(__uint2float_rn(w >> 8), 5.9604644775390625e-08f);
}

// x = fl(fl(g + e) + 0): canonical gradient-plus-EF (R2)
__device__ __forceinline__ float canon(float g, float e) {
  return __fadd_rn(__fadd_rn(g, e), 0.0f);
}

__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(LG_FULL, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(LG_FULL, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(LG_FULL, v, o);
  return v;
}

// floor(v) for 0 <= v < 2^23 without the conversion pipe: RD(v + 2^23) - 2^23 (exact)
__device__ __forceinline__ float floor_pos(float v) {
  return __fsub_rn(__fadd_rd(v, 8388608.0f), 8388608.0f);
}

// Layer of global record gb: largest l with bucket0[l] <= gb (bucket0 ascending, L+1 entries)
__device__ __forceinline__ int find_layer(const int64_t* b0, int L, int64_t gb) {
  int lo = 0, hi = L - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (b0[mid] <= gb) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may be
// scheduled while its predecessor in the stream drains; it must call pdl_wait() before
// touching anything the predecessor writes (griddepcontrol.wait returns once the
// predecessor grid has completed and its memory is visible).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Let the next PDL-launched kernel of the stream be scheduled now (on the SMs this grid
// leaves free) instead of at this grid's completion; it still sees this grid's memory
// only after its own pdl_wait().
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

}  // namespace lg

// host-side error helpers ------------------------------------------------------
void lg_set_error(const char* fmt, ...);
#define LG_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess) {                                                           \
      lg_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
      return LGRECO_ECUDA;                                                             \
    }                                                                                  \
  } while (0)
