// accum.cu -- K0: the paper-mode gradient accumulation G += g.
//
// PAPER.md:313 "we accumulate per-layer gradients in auxiliary buffers" and :318 (the
// memory cost is one copy of the model): between two replans every step adds its local
// gradient into G; lgreco_profile then reads G with d_ef = NULL (R2).
// Arithmetic: one IEEE fp32 round-to-nearest add per element, G[i] = fl(G[i] + g[i]).
//
// HBM-bound: 12 B per element (read G, read g, write G).  128-bit loads / stores when
// both pointers share their alignment mod 16 (scalar head up to the 16-byte boundary,
// scalar tail), else a scalar grid-stride loop.  Grid = SMs x 4 CTAs of 512 threads,
// 4 float4 per thread in flight per iteration.
#include "common.cuh"

namespace {

__global__ void __launch_bounds__(512) k_accumulate(float* __restrict__ G, const float* __restrict__ g, int64_t n,
                                                    int64_t head, int vec) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  if (!vec) {
    for (int64_t i = tid; i < n; i += nthr) G[i] = __fadd_rn(G[i], g[i]);
    return;
  }
  // scalar head [0, head) and tail, vector body
  if (tid < head) G[tid] = __fadd_rn(G[tid], g[tid]);
  const int64_t nv = (n - head) >> 2;
  float4* __restrict__ Gv = reinterpret_cast<float4*>(G + head);
  const float4* __restrict__ gv = reinterpret_cast<const float4*>(g + head);
  int64_t i = tid;
  for (; i + 3 * nthr < nv; i += 4 * nthr) {
    float4 a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { a[u] = Gv[i + u * nthr]; b[u] = __ldcs(gv + i + u * nthr); }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u].x = __fadd_rn(a[u].x, b[u].x); a[u].y = __fadd_rn(a[u].y, b[u].y);
      a[u].z = __fadd_rn(a[u].z, b[u].z); a[u].w = __fadd_rn(a[u].w, b[u].w);
      Gv[i + u * nthr] = a[u];
    }
  }
  for (; i < nv; i += nthr) {
    float4 a = Gv[i];
    const float4 b = __ldcs(gv + i);
    a.x = __fadd_rn(a.x, b.x); a.y = __fadd_rn(a.y, b.y); a.z = __fadd_rn(a.z, b.z); a.w = __fadd_rn(a.w, b.w);
    Gv[i] = a;
  }
  const int64_t t0 = head + (nv << 2);
  if (tid < n - t0) G[t0 + tid] = __fadd_rn(G[t0 + tid], g[t0 + tid]);
}

}  // namespace

extern "C" int lgreco_accumulate(float* d_G, const float* d_g, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!d_G || !d_g))) {
    lg_set_error("accumulate: bad argument (n = %lld)", (long long)n);
    return LGRECO_EINVAL;
  }
  if (n == 0) return LGRECO_OK;
  const uintptr_t aG = reinterpret_cast<uintptr_t>(d_G), ag = reinterpret_cast<uintptr_t>(d_g);
  if ((aG & 3) || (ag & 3)) {
    lg_set_error("accumulate: pointers must be 4-byte aligned");
    return LGRECO_EINVAL;
  }
  int dev = 0, nsm = 148;
  LG_CUDA(cudaGetDevice(&dev));
  LG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int vec = (aG & 15) == (ag & 15);
  int64_t head = vec ? (int64_t)(((16 - (aG & 15)) & 15) >> 2) : 0;
  if (head > n) head = n;
  const int64_t work = vec ? (n - head) / 4 : n;
  int64_t blocks = (work + 511) / 512;
  if (blocks > (int64_t)nsm * 4) blocks = (int64_t)nsm * 4;
  if (blocks < 1) blocks = 1;
  k_accumulate<<<(unsigned)blocks, 512, 0, (cudaStream_t)stream>>>(d_G, d_g, n, head, vec);
  LG_CUDA(cudaGetLastError());
  return LGRECO_OK;
}
