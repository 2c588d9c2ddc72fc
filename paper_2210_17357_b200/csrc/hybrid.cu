// hybrid.cu -- NEXT-4: mixed-family plans ("combining different compression
// techniques inside the same model").  Two tiny device kernels around the unchanged
// solver: the families' (err, bits) tables side by side in one table (Algorithm 1 then
// picks a (family, parameter) column per layer), and the chosen columns split back into
// per-family choice vectors (LGRECO_CHOICE_SKIP where another family owns the layer).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "ctx.h"

namespace lg {

constexpr int HY_MAXF = 8;
struct HyTabs { const double* err[HY_MAXF]; const int64_t* bits[HY_MAXF]; int32_t K[HY_MAXF]; int32_t c0[HY_MAXF + 1]; };
struct HyOut { int32_t* ch[HY_MAXF]; int32_t K[HY_MAXF]; int32_t c0[HY_MAXF + 1]; };

__global__ void k_hybrid_table(HyTabs t, int F, int L, double* __restrict__ err, int64_t* __restrict__ bits) {
  const int Kt = t.c0[F];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)L * Kt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / Kt), col = (int)(i - (int64_t)l * Kt);
    int f = 0;
    while (f + 1 < F && col >= t.c0[f + 1]) ++f;
    const int j = col - t.c0[f];
    err[i] = t.err[f][(int64_t)l * t.K[f] + j];
    bits[i] = t.bits[f][(int64_t)l * t.K[f] + j];
  }
}

__global__ void k_hybrid_split(const int32_t* __restrict__ choice, HyOut o, int F, int L) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < L; l += gridDim.x * blockDim.x) {
    const int col = choice[l];
    for (int f = 0; f < F; ++f) {
      int v;
      if (col < 0) v = (f == 0) ? col : LGRECO_CHOICE_SKIP;  // lossless layers: family 0's alone
      else if (col >= o.c0[f] && col < o.c0[f + 1]) v = col - o.c0[f];
      else v = LGRECO_CHOICE_SKIP;
      o.ch[f][l] = v;
    }
  }
}

}  // namespace lg

extern "C" int lgreco_hybrid_table(const double* const* h_err_f, const int64_t* const* h_bits_f, const int32_t* h_K,
                                   int32_t F, int32_t L, double* d_err_out, int64_t* d_bits_out, void* stream) {
  if (!h_err_f || !h_bits_f || !h_K || !d_err_out || !d_bits_out || F < 1 || F > lg::HY_MAXF || L < 0) {
    lg_set_error("hybrid_table: bad arguments");
    return LGRECO_EINVAL;
  }
  lg::HyTabs t{};
  t.c0[0] = 0;
  for (int f = 0; f < F; ++f) {
    if (!h_err_f[f] || !h_bits_f[f] || h_K[f] < 1) { lg_set_error("hybrid_table: family %d", f); return LGRECO_EINVAL; }
    t.err[f] = h_err_f[f];
    t.bits[f] = h_bits_f[f];
    t.K[f] = h_K[f];
    t.c0[f + 1] = t.c0[f] + h_K[f];
  }
  const int64_t n = (int64_t)L * t.c0[F];
  if (n == 0) return LGRECO_OK;
  lg::k_hybrid_table<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, (cudaStream_t)stream>>>(
      t, F, L, d_err_out, d_bits_out);
  return cudaGetLastError() == cudaSuccess ? LGRECO_OK : LGRECO_ECUDA;
}

extern "C" int lgreco_hybrid_split(const int32_t* d_choice, const int32_t* h_K, int32_t F, int32_t L,
                                   int32_t* const* h_choice_f, void* stream) {
  if (!d_choice || !h_K || !h_choice_f || F < 1 || F > lg::HY_MAXF || L < 0) {
    lg_set_error("hybrid_split: bad arguments");
    return LGRECO_EINVAL;
  }
  lg::HyOut o{};
  o.c0[0] = 0;
  for (int f = 0; f < F; ++f) {
    if (!h_choice_f[f] || h_K[f] < 1) { lg_set_error("hybrid_split: family %d", f); return LGRECO_EINVAL; }
    o.ch[f] = h_choice_f[f];
    o.K[f] = h_K[f];
    o.c0[f + 1] = o.c0[f] + h_K[f];
  }
  if (L == 0) return LGRECO_OK;
  lg::k_hybrid_split<<<(L + 255) / 256, 256, 0, (cudaStream_t)stream>>>(d_choice, o, F, L);
  return cudaGetLastError() == cudaSuccess ? LGRECO_OK : LGRECO_ECUDA;
}
