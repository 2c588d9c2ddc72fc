// dp.cu -- K4: Algorithm 1 of L-GreCo on one CTA.
//
// DP[l][e] = min_c DP[l-1][e - disc[l][c]] + bits[l][c] over discretised error
// bins e in [0, D], step Emax/D (Alg.1 lines 2-22), argmin over the last row
// (line 23) and backtracking through PD (lines 24-27).  Readings: R16 ceil
// discretisation, R17 disc > D skipped, R18 min-update init through a virtual
// layer 0, R19 strict < in candidate order and smallest e on argmin ties, R20
// fallback to the defaults.  The layer loop is sequential (a barrier per row);
// the D+1 cells of a row are spread over 1024 threads; both rows live in shared
// memory, PD (one byte per cell) in global memory.
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace lg {

constexpr int DP_THREADS = 1024;
constexpr int64_t DP_INF = INT64_MAX;

__device__ __forceinline__ double metric(double v, uint32_t flags) {
  return (flags & LGRECO_METRIC_SQ) ? __dmul_rn(v, v) : v;
}

__device__ __forceinline__ int32_t discretise(double m, double emax, int D, uint32_t flags) {
  if (emax == 0.0) return (m == 0.0) ? 0 : -1;
  const double q = __ddiv_rn(__dmul_rn(m, (double)D), emax);
  const double r = (flags & LGRECO_DISC_FLOOR) ? floor(q) : ceil(q);
  return (r > (double)D) ? -1 : (int32_t)r;
}

__global__ void __launch_bounds__(DP_THREADS, 1)
k_solve(const double* __restrict__ err, const int64_t* __restrict__ bits, int L, int K,
        const int32_t* __restrict__ default_idx, const int32_t* __restrict__ compress, int D, uint32_t flags,
        int32_t* __restrict__ choice, lgreco_solve_info* __restrict__ info, uint8_t* __restrict__ PD,
        int32_t* __restrict__ act, int64_t* __restrict__ grows, int rows_in_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int32_t s_disc[256];
  __shared__ int64_t s_bits[256];
  __shared__ int s_La, s_status;
  __shared__ double s_emax;
  __shared__ int64_t s_defbits;
  __shared__ int64_t s_redv[DP_THREADS / 32];
  __shared__ int s_rede[DP_THREADS / 32];
  const int tid = threadIdx.x;

  // ---- Alg.1 lines 1-2: active layers, Emax of the defaults (layer order, fp64)
  if (tid == 0) {
    int La = 0, status = LGRECO_OK;
    double emax = 0.0;
    int64_t defb = 0;
    for (int l = 0; l < L; ++l) {
      choice[l] = -1;
      if (compress && !compress[l]) continue;
      const int d = default_idx[l];
      if (d < 0 || d >= K) { status = LGRECO_EINVAL; continue; }
      for (int c = 0; c < K; ++c) {
        const double v = err[(int64_t)l * K + c];
        if (!isfinite(v) || v < 0.0) status = LGRECO_ENONFINITE;
        if (bits[(int64_t)l * K + c] < 0) status = LGRECO_EINVAL;
      }
      act[La++] = l;
      emax = __dadd_rn(emax, metric(err[(int64_t)l * K + d], flags));
      defb += bits[(int64_t)l * K + d];
    }
    s_La = La; s_status = status; s_emax = emax; s_defbits = defb;
  }
  __syncthreads();
  const int La = s_La;
  const double emax = s_emax;
  if (s_status != LGRECO_OK || La == 0) {
    if (tid == 0) {
      lgreco_solve_info inf = {};
      inf.n_active = La;
      inf.status = s_status;
      *info = inf;
    }
    return;
  }
  int64_t* rowA = rows_in_smem ? reinterpret_cast<int64_t*>(smem_raw) : grows;
  int64_t* rowB = rowA + (D + 1);
  for (int e = tid; e <= D; e += DP_THREADS) rowA[e] = (e == 0) ? 0 : DP_INF;  // virtual layer 0
  int64_t* prev = rowA;
  int64_t* cur = rowB;

  // ---- Alg.1 lines 13-22 (with the min-update init of line 10, R18)
  for (int a = 0; a < La; ++a) {
    const int l = act[a];
    if (tid < K) {
      s_disc[tid] = discretise(metric(err[(int64_t)l * K + tid], flags), emax, D, flags);
      s_bits[tid] = bits[(int64_t)l * K + tid];
    }
    __syncthreads();
    uint8_t* pdrow = PD + (int64_t)a * (D + 1);
    for (int e = tid; e <= D; e += DP_THREADS) {
      int64_t best = DP_INF;
      int pd = 0;
      for (int c = 0; c < K; ++c) {
        const int d = s_disc[c];
        if (d < 0 || d > e) continue;
        const int64_t p = prev[e - d];
        if (p == DP_INF) continue;
        const int64_t t = p + s_bits[c];
        if (t < best) { best = t; pd = c; }
      }
      cur[e] = best;
      pdrow[e] = (uint8_t)pd;
    }
    __syncthreads();
    int64_t* sw = prev; prev = cur; cur = sw;
  }

  // ---- line 23: argmin over the last row, smallest e on ties (R19)
  int64_t bv = DP_INF;
  int be = 0x7fffffff;
  for (int e = tid; e <= D; e += DP_THREADS)
    if (prev[e] < bv) { bv = prev[e]; be = e; }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t ov = __shfl_xor_sync(LG_FULL, bv, o);
    const int oe = __shfl_xor_sync(LG_FULL, be, o);
    if (ov < bv || (ov == bv && oe < be)) { bv = ov; be = oe; }
  }
  if ((tid & 31) == 0) { s_redv[tid >> 5] = bv; s_rede[tid >> 5] = be; }
  __syncthreads();

  // ---- lines 24-27: backtrack; R20 fallback; summary
  if (tid == 0) {
    bv = DP_INF; be = 0x7fffffff;
    for (int w = 0; w < DP_THREADS / 32; ++w)
      if (s_redv[w] < bv || (s_redv[w] == bv && s_rede[w] < be)) { bv = s_redv[w]; be = s_rede[w]; }
    int used_default = 0;
    if (bv == DP_INF) {
      used_default = 1;
    } else {
      int e = be;
      for (int a = La - 1; a >= 0; --a) {
        const int l = act[a];
        const int c = PD[(int64_t)a * (D + 1) + e];
        choice[l] = c;
        e -= discretise(metric(err[(int64_t)l * K + c], flags), emax, D, flags);
      }
      int64_t pb = 0;
      double pe = 0.0;
      for (int a = 0; a < La; ++a) {
        const int l = act[a];
        pb += bits[(int64_t)l * K + choice[l]];
        pe = __dadd_rn(pe, metric(err[(int64_t)l * K + choice[l]], flags));
      }
      if (pb > s_defbits || pe > emax) used_default = 1;
    }
    if (used_default)
      for (int a = 0; a < La; ++a) choice[act[a]] = default_idx[act[a]];
    int64_t tb = 0;
    double te = 0.0;
    for (int a = 0; a < La; ++a) {
      const int l = act[a];
      tb += bits[(int64_t)l * K + choice[l]];
      te = __dadd_rn(te, metric(err[(int64_t)l * K + choice[l]], flags));
    }
    lgreco_solve_info inf = {};
    inf.emax = emax;
    inf.total_err = te;
    inf.total_bits = tb;
    inf.default_bits = s_defbits;
    inf.used_default = used_default;
    inf.n_active = La;
    inf.status = LGRECO_OK;
    *info = inf;
  }
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

size_t solve_workspace_bytes(int L, int K, int D) {
  (void)K;
  return align_up((size_t)L * (D + 1)) + align_up(sizeof(int32_t) * (size_t)(L + 1)) +
         align_up(sizeof(int64_t) * 2 * (size_t)(D + 1));
}

cudaError_t launch_solve(const SolveArgs& a, void* ws, cudaStream_t st) {
  uint8_t* base = static_cast<uint8_t*>(ws);
  uint8_t* pd = base;
  int32_t* act = reinterpret_cast<int32_t*>(base + align_up((size_t)a.L * (a.D + 1)));
  int64_t* grows = reinterpret_cast<int64_t*>(base + align_up((size_t)a.L * (a.D + 1)) +
                                              align_up(sizeof(int32_t) * (size_t)(a.L + 1)));
  const size_t row_bytes = sizeof(int64_t) * 2 * (size_t)(a.D + 1);
  const int in_smem = row_bytes <= 200 * 1024;
  const size_t smem = in_smem ? row_bytes : 0;
  cudaError_t e = cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(200 * 1024));
  if (e != cudaSuccess) return e;
  k_solve<<<1, DP_THREADS, smem, st>>>(a.err, a.bits, a.L, a.K, a.default_idx, a.compress, a.D, a.flags,
                                       a.choice, a.info, pd, act, grows, in_smem);
  return cudaGetLastError();
}

}  // namespace lg
