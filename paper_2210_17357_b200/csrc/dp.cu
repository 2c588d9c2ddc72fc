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

#include <algorithm>

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
k_solve_generic(const double* __restrict__ err, const int64_t* __restrict__ bits, int L, int K,
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


// ---------------------------------------------------------------------------
// Fast path: cells in registers, packed (value << cbits | c) keys.
// Costs are divided by g = gcd of all active costs (an exact order-preserving
// rescale), so the DP runs on 32-bit keys whenever the largest possible plan
// cost fits in 31 - cbits bits, else on 64-bit keys.  min() over packed keys
// picks the smallest cost and, among equal costs, the first candidate in list
// order -- exactly Alg.1's strict-< update in candidate order (R19).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t gcd64(uint64_t a, uint64_t b) {
  while (b) { const uint64_t t = a % b; a = b; b = t; }
  return a;
}

template <int CPT, int KT>
__global__ void __launch_bounds__(DP_THREADS, 1)
k_solve_fast(const double* __restrict__ err, const int64_t* __restrict__ bits, int L, int K,
             const int32_t* __restrict__ default_idx, const int32_t* __restrict__ compress, int D, uint32_t flags,
             int32_t* __restrict__ choice, lgreco_solve_info* __restrict__ info, uint8_t* __restrict__ PD,
             int32_t* __restrict__ act, int32_t* __restrict__ wdisc, uint64_t* __restrict__ wadd) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int32_t s_disc[2][256];
  __shared__ uint64_t s_add[2][256];
  __shared__ int s_La, s_status, s_wide, s_cbits;
  __shared__ double s_emax;
  __shared__ int64_t s_defbits;
  __shared__ unsigned long long s_mx;
  __shared__ uint64_t s_g[DP_THREADS / 32];
  __shared__ uint64_t s_redk[DP_THREADS / 32];
  __shared__ int s_rede[DP_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W1 = D + 1;

  // ---- prelude, parallel: stage flags/defaults in smem (row area is free yet)
  int32_t* sm_flag = reinterpret_cast<int32_t*>(smem_raw);   // [L]
  int32_t* sm_def = sm_flag + L;                             // [L]
  double* sm_de = reinterpret_cast<double*>(sm_def + L);  // [L] metric(err[l][def]) (8L bytes in: aligned)
  int64_t* sm_db = reinterpret_cast<int64_t*>(sm_de + L);    // [L] bits[l][def]
  if (tid == 0) { s_status = LGRECO_OK; s_mx = 0; }
  __syncthreads();
  for (int l = tid; l < L; l += DP_THREADS) {
    const int f = compress ? (compress[l] != 0) : 1;
    const int d = default_idx[l];
    sm_flag[l] = f;
    sm_def[l] = d;
    choice[l] = -1;
    if (f) {
      if (d < 0 || d >= K) { atomicExch(&s_status, LGRECO_EINVAL); sm_de[l] = 0.0; sm_db[l] = 0; }
      else { sm_de[l] = metric(err[(int64_t)l * K + d], flags); sm_db[l] = bits[(int64_t)l * K + d]; }
    }
  }
  __syncthreads();
  // ---- Alg.1 lines 1-2 (thread 0, layer order, from shared memory)
  if (tid == 0) {
    int La = 0;
    double emax = 0.0;
    int64_t defb = 0;
    for (int l = 0; l < L; ++l) {
      if (!sm_flag[l]) continue;
      act[La++] = l;
      emax = __dadd_rn(emax, sm_de[l]);
      defb += sm_db[l];
    }
    s_La = La; s_emax = emax; s_defbits = defb;
    int cb = 0;
    while ((1 << cb) < K) ++cb;
    s_cbits = cb;
  }
  __syncthreads();
  const int La = s_La;
  const double emax = s_emax;
  // ---- validation + gcd of costs + largest plan cost (parallel)
  uint64_t gg = 0;
  int bad = 0;
  for (int i = tid; i < La * K; i += DP_THREADS) {
    const int l = act[i / K];
    const double v = err[(int64_t)l * K + (i % K)];
    const int64_t b = bits[(int64_t)l * K + (i % K)];
    if (!isfinite(v) || v < 0.0) bad |= 1;
    if (b < 0) bad |= 2;
    gg = gcd64(gg, (uint64_t)(b < 0 ? 0 : b));
  }
  bad = __reduce_or_sync(LG_FULL, bad);
#pragma unroll
  for (int o = 16; o; o >>= 1) gg = gcd64(gg, __shfl_xor_sync(LG_FULL, gg, o));
  if (lane == 0) {
    s_g[warp] = gg;
    if (bad & 1) atomicExch(&s_status, LGRECO_ENONFINITE);
    else if (bad & 2) atomicExch(&s_status, LGRECO_EINVAL);
  }
  __syncthreads();
  if (tid == 0) {
    uint64_t g = 0;
    for (int w = 0; w < DP_THREADS / 32; ++w) g = gcd64(g, s_g[w]);
    s_g[0] = g ? g : 1;
  }
  __syncthreads();
  const uint64_t g = s_g[0];
  for (int a = tid; a < La; a += DP_THREADS) {
    uint64_t m = 0;
    for (int c = 0; c < K; ++c) m = max(m, (uint64_t)max((int64_t)0, bits[(int64_t)act[a] * K + c]) / g);
    atomicAdd(&s_mx, (unsigned long long)m);
  }
  __syncthreads();
  if (tid == 0) {
    s_wide = (s_mx >= (1ull << (30 - s_cbits))) ? 1 : 0;  // 32-bit keys < 2^30 < INF32
    if (s_mx >= (1ull << (62 - s_cbits)) && s_status == LGRECO_OK) s_status = LGRECO_EINVAL;
  }
  __syncthreads();
  if (s_status != LGRECO_OK || La == 0) {
    if (tid == 0) {
      lgreco_solve_info inf = {};
      inf.n_active = La;
      inf.status = s_status;
      *info = inf;
    }
    return;
  }
  const int cbits = s_cbits;
  const uint64_t cmask = (1ull << cbits) - 1;
  const bool wide = s_wide;
  // ---- Alg.1 lines 3-5 for every (layer, candidate), in parallel, to the workspace
  for (int i = tid; i < La * K; i += DP_THREADS) {
    const int a = i / K, c = i % K;
    const int l = act[a];
    wdisc[i] = discretise(metric(err[(int64_t)l * K + c], flags), emax, D, flags);
    wadd[i] = (((uint64_t)bits[(int64_t)l * K + c] / g) << cbits) | (uint64_t)c;
  }
  __syncthreads();
  // rows: 32-bit keys -> two rows padded with W1 INF entries in front (no bounds test);
  //       64-bit keys -> two rows with one INF sentinel at index -1 (clamped index)
  // (+ DP_THREADS tail entries: the last register cell of a thread may lie past D)
  const int row32 = 2 * W1 + DP_THREADS, row64 = W1 + 1 + DP_THREADS;
  uint32_t* r32a = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* r32b = r32a + row32;
  uint64_t* r64a = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* r64b = r64a + row64;
  const uint32_t INF32 = 0x7FFFFF00u;  // > every 32-bit key; INF32 + addend < 2^32
  const uint64_t INF64 = 1ull << 62;
  if (!wide) {
    for (int i = tid; i < row32; i += DP_THREADS) { r32a[i] = (i == W1) ? 0u : INF32; r32b[i] = INF32; }
  } else {
    for (int i = tid; i < row64; i += DP_THREADS) { r64a[i] = (i == 1) ? 0ull : INF64; r64b[i] = INF64; }
  }
  if (tid < K) { s_disc[0][tid] = wdisc[tid]; s_add[0][tid] = wadd[tid]; }
  __syncthreads();
  int cur_is_b = 1;
  for (int a = 0; a < La; ++a) {
    const int sb = a & 1;
    // prefetch the next layer's candidate row (published by the barrier below)
    int32_t nd = -1;
    uint64_t na = 0;
    if (tid < K && a + 1 < La) { nd = wdisc[(a + 1) * K + tid]; na = wadd[(a + 1) * K + tid]; }
    uint8_t* pdrow = PD + (int64_t)a * W1;
    if (!wide) {
      const uint32_t* prev = (cur_is_b ? r32a : r32b) + W1;  // index e-d >= -W1 is padded
      uint32_t* cur = (cur_is_b ? r32b : r32a) + W1;
      uint32_t best[CPT];
#pragma unroll
      for (int i = 0; i < CPT; ++i) best[i] = 0xFFFFFFFFu;
      if (KT > 0) {
        // compile-time candidate bound: every prev[] read is an LDS with an immediate offset
#pragma unroll
        for (int c = 0; c < (KT > 0 ? KT : 1); ++c) {
          if (c < K) {
            const int d = s_disc[sb][c];
            if (d >= 0) {
              const uint32_t ak = (uint32_t)s_add[sb][c];
              const uint32_t* pv = prev - d + tid;
#pragma unroll
              for (int i = 0; i < CPT; ++i) best[i] = min(best[i], pv[i * DP_THREADS] + ak);
            }
          }
        }
      } else {
        for (int c = 0; c < K; ++c) {
          const int d = s_disc[sb][c];
          if (d < 0) continue;
          const uint32_t ak = (uint32_t)s_add[sb][c];
          const uint32_t* pv = prev - d + tid;
#pragma unroll
          for (int i = 0; i < CPT; ++i) best[i] = min(best[i], pv[i * DP_THREADS] + ak);
        }
      }
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const int e = tid + i * DP_THREADS;
        if (e < W1) {
          const uint32_t k = best[i];
          cur[e] = min(k, INF32) & ~(uint32_t)cmask;  // unreachable stays >= INF32
          pdrow[e] = (uint8_t)(k & (uint32_t)cmask);   // read only on the backtrack path
        }
      }
    } else {
      const uint64_t* prev = (cur_is_b ? r64a : r64b) + 1;  // index -1 is the INF sentinel
      uint64_t* cur = (cur_is_b ? r64b : r64a) + 1;
      uint64_t best[CPT];
#pragma unroll
      for (int i = 0; i < CPT; ++i) best[i] = ~0ull;
      for (int c = 0; c < K; ++c) {
        const int d = s_disc[sb][c];
        if (d < 0) continue;
        const uint64_t ak = s_add[sb][c];
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
          const int idx = max(tid + i * DP_THREADS - d, -1);
          best[i] = min(best[i], prev[idx] + ak);
        }
      }
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const int e = tid + i * DP_THREADS;
        if (e < W1) {
          const uint64_t k = best[i];
          cur[e] = (k >= INF64) ? INF64 : (k & ~cmask);
          pdrow[e] = (uint8_t)((k >= INF64) ? 0 : (k & cmask));
        }
      }
    }
    if (tid < K) { s_disc[sb ^ 1][tid] = nd; s_add[sb ^ 1][tid] = na; }
    cur_is_b ^= 1;
    __syncthreads();
  }
  // ---- line 23: argmin of the last row, smallest e on ties
  uint64_t bk = ~0ull;
  int be = 0x7fffffff;
  for (int e = tid; e < W1; e += DP_THREADS) {
    uint64_t v;
    if (!wide) { const uint32_t x = ((cur_is_b ? r32a : r32b) + W1)[e]; v = (x >= INF32) ? ~0ull : x; }
    else { const uint64_t x = ((cur_is_b ? r64a : r64b) + 1)[e]; v = (x >= INF64) ? ~0ull : x; }
    if (v < bk) { bk = v; be = e; }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t ov = __shfl_xor_sync(LG_FULL, bk, o);
    const int oe = __shfl_xor_sync(LG_FULL, be, o);
    if (ov < bk || (ov == bk && oe < be)) { bk = ov; be = oe; }
  }
  if (lane == 0) { s_redk[warp] = bk; s_rede[warp] = be; }
  __syncthreads();
  // stage the discretised table in shared memory for the serial backtrack
  int32_t* sdisc_all = reinterpret_cast<int32_t*>(smem_raw);
  const bool disc_in_smem = (size_t)La * K * 4 <= (size_t)4 * (wide ? 2 * row64 * 2 : 2 * row32);
  if (disc_in_smem)
    for (int i = tid; i < La * K; i += DP_THREADS) sdisc_all[i] = wdisc[i];
  __syncthreads();
  const int32_t* bdisc = disc_in_smem ? sdisc_all : wdisc;
  // ---- lines 24-27 backtrack + R20 (thread 0)
  if (tid == 0) {
    bk = ~0ull; be = 0x7fffffff;
    for (int w = 0; w < DP_THREADS / 32; ++w)
      if (s_redk[w] < bk || (s_redk[w] == bk && s_rede[w] < be)) { bk = s_redk[w]; be = s_rede[w]; }
    int used_default = 0;
    if (bk == ~0ull) {
      used_default = 1;
    } else {
      int e = be;
      for (int a = La - 1; a >= 0; --a) {
        const int c = PD[(int64_t)a * W1 + e];
        choice[act[a]] = c;
        e -= bdisc[a * K + c];
      }
    }
    s_La = used_default;
  }
  __syncthreads();
  // R20 check and the summary (parallel gathers, ordered fp64 sum by thread 0)
  double* sm_ce = reinterpret_cast<double*>(smem_raw);         // [La] metric(err[choice])
  int64_t* sm_cb = reinterpret_cast<int64_t*>(sm_ce + La);    // [La] bits[choice]
  int used_default = s_La;
  if (used_default) {
    for (int a = tid; a < La; a += DP_THREADS) choice[act[a]] = default_idx[act[a]];
    __syncthreads();
  }
  for (int pass = 0; pass < 2; ++pass) {
    for (int a = tid; a < La; a += DP_THREADS) {
      const int l = act[a];
      const int c = used_default ? default_idx[l] : choice[l];
      sm_ce[a] = metric(err[(int64_t)l * K + c], flags);
      sm_cb[a] = bits[(int64_t)l * K + c];
    }
    __syncthreads();
    if (tid == 0) {
      int64_t pb = 0;
      double pe = 0.0;
      for (int a = 0; a < La; ++a) { pb += sm_cb[a]; pe = __dadd_rn(pe, sm_ce[a]); }
      if (!used_default && (pb > s_defbits || pe > emax)) {
        s_La = 1;  // fall back; recompute the summary for the defaults
      } else {
        lgreco_solve_info inf = {};
        inf.emax = emax;
        inf.total_err = pe;
        inf.total_bits = pb;
        inf.default_bits = s_defbits;
        inf.used_default = used_default;
        inf.n_active = La;
        inf.status = LGRECO_OK;
        *info = inf;
        s_La = -1;  // done
      }
    }
    __syncthreads();
    if (s_La < 0) break;
    used_default = 1;
    for (int a = tid; a < La; a += DP_THREADS) choice[act[a]] = default_idx[act[a]];
    __syncthreads();
  }
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

size_t solve_workspace_bytes(int L, int K, int D) {
  return align_up((size_t)L * (D + 1)) + align_up(sizeof(int32_t) * (size_t)(L + 1)) +
         align_up(sizeof(int64_t) * 2 * (size_t)(D + 1)) + align_up(sizeof(int32_t) * (size_t)L * K) +
         align_up(sizeof(uint64_t) * (size_t)L * K);
}

cudaError_t launch_solve(const SolveArgs& a, void* ws, cudaStream_t st) {
  uint8_t* base = static_cast<uint8_t*>(ws);
  uint8_t* pd = base;
  int32_t* act = reinterpret_cast<int32_t*>(base + align_up((size_t)a.L * (a.D + 1)));
  int64_t* grows = reinterpret_cast<int64_t*>(base + align_up((size_t)a.L * (a.D + 1)) +
                                              align_up(sizeof(int32_t) * (size_t)(a.L + 1)));
  int32_t* wdisc = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(grows) +
                                              align_up(sizeof(int64_t) * 2 * (size_t)(a.D + 1)));
  uint64_t* wadd = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(wdisc) +
                                               align_up(sizeof(int32_t) * (size_t)a.L * a.K));
  const int W1 = a.D + 1;
  const int cpt = (W1 + DP_THREADS - 1) / DP_THREADS;
  // fast path: two padded 32-bit rows or two 64-bit rows in smem (see k_solve_fast)
  const size_t fast_smem = std::max((size_t)8 * (2 * W1 + DP_THREADS), (size_t)16 * (W1 + 1 + DP_THREADS));
  // the prelude stages 24 bytes per layer in the same shared memory
  if (cpt <= 12 && fast_smem <= 200 * 1024 && (size_t)24 * a.L + 64 <= fast_smem) {
    cudaError_t e = cudaSuccess;
#define LG_SF2(C, KT)                                                                                      \
  {                                                                                                          \
    e = cudaFuncSetAttribute(k_solve_fast<C, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);  \
    if (e != cudaSuccess) return e;                                                                          \
    k_solve_fast<C, KT><<<1, DP_THREADS, fast_smem, st>>>(a.err, a.bits, a.L, a.K, a.default_idx, a.compress, \
                                                          a.D, a.flags, a.choice, a.info, pd, act, wdisc, wadd); \
  }
#define LG_SF(C)                                       \
  case C:                                              \
    if (a.K <= 8) LG_SF2(C, 8) else if (a.K <= 16) LG_SF2(C, 16) else LG_SF2(C, 0) \
    break;
    switch (cpt) { LG_SF(1) LG_SF(2) LG_SF(3) LG_SF(4) LG_SF(5) LG_SF(6) LG_SF(7) LG_SF(8) LG_SF(9) LG_SF(10)
                   LG_SF(11) LG_SF(12) }
#undef LG_SF
    return cudaGetLastError();
  }
  const size_t row_bytes = sizeof(int64_t) * 2 * (size_t)(a.D + 1);
  const int in_smem = row_bytes <= 200 * 1024;
  const size_t smem = in_smem ? row_bytes : 0;
  cudaError_t e = cudaFuncSetAttribute(k_solve_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(200 * 1024));
  if (e != cudaSuccess) return e;
  k_solve_generic<<<1, DP_THREADS, smem, st>>>(a.err, a.bits, a.L, a.K, a.default_idx, a.compress, a.D, a.flags,
                                               a.choice, a.info, pd, act, grows, in_smem);
  return cudaGetLastError();
}

}  // namespace lg
