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
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <time.h>
#include <unistd.h>

#include "common.cuh"
#include "kernels.h"
#include "memo.h"

namespace lg {

constexpr int DP_THREADS = 1024;
constexpr int64_t DP_INF = INT64_MAX;

// saturating sum of costs (the width guard: a wrapped sum would skip the EINVAL check)
__device__ __forceinline__ unsigned long long sat_add(unsigned long long a, unsigned long long b) {
  const unsigned long long s = a + b;
  return s < a ? ~0ull : s;
}

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
// Fast path: cells in registers, packed (value << kb | c) keys.
// Costs are divided by g = the largest power of two dividing every active cost (an
// exact order- and sum-preserving rescale: one OR-reduction, a shift per cost).  min() over packed keys picks the smallest cost and, among equal costs,
// the first candidate in list order -- exactly Alg.1's strict-< update in candidate
// order (R19).  32-bit keys (one LDS + one VIADDMNMX, DPX add-min, per cell and
// candidate) whenever the largest plan cost fits 30 - kb bits:
//   K <= 16 (KT > 0): kb = ceil(log2 K), key = value << kb | c;
//   K > 16 (KT = 0):  candidates in groups of 16, kb = 4, key = value << 4 | (c % 16);
//                     the min over a group is merged into the running best by value
//                     with strict < (earlier group wins ties), the group kept aside.
// Otherwise 64-bit keys value << cbits | c.
//
// A warp owns 32*CPT consecutive cells; row arrays carry 32*CPT INF cells in front.
// A candidate shift d > wbase + 32*CPT (the warp's whole window below cell 0) is
// clamped to wbase + 32*CPT, so every read lands in the row or in the INF pad.
// PD is stored thread-major, one 16-byte word per thread and layer (byte i =
// register i): PD byte of (layer a, cell e) = PD[a*16384 + tid(e)*16 + i(e)].
// ---------------------------------------------------------------------------
constexpr int PD_ROW = DP_THREADS * 16;

// Cell e lives in warp w = e / (32*CPT), register i = (e % (32*CPT)) / 32, lane e % 32:
// a warp owns one contiguous range of 32*CPT cells (so a warp wholly outside the
// reachable band skips its row at once).
template <int CPT>
__device__ __forceinline__ int pd_byte(const uint8_t* PD, int a, int e) {
  const int w = e / (32 * CPT), r = e - w * (32 * CPT);
  return __ldcg(PD + (int64_t)a * PD_ROW + (w * 32 + (r & 31)) * 16 + (r >> 5));  // L2 (written this kernel)
}

// byte p of x replaced by the low byte of y
__device__ __forceinline__ uint32_t put_byte(uint32_t x, uint32_t y, int p) {
  return __byte_perm(x, y, p == 0 ? 0x3214 : p == 1 ? 0x3240 : p == 2 ? 0x3410 : 0x4210);
}

#ifdef LG_DP_TIMING
#define LG_T(i) do { if (tid == 0) tstamp[i] = clock64(); } while (0)
#else
#define LG_T(i) do { } while (0)
#endif

template <int CPT, int KT>
__global__ void __launch_bounds__(DP_THREADS, 1)
k_solve_fast(const double* __restrict__ err, const int64_t* __restrict__ bits, int L, int K,
             const int32_t* __restrict__ default_idx, const int32_t* __restrict__ compress, int D, uint32_t flags,
             int32_t* __restrict__ choice, lgreco_solve_info* __restrict__ info, uint8_t* __restrict__ PD,
             int32_t* __restrict__ act, int32_t* __restrict__ wdisc, uint64_t* __restrict__ wadd) {
  static_assert(CPT >= 1 && CPT <= 16, "PD word holds 16 cells");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(16) uint2 s_cand[2][256];  // {disc, 32-bit key addend} per candidate, double-buffered
  __shared__ uint64_t s_add[2][256];  // 64-bit key addend
  __shared__ int2 s_band[2];
  __shared__ int s_La, s_status, s_wide, s_cbits;
  __shared__ double s_emax;
  __shared__ int64_t s_defbits;
  __shared__ unsigned long long s_mx;
  __shared__ uint64_t s_g[DP_THREADS / 32];
  __shared__ uint64_t s_redk[DP_THREADS / 32];
  __shared__ int s_rede[DP_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W1 = D + 1;
#ifdef LG_DP_TIMING
  long long tstamp[10];
  long long t_ldg = 0, t_rest = 0;
  int n_rounds = 0;
#endif
  LG_T(0);

  // ---- prelude, parallel: stage flags/defaults in smem (row area is free yet)
  int32_t* sm_flag = reinterpret_cast<int32_t*>(smem_raw);   // [L]
  int32_t* sm_act = sm_flag + L;                             // [L] compacted active layer ids
  double* sm_de = reinterpret_cast<double*>(sm_act + L);     // [L] metric(err[l][def]), by layer (8L bytes in)
  double* sm_dea = sm_de + L;                                // [L] the same, compacted
  if (tid == 0) { s_status = LGRECO_OK; s_mx = 0; }
  __syncthreads();
  int64_t db_part = 0;
  int bad_def = 0;
  for (int l = tid; l < L; l += DP_THREADS) {
    const int f = compress ? (compress[l] != 0) : 1;
    const int d = default_idx[l];
    sm_flag[l] = f;
    choice[l] = -1;
    if (f) {
      if (d < 0 || d >= K) { bad_def = 1; sm_de[l] = 0.0; }
      else { sm_de[l] = metric(err[(int64_t)l * K + d], flags); db_part += bits[(int64_t)l * K + d]; }
    }
  }
  if (__any_sync(LG_FULL, bad_def) && lane == 0) atomicExch(&s_status, LGRECO_EINVAL);
#pragma unroll
  for (int o = 16; o; o >>= 1) db_part += __shfl_xor_sync(LG_FULL, db_part, o);
  if (lane == 0) s_redk[warp] = (uint64_t)db_part;
  __syncthreads();
  // ---- Alg.1 lines 1-2 (warp 0): ordered compaction by ballot, Emax in layer order
  if (warp == 0) {
    int La = 0;
    for (int base = 0; base < L; base += 32) {
      const int l = base + lane;
      const int f = (l < L) ? sm_flag[l] : 0;
      const unsigned m = __ballot_sync(LG_FULL, f);
      if (f) {
        const int pos = La + __popc(m & ((1u << lane) - 1u));
        sm_act[pos] = l;
        act[pos] = l;
        sm_dea[pos] = sm_de[l];
      }
      La += __popc(m);
    }
    __syncwarp();
    if (lane == 0) {
      double emax = 0.0;
      int a = 0;
      for (; a + 4 <= La; a += 4) {  // loads hoisted, the fp64 chain stays in layer order
        const double v0 = sm_dea[a], v1 = sm_dea[a + 1], v2 = sm_dea[a + 2], v3 = sm_dea[a + 3];
        emax = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(emax, v0), v1), v2), v3);
      }
      for (; a < La; ++a) emax = __dadd_rn(emax, sm_dea[a]);
      int64_t defb = 0;
      for (int w = 0; w < DP_THREADS / 32; ++w) defb += (int64_t)s_redk[w];
      s_La = La; s_emax = emax; s_defbits = defb;
      int cb = 0;
      while ((1 << cb) < K) ++cb;
      s_cbits = cb;
    }
  }
  __syncthreads();
  LG_T(1);
  const int La = s_La;
  const double emax = s_emax;
  // ---- one pass over every (layer, candidate): validation, Alg.1 lines 3-5 (discretise
  //      to the workspace), OR of the costs, per-layer largest cost (for the key width)
  uint64_t gg = 0, mx_part = 0;
  int bad = 0;
  for (int a = warp; a < La; a += DP_THREADS / 32) {
    const int l = sm_act[a];
    uint64_t m = 0;
    for (int c = lane; c < K; c += 32) {
      const double v = err[(int64_t)l * K + c];
      const int64_t b = bits[(int64_t)l * K + c];
      if (!isfinite(v) || v < 0.0) bad |= 1;
      if (b < 0) bad |= 2;
      const uint64_t ub = (uint64_t)(b < 0 ? 0 : b);
      gg |= ub;
      m = max(m, ub);
      wdisc[a * K + c] = discretise(metric(v, flags), emax, D, flags);
      wadd[a * K + c] = ub;  // raw cost; keyed (cost/g << cbits | c) when staged per layer
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(LG_FULL, m, o));
    mx_part = sat_add(mx_part, m);  // sum_a max_c cost (lane-replicated)
  }
  bad = __reduce_or_sync(LG_FULL, bad);
#pragma unroll
  for (int o = 16; o; o >>= 1) gg |= __shfl_xor_sync(LG_FULL, gg, o);
  if (lane == 0) {
    s_g[warp] = gg;
    s_redk[warp] = mx_part;
    if (bad & 1) atomicExch(&s_status, LGRECO_ENONFINITE);
    else if (bad & 2) atomicExch(&s_status, LGRECO_EINVAL);
  }
  __syncthreads();
  if (warp == 0) {
    uint64_t g = s_g[lane];
    unsigned long long mxs = s_redk[lane];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      g |= __shfl_xor_sync(LG_FULL, g, o);
      mxs = sat_add(mxs, __shfl_xor_sync(LG_FULL, mxs, o));
    }
    if (lane == 0) {
      g = g ? (g & (~g + 1)) : 1;  // lowest set bit of the OR = 2^min ctz(cost)
      s_g[0] = g;
      // every cost is a multiple of g, so sum_a max_c cost/g = (sum_a max_c cost)/g exactly
      const uint64_t mx = mxs >> (__ffsll((long long)g) - 1);
      const int kb = (KT > 0) ? s_cbits : 4;
      s_wide = (mx >= (1ull << (30 - kb))) ? 1 : 0;  // 32-bit keys < 2^30 < INF32
      if (mx >= (1ull << (62 - s_cbits)) && s_status == LGRECO_OK) s_status = LGRECO_EINVAL;
    }
  }
  __syncthreads();
  const uint64_t g = s_g[0];
  const int gsh = __ffsll((long long)g) - 1;
  const int cbits = s_cbits;
  LG_T(2);
  if (s_status != LGRECO_OK || La == 0) {
    if (tid == 0) {
      lgreco_solve_info inf = {};
      inf.n_active = La;
      inf.status = s_status;
      *info = inf;
    }
    return;
  }
  const bool wide = s_wide;
  const int kb = wide ? cbits : ((KT > 0) ? cbits : 4);  // key bits below the value
  const uint64_t kmask = (1ull << kb) - 1;
  const int pdmask = (!wide && KT == 0) ? 0xFF : (int)((1u << cbits) - 1u);  // PD byte -> c
  auto keyed = [&](uint64_t ub, int c) -> uint64_t {
    return ((ub >> gsh) << kb) | (uint64_t)(c & (int)kmask);
  };
  // two rows of 32*CPT INF pad cells + CPT*1024 cells (cells past D are computed
  // too; a cell <= D never reads one)
  constexpr int PAD = 32 * CPT;
  const int row = PAD + CPT * DP_THREADS;
  uint32_t* r32a = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* r32b = r32a + row;
  uint64_t* r64a = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* r64b = r64a + row;
  const uint32_t INF32 = 0x7FFFFF00u;  // > every 32-bit key; INF32 + addend < 2^32
  const uint64_t INF64 = 1ull << 62;
  if (!wide) {
    for (int i = tid; i < row; i += DP_THREADS) { r32a[i] = (i == PAD) ? 0u : INF32; r32b[i] = INF32; }
  } else {
    for (int i = tid; i < row; i += DP_THREADS) { r64a[i] = (i == PAD) ? 0ull : INF64; r64b[i] = INF64; }
  }
  // Reachable band: a cell e of row a is finite only if lo_a <= e <= hi_a, with lo/hi the
  // running sums of the smallest/largest admissible disc (exact: every path to e sums
  // one admissible disc per layer).  A warp whose cells lie wholly outside the band
  // skips the row (its cells reset to INF).  Tracked for K <= 32 (warp 0).
  const bool track_band = K <= 32;
  int lo = 0, hi = 0;  // band of the virtual layer 0 (warp 0 lanes keep it)
  // Candidates of active layer a (lanes c < K loaded d, ub earlier) into slot, and the
  // band update.  Inadmissible candidates (disc < 0) and the padding up to KT become
  // {disc 0, addend INF}: they never win a min, so the inner loop has no branches.
  const int KP = (KT > 0) ? KT : K;
  auto stage = [&](int32_t d, uint64_t ub, int slot, int& blo, int& bhi) {
    if (tid < KP) {
      const bool ok = tid < K && d >= 0;
      const uint64_t k = ok ? keyed(ub, tid) : 0;
      s_cand[slot][tid] = make_uint2(ok ? (uint32_t)d : 0u, ok ? (uint32_t)k : INF32);
      s_add[slot][tid] = ok ? k : INF64;
    }
    if (track_band && warp == 0) {
      const unsigned ok = (tid < K && d >= 0) ? 1u : 0u;
      const unsigned mn = __reduce_min_sync(LG_FULL, ok ? (unsigned)d : 0x7fffffffu);
      const unsigned mxd = __reduce_max_sync(LG_FULL, ok ? (unsigned)d : 0u);
      const bool any = __any_sync(LG_FULL, ok);
      blo = any ? min(blo + (int)mn, 0x3fffffff) : 0x3fffffff;
      bhi = any ? min(bhi + (int)mxd, D) : -1;
      if (lane == 0) s_band[slot] = make_int2(blo, bhi);
    }
  };
  if (!track_band && tid == 0) { s_band[0] = make_int2(0, D); s_band[1] = make_int2(0, D); }
  {
    const int32_t d0 = (tid < K) ? wdisc[tid] : -1;
    const uint64_t u0 = (tid < K) ? wadd[tid] : 0;
    stage(d0, u0, 0, lo, hi);
  }
  __syncthreads();
  LG_T(3);
  int cur_is_b = 1;
  const int wbase = warp * (32 * CPT);
  const int dclamp = wbase + PAD;  // shifts beyond this read only INF (whole window < 0)
  for (int a = 0; a < La; ++a) {
    const int sb = a & 1;
    const int2 band = s_band[sb];
    // prefetch the next layer's candidates (staged after this row, before the barrier)
    int32_t nd = -1;
    uint64_t nub = 0;
    if (tid < K && a + 1 < La) { nd = wdisc[(a + 1) * K + tid]; nub = wadd[(a + 1) * K + tid]; }
    uint32_t pdw[4] = {0u, 0u, 0u, 0u};
    const bool live = (wbase + 32 * CPT - 1 >= band.x) && (wbase <= band.y);  // warp-uniform
    if (!wide) {
      const uint32_t* prev = (cur_is_b ? r32a : r32b) + PAD + wbase + lane;
      uint32_t* cur = (cur_is_b ? r32b : r32a) + PAD + wbase + lane;
      if (live) {
        uint32_t best[CPT];
        if (KT > 0) {
          // compile-time candidate count: every prev[] read is an LDS with an immediate offset
#pragma unroll
          for (int c = 0; c < (KT > 0 ? KT : 2); c += 2) {
            const uint4 q = *reinterpret_cast<const uint4*>(&s_cand[sb][c]);
            const uint32_t* pv = prev - min((int)q.x, dclamp);
#pragma unroll
            for (int i = 0; i < CPT; ++i)
              best[i] = (c == 0) ? pv[i * 32] + q.y : __viaddmin_u32(pv[i * 32], q.y, best[i]);
            if (c + 1 < KT) {
              const uint32_t* pw = prev - min((int)q.z, dclamp);
#pragma unroll
              for (int i = 0; i < CPT; ++i) best[i] = __viaddmin_u32(pw[i * 32], q.w, best[i]);
            }
          }
#pragma unroll
          for (int i = 0; i < CPT; ++i) {
            const uint32_t k = best[i];
            cur[i * 32] = min(k, INF32) & ~(uint32_t)kmask;  // unreachable stays >= INF32
            pdw[i >> 2] = put_byte(pdw[i >> 2], k, i & 3);   // low bits = candidate (backtrack only)
          }
        } else {
          uint32_t bgrp[CPT];
#pragma unroll
          for (int i = 0; i < CPT; ++i) { best[i] = 0xFFFFFFFFu; bgrp[i] = 0; }
          for (int c0 = 0; c0 < K; c0 += 16) {
            const int cn = min(16, K - c0);
            uint32_t gk[CPT];
#pragma unroll
            for (int i = 0; i < CPT; ++i) gk[i] = 0xFFFFFFFFu;
            for (int c = 0; c < cn; ++c) {
              const uint2 cd = s_cand[sb][c0 + c];
              const uint32_t* pv = prev - min((int)cd.x, dclamp);
#pragma unroll
              for (int i = 0; i < CPT; ++i) gk[i] = __viaddmin_u32(pv[i * 32], cd.y, gk[i]);
            }
#pragma unroll
            for (int i = 0; i < CPT; ++i)
              if ((gk[i] & ~15u) < (best[i] & ~15u)) { best[i] = gk[i]; bgrp[i] = (uint32_t)c0; }
          }
#pragma unroll
          for (int i = 0; i < CPT; ++i) {
            const uint32_t k = best[i];
            cur[i * 32] = min(k, INF32) & ~15u;
            pdw[i >> 2] = put_byte(pdw[i >> 2], bgrp[i] + (k & 15u), i & 3);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < CPT; ++i) cur[i * 32] = INF32;
      }
    } else {
      const uint64_t* prev = (cur_is_b ? r64a : r64b) + PAD + wbase + lane;
      uint64_t* cur = (cur_is_b ? r64b : r64a) + PAD + wbase + lane;
      uint64_t best[CPT];
#pragma unroll
      for (int i = 0; i < CPT; ++i) best[i] = ~0ull;
      if (live) {
        for (int c = 0; c < KP; ++c) {
          const uint64_t* pv = prev - min((int)s_cand[sb][c].x, dclamp);
          const uint64_t ak = s_add[sb][c];
#pragma unroll
          for (int i = 0; i < CPT; ++i) best[i] = min(best[i], pv[i * 32] + ak);
        }
      }
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const uint64_t k = best[i];
        cur[i * 32] = (k >= INF64) ? INF64 : (k & ~kmask);
        pdw[i >> 2] = put_byte(pdw[i >> 2], (uint32_t)k, i & 3);
      }
    }
    if (live)
      *reinterpret_cast<uint4*>(PD + (int64_t)a * PD_ROW + tid * 16) = make_uint4(pdw[0], pdw[1], pdw[2], pdw[3]);
    if (a + 1 < La) stage(nd, nub, sb ^ 1, lo, hi);
    cur_is_b ^= 1;
    __syncthreads();
  }
  LG_T(4);
  // ---- line 23: argmin of the last row, smallest e on ties
  uint64_t bk = ~0ull;
  int be = 0x7fffffff;
  for (int e = tid; e < W1; e += DP_THREADS) {
    uint64_t v;
    if (!wide) { const uint32_t x = ((cur_is_b ? r32a : r32b) + PAD)[e]; v = (x >= INF32) ? ~0ull : x; }
    else { const uint64_t x = ((cur_is_b ? r64a : r64b) + PAD)[e]; v = (x >= INF64) ? ~0ull : x; }
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
  LG_T(7);
  // stage the discretised table and the active list in shared memory for the backtrack
  int32_t* sdisc_all = reinterpret_cast<int32_t*>(smem_raw);
  const size_t rows_bytes = (size_t)16 * row;  // allocated for two 64-bit rows
  const bool disc_in_smem = (size_t)(La * K + 2 * La) * 4 <= rows_bytes;
  if (disc_in_smem) {
    for (int i = tid; i < La * K; i += DP_THREADS) sdisc_all[i] = wdisc[i];
    for (int i = tid; i < La; i += DP_THREADS) sdisc_all[La * K + i] = act[i];
  }
  __syncthreads();
  LG_T(8);
  const int32_t* bdisc = disc_in_smem ? sdisc_all : wdisc;
  int32_t* bch = disc_in_smem ? sdisc_all + La * K + La : nullptr;  // chosen c per active layer
  // ---- lines 24-27 backtrack (warp 0).  Speculative: one PD round trip resolves up to
  //      three layers.  Entry 0 is PD(a, e); entry 1+c1 is PD(a-1, e - disc[a][c1]);
  //      entry 1+K+c1*K+c2 is PD(a-2, e - disc[a][c1] - disc[a-1][c2]); two entries
  //      per lane.  The disc rows are loaded before e is known.
  if (warp == 0) {
    uint64_t k = s_redk[lane];
    int ee = s_rede[lane];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint64_t ov = __shfl_xor_sync(LG_FULL, k, o);
      const int oe = __shfl_xor_sync(LG_FULL, ee, o);
      if (ov < k || (ov == k && oe < ee)) { k = ov; ee = oe; }
    }
    const int used_default = (k == ~0ull);
    const int cm = pdmask;
    auto put = [&](int a, int c) {
      if (lane == 0) {
        if (bch) bch[a] = c;
        else choice[act[a]] = c;
      }
    };
    if (!used_default) {
      const int depth = (K < 32 && 1 + K + K * K <= 64) ? 3 : ((K < 32) ? 2 : 1);
      // per lane slot r: level and candidate pair of entry j = lane + 32 r
      int lev[2], c1s[2], c2s[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int j = lane + 32 * r;
        lev[r] = -1; c1s[r] = 0; c2s[r] = 0;
        if (j == 0) lev[r] = 0;
        else if (depth >= 2 && j <= K) { lev[r] = 1; c1s[r] = j - 1; }
        else if (depth >= 3 && j < 1 + K + K * K) { lev[r] = 2; c1s[r] = (j - 1 - K) / K; c2s[r] = (j - 1 - K) % K; }
      }
      int e = ee, a = La - 1;
      // the disc rows of a round do not depend on e: the next round's are loaded
      // (and its speculative offsets formed) while this round's PD loads are in flight
      auto disc_rows = [&](int ar, int& da, int& db, int& dc, int* off) {
        da = (lane < K) ? bdisc[ar * K + lane] : 0;
        db = (lane < K) ? bdisc[(ar - 1) * K + lane] : 0;
        dc = (lane < K && depth >= 3) ? bdisc[(ar - 2) * K + lane] : 0;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int d1 = __shfl_sync(LG_FULL, da, c1s[r]);
          const int d2 = __shfl_sync(LG_FULL, db, c2s[r]);
          off[r] = (lev[r] == 0) ? 0 : (lev[r] == 1) ? ((d1 >= 0) ? d1 : -1)
                 : (lev[r] == 2) ? ((d1 >= 0 && d2 >= 0) ? d1 + d2 : -1) : -1;
        }
      };
      if (depth > 1 && a >= depth - 1) {
        int da, db, dc, off[2];
        disc_rows(a, da, db, dc, off);
        for (;;) {
          int v[2];
#ifdef LG_DP_TIMING
          const long long tq0 = clock64();
#endif
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            v[r] = 0;
            if (off[r] >= 0 && e - off[r] >= 0) v[r] = pd_byte<CPT>(PD, a - lev[r], e - off[r]);
          }
          const int an = a - depth;
          int nda = 0, ndb = 0, ndc = 0, noff[2] = {-1, -1};
          if (an >= depth - 1) disc_rows(an, nda, ndb, ndc, noff);
#ifdef LG_DP_TIMING
          {
            const int vv = __shfl_sync(LG_FULL, v[0] + v[1], 0);
            const long long tq1 = clock64();
            t_ldg += tq1 - tq0 + (vv & 0);
            ++n_rounds;
          }
#endif
          auto val = [&](int j) {
            const int x0 = __shfl_sync(LG_FULL, v[0], j & 31), x1 = __shfl_sync(LG_FULL, v[1], j & 31);
            return (j < 32 ? x0 : x1) & cm;
          };
          const int c0 = val(0);
          const int c1 = val(1 + c0);
          put(a, c0);
          put(a - 1, c1);
          int de = __shfl_sync(LG_FULL, da, c0) + __shfl_sync(LG_FULL, db, c1);
          if (depth >= 3) {
            const int c2 = val(1 + K + c0 * K + c1);
            put(a - 2, c2);
            de += __shfl_sync(LG_FULL, dc, c2);
          }
          e -= de;
          a = an;
          if (a < depth - 1) break;
          da = nda; db = ndb; dc = ndc; off[0] = noff[0]; off[1] = noff[1];
        }
      }
      for (; a >= 0; --a) {
        const int c = pd_byte<CPT>(PD, a, e) & cm;
        put(a, c);
        e -= bdisc[a * K + c];
      }
    }
    if (lane == 0) s_La = used_default;
  }
  __syncthreads();
  if (bch && !s_La)
    for (int a = tid; a < La; a += DP_THREADS) choice[bdisc[La * K + a]] = bch[a];
  __syncthreads();
  LG_T(5);
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
      int a = 0;
      for (; a + 4 <= La; a += 4) {
        const double v0 = sm_ce[a], v1 = sm_ce[a + 1], v2 = sm_ce[a + 2], v3 = sm_ce[a + 3];
        pb += sm_cb[a] + sm_cb[a + 1] + sm_cb[a + 2] + sm_cb[a + 3];
        pe = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(pe, v0), v1), v2), v3);
      }
      for (; a < La; ++a) { pb += sm_cb[a]; pe = __dadd_rn(pe, sm_ce[a]); }
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
  LG_T(6);
#ifdef LG_DP_TIMING
  if (tid == 0)
    printf("dp timing (cycles): prelude %lld gcd/disc %lld rows %lld loop %lld (%lld/layer) argmin %lld stage %lld "
           "back %lld (rounds %d, ldg %lld/round) summary %lld\n",
           tstamp[1] - tstamp[0], tstamp[2] - tstamp[1], tstamp[3] - tstamp[2], tstamp[4] - tstamp[3],
           (tstamp[4] - tstamp[3]) / (La ? La : 1), tstamp[7] - tstamp[4], tstamp[8] - tstamp[7],
           tstamp[5] - tstamp[8], n_rounds, n_rounds ? t_ldg / n_rounds : 0LL, tstamp[6] - tstamp[5]);
#endif
}

// ---------------------------------------------------------------------------
// Cluster path: the row recursion of Alg.1 (lines 13-22) spread over a thread-block
// cluster of NC CTAs (one per SM).  A single SM is bound by shared-memory bandwidth
// (one 4-byte LDS per cell and candidate: 10,001 x 7 x 4 B / 128 B/clk ~ 2.2 K cycles
// per row); NC SMs each own a contiguous slice of S cells and keep a full-length copy
// of the two rows.  Cell e of row a reads row a-1 at e - d (d >= 0), i.e. only cells
// at or below e, so CTA r needs, besides its own slice, the cells [r S - maxd, r S) of
// lower CTAs, where maxd is the largest admissible disc of the next layer (exact: no
// read of row a+1 reaches further down).  Every warp pushes the cells of its slice that
// a higher CTA will read straight from its registers into that CTA's copy of the row
// (st.shared::cluster), then one cluster barrier (release/acquire) per row publishes
// them; the same barrier orders the reuse of the double-buffered rows (no CTA writes
// row a+2 before every CTA has finished reading row a).  Keys, tie-breaks, the band
// skip and the PD bytes are those of k_solve_fast; the argmin is reduced per CTA and
// gathered in rank 0 over DSMEM; rank 0 backtracks through PD (global, L2).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_map(const void* p, uint32_t rank) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cl_st(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_st(uint32_t addr, uint64_t v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}

// Cross-cluster handshake of the two layer groups (workspace): group 0's CTAs publish
// the launch's token after writing their slice of F.
struct JoinMeta {
  uint64_t tok[16];
};
__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// PD byte of (layer a, cell e): cell-major rows of PDR bytes, in L2 (written by the
// row kernel: __ldcg)
__device__ __forceinline__ int pd_cm(const uint8_t* PD, int64_t PDR, int a, int e) {
  return __ldcg(PD + (int64_t)a * PDR + e);
}

// Backtrack (Alg.1 lines 24-27) of the active layers a_hi, a_hi - 1, ..., a_lo from cell e
// by one warp: bch[a] = PD(a, e) & cm, e -= disc[a][bch[a]].  Speculative: one PD round
// trip resolves up to three layers (entry 0 = PD(a, e); entry 1 + c1 = PD(a - 1, e -
// disc[a][c1]); entry 1 + K + c1 K + c2 = PD(a - 2, e - disc[a][c1] - disc[a-1][c2]); two
// entries per lane); the disc rows are loaded before e is known.  bdisc: [La][K].
__device__ __noinline__ void bt_warp(const uint8_t* __restrict__ PD, int64_t PDR, const int32_t* bdisc, int K, int cm,
                                     int a_hi, int a_lo, int e, int32_t* bch) {
  const int lane = threadIdx.x & 31;
  auto put = [&](int a, int c) {
    if (lane == 0) bch[a] = c;
  };
  const int depth = (K < 32 && 1 + K + K * K <= 64) ? 3 : ((K < 32) ? 2 : 1);
  int lev[2], c1s[2], c2s[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int j = lane + 32 * r;
    lev[r] = -1; c1s[r] = 0; c2s[r] = 0;
    if (j == 0) lev[r] = 0;
    else if (depth >= 2 && j <= K) { lev[r] = 1; c1s[r] = j - 1; }
    else if (depth >= 3 && j < 1 + K + K * K) { lev[r] = 2; c1s[r] = (j - 1 - K) / K; c2s[r] = (j - 1 - K) % K; }
  }
  int a = a_hi;
  auto disc_rows = [&](int ar, int& da, int& db, int& dc, int* off) {
    da = (lane < K) ? bdisc[ar * K + lane] : 0;
    db = (lane < K) ? bdisc[(ar - 1) * K + lane] : 0;
    dc = (lane < K && depth >= 3) ? bdisc[(ar - 2) * K + lane] : 0;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int d1 = __shfl_sync(LG_FULL, da, c1s[r]);
      const int d2 = __shfl_sync(LG_FULL, db, c2s[r]);
      off[r] = (lev[r] == 0) ? 0 : (lev[r] == 1) ? ((d1 >= 0) ? d1 : -1)
             : (lev[r] == 2) ? ((d1 >= 0 && d2 >= 0) ? d1 + d2 : -1) : -1;
    }
  };
  if (depth > 1 && a - (depth - 1) >= a_lo) {
    int da, db, dc, off[2];
    disc_rows(a, da, db, dc, off);
    for (;;) {
      int v[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        v[r] = 0;
        if (off[r] >= 0 && e - off[r] >= 0) v[r] = pd_cm(PD, PDR, a - lev[r], e - off[r]);
      }
      const int an = a - depth;
      int nda = 0, ndb = 0, ndc = 0, noff[2] = {-1, -1};
      if (an - (depth - 1) >= a_lo) disc_rows(an, nda, ndb, ndc, noff);
      auto val = [&](int j) {
        const int x0 = __shfl_sync(LG_FULL, v[0], j & 31), x1 = __shfl_sync(LG_FULL, v[1], j & 31);
        return (j < 32 ? x0 : x1) & cm;
      };
      const int c0 = val(0);
      const int c1 = val(1 + c0);
      put(a, c0);
      put(a - 1, c1);
      int de = __shfl_sync(LG_FULL, da, c0) + __shfl_sync(LG_FULL, db, c1);
      if (depth >= 3) {
        const int c2 = val(1 + K + c0 * K + c1);
        put(a - 2, c2);
        de += __shfl_sync(LG_FULL, dc, c2);
      }
      e -= de;
      a = an;
      if (a - (depth - 1) < a_lo) break;
      da = nda; db = ndb; dc = ndc; off[0] = noff[0]; off[1] = noff[1];
    }
  }
  for (; a >= a_lo; --a) {
    const int c = pd_cm(PD, PDR, a, e) & cm;
    put(a, c);
    e -= bdisc[a * K + c];
  }
  __syncwarp();
}

// R20 check and summary (whole CTA): choice[act[a]] = bch[a] (or the defaults when
// used_default), the plan's bits and raw error summed in layer order; the defaults are
// returned instead when the plan is not within the default bits and Emax.  sm_ce:
// 16 * La bytes of shared scratch; s_flag: a shared int.
__device__ __noinline__ void finish_plan(int used_default, const int32_t* bch, int La, const int32_t* __restrict__ act,
                                         const int32_t* __restrict__ default_idx, const double* __restrict__ err,
                                         const int64_t* __restrict__ bits, int K, uint32_t flags, double emax,
                                         int64_t defbits, int32_t* __restrict__ choice,
                                         lgreco_solve_info* __restrict__ info, double* sm_ce, int* s_flag) {
  const int tid = threadIdx.x, NT = blockDim.x;
#ifdef LG_DP_TIMING
  long long fp0 = clock64(), fp1 = 0, fp2 = 0, fp3 = 0;
#endif
  if (!used_default)
    for (int a = tid; a < La; a += NT) choice[act[a]] = bch[a];
  __syncthreads();
#ifdef LG_DP_TIMING
  fp1 = clock64();
#endif
  int64_t* sm_cb = reinterpret_cast<int64_t*>(sm_ce + La);
  if (used_default) {
    for (int a = tid; a < La; a += NT) choice[act[a]] = default_idx[act[a]];
    __syncthreads();
  }
  for (int pass = 0; pass < 2; ++pass) {
    for (int a = tid; a < La; a += NT) {
      const int l = act[a];
      const int c = used_default ? default_idx[l] : bch[a];
      sm_ce[a] = metric(err[(int64_t)l * K + c], flags);
      sm_cb[a] = bits[(int64_t)l * K + c];
    }
    __syncthreads();
#ifdef LG_DP_TIMING
    if (pass == 0) fp2 = clock64();
#endif
    if (tid < 32) {
      // lane 0: the serial fp64 chain in layer order; 16 terms staged in registers ahead
      // of each run of dependent adds; the int64 bits sum over the warp (order-free)
      int64_t pb = 0;
      for (int a = tid; a < La; a += 32) pb += sm_cb[a];
#pragma unroll
      for (int o = 16; o; o >>= 1) pb += __shfl_xor_sync(LG_FULL, pb, o);
      double pe = 0.0;
      if (tid == 0) {
        int a = 0;
        for (; a + 16 <= La; a += 16) {
          double v[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = sm_ce[a + q];
#pragma unroll
          for (int q = 0; q < 16; ++q) pe = __dadd_rn(pe, v[q]);
        }
        for (; a < La; ++a) pe = __dadd_rn(pe, sm_ce[a]);
      }
      if (tid != 0) {
      } else if (!used_default && (pb > defbits || pe > emax)) {
        *s_flag = 1;
      } else {
        lgreco_solve_info inf = {};
        inf.emax = emax;
        inf.total_err = pe;
        inf.total_bits = pb;
        inf.default_bits = defbits;
        inf.used_default = used_default;
        inf.n_active = La;
        inf.status = LGRECO_OK;
        *info = inf;
        *s_flag = -1;
      }
    }
    __syncthreads();
#ifdef LG_DP_TIMING
    if (pass == 0) fp3 = clock64();
#endif
    if (*s_flag < 0) break;
    used_default = 1;
    for (int a = tid; a < La; a += NT) choice[act[a]] = default_idx[act[a]];
    __syncthreads();
  }
#ifdef LG_DP_TIMING
  if (tid == 0) printf("finish_plan: choice %lld gather %lld sum %lld rest %lld\n", fp1 - fp0, fp2 - fp1, fp3 - fp2, clock64() - fp3);
#endif
}

#ifndef QP_DP_CPT0
#define QP_DP_CPT0 2  // smallest cells-per-thread of the cluster solve (more warps below that)
#endif
constexpr int CL_MAX = 16;  // CTAs per cluster (16: non-portable size; 8 is the portable maximum)

template <int CPT, int KT>
__global__ void __launch_bounds__(DP_THREADS, 1)
k_solve_cl(const double* __restrict__ err, const int64_t* __restrict__ bits, int L, int K,
           const int32_t* __restrict__ default_idx, const int32_t* __restrict__ compress, int D, uint32_t flags,
           int32_t* __restrict__ choice, lgreco_solve_info* __restrict__ info, uint8_t* __restrict__ PD,
           int32_t* __restrict__ act, int32_t* __restrict__ wdisc, uint64_t* __restrict__ wadd,
           int32_t* __restrict__ wmaxd, int ngroups, uint64_t* __restrict__ rowout, JoinMeta* __restrict__ jmeta,
           uint64_t tok) {
  static_assert(KT >= 0 && KT <= 16 && (CPT == 1 || CPT == 2 || CPT == 4 || CPT == 8 || CPT == 16), "cluster DP");
  // KT > 0: K <= KT candidates, tables of the whole recursion in shared memory;
  // KT == 0: K <= 256 candidates in groups of 16 (k_solve_fast's grouped keys), tables
  // in global memory (this CTA's copy of the workspace), staged per row
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_La, s_status, s_wide, s_cbits;
  __shared__ double s_emax;
  __shared__ int64_t s_defbits;
  __shared__ uint64_t s_g[32];
  __shared__ uint64_t s_redk[32];
  __shared__ int s_rede[32];
  __shared__ uint64_t s_clk[CL_MAX];
  __shared__ int s_cle[CL_MAX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = blockDim.x, NW = NT >> 5;
  // ngroups == 2: two clusters, each running the row recursion of one half of the active
  // layers from the zero row; k_solve_join combines them (see "Layer groups" below)
  const uint32_t rank = cl_rank(), NC = gridDim.x / ngroups;
  const int grp = (ngroups > 1) ? (int)(blockIdx.x / NC) : 0;
  const int S = NW * 32 * CPT;     // cells per CTA
  const int cbase = (int)rank * S; // first cell of this CTA
#ifdef LG_DP_TIMING
  long long tstamp[20] = {0};
  long long t_push = 0, t_c = 0, t_p = 0, t_s = 0, t_cl = 0;
#endif
  LG_T(0);
  pdl_wait();  // the error / size tables of the profile
  // the next kernel may be scheduled beside the solve now: a compress that reads this
  // plan waits for it (pdl_wait), the concurrent fused pass of the next step reads an
  // older plan (LGRECO_PC_CONCURRENT)
  pdl_trigger();
  LG_T(10);

  // ---- prelude (every CTA, identical).  Latency-bound: a handful of block-wide steps,
  //      one thread per layer (or per (layer, candidate) pair) in each, no atomics on the
  //      critical values; only Emax is a serial chain (layer order, fp64: R20).
  int32_t* sm_act = reinterpret_cast<int32_t*>(smem_raw);
  double* sm_dea = reinterpret_cast<double*>(sm_act + ((L + 1) & ~1));
  // the whole (err, bits) table in one global round trip (every later prelude read is
  // shared memory) when it fits in front of the rows' space
  constexpr int PADC = 32 * CPT;
  const bool pre = (size_t)(12 + 16 * K) * L + 64 <= (size_t)16 * (PADC + (int)NC * S);
  double* sm_err = sm_dea + L;
  int64_t* sm_bits = reinterpret_cast<int64_t*>(sm_err + (pre ? (size_t)L * K : 0));
  __shared__ long long s_scan[32];
  __shared__ int s_bad;  // bit 0: non-finite or negative error, bit 1: bad default / cost, bit 2: key width
  __shared__ unsigned long long s_or[32];
  // block-wide inclusive sum over the threads (int64); *tot = the block's total
  auto bscan = [&](long long v, long long* tot) -> long long {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(LG_FULL, v, o);
      if (lane >= o) v += t;
    }
    if (lane == 31) s_scan[warp] = v;
    __syncthreads();
    if (warp == 0) {
      long long x = (lane < NW) ? s_scan[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(LG_FULL, x, o);
        if (lane >= o) x += t;
      }
      s_scan[lane] = x;
    }
    __syncthreads();
    const long long r = v + ((warp > 0) ? s_scan[warp - 1] : 0);
    *tot = s_scan[NW - 1];
    __syncthreads();
    return r;
  };
  // (1) the table, the flags and the defaults: one round trip
  {
    int fl[4], df[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int l = tid + j * NT;
      fl[j] = (l < L) ? (compress ? (__ldg(compress + l) != 0) : 1) : 0;
      df[j] = (l < L) ? __ldg(default_idx + l) : 0;
    }
    if (pre) {
#pragma unroll 4
      for (int i = tid; i < L * K; i += NT) { sm_err[i] = __ldg(err + i); sm_bits[i] = __ldg(bits + i); }
    }
    if (tid == 0) s_bad = 0;
    __syncthreads();
    const double* t_err0 = pre ? sm_err : err;
    const int64_t* t_bits0 = pre ? sm_bits : bits;
    // (2) active list (block scan of the flags, layer order), Emax terms, default bits
    long long db = 0, base = 0;
    int bad_def = 0;
    for (int t0 = 0; t0 < L; t0 += NT) {
      const int j = t0 / NT;
      const int l = t0 + tid;
      int f = 0, d = 0;
      if (j < 4) { f = fl[j]; d = df[j]; }
      else if (l < L) { f = compress ? (compress[l] != 0) : 1; d = default_idx[l]; }
      if (l < L && rank == 0 && grp == 0) choice[l] = -1;
      double de = 0.0;
      if (f) {
        if (d < 0 || d >= K) bad_def = 1;
        else { de = metric(t_err0[(int64_t)l * K + d], flags); db += t_bits0[(int64_t)l * K + d]; }
      }
      long long tot;
      const long long pos = bscan(f, &tot) - f + base;
      if (f) {
        sm_act[pos] = l;
        sm_dea[pos] = de;
        if (rank == 0 && grp == 0) act[pos] = l;
      }
      base += tot;
    }
    if (__any_sync(LG_FULL, bad_def) && lane == 0) atomicOr(&s_bad, 2);
    long long dbt;
    bscan(db, &dbt);  // (the inclusive value is not needed: the total)
    if (tid == 0) { s_La = (int)base; s_defbits = dbt; }
    __syncthreads();
  }
  const int La = s_La;
  const double* t_err = pre ? sm_err : err;
  const int64_t* t_bits = pre ? sm_bits : bits;
  LG_T(6);
  // (3) Emax = sum of the defaults' errors in layer order (warp 0, lane 0: a serial fp64
  //     chain, loads batched 8 ahead) || the other warps: per active layer the largest
  //     cost, the OR of all costs (their lowest set bit is the exact rescale g), and the
  //     sum of the largest costs (the key width check; saturating)
  constexpr int PAD = 32 * CPT;
  const int row = PAD + (int)NC * S;
  unsigned char* tail = smem_raw + (size_t)16 * row;
  uint64_t* my_wadd;  // [La*K] raw costs
  int32_t* my_wdisc;  // [La*K] discretised errors
  int32_t* my_wmaxd;  // [La+1] largest admissible disc per layer (0 past the end)
  if constexpr (KT > 0) {
    my_wadd = reinterpret_cast<uint64_t*>(tail);
    my_wdisc = reinterpret_cast<int32_t*>(my_wadd + (size_t)La * K);
    my_wmaxd = my_wdisc + (size_t)La * K;
  } else {
    my_wadd = wadd + (size_t)rank * L * K;
    my_wdisc = wdisc + (size_t)rank * L * K;
    my_wmaxd = reinterpret_cast<int32_t*>(tail);
  }
  constexpr int KP2 = (KT + 2) & ~1;
  uint2* cand_all = reinterpret_cast<uint2*>(
      (reinterpret_cast<uintptr_t>(my_wmaxd + La + 1) + 15) & ~static_cast<uintptr_t>(15));  // [La][KP2], 16-B aligned
  uint64_t* add_all = reinterpret_cast<uint64_t*>(cand_all + (size_t)La * (KT > 0 ? KP2 : 0));  // [La][KT]
  int2* band_all = reinterpret_cast<int2*>(add_all + (size_t)La * KT);          // [La]
  {
    uint64_t gg = 0, mxp = 0;
    int bad = 0;
    if (warp == 0) {
      if (lane == 0) {
        double emax = 0.0;
        int a = 0;
        for (; a + 8 <= La; a += 8) {
          double v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = sm_dea[a + j];
#pragma unroll
          for (int j = 0; j < 8; ++j) emax = __dadd_rn(emax, v[j]);
        }
        for (; a < La; ++a) emax = __dadd_rn(emax, sm_dea[a]);
        s_emax = emax;
        int cb = 0;
        while ((1 << cb) < K) ++cb;
        s_cbits = cb;
      }
    }
    if (warp > 0 || NW == 1) {  // (a one-warp CTA: warp 0 after the chain)
      const int t1 = (NW > 1) ? tid - 32 : tid, st1 = (NW > 1) ? NT - 32 : NT;
      for (int a = t1; a < La; a += st1) {
        const int l = sm_act[a];
        uint64_t m = 0;
        for (int c = 0; c < K; ++c) {
          const int64_t b = t_bits[(int64_t)l * K + c];
          if (b < 0) bad |= 2;
          const uint64_t ub = (uint64_t)(b < 0 ? 0 : b);
          gg |= ub;
          m = max(m, ub);
          my_wadd[a * K + c] = ub;  // raw cost; keyed (cost/g << cbits | c) when staged per layer
        }
        mxp = sat_add(mxp, m);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      gg |= __shfl_xor_sync(LG_FULL, gg, o);
      mxp = sat_add(mxp, __shfl_xor_sync(LG_FULL, mxp, o));
    }
    bad = __reduce_or_sync(LG_FULL, bad);
    if (lane == 0) {
      s_or[warp] = gg;
      s_redk[warp] = mxp;
      if (bad) atomicOr(&s_bad, bad);
    }
    __syncthreads();
  }
  const double emax = s_emax;
  const int cbits = s_cbits;
  LG_T(7);
  // (4) one thread per active layer: its K discretised errors (Alg.1 lines 3-5, K
  //     independent divisions in flight), the largest / smallest admissible disc, the
  //     split weight; warp 0 meanwhile reduces the cost facts to g, the key width and the
  //     width check
  {
    int bad = 0;
    if (warp == 0) {
      uint64_t g = (lane < NW) ? s_or[lane] : 0;
      unsigned long long mxs = (lane < NW) ? s_redk[lane] : 0;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        g |= __shfl_xor_sync(LG_FULL, g, o);
        mxs = sat_add(mxs, __shfl_xor_sync(LG_FULL, mxs, o));
      }
      if (lane == 0) {
        g = g ? (g & (~g + 1)) : 1;  // lowest set bit of the OR = 2^min ctz(cost)
        s_g[0] = g;
        // every cost is a multiple of g, so sum_a max_c cost/g = (sum_a max_c cost)/g exactly
        const uint64_t mx = mxs >> (__ffsll((long long)g) - 1);
        s_wide = (mx >= (1ull << (30 - ((KT > 0) ? cbits : 4)))) ? 1 : 0;
        if (mx >= (1ull << (62 - cbits))) atomicOr(&s_bad, 4);
      }
    }
    for (int a = tid; a < La; a += NT) {
      const int l = sm_act[a];
      int mn = 0x7fffffff, mxd = -1;
      for (int c = 0; c < K; ++c) {
        const double v = t_err[(int64_t)l * K + c];
        if (!isfinite(v) || v < 0.0) bad |= 1;
        const int dd = discretise(metric(v, flags), emax, D, flags);
        my_wdisc[a * K + c] = dd;
        if (dd >= 0) { mn = min(mn, dd); mxd = max(mxd, dd); }
      }
      my_wmaxd[a] = max(mxd, 0);
      band_all[a] = make_int2(mxd >= 0 ? mn : -1, max(mxd, 0));  // per-layer (min, max) admissible disc
    }
    if (tid == 0) my_wmaxd[La] = 0;
    bad = __reduce_or_sync(LG_FULL, bad);
    if (lane == 0 && bad) atomicOr(&s_bad, bad);
    __syncthreads();
    if (tid == 0) s_status = (s_bad & 1) ? LGRECO_ENONFINITE : (s_bad ? LGRECO_EINVAL : LGRECO_OK);
    __syncthreads();
  }
  const uint64_t g = s_g[0];
  const int gsh = __ffsll((long long)g) - 1;
  LG_T(8);
  if (s_status != LGRECO_OK || La == 0) {  // identical in every CTA: no cluster barrier is pending
    if (rank == 0 && tid == 0 && grp == 0) {
      lgreco_solve_info inf = {};
      inf.n_active = La;
      inf.status = s_status;
      *info = inf;
    }
    return;
  }
  const bool wide = s_wide;
  const int kb = (wide || KT > 0) ? cbits : 4;  // key bits below the value
  const uint64_t kmask = (1ull << kb) - 1;
  const int pdmask = (!wide && KT == 0) ? 0xFF : (int)((1u << cbits) - 1u);  // PD byte -> c
  auto keyed = [&](uint64_t ub, int c) -> uint64_t { return ((ub >> gsh) << kb) | (uint64_t)(c & (int)kmask); };
  uint32_t* r32a = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* r32b = r32a + row;
  uint64_t* r64a = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* r64b = r64a + row;
  const uint32_t INF32 = 0x7FFFFF00u;
  const uint64_t INF64 = 1ull << 62;
  // (5) the layer split (ngroups == 2: a bottom group [0, h) and a top group [h, La) of
  //     about equal estimated row cost -- a row costs ~1.8 K cycles plus its DSMEM pushes,
  //     ~maxd / 16 cycles, C4 measured; every CTA computes the same h), the reachable
  //     bands of this group's layers (exact: running sums of the smallest / largest
  //     admissible disc from the zero row, saturating at D; a layer with no admissible
  //     candidate empties every later band), the keyed candidate pairs, the rows
  __shared__ int s_a0, s_a1;
  __shared__ unsigned s_ns;
  if (ngroups > 1) {
    long long tot = 0, wsum = 0;
    for (int t0 = 0; t0 < La; t0 += NT) wsum += (t0 + tid < La) ? 1800 + my_wmaxd[t0 + tid] / 16 : 0;
    bscan(wsum, &tot);
    const long long half = (tot + 1) / 2;
    long long carry = 0;
    for (int t0 = 0; t0 < La; t0 += NT) {
      const int a = t0 + tid;
      const long long w = (a < La) ? 1800 + my_wmaxd[a] / 16 : 0;
      long long tt;
      const long long inc = bscan(w, &tt) + carry;
      if (a < La && inc >= half && inc - w < half) {
        const int h = min(max(a + 1, La > 1 ? 1 : 0), La > 1 ? La - 1 : La);
        s_a0 = grp ? h : 0;
        s_a1 = grp ? La : h;
      }
      carry += tt;
    }
    if (tid == 0) s_ns = 0;  // E2 list count (rank 0's is used; ordered by the init cluster barrier)
  } else if (tid == 0) {
    s_a0 = 0;
    s_a1 = La;
  }
  __syncthreads();
  const int a0 = s_a0, a1 = s_a1;
  LG_T(15);
  {
    long long clo = 0, chi = 0, cdead = 0;
    for (int t0 = a0; t0 < a1; t0 += NT) {
      const int a = t0 + tid;
      const int2 mm = (a < a1) ? band_all[a] : make_int2(0, 0);
      long long lo = (mm.x >= 0) ? mm.x : 0, hi = mm.y, dd = (mm.x < 0) ? 1 : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long t1 = __shfl_up_sync(LG_FULL, lo, o), t2 = __shfl_up_sync(LG_FULL, hi, o),
                        t3 = __shfl_up_sync(LG_FULL, dd, o);
        if (lane >= o) { lo += t1; hi += t2; dd += t3; }
      }
      __shared__ long long s_b3[3][32];
      if (lane == 31) { s_b3[0][warp] = lo; s_b3[1][warp] = hi; s_b3[2][warp] = dd; }
      __syncthreads();
      long long plo = clo, phi = chi, pdd = cdead;
      for (int w2 = 0; w2 < warp; ++w2) { plo += s_b3[0][w2]; phi += s_b3[1][w2]; pdd += s_b3[2][w2]; }
      long long tlo = clo, thi = chi, tdd = cdead;
      for (int w2 = 0; w2 < NW; ++w2) { tlo += s_b3[0][w2]; thi += s_b3[1][w2]; tdd += s_b3[2][w2]; }
      __syncthreads();
      if (a < a1) {
        lo += plo; hi += phi; dd += pdd;
        band_all[a] = make_int2(dd ? 0x3fffffff : (int)min(lo, 0x3fffffffll), (int)min(hi, (long long)D));
      }
      clo = tlo; chi = thi; cdead = tdd;
    }
  }
  for (int i = tid; KT > 0 && i < La * KP2; i += NT) {
    const int aa = i / KP2, c = i - aa * KP2;
    const int32_t d = (c < K) ? my_wdisc[aa * K + c] : -1;
    const bool ok = c < K && d >= 0;
    const uint64_t k = ok ? keyed(my_wadd[aa * K + c], c) : 0;
    cand_all[i] = make_uint2(ok ? (uint32_t)d : 0u, ok ? (uint32_t)k : INF32);
    if (c < KT) add_all[aa * KT + c] = ok ? k : INF64;
  }
  LG_T(16);
  if (!wide) {  // three row buffers (the 16-byte-per-cell region holds four u32 rows)
    for (int i = tid; i < row; i += NT) { r32a[i] = (i == PAD) ? 0u : INF32; r32b[i] = INF32; r32b[row + i] = INF32; }
  } else {
    for (int i = tid; i < row; i += NT) { r64a[i] = (i == PAD) ? 0ull : INF64; r64b[i] = INF64; }
  }
  // s_bar[i]: completion of the remote cells of the row in buffer i (st.async complete_tx)
  __shared__ __align__(8) uint64_t s_bar[3];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_bar[1])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_bar[2])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // KT == 0: the candidates of row a staged in s_ck/s_ak[a & 1] (keyed as above)
  __shared__ __align__(16) uint2 s_ck[2][KT > 0 ? 2 : 256];
  __shared__ uint64_t s_ak[2][KT > 0 ? 1 : 256];
  auto stage0 = [&](int32_t d, uint64_t ub, int slot) {
    if (tid < K) {
      const bool ok = d >= 0;
      const uint64_t k = ok ? keyed(ub, tid) : 0;
      s_ck[slot][tid] = make_uint2(ok ? (uint32_t)d : 0u, ok ? (uint32_t)k : INF32);
      s_ak[slot][tid] = ok ? k : INF64;
    }
  };
  LG_T(17);
  if (KT == 0 && a0 < a1) stage0((tid < K) ? my_wdisc[a0 * K + tid] : -1, (tid < K) ? my_wadd[a0 * K + tid] : 0, 0);
  LG_T(1);
  __syncthreads();  // (cl_sync orders these too; the explicit CTA barrier keeps racecheck exact)
  cl_sync();  // every CTA's rows and barriers initialised before any remote push lands
  if (!wide) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // "row -1 done"
  LG_T(2);
  // Row buffers: row a in buffer bc, row a-1 in bp (row -1 = the initial row, buffer 0).
  // Narrow keys: NB = 3 buffers, so the cluster barrier that keeps a CTA from pushing
  // into a buffer a peer still reads is split: the wait for "every CTA finished row a-1"
  // happens after this CTA computed row a (arrive after row a-1, wait after row a) and
  // its latency hides behind a row; a push of row a then lands in the buffer of row
  // a-3, last read while computing row a-2, which every CTA finished (waited for before
  // row a).  Wide keys (64-bit rows): NB = 2 and the full barrier per row.
  const int NB = wide ? 2 : 3;
  int bc = 1, bp = 0;
  uint32_t bph = 0u;  // bit i: parity of s_bar[i]'s next phase
  const int wbase = cbase + warp * (32 * CPT);
  const int dclamp = wbase + PAD;
  const int64_t PDR = (int64_t)NC * NT * CPT;  // PD bytes per layer
  const uint32_t vb = wide ? 8u : 4u;
  // row a's candidate pairs, band and max shift, loaded during row a-1 (off the
  // critical path of the row)
  uint4 cq[KP2 / 2];
#pragma unroll
  for (int c = 0; c < KP2 / 2; ++c)
    cq[c] = (KT > 0 && a0 < a1) ? reinterpret_cast<const uint4*>(cand_all + (size_t)a0 * KP2)[c] : make_uint4(0, 0, 0, 0);
  int2 band = (a0 < a1) ? band_all[a0] : make_int2(0, 0);
  int maxd = (a0 + 1 < a1) ? my_wmaxd[a0 + 1] : 0;  // the next row's largest shift (0: no next row)
  for (int a = a0; a < a1; ++a) {
    const int sb = bc;     // barrier of row a's buffer
    const int sk = (a - a0) & 1;  // KT == 0 candidate staging slot of row a
    // cells of row a this CTA receives: [cbase - maxd, cbase) (clipped at 0)
    if (tid == 0) {
      uint32_t bytes = (uint32_t)min(maxd, cbase) * vb;
#ifdef LG_DP_TIMING
      if (flags & (1u << 30)) bytes = 0;  // diagnostic: no pushes (wrong result)
#endif
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&s_bar[sb])),
                   "r"(bytes)
                   : "memory");
    }
#ifdef LG_DP_TIMING
    const long long tr0 = clock64();
#endif
    const uint2* cnd = cand_all + (size_t)a * KP2;
    int32_t nd = -1;  // KT == 0: next layer's candidate tid, staged after this row
    uint64_t nub = 0;
    if (KT == 0 && tid < K && a + 1 < a1) { nd = my_wdisc[(a + 1) * K + tid]; nub = my_wadd[(a + 1) * K + tid]; }
    uint32_t pdw[4] = {0u, 0u, 0u, 0u};
    const bool live = (wbase + 32 * CPT - 1 >= band.x) && (wbase <= band.y);
    // highest CTA that reads any cell of this warp in the next row
    int rtop = min((int)NC - 1, (wbase + 32 * CPT - 1 + maxd) / S);
#ifdef LG_DP_TIMING
    if (flags & (1u << 30)) rtop = -1;  // diagnostic only: no pushes (wrong result)
#endif
    if (!wide) {
      const uint32_t* prev = r32a + (size_t)bp * row + PAD + wbase + lane;
      uint32_t* cur = r32a + (size_t)bc * row + PAD + wbase + lane;
      uint32_t best[CPT];
      if (live && KT == 0) {
        uint32_t bgrp[CPT];
#pragma unroll
        for (int i = 0; i < CPT; ++i) { best[i] = 0xFFFFFFFFu; bgrp[i] = 0; }
        for (int c0 = 0; c0 < K; c0 += 16) {
          const int cn = min(16, K - c0);
          uint32_t gk[CPT];
#pragma unroll
          for (int i = 0; i < CPT; ++i) gk[i] = 0xFFFFFFFFu;
          for (int c = 0; c < cn; ++c) {
            const uint2 cd = s_ck[sk][c0 + c];
            const uint32_t* pv = prev - min((int)cd.x, dclamp);
#pragma unroll
            for (int i = 0; i < CPT; ++i) gk[i] = __viaddmin_u32(pv[i * 32], cd.y, gk[i]);
          }
#pragma unroll
          for (int i = 0; i < CPT; ++i)
            if ((gk[i] & ~15u) < (best[i] & ~15u)) { best[i] = gk[i]; bgrp[i] = (uint32_t)c0; }
        }
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
          const uint32_t k = best[i];
          best[i] = min(k, INF32) & ~15u;
          pdw[i >> 2] = put_byte(pdw[i >> 2], bgrp[i] + (k & 15u), i & 3);
        }
      } else if (live) {
#pragma unroll
        for (int c = 0; c < KT; c += 2) {
          const uint4 q = cq[c >> 1];
          const uint32_t* pv = prev - min((int)q.x, dclamp);
#pragma unroll
          for (int i = 0; i < CPT; ++i)
            best[i] = (c == 0) ? pv[i * 32] + q.y : __viaddmin_u32(pv[i * 32], q.y, best[i]);
          if (c + 1 < KT) {
            const uint32_t* pw = prev - min((int)q.z, dclamp);
#pragma unroll
            for (int i = 0; i < CPT; ++i) best[i] = __viaddmin_u32(pw[i * 32], q.w, best[i]);
          }
        }
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
          const uint32_t k = best[i];
          best[i] = min(k, INF32) & ~(uint32_t)kmask;
          pdw[i >> 2] = put_byte(pdw[i >> 2], k, i & 3);
        }
      } else {
#pragma unroll
        for (int i = 0; i < CPT; ++i) best[i] = INF32;
      }
#pragma unroll
      for (int i = 0; i < CPT; ++i) cur[i * 32] = best[i];
#ifdef LG_DP_TIMING
      t_c += clock64() - tr0 + (best[0] & 0);
#endif
      for (int r2 = (int)rank + 1; r2 <= rtop; ++r2) {  // warp-uniform bounds
        const int need = r2 * S - maxd;                   // r2 reads cells >= need
        const uint32_t rbar = cl_map(&s_bar[sb], (uint32_t)r2);
#pragma unroll
        for (int i = 0; i < CPT; ++i)
          if (wbase + 32 * i + lane >= need)
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                             cl_map(cur + i * 32, (uint32_t)r2)),
                         "r"(best[i]), "r"(rbar)
                         : "memory");
      }
    } else {
      const uint64_t* prev = r64a + (size_t)bp * row + PAD + wbase + lane;
      uint64_t* cur = r64a + (size_t)bc * row + PAD + wbase + lane;
      const uint64_t* add = add_all + (size_t)a * KT;
      uint64_t best[CPT];
#pragma unroll
      for (int i = 0; i < CPT; ++i) best[i] = ~0ull;
      if (live) {
        for (int c = 0; c < (KT > 0 ? KT : K); ++c) {
          const uint64_t* pv = prev - min((int)(KT > 0 ? cnd[c].x : s_ck[sk][c].x), dclamp);
          const uint64_t ak = (KT > 0) ? add[c] : s_ak[sk][c];
#pragma unroll
          for (int i = 0; i < CPT; ++i) best[i] = min(best[i], pv[i * 32] + ak);
        }
      }
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const uint64_t k = best[i];
        best[i] = (k >= INF64) ? INF64 : (k & ~kmask);
        pdw[i >> 2] = put_byte(pdw[i >> 2], (uint32_t)k, i & 3);
        cur[i * 32] = best[i];
      }
      for (int r2 = (int)rank + 1; r2 <= rtop; ++r2) {
        const int need = r2 * S - maxd;
        const uint32_t rbar = cl_map(&s_bar[sb], (uint32_t)r2);
#pragma unroll
        for (int i = 0; i < CPT; ++i)
          if (wbase + 32 * i + lane >= need)
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                             cl_map(cur + i * 32, (uint32_t)r2)),
                         "l"(best[i]), "r"(rbar)
                         : "memory");
      }
    }
    bp = bc;
    bc = (bc + 1 == NB) ? 0 : bc + 1;
    if (KT == 0 && a + 1 < a1) stage0(nd, nub, sk ^ 1);  // slot last read in row a-1
    if (a + 1 < a1) {
      const uint4* nq = reinterpret_cast<const uint4*>(cand_all + (size_t)(a + 1) * KP2);
#pragma unroll
      for (int c = 0; c < KP2 / 2; ++c) if (KT > 0) cq[c] = nq[c];
      band = band_all[a + 1];
      maxd = (a + 2 < a1) ? my_wmaxd[a + 2] : 0;
    }
#ifdef LG_DP_TIMING
    const long long tp0 = clock64();
    t_p += tp0 - tr0;
#endif
    // local cells of row a visible to every warp of this CTA
    __syncthreads();
#ifdef LG_DP_TIMING
    const long long ts1 = clock64();
    t_s += ts1 - tp0;
#endif
    // back-pressure only (no CTA runs a row ahead, so no push lands in a row buffer a
    // peer still reads); the data itself is ordered by the st.async -> mbarrier path
    if (NB == 3) {
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every CTA finished row a-1
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    if (live) {  // cell-major PD row (byte of cell e at a * PDR + e): 32 B per warp store
      uint8_t* dst = PD + (int64_t)a * PDR + cbase + warp * 32 * CPT + lane;
#pragma unroll
      for (int i = 0; i < CPT; ++i) __stcg(dst + 32 * i, (uint8_t)(pdw[i >> 2] >> (8 * (i & 3))));
    }
    if (NB == 2) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
#ifdef LG_DP_TIMING
    t_cl += clock64() - ts1;
#endif
    // remote cells of row a landed
    {
      const uint32_t ba = (uint32_t)__cvta_generic_to_shared(&s_bar[sb]);
      const uint32_t par = (bph >> sb) & 1u;
      asm volatile(
          "{\n\t.reg .pred done;\n\t"
          "DPW_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
          "@!done bra DPW_%=;\n\t}\n" ::"r"(ba),
          "r"(par)
          : "memory");
      bph ^= 1u << sb;
    }
#ifdef LG_DP_TIMING
    t_push += clock64() - tp0;
#endif
  }
  if (!wide) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // pairs the last arrive
  LG_T(3);
  if (ngroups > 1) {
    // ---- the join of the two layer groups (see "Layer groups" below), in the top
    //      group's cluster: its last row P stays in its CTAs' shared memory
    const uint64_t NONE = ~0ull;
    auto rowv = [&](int e) -> uint64_t {  // last row's value at cell e (units of 2^gsh bits)
      if (e > D) return NONE;
      if (!wide) {
        const uint32_t x = (r32a + (size_t)bp * row + PAD)[e];
        return (x >= INF32) ? NONE : (uint64_t)(x >> kb);
      }
      const uint64_t x = (r64a + (size_t)bp * row + PAD)[e];
      return (x >= INF64) ? NONE : (x >> kb);
    };
    uint64_t* F = rowout;                                           // group 0's last row
    if (grp == 0) {
      for (int el = tid; el < S; el += NT) {
        const int e = cbase + el;
        if (e > D) break;
        __stcg(F + e, rowv(e));
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        st_release_gpu(&jmeta->tok[rank], tok);  // this slice of F (and every PD row) is written
      }
      return;
    }
    // (1) prefix minima of P with their first index: a chunk of CPT cells per thread,
    //     block scan, then the slices below this CTA's (their totals over DSMEM)
    __shared__ uint64_t s_slv[CL_MAX];
    __shared__ int s_sli[CL_MAX];
    uint64_t* PMs = reinterpret_cast<uint64_t*>(smem_raw + (size_t)(wide ? 8 : 4) * bc * row);  // a free row buffer
    int32_t* PAs = reinterpret_cast<int32_t*>(PMs + S);
    const int c0 = tid * CPT;
    uint64_t pv[CPT];
    uint64_t mv = NONE;
    int mi = -1;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      pv[j] = rowv(cbase + c0 + j);
      if (pv[j] < mv) { mv = pv[j]; mi = cbase + c0 + j; }
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {  // inclusive scan, the earlier operand winning ties
      const uint64_t ov = __shfl_up_sync(LG_FULL, mv, o);
      const int oi = __shfl_up_sync(LG_FULL, mi, o);
      if (lane >= o && ov <= mv) { mv = ov; mi = oi; }
    }
    if (lane == 31) { s_redk[warp] = mv; s_rede[warp] = mi; }
    __syncthreads();
    if (warp == 0) {
      uint64_t wv = (lane < NW) ? s_redk[lane] : NONE;
      int wi = (lane < NW) ? s_rede[lane] : -1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t ov = __shfl_up_sync(LG_FULL, wv, o);
        const int oi = __shfl_up_sync(LG_FULL, wi, o);
        if (lane >= o && ov <= wv) { wv = ov; wi = oi; }
      }
      s_redk[lane] = wv;  // inclusive over warps 0..lane
      s_rede[lane] = wi;
      const uint64_t tv = __shfl_sync(LG_FULL, wv, NW - 1);  // the slice's minimum
      const int ti = __shfl_sync(LG_FULL, wi, NW - 1);
      if (lane < (int)NC) {
        cl_st(cl_map(&s_slv[rank], (uint32_t)lane), tv);
        cl_st(cl_map(&s_sli[rank], (uint32_t)lane), (uint32_t)ti);
      }
    }
    cl_sync();  // the slice minima of every CTA landed; s_redk / s_rede complete
    {
      uint64_t cv = NONE;  // prefix over the lower slices, then the lower threads of this one
      int ci = -1;
      for (uint32_t r2 = 0; r2 < rank; ++r2)
        if (s_slv[r2] < cv) { cv = s_slv[r2]; ci = s_sli[r2]; }
      uint64_t ev = (warp > 0) ? s_redk[warp - 1] : NONE;
      int ei = (warp > 0) ? s_rede[warp - 1] : -1;
      const uint64_t lv = __shfl_up_sync(LG_FULL, mv, 1);
      const int li = __shfl_up_sync(LG_FULL, mi, 1);
      if (lane > 0 && lv < ev) { ev = lv; ei = li; }
      if (ev < cv) { cv = ev; ci = ei; }
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        if (pv[j] < cv) { cv = pv[j]; ci = cbase + c0 + j; }
        PMs[c0 + j] = cv;
        PAs[c0 + j] = ci;
      }
    }
    // (2) group 0's F: wait for its 16 slices
    if (tid < (int)NC)
      while (ld_acquire_gpu(&jmeta->tok[tid]) != tok) __nanosleep(64);
    __syncthreads();
    LG_T(4);
    // (3) C* = min_{e1} F[e1] + PM[D - e1] and e* = the smallest e1 + PA[D - e1] attaining
    //     it: x = D - e1 runs over this CTA's cells (order-free: a lexicographic minimum)
    uint64_t bv = NONE;
    int be = 0x7fffffff;
    uint64_t fv[CPT];  // F[D - x] over this CTA's cells (reused by (4) when e* = D)
    {
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int x = cbase + c0 + j;
        fv[j] = (x <= D) ? __ldcg(F + (D - x)) : NONE;
      }
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const uint64_t pm = PMs[c0 + j];
        if (fv[j] == NONE || pm == NONE) continue;
        const uint64_t v = fv[j] + pm;
        const int e = D - (cbase + c0 + j) + PAs[c0 + j];
        if (v < bv || (v == bv && e < be)) { bv = v; be = e; }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint64_t ov = __shfl_xor_sync(LG_FULL, bv, o);
      const int oe = __shfl_xor_sync(LG_FULL, be, o);
      if (ov < bv || (ov == bv && oe < be)) { bv = ov; be = oe; }
    }
    __syncthreads();  // s_redk / s_rede reads of (1) done
    if (lane == 0) { s_redk[warp] = bv; s_rede[warp] = be; }
    __syncthreads();
    if (warp == 0) {
      bv = (lane < NW) ? s_redk[lane] : NONE;
      be = (lane < NW) ? s_rede[lane] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint64_t ov = __shfl_xor_sync(LG_FULL, bv, o);
        const int oe = __shfl_xor_sync(LG_FULL, be, o);
        if (ov < bv || (ov == bv && oe < be)) { bv = ov; be = oe; }
      }
      if (lane < (int)NC) {
        cl_st(cl_map(&s_clk[rank], (uint32_t)lane), bv);
        cl_st(cl_map(&s_cle[rank], (uint32_t)lane), (uint32_t)be);
      }
    }
    cl_sync();
    uint64_t Cs = NONE;
    int es = 0x7fffffff;
    for (int r2 = 0; r2 < (int)NC; ++r2)
      if (s_clk[r2] < Cs || (s_clk[r2] == Cs && s_cle[r2] < es)) { Cs = s_clk[r2]; es = s_cle[r2]; }
    const int used_default = (Cs == NONE);
    // (4) E2 = {e2 <= e* : F[e* - e2] + P[e2] == C*} over this CTA's cells, appended to
    //     rank 0's list over DSMEM (rank 0's row space is dead from here: (3) is done)
    int2* const sv0 = reinterpret_cast<int2*>(smem_raw + (((size_t)La * 4 + 15) & ~(size_t)15));
    if (!used_default) {
      if (es != D) {  // (e* = D, the usual case: the F window of (3))
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
          const int x = cbase + c0 + j;
          fv[j] = (x <= es && pv[j] != NONE) ? __ldcg(F + (es - x)) : NONE;
        }
      }
#pragma unroll
      for (int j = 0; j < CPT; ++j)
        if (fv[j] != NONE && pv[j] != NONE && fv[j] + pv[j] == Cs) {
          uint32_t idx;
          asm volatile("atom.shared::cluster.add.u32 %0, [%1], 1;" : "=r"(idx) : "r"(cl_map(&s_ns, 0)) : "memory");
          const int e2 = cbase + c0 + j;
          asm volatile("st.shared::cluster.v2.s32 [%0], {%1, %2};" ::"r"(cl_map(sv0 + idx, 0)), "r"(e2), "r"(e2)
                       : "memory");
        }
    }
    cl_sync();
    LG_T(18);
#ifdef LG_DP_TIMING
    if ((rank == NC - 1 || rank == NC / 2) && tid == 0)
      printf("dp group 1 rank %d per row: compute %lld push %lld syncthreads %lld cluster %lld all-waits %lld\n",
             (int)rank, t_c / (a1 - a0), (t_p - t_c) / (a1 - a0), t_s / (a1 - a0), t_cl / (a1 - a0),
             t_push / (a1 - a0));
#endif
    if (rank != 0) return;
    // (5) rank 0: the lexicographic walk of the top group while several E2 entries
    //     survive, the two backtracks (one warp each), R20 check and summary
    __shared__ int s_cnt[2], s_m;
    int32_t* bch = reinterpret_cast<int32_t*>(smem_raw);  // [La] (the rows are dead)
    int2* const sv1 = sv0 + (D + 1);
    double* sm_ce = reinterpret_cast<double*>(sv0);  // finish_plan's scratch (after the walk)
    const int h = a0;
    if (!used_default) {
      const int ns0 = (int)s_ns;
      int ns = ns0, cur = 0, a = La - 1;
      if (tid == 0) { s_cnt[0] = ns0; s_m = 0x7fffffff; }
      __syncthreads();
      while (ns > 1 && a >= h) {
        const int2* svc = cur ? sv1 : sv0;
        int2* svn = cur ? sv0 : sv1;
        for (int i = tid; i < ns; i += NT) atomicMin(&s_m, pd_cm(PD, PDR, a, svc[i].x) & pdmask);
        if (tid == 0) s_cnt[cur ^ 1] = 0;
        __syncthreads();
        const int m = s_m;
        const int dm = my_wdisc[a * K + m];
        for (int i = tid; i < ns; i += NT) {
          const int2 w = svc[i];
          if ((pd_cm(PD, PDR, a, w.x) & pdmask) == m) svn[atomicAdd(&s_cnt[cur ^ 1], 1)] = make_int2(w.x - dm, w.y);
        }
        if (tid == 0) bch[a] = m;
        __syncthreads();
        ns = s_cnt[cur ^ 1];
        cur ^= 1;
        if (tid == 0) s_m = 0x7fffffff;
        --a;
        __syncthreads();
      }
      const int2 w = (cur ? sv1 : sv0)[0];
      LG_T(19);
      if (warp == 0 && a >= h) bt_warp(PD, PDR, my_wdisc, K, pdmask, a, h, w.x, bch);
      if (warp == (NW > 1 ? 1 : 0) && h > 0) bt_warp(PD, PDR, my_wdisc, K, pdmask, h - 1, 0, es - w.y, bch);
    }
    __syncthreads();
    LG_T(5);
    __shared__ int s_fl;
    finish_plan(used_default, bch, La, act, default_idx, err, bits, K, flags, emax, s_defbits, choice, info, sm_ce,
                &s_fl);
#ifdef LG_DP_TIMING
    if (tid == 0)
      printf("dp prelude detail: pdl %lld table+active %lld emax||costs %lld disc %lld split %lld band+cand %lld "
             "rowinit+bars %lld sync %lld\n", tstamp[10] - tstamp[0], tstamp[6] - tstamp[10], tstamp[7] - tstamp[6],
             tstamp[8] - tstamp[7], tstamp[15] - tstamp[8], tstamp[16] - tstamp[15], tstamp[17] - tstamp[16],
             tstamp[2] - tstamp[17]);
    if (tid == 0)
      printf("dp join detail: join %lld walk-setup %lld backtrack %lld | per row: compute %lld push %lld "
             "syncthreads %lld cluster %lld all-waits %lld\n", tstamp[18] - tstamp[4],
             tstamp[19] - tstamp[18], tstamp[5] - tstamp[19], t_c / (a1 - a0), (t_p - t_c) / (a1 - a0),
             t_s / (a1 - a0), t_cl / (a1 - a0), t_push / (a1 - a0));
    if (tid == 0)
      printf("dp group 1 (join in-cluster): layers [%d, %d) of %d: prelude %lld init %lld rows %lld (%lld/layer) "
             "P-scan+F-wait %lld join+backtrack %lld summary %lld\n", a0, a1, La, tstamp[1] - tstamp[0],
             tstamp[2] - tstamp[1], tstamp[3] - tstamp[2], (tstamp[3] - tstamp[2]) / (a1 > a0 ? a1 - a0 : 1),
             tstamp[4] - tstamp[3], tstamp[5] - tstamp[4], clock64() - tstamp[5]);
#endif
    return;
  }
  // ---- line 23: argmin of the last row over this CTA's cells, gathered in rank 0
  {
    uint64_t bk = ~0ull;
    int be = 0x7fffffff;
    for (int el = tid; el < S; el += NT) {
      const int e = cbase + el;
      if (e > D) break;
      uint64_t v;
      if (!wide) { const uint32_t x = (r32a + (size_t)bp * row + PAD)[e]; v = (x >= INF32) ? ~0ull : x; }
      else { const uint64_t x = (r64a + (size_t)bp * row + PAD)[e]; v = (x >= INF64) ? ~0ull : x; }
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
    if (warp == 0) {
      bk = (lane < NW) ? s_redk[lane] : ~0ull;
      be = (lane < NW) ? s_rede[lane] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint64_t ov = __shfl_xor_sync(LG_FULL, bk, o);
        const int oe = __shfl_xor_sync(LG_FULL, be, o);
        if (ov < bk || (ov == bk && oe < be)) { bk = ov; be = oe; }
      }
      if (lane == 0) {
        cl_st(cl_map(&s_clk[rank], 0), bk);
        cl_st(cl_map(&s_cle[rank], 0), (uint32_t)be);
      }
    }
  }
  cl_sync();  // PD (global) and the gathered argmins visible; peers may exit after this
  LG_T(4);
  if (rank != 0) return;
  // ---- rank 0: backtrack (lines 24-27) through PD, R20 check and summary
  const int32_t* bdisc = my_wdisc;  // the discretised table (shared memory)
  int32_t* bch = reinterpret_cast<int32_t*>(smem_raw);  // [La] chosen c per active layer (rows are dead)
  __syncthreads();
  if (warp == 0) {
    uint64_t k = (lane < (int)NC) ? s_clk[lane] : ~0ull;
    int ee = (lane < (int)NC) ? s_cle[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint64_t ov = __shfl_xor_sync(LG_FULL, k, o);
      const int oe = __shfl_xor_sync(LG_FULL, ee, o);
      if (ov < k || (ov == k && oe < ee)) { k = ov; ee = oe; }
    }
    const int used_default = (k == ~0ull);
    if (!used_default) bt_warp(PD, PDR, bdisc, K, pdmask, La - 1, 0, ee, bch);
    if (lane == 0) s_La = used_default;
  }
  __syncthreads();
  double* sm_ce = reinterpret_cast<double*>(smem_raw + (((size_t)La * 4 + 15) & ~(size_t)15));  // after bch
  finish_plan(s_La, bch, La, act, default_idx, err, bits, K, flags, emax, s_defbits, choice, info, sm_ce, &s_La);
#ifdef LG_DP_TIMING
  LG_T(5);
  if (tid == 0)
    printf("dp cluster prelude phases: flags %lld compact+emax %lld disc %lld gcd+cand %lld\n", tstamp[6] - tstamp[0],
           tstamp[7] - tstamp[6], tstamp[8] - tstamp[7], tstamp[9] - tstamp[8]);
  if (tid == 0)
    printf("dp cluster timing (cycles, rank 0): prelude %lld init %lld rows %lld (%lld/layer: compute %lld push %lld "
           "syncthreads %lld cluster %lld all-waits %lld) argmin %lld back+summary %lld\n", tstamp[1] - tstamp[0],
           tstamp[2] - tstamp[1], tstamp[3] - tstamp[2], (tstamp[3] - tstamp[2]) / (La ? La : 1), t_c / La,
           (t_p - t_c) / La, t_s / La, t_cl / La, t_push / (La ? La : 1), tstamp[4] - tstamp[3], tstamp[5] - tstamp[4]);
#endif
}

// ---------------------------------------------------------------------------
// Layer groups.  With ngroups == 2, k_solve_cl's two clusters run Alg.1's row recursion
// for the bottom active layers [0, h) and for the top layers [h, La) concurrently, each
// from the zero row: the critical path of the solve halves.  The bottom cluster writes its
// last row F to global memory and releases the launch's token per CTA; the top cluster
// keeps its last row P in its CTAs' shared memory (a slice per CTA), waits for the 16
// tokens and joins (the bottom cluster never waits, so co-scheduling is not required).
// The whole recursion's last row is their min-plus convolution, DP[e] = min_{e1} F[e1] +
// P[e - e1] (min-plus is associative), and the join returns exactly Alg.1's plan without
// forming it:
//  * C* = min_{e <= D} DP[e] = min_{e1} F[e1] + PM[D - e1], PM = prefix minima of P;
//  * e* = the smallest e attaining C* (line 23, R19) = the smallest e1 + PA[D - e1] over
//    the e1 attaining C*, PA[x] = the first index of P's minimum over [0, x];
//  * lines 24-27: from (La - 1, e*) Alg.1's PD takes, layer by layer from the top, the
//    first candidate (strict <, R19) that still has an optimal completion -- the
//    lexicographically smallest (c_{La-1}, ..., c_0) among the optimal plans of total
//    disc e*.  An optimal plan is optimal within each group at its split (e* - e2, e2),
//    so its top part is the top group's own backtrack from some e2 in
//    E2 = {e2 : F[e* - e2] + P[e2] = C*}: every e2 of E2 walks down the top group's PD
//    at once and, layer by layer, only the walks with the smallest candidate survive;
//    the last survivor's e2 fixes e1 = e* - e2 and the bottom group's own backtrack from
//    e1 gives the bottom layers.  (Usually |E2| = 1 and both backtracks run at once on
//    two warps, PD read from L2.)
// Checked against a sequential reference on 600 random tie-heavy instances for every
// split point (K4), and bit-exact against the oracle in tests/test_gpu_dp.py.
// ---------------------------------------------------------------------------
// Weighted costs (NEXT-1): out = bits * w[l], exact in int64; -1 on a negative input or
// overflow (lgreco_solve rejects negative costs with LGRECO_EINVAL).
__global__ void k_weight_costs(const int64_t* __restrict__ bits, const int64_t* __restrict__ w, int L, int K,
                               int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)L * K;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = bits[i], x = w[i / K];
    int64_t r = -1;
    if (b >= 0 && x >= 0) {
      const unsigned long long hi = __umul64hi((unsigned long long)b, (unsigned long long)x);
      const unsigned long long lo = (unsigned long long)b * (unsigned long long)x;
      if (hi == 0 && lo <= (unsigned long long)INT64_MAX) r = (int64_t)lo;
    }
    out[i] = r;
  }
}

cudaError_t launch_weight_costs(const int64_t* bits, const int64_t* w, int L, int K, int64_t* out, cudaStream_t st) {
  const int64_t n = (int64_t)L * K;
  if (n <= 0) return cudaSuccess;
  k_weight_costs<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, st>>>(bits, w, L, K, out);
  return cudaGetLastError();
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

size_t solve_workspace_bytes(int L, int K, int D) {
  return align_up((size_t)L * std::max(D + 1 + CL_MAX * 32 * 8, PD_ROW)) + align_up(sizeof(int32_t) * (size_t)(L + 1)) +
         align_up(sizeof(int64_t) * 2 * (size_t)(D + 1)) + align_up(sizeof(int32_t) * (size_t)L * K * CL_MAX) +
         align_up(sizeof(uint64_t) * (size_t)L * K * CL_MAX) + align_up(sizeof(int32_t) * (size_t)(L + 1) * CL_MAX) +
         align_up(sizeof(JoinMeta));
}

// Cluster launch (k_solve_cl) when the shapes fit: K <= 16, CPT in {2, 4, 8}, two
// 64-bit full-length rows within 200 KB of shared memory, and an 8-CTA cluster of that
// size can be resident.  Returns cudaErrorNotSupported (nothing launched) otherwise.
static cudaError_t launch_solve_cluster(const SolveArgs& a, uint8_t* pd, int32_t* act, int32_t* wdisc, uint64_t* wadd,
                                        int32_t* wmaxd, int NC, int ngroups, uint64_t* rowout, JoinMeta* jmeta,
                                        cudaStream_t st) {
  if (a.K < 1 || a.K > 256) return cudaErrorNotSupported;
  if (const char* env = getenv("LGRECO_DP_NC")) NC = std::max(2, std::min(CL_MAX, atoi(env)));
  int cpt = 1;
  if (const char* env = getenv("LGRECO_DP_CPT")) cpt = std::max(1, std::min(8, atoi(env)));
  else cpt = QP_DP_CPT0;
  while (cpt <= 8 && (int64_t)NC * DP_THREADS * cpt < (int64_t)a.D + 1) cpt *= 2;
  if (cpt > 8) return cudaErrorNotSupported;
  // (KT == 0 stages one candidate per thread: at least K threads)
  const int nw = std::max((int)(((int64_t)a.D + 1 + NC * 32 * cpt - 1) / (NC * 32 * cpt)), (a.K + 31) / 32);
  const int nt = nw * 32;
  const int S = nt * cpt;
  // two 64-bit rows, then the per-layer tables: costs (8 B), disc (4 B), max disc (4 B),
  // candidate pairs (8 B x KP2), 64-bit keys (8 B x KT), band (8 B)
  int kt0 = a.K <= 4 ? 4 : a.K == 5 ? 5 : a.K <= 7 ? 7 : a.K <= 8 ? 8 : a.K <= 16 ? 16 : 0;
  const size_t rows_b = (size_t)16 * (32 * cpt + (size_t)NC * S);
  // KT == 0: only the max-disc and band tables live in shared memory
  auto smem_of = [&](int k) {
    return rows_b + (size_t)4 * (a.L + 4) + 16 + (size_t)8 * a.L +
           (k > 0 ? (size_t)12 * a.L * a.K + (size_t)a.L * (8 * ((k + 2) & ~1) + 8 * k) : 0);
  };
  if (kt0 > 0 && smem_of(kt0) > 220 * 1024) kt0 = 0;  // many layers: per-row staged tables (grouped keys)
  const size_t smem = smem_of(kt0);
  if (smem > 220 * 1024 || (size_t)24 * a.L + 64 > rows_b) return cudaErrorNotSupported;
  const int kt = kt0;
  // layer groups: K <= 16 (tables in shared memory); the top group's rank 0 walks the
  // E2 list in the row space ([La] choices, two (D + 1)-entry int2 lists)
  if (ngroups > 1 && (size_t)4 * a.L + 16 + (size_t)16 * (a.D + 1) > rows_b) return cudaErrorNotSupported;
  if (ngroups > 1 && kt == 0) return cudaErrorNotSupported;
  void (*fn)(const double*, const int64_t*, int, int, const int32_t*, const int32_t*, int, uint32_t, int32_t*,
             lgreco_solve_info*, uint8_t*, int32_t*, int32_t*, uint64_t*, int32_t*, int, uint64_t*, JoinMeta*,
             uint64_t) = nullptr;
#define LG_CL(C, KT) if (cpt == C && kt == KT) fn = k_solve_cl<C, KT>;
#define LG_CL_K(C) LG_CL(C, 4) LG_CL(C, 5) LG_CL(C, 7) LG_CL(C, 8) LG_CL(C, 16) LG_CL(C, 0)
  LG_CL_K(1) LG_CL_K(2) LG_CL_K(4) LG_CL_K(8)
#undef LG_CL_K
#undef LG_CL
  if (!fn) return cudaErrorNotSupported;
  // attribute + cluster-occupancy checks are host-side driver calls (tens of us): done
  // once per (device, kernel, shared memory, block) configuration and memoised (memo.h)
  long long okm = -1;
  const bool cached = memo_get((const void*)fn, (long long)smem, nt, NC, ngroups, &okm);
  if (cached && !okm) return cudaErrorNotSupported;
  cudaError_t e = cudaSuccess;
  if (!cached) {
    if (NC > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      return cudaErrorNotSupported;
    }
    e = memo_smem_attr((const void*)fn, smem);
    if (e != cudaSuccess) { cudaGetLastError(); return cudaErrorNotSupported; }
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = NC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(NC * ngroups, 1, 1);
  cfg.blockDim = dim3(nt, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (!cached) {
    int nclusters = 0;
    e = cudaOccupancyMaxActiveClusters(&nclusters, (const void*)fn, &cfg);
    const int ok = (e == cudaSuccess && nclusters >= ngroups) ? 1 : 0;
    memo_put((const void*)fn, (long long)smem, nt, NC, ngroups, ok);
    if (!ok) {
      if (getenv("LGRECO_DEBUG")) fprintf(stderr, "lgreco: cluster occupancy %d (%s)\n", nclusters, cudaGetErrorString(e));
      cudaGetLastError();
      return cudaErrorNotSupported;
    }
  }
  // a plain launch (no PDL attribute): the solve waits for ALL prior work of the stream --
  // in the pipelined schedule that is the previous solve too, whose plan the concurrent
  // fused pass before this call reads (include/lgreco.h, LGRECO_PC_CONCURRENT)
  cfg.numAttrs = 1;
  // the launch's token (the group handshake): unique per launch in this process
  static std::atomic<uint64_t> g_tok{0x9E3779B97F4A7C15ull ^ ((uint64_t)time(nullptr) << 24) ^ (uint64_t)getpid()};
  const uint64_t tok = g_tok.fetch_add(2) | 1ull;
  return cudaLaunchKernelEx(&cfg, fn, a.err, a.bits, a.L, a.K, a.default_idx, a.compress, a.D, a.flags, a.choice, a.info,
                            pd, act, wdisc, wadd, wmaxd, ngroups, rowout, jmeta, tok);
}

cudaError_t launch_solve(const SolveArgs& a, void* ws, cudaStream_t st) {
  uint8_t* base = static_cast<uint8_t*>(ws);
  uint8_t* pd = base;
  const size_t pd_bytes = align_up((size_t)a.L * std::max(a.D + 1 + CL_MAX * 32 * 8, PD_ROW));
  int32_t* act = reinterpret_cast<int32_t*>(base + pd_bytes);
  int64_t* grows = reinterpret_cast<int64_t*>(base + pd_bytes +
                                              align_up(sizeof(int32_t) * (size_t)(a.L + 1)));
  int32_t* wdisc = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(grows) +
                                              align_up(sizeof(int64_t) * 2 * (size_t)(a.D + 1)));
  uint64_t* wadd = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(wdisc) +
                                               align_up(sizeof(int32_t) * (size_t)a.L * a.K * CL_MAX));
  int32_t* wmaxd = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(wadd) +
                                              align_up(sizeof(uint64_t) * (size_t)a.L * a.K * CL_MAX));
  JoinMeta* jmeta = reinterpret_cast<JoinMeta*>(reinterpret_cast<uint8_t*>(wmaxd) +
                                                align_up(sizeof(int32_t) * (size_t)(a.L + 1) * CL_MAX));
  uint64_t* rowout = reinterpret_cast<uint64_t*>(grows);
  if (!(a.flags & LGRECO_SOLVE_SINGLE_CTA)) {
    // two layer groups on two 16-CTA clusters when the table is long enough to pay for the
    // join (LGRECO_DP_GROUPS=1|2 overrides); else one cluster of 16 SMs, else 8
    int ng = a.L >= 32 ? 2 : 1;
    if (const char* env = getenv("LGRECO_DP_GROUPS")) ng = atoi(env) == 2 ? 2 : 1;
    cudaError_t ce = cudaErrorNotSupported;
    // LGRECO_SOLVE_NARROW: 8-CTA clusters (beside the fused pass: 2 x 8 SMs for 62 us took
    // less from it than 2 x 16 SMs for 55 us -- C4 pipelined step 96.5 vs 100.2 us)
    const int nc = (a.flags & LGRECO_SOLVE_NARROW) ? 8 : 16;
    if (ng == 2) ce = launch_solve_cluster(a, pd, act, wdisc, wadd, wmaxd, nc, 2, rowout, jmeta, st);
    if (ce == cudaErrorNotSupported) ce = launch_solve_cluster(a, pd, act, wdisc, wadd, wmaxd, nc, 1, rowout, jmeta, st);
    if (ce == cudaErrorNotSupported) ce = launch_solve_cluster(a, pd, act, wdisc, wadd, wmaxd, 8, 1, rowout, jmeta, st);
    if (ce != cudaErrorNotSupported) return ce;
    if (getenv("LGRECO_DEBUG")) fprintf(stderr, "lgreco: cluster solve not used (L=%d K=%d D=%d)\n", a.L, a.K, a.D);
  }
  const int W1 = a.D + 1;
  const int cpt = (W1 + DP_THREADS - 1) / DP_THREADS;
  // fast path: two padded 32-bit rows or two 64-bit rows in smem (see k_solve_fast)
  const size_t fast_smem = (size_t)16 * (32 * cpt + cpt * DP_THREADS);  // two 64-bit rows (>= two 32-bit rows)
  // the prelude stages 24 bytes per layer in the same shared memory
  if (cpt <= 16 && fast_smem <= 200 * 1024 && (size_t)24 * a.L + 64 <= fast_smem) {
    cudaError_t e = cudaSuccess;
#define LG_SF2(C, KT)                                                                                      \
  {                                                                                                          \
    e = memo_smem_attr((const void*)k_solve_fast<C, KT>, 200 * 1024);                                     \
    if (e != cudaSuccess) return e;                                                                          \
    k_solve_fast<C, KT><<<1, DP_THREADS, fast_smem, st>>>(a.err, a.bits, a.L, a.K, a.default_idx, a.compress, \
                                                          a.D, a.flags, a.choice, a.info, pd, act, wdisc, wadd); \
  }
#define LG_SF(C)                                       \
  case C:                                              \
    if (C == 10 && a.K == 5) LG_SF2(C, (C == 10 ? 5 : 8)) else if (C == 10 && a.K == 7) LG_SF2(C, (C == 10 ? 7 : 8)) \
    else if (a.K <= 8) LG_SF2(C, 8) else if (a.K <= 16) LG_SF2(C, 16) else LG_SF2(C, 0) \
    break;
    switch (cpt) { LG_SF(1) LG_SF(2) LG_SF(3) LG_SF(4) LG_SF(5) LG_SF(6) LG_SF(7) LG_SF(8) LG_SF(9) LG_SF(10)
                   LG_SF(11) LG_SF(12) LG_SF(13) LG_SF(14) LG_SF(15) LG_SF(16) }
#undef LG_SF
    return cudaGetLastError();
  }
  const size_t row_bytes = sizeof(int64_t) * 2 * (size_t)(a.D + 1);
  const int in_smem = row_bytes <= 200 * 1024;
  const size_t smem = in_smem ? row_bytes : 0;
  cudaError_t e = memo_smem_attr((const void*)k_solve_generic, 200 * 1024);
  if (e != cudaSuccess) return e;
  k_solve_generic<<<1, DP_THREADS, smem, st>>>(a.err, a.bits, a.L, a.K, a.default_idx, a.compress, a.D, a.flags,
                                               a.choice, a.info, pd, act, grows, in_smem);
  return cudaGetLastError();
}

}  // namespace lg
