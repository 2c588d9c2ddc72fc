// qsgd.cu -- QSGD-style bucketed min/max stochastic quantisation on sm_100a.
//
//   K1  k_qprofile   (a2)  one HBM pass over x = g + e; per bucket min/max by warp
//                          shuffles, then the realised squared error of EVERY
//                          candidate bit-width from the same Philox uniforms
//                          (R5, R6).  Deterministic:
//                          fixed chunk -> per-chunk partial -> ordered reduce.
//   K1+K5 k_qprofile_q<K, 1|2>  the fused per-step pass (lgreco_profile_compress): K1
//                          plus the planned candidate's quantisation from the same
//                          registers and uniforms -- out and e' (W = 1) or the stage-1
//                          records straight into the owners' windows (W > 1, peer memory).
//   K1b k_qprofile_reduce  per-layer fixed-order fp64 sum of chunk partials, sqrt.
//   K5  k_qpack      (a8)  quantise with the chosen bits, bit-plane pack via
//                          __ballot_sync, fused error feedback e <- x - dec
//                          (and, for W == 1, the decoded output).
//   K8  k_qreduce    (a9)  owner shard: decode W stage-1 records, ordered fp32 sum,
//                          x fl(1/W), requantise (stream 1) and pack stage 2.
//   K9  k_qunpack    (a10) decode a payload into the fp32 mean gradient.
//
// One warp owns one bucket (record) of B = 128*m elements; lane l holds elements
// 128t + 4l .. 4l+3 of sub-block t.  Every CTA owns a fixed chunk of <= 64 buckets
// of ONE layer (no per-record layer search).  Full buckets of 16B-aligned layers
// at B = 128 take a branch-free float4 fast path; the ragged last bucket of a layer,
// misaligned layers and B > 128 take the generic path.
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "memo.h"

namespace lg {

constexpr int QP_THREADS = 256;
constexpr int QP_WARPS = QP_THREADS / 32;
#ifndef Q1_TRIGGER
#define Q1_TRIGGER 0  // K1 / the fused pass trigger their dependents (K1b) as each warp runs out of quads
#endif
#ifndef QF_MAGIC
#define QF_MAGIC 1  // fused pass: the planned candidate's ceil by the FADD2 magic (1) or FRND.CEIL (0); A/B 96.5 -> 95.0 us per pipelined step (the XU pipe carries the profile's ceils)
#endif
#ifndef QP_XU_CEIL
#define QP_XU_CEIL 5  // candidates of the K1 fast path whose ceil runs on the XU pipe (others: FADD2 magic; A/B: 0-5 equal, 7 +2 %)
#endif

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
// three-input forms (FMNMX3, sm_100)
__device__ __forceinline__ float fmin3_nan(float a, float b, float c) {
  float r;
  asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmax3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ void warp_minmax_nan(float& mn, float& mx) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = fmin_nan(mn, __shfl_xor_sync(LG_FULL, mn, o));
    mx = fmax_nan(mx, __shfl_xor_sync(LG_FULL, mx, o));
  }
}

struct X4 { float v[4]; };

__device__ __forceinline__ X4 canon4(float4 a, float4 b) {
  X4 r;
  r.v[0] = canon(a.x, b.x); r.v[1] = canon(a.y, b.y);
  r.v[2] = canon(a.z, b.z); r.v[3] = canon(a.w, b.w);
  return r;
}

__device__ __forceinline__ float4 ld4(const float* __restrict__ p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

// Generic load: 4 elements of the lane starting at flat index base, nv valid.
__device__ __forceinline__ X4 load_x4(const float* __restrict__ g, const float* __restrict__ e,
                                      int64_t base, int nv, bool aligned) {
  X4 r;
  if (nv >= 4 && aligned) {
    r = canon4(ld4(g + base), e ? ld4(e + base) : make_float4(0.f, 0.f, 0.f, 0.f));
  } else {
#pragma unroll
    for (int s = 0; s < 4; ++s)
      r.v[s] = (s < nv) ? canon(__ldg(g + base + s), e ? __ldg(e + base + s) : 0.f) : 0.f;
  }
  return r;
}

__device__ __forceinline__ void store_x4(float* __restrict__ dst, int64_t base, int nv, bool aligned,
                                         const float* v) {
  if (nv >= 4 && aligned) {
    *reinterpret_cast<float4*>(dst + base) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
#pragma unroll
    for (int s = 0; s < 4; ++s)
      if (s < nv) dst[base + s] = v[s];
  }
}

// Per-bucket quantiser parameters for s = 2^b - 1 (R5): inv = RD(s/range) (so t·inv <= s
// for every t <= range: the code never exceeds s), unit = RN(range/s); constant
// (mx == mn) or s/range >= FLT_MAX (inv = FLT_MAX) -> inv = 0 (q = 0).
__device__ __forceinline__ void qparams(float mn, float mx, float s, float& inv, float& unit) {
  if (mx == mn) { inv = 0.f; unit = 0.f; return; }
  const float range = __fsub_rn(mx, mn);
  // RD from the RN quotient (div.rd is a slow path): step down one ulp when inv·range > s;
  // the FMA's sign is exact (the residual is far above the subnormal range)
  inv = __fdiv_rn(s, range);
  if (__fmaf_rn(inv, range, -s) > 0.f) inv = __int_as_float(__float_as_int(inv) - 1);
  unit = __fdiv_rn(range, s);
  if (!(inv < 3.40282347e+38f)) inv = 0.f;
}

// Stochastic rounding of t = x - mn (R6): q = min(floor(v) + [u < frac(v)], s) with
// v = t·inv exact.  r = t·inv - u is formed exactly inside one FFMA and rounded up once:
// for r in (n-1, n], RU(r) stays in (n-1, n] (every integer below 2^24 is a float), so
// ceil(RU(r)) = ceil(r) = floor(v) + [u < frac(v)] bit for bit (u = frac(v) -> floor(v)).
// r in (-1, 0] gives q = -0: (uint32_t) and fmaf(q, unit, mn) treat it as +0 (mn != -0,
// x is canonical).  With inv = RD(s/range) (R5) v <= s always, so the min with s never
// binds; the pack/decode kernels (HBM-bound) keep R6's literal min, the profile's paired
// loop (issue-bound) drops it.
__device__ __forceinline__ float qcode(float t, float inv, float u, float s) {
  return fminf(ceilf(__fmaf_ru(t, inv, -u)), s);
}

__device__ __forceinline__ void uniforms4(uint32_t c0, uint32_t rankfield, uint32_t step, uint32_t stream,
                                          uint32_t k0, uint32_t k1, float* u) {
  const U4 r = philox10(c0, rankfield, step, stream, k0, k1);
  u[0] = word_u(r.x); u[1] = word_u(r.y); u[2] = word_u(r.z); u[3] = word_u(r.w);
}

// ---------------------------------------------------------------------------
// K1 profile
// ---------------------------------------------------------------------------
// Quantise 4 elements with every candidate and accumulate the lane's SSE (fp32, of
// d * S: see bucket_scale).
template <int KT>
__device__ __forceinline__ void prof_candidates(const float* x, float mn, const float* u, float my_inv,
                                                float my_unit, const CandS& cs, int K, float S, float* acc) {
  float tt[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) tt[s] = __fsub_rn(x[s], mn);
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    if (j < K) {
      const float inv = __shfl_sync(LG_FULL, my_inv, j);
      const float unit = __shfl_sync(LG_FULL, my_unit, j);
      float sse = 0.f;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const float q = qcode(tt[s], inv, u[s], cs.s[j]);
        const float d = __fmul_rn(__fsub_rn(x[s], __fmaf_rn(q, unit, mn)), S);
        sse = __fmaf_rn(d, d, sse);
      }
      acc[j] = __fadd_rn(acc[j], sse);
    }
  }
}

// Fast-path candidate loop (full aligned buckets of 128, 8 lanes per bucket, 16
// elements per lane).  q is the pinned code (R6) computed as in qcode:
//   q = min(ceil(RU(t * inv - u)), s)   (t * inv - u exact inside one FFMA.RU),
// which equals min(floor(v) + [u < v - floor(v)], s) for the exact v = t * inv: for
// real r = v - u in (n-1, n], RU(r) lies in (n-1, n] because every integer below 2^24
// is a float, so ceil(RU(r)) = ceil(r) = floor(v) + [u < frac(v)] (u = frac(v) gives
// floor(v)).  The ceil is FRND.CEIL on the conversion pipe, or RU(w + (2^23 + 1)) -
// (2^23 + 1) on the FMA pipe (exact for w in (-1, 2^23 - 1)).  -u = (w >> 8) * -2^-24 is
// one exact FMUL per element shared by all candidates.  dec = fmaf(q, unit, mn) and
// d = x - dec are the pinned decode, so the SSE is
// that of the realised reconstruction.
#ifndef QP_F32X2
#define QP_F32X2 1  // K1 candidate loop on the paired fp32 instructions (FFMA2 / FADD2 / FMUL2)
#endif
// Paired fp32 (sm_100: FFMA2/FADD2/FMUL2 -- two independent IEEE fp32 operations, each
// rounded as its scalar form, one issue slot; a scalar operand is broadcast).
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2pk(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2up(f2_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2fma_rp(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rp.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2_t f2fma(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2_t f2add(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2add_rp(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rp.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2mul(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// The same loop on element pairs (s = 0,1 and 2,3): per pair and candidate one FFMA2.RP
// (w), two ceils, no clamp (inv = RD(s/range) keeps v <= s, R5), one FFMA2 for -dec =
// fma(q, -unit, -mn) (exactly -RN(q unit + mn): RN is symmetric), one FADD2 for d = x +
// (-dec) (= RN(x - dec)), one FFMA2 for the square: 3 issue slots per element and
// candidate instead of 6, every result bit-identical to the scalar form.  The SSE is kept as two fp32 partial sums
// (even / odd elements) per candidate, added at the end.
__device__ __forceinline__ f2_t f2sub(f2_t a, f2_t b) {
  f2_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Fused profile + compress (QFuse): the lane's part of the planned candidate's
// quantisation of its 16 elements -- K5's arithmetic (qcode, dec = fmaf(q, unit, mn),
// e' = x - dec, x canonical), from the uniforms the profile draws anyway.
struct FuseW {
  float invc, unitc;  // the planned candidate's inv / unit of this bucket
  int64_t ebase;      // flat index of the lane's element 0 (element 32i + s at ebase + 32i + s)
  int lim;            // element offsets 32i + s < lim are valid
  bool vec;           // 16-byte stores (regular quad)
  bool wr;            // write at all (valid bucket, layer not skipped)
};

// FUSE: 0 profile only, 1 + compress with the decoded output (W = 1), 2 + compress
// keeping the codes for the stage-1 records (W > 1; codes[i] = the lane's 4 codes of
// sub-block i, one per byte)
template <int KT, bool SCALED, int FUSE = 0>
__device__ __forceinline__ void prof_cand16x2(const float* x, float mn, uint32_t c0, uint32_t rankfield, uint32_t step,
                                              const PhiloxRK& rk, const float* inv, const float* unit,
                                              const CandS& cs, float S, float* acc, const FuseW& fw = FuseW{},
                                              float* __restrict__ out = nullptr, float* __restrict__ ef = nullptr,
                                              uint32_t* codes = nullptr) {
  constexpr float MAGIC = 8388609.0f;  // 2^23 + 1
  constexpr float NEG_2M24 = -5.9604644775390625e-08f;
  f2_t a2[KT];
#pragma unroll
  for (int j = 0; j < KT; ++j) a2[j] = f2pk(0.f, 0.f);
  const f2_t nmn = f2pk(-mn, -mn);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const U4 r = philox10_rk(c0 + 8 * i, rankfield, step, 0u, rk);
    const f2_t nu[2] = {f2mul(f2pk(__uint2float_rn(r.x >> 8), __uint2float_rn(r.y >> 8)), f2pk(NEG_2M24, NEG_2M24)),
                        f2mul(f2pk(__uint2float_rn(r.z >> 8), __uint2float_rn(r.w >> 8)), f2pk(NEG_2M24, NEG_2M24))};
    const f2_t xp[2] = {f2pk(x[4 * i], x[4 * i + 1]), f2pk(x[4 * i + 2], x[4 * i + 3])};
    const f2_t tp[2] = {f2add(xp[0], nmn), f2add(xp[1], nmn)};
#pragma unroll
    for (int j = 0; j < KT; ++j) {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const f2_t w = f2fma_rp(tp[p], f2pk(inv[j], inv[j]), nu[p]);
        // no clamp: inv = RD(s/range) makes t·inv - u <= s, so ceil <= s (R5)
        float q0, q1;
        if (j >= KT - QP_XU_CEIL) {
          float w0, w1;
          f2up(w, w0, w1);
          q0 = ceilf(w0);
          q1 = ceilf(w1);
        } else {
          f2up(f2add(f2add_rp(w, f2pk(MAGIC, MAGIC)), f2pk(-MAGIC, -MAGIC)), q0, q1);
        }
        f2_t d = f2add(xp[p], f2fma(f2pk(q0, q1), f2pk(-unit[j], -unit[j]), nmn));
        if (SCALED) d = f2mul(d, f2pk(S, S));
        a2[j] = f2fma(d, d, a2[j]);
      }
    }
    if constexpr (FUSE != 0) {
      if (fw.wr) {
        float dv[4], ev[4];
        uint32_t cw = 0;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const f2_t w = f2fma_rp(tp[p], f2pk(fw.invc, fw.invc), nu[p]);
          f2_t q;
          if (QF_MAGIC || FUSE == 2) {  // ceil on the FMA pipe (the conversion pipe carries the profile's ceils)
            const f2_t y = f2add_rp(w, f2pk(MAGIC, MAGIC));  // = ceil(w) + 2^23 + 1, exact
            q = f2add(y, f2pk(-MAGIC, -MAGIC));
            if (FUSE == 2) {  // the code as an integer: y's mantissa = ceil(w) + 1 (w > -1)
              float y0, y1;
              f2up(y, y0, y1);
              cw |= ((__float_as_uint(y0) & 0x7fffffu) - 1u) << (16 * p);
              cw |= ((__float_as_uint(y1) & 0x7fffffu) - 1u) << (16 * p + 8);
            }
          } else {
            float w0, w1;
            f2up(w, w0, w1);
            q = f2pk(ceilf(w0), ceilf(w1));
          }
          const f2_t dec = f2fma(q, f2pk(fw.unitc, fw.unitc), f2pk(mn, mn));
          f2up(dec, dv[2 * p], dv[2 * p + 1]);
          f2up(f2sub(xp[p], dec), ev[2 * p], ev[2 * p + 1]);
        }
        const int64_t o = fw.ebase + 32 * i;
        if (fw.vec) {
          if (FUSE == 1) *reinterpret_cast<float4*>(out + o) = make_float4(dv[0], dv[1], dv[2], dv[3]);
          *reinterpret_cast<float4*>(ef + o) = make_float4(ev[0], ev[1], ev[2], ev[3]);
        } else {
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2)
            if (32 * i + s2 < fw.lim) {
              if (FUSE == 1) out[o + s2] = dv[s2];
              ef[o + s2] = ev[s2];
            }
        }
        if (FUSE == 2) {  // codes beyond the layer's end are 0 (x = mn there: t = 0)
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2)
            if (!(32 * i + s2 < fw.lim)) cw &= ~(0xffu << (8 * s2));
          codes[i] = cw;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    float lo, hi;
    f2up(a2[j], lo, hi);
    acc[j] = __fadd_rn(lo, hi);
  }
}

template <int KT, bool SCALED>
__device__ __forceinline__ void prof_cand16(const float* x, float mn, uint32_t c0, uint32_t rankfield, uint32_t step,
                                            uint32_t k0, uint32_t k1, const float* inv, const float* unit,
                                            const CandS& cs, float S, float* acc) {
  constexpr float MAGIC = 8388609.0f;  // 2^23 + 1
#pragma unroll
  for (int j = 0; j < KT; ++j) acc[j] = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const U4 r = philox10(c0 + 8 * i, rankfield, step, 0u, k0, k1);
    constexpr float NEG_2M24 = -5.9604644775390625e-08f;  // -u = (w >> 8) * -2^-24, exact
    const float nu[4] = {__fmul_rn(__uint2float_rn(r.x >> 8), NEG_2M24), __fmul_rn(__uint2float_rn(r.y >> 8), NEG_2M24),
                         __fmul_rn(__uint2float_rn(r.z >> 8), NEG_2M24), __fmul_rn(__uint2float_rn(r.w >> 8), NEG_2M24)};
    float t[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) t[s] = __fsub_rn(x[4 * i + s], mn);
#pragma unroll
    for (int j = 0; j < KT; ++j) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const float xv = x[4 * i + s];
        const float w = __fmaf_ru(t[s], inv[j], nu[s]);  // RU(t·inv - u), one rounding (qcode)
        // ceil(w): the last QP_XU_CEIL candidates use FRND.CEIL on the conversion
        // pipe (idle otherwise), the others the two-FADD magic on the FMA pipe (the
        // kernel's bottleneck): both are exact; -0 from FRND changes no error
        const float cw = (j >= KT - QP_XU_CEIL) ? ceilf(w) : __fsub_rn(__fadd_ru(w, MAGIC), MAGIC);
        const float q = fminf(cw, cs.s[j]);
        float d = __fsub_rn(xv, __fmaf_rn(q, unit[j], mn));
        if (SCALED) d = __fmul_rn(d, S);  // exact power-of-two rescale: d^2 stays normal
        acc[j] = __fmaf_rn(d, d, acc[j]);
      }
    }
  }
}

// Per-bucket rescale of the error terms.  d = x - dec is exact-as-rounded; its square
// in fp32 underflows (or loses bits as a subnormal) once |d| < 2^-63, which the fp64
// oracle does not.  Buckets with range < 2^-20 therefore square d * 2^k (k = 127 -
// biased exponent of the range, so range * 2^k is in [1, 2)) and add the fp32 sum times
// 2^-2k in fp64.  Other buckets: k = 0.
__device__ __forceinline__ bool bucket_scale(float mn, float mx, float& S, double& S2inv) {
  const int eb = (int)((__float_as_uint(__fsub_rn(mx, mn)) >> 23) & 0xffu);
  if (eb >= 107) { S = 1.f; S2inv = 1.0; return false; }
  const int k = 127 - eb;  // 21..127
  S = __uint_as_float((uint32_t)(127 + k) << 23);
  S2inv = __longlong_as_double((long long)(1023 - 2 * k) << 52);
  return true;
}

template <int KT>
__global__ void __launch_bounds__(QP_THREADS, 3)
k_qprofile(const float* __restrict__ g, const float* __restrict__ e, const DevLayer* __restrict__ layers,
           const ProfChunk* __restrict__ chunks, int B, const CandS cs, int K, uint32_t k0, uint32_t k1,
           uint32_t rankfield, uint32_t step, double* __restrict__ partial) {
  __shared__ double red[QP_WARPS][KT];
  const ProfChunk ch = chunks[blockIdx.x];
  const DevLayer ly = layers[ch.layer];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool fast_layer = ((ly.offset & 3) == 0) && B == 128;
  const int M = B >> 7;
  const float my_s = (lane < K) ? cs.s[lane] : 1.f;
  double acc[KT];
#pragma unroll
  for (int j = 0; j < KT; ++j) acc[j] = 0.0;

  int bi = warp;
  if (fast_layer) {
    // ---- fast path: full aligned buckets of 128; lane group grp (8 lanes) owns one
    //      bucket, lane l8 holds elements 32i + 4*l8 + s (i, s < 4) = Philox counter
    //      gb*32 + 8i + l8, words s (R3).  Per-candidate inv/unit computed by lane j of
    //      the group and kept in registers for the bucket's 16 elements.
    const int grp = lane >> 3, l8 = lane & 7;
    const float gs = (l8 < K) ? cs.s[l8] : 1.f;
    const float gs2 = (KT > 8 && l8 + 8 < K) ? cs.s[(l8 + 8) & 15] : 1.f;
    const int64_t nfull = min((int64_t)ch.nbk, ly.numel / 128 - ch.first);
    for (int b0 = warp * 4; b0 < nfull; b0 += QP_WARPS * 4) {
      const int bq = b0 + grp;
      const bool valid = bq < nfull;
      const int64_t jb = ch.first + (valid ? bq : b0);
      const int64_t base = ly.offset + jb * 128 + 4 * l8;
      float x[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 a = ld4(g + base + 32 * i);
        if (e) {
          const float4 c = ld4(e + base + 32 * i);
          x[4 * i] = __fadd_rn(a.x, c.x); x[4 * i + 1] = __fadd_rn(a.y, c.y);
          x[4 * i + 2] = __fadd_rn(a.z, c.z); x[4 * i + 3] = __fadd_rn(a.w, c.w);
        } else {
          x[4 * i] = a.x; x[4 * i + 1] = a.y; x[4 * i + 2] = a.z; x[4 * i + 3] = a.w;
        }
      }
      // (the +0 of canon() only turns -0 into +0, which changes no error: omitted here)
      float mn = fmin_nan(x[0], x[1]), mx = fmax_nan(x[0], x[1]);
#pragma unroll
      for (int s = 2; s < 16; ++s) { mn = fmin_nan(mn, x[s]); mx = fmax_nan(mx, x[s]); }
#pragma unroll
      for (int o = 4; o; o >>= 1) {
        mn = fmin_nan(mn, __shfl_xor_sync(LG_FULL, mn, o));
        mx = fmax_nan(mx, __shfl_xor_sync(LG_FULL, mx, o));
      }
      float my_inv, my_unit, my_inv2 = 0.f, my_unit2 = 0.f;
      qparams(mn, mx, gs, my_inv, my_unit);
      if (KT > 8) qparams(mn, mx, gs2, my_inv2, my_unit2);
      float inv[KT], unit[KT];
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        inv[j] = __shfl_sync(LG_FULL, j < 8 ? my_inv : my_inv2, (lane & ~7) + (j & 7));
        unit[j] = __shfl_sync(LG_FULL, j < 8 ? my_unit : my_unit2, (lane & ~7) + (j & 7));
      }
      const uint32_t c0 = (uint32_t)((ly.bucket0 + jb) * 32 + l8);
      float S;
      double S2inv;
      const bool small = bucket_scale(mn, mx, S, S2inv);
      float a2[KT];
#if QP_F32X2
      const PhiloxRK rk = philox_rk(k0, k1);
      if (__any_sync(LG_FULL, small)) prof_cand16x2<KT, true>(x, mn, c0, rankfield, step, rk, inv, unit, cs, S, a2);
      else prof_cand16x2<KT, false>(x, mn, c0, rankfield, step, rk, inv, unit, cs, 1.f, a2);
#else
      if (__any_sync(LG_FULL, small)) prof_cand16<KT, true>(x, mn, c0, rankfield, step, k0, k1, inv, unit, cs, S, a2);
      else prof_cand16<KT, false>(x, mn, c0, rankfield, step, k0, k1, inv, unit, cs, 1.f, a2);
#endif
      if (valid) {
#pragma unroll
        for (int j = 0; j < KT; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn((double)a2[j], S2inv));
      }
    }
    // ragged last bucket of the layer (if in this chunk): the generic path, warp 0
    bi = (nfull < ch.nbk && warp == 0) ? (int)nfull : ch.nbk;
  }
  for (; bi < ch.nbk; bi += QP_WARPS) {
    const int64_t jb = ch.first + bi;
    const int64_t gb = ly.bucket0 + jb;
    const int64_t e0 = jb * (int64_t)B;
    {
      // ---- generic path: ragged / misaligned / B > 128
      const bool aligned = (ly.offset & 3) == 0;
      float mn = INFINITY, mx = -INFINITY;
      X4 xs;
      for (int t = 0; t < M; ++t) {
        const int64_t i0 = e0 + 128 * t + 4 * lane;
        const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
        xs = load_x4(g, e, ly.offset + i0, nv, aligned);
#pragma unroll
        for (int s = 0; s < 4; ++s)
          if (s < nv) { mn = fmin_nan(mn, xs.v[s]); mx = fmax_nan(mx, xs.v[s]); }
      }
      warp_minmax_nan(mn, mx);
      float my_inv, my_unit;
      qparams(mn, mx, my_s, my_inv, my_unit);
      float S;
      double S2inv;
      bucket_scale(mn, mx, S, S2inv);
      float a2[KT];
#pragma unroll
      for (int j = 0; j < KT; ++j) a2[j] = 0.f;
      for (int t = 0; t < M; ++t) {
        const int64_t i0 = e0 + 128 * t + 4 * lane;
        const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
        if (M > 1) xs = load_x4(g, e, ly.offset + i0, nv, aligned);
        float u[4], x[4];
        uniforms4((uint32_t)(gb * (B >> 2) + 32 * t + lane), rankfield, step, 0u, k0, k1, u);
#pragma unroll
        for (int s = 0; s < 4; ++s) x[s] = (s < nv) ? xs.v[s] : mn;  // invalid -> d = 0
        prof_candidates<KT>(x, mn, u, my_inv, my_unit, cs, K, S, a2);
      }
#pragma unroll
      for (int j = 0; j < KT; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn((double)a2[j], S2inv));
    }
  }
  // ---- deterministic block reduction (fp64)
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    if (j < K) {
      const double v = warp_sum_d(acc[j]);
      if (lane == 0) red[warp][j] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < QP_WARPS; ++w) s += red[w][threadIdx.x];
    partial[(int64_t)blockIdx.x * K + threadIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// K1 (B = 128): persistent warps over chunks of <= 32 buckets of one layer, handed
// out dynamically (one global ticket counter; a warp holds its next chunk while
// computing the current one).  A chunk is walked in "quads" of 4 consecutive buckets
// (one per 8-lane group), staged into shared memory by the bulk-copy engine
// (cp.async.bulk, TMA 1-D) with an mbarrier per stage: while a warp computes quad q,
// the next quad (of this chunk or of its next chunk) is in flight.  Each chunk's fp64
// SSE goes to its own partial slot, so K1b's fixed-order per-layer sum is
// deterministic whatever warp took the chunk.  Dynamic hand-out balances the warps of
// an SM (the issue arbiter favours high warp ids, so static equal ranges leave a
// tail of low-id warps).  Quads of misaligned layers or with a ragged bucket are
// loaded directly (masked).  The last warp to finish resets the counter, so the
// launch is stream- and graph-replay safe.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t sm_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "QW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra QW_%=;\n\t}\n" ::"r"(sm_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bar_expect_tx_a(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait_a(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "QWA_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra QWA_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_a(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sm_addr(dst)),
               "l"(src), "r"(bytes), "r"(sm_addr(bar))
               : "memory");
}

#ifndef QK_UNROLL
#define QK_UNROLL 4  // K5 fast path: buckets per warp iteration (loads in flight)
#endif
constexpr int QP_NPART = 16;  // K1 ticket counters (parts of the quad range), 256 B apart
constexpr int QR_ROWS = 256;  // K1b segment: rows of one layer reduced by one fixed tree
#ifndef Q1_WARPS
#define Q1_WARPS 8  // warps per CTA of the K1 fast kernel (each double-buffers 4 KB quads: 8 KB of shared memory)
#endif
#ifndef Q1_STAGES
#define Q1_STAGES 2  // quad buffers per warp (1: the next quad is fetched once the current one is in registers)
#endif
#ifndef Q1_MINB
#define Q1_MINB 3   // resident CTAs per SM of the K1 fast kernel (register budget 65536 / (32 Q1_WARPS Q1_MINB))
#endif
constexpr int Q1_THREADS = 32 * Q1_WARPS;
#ifndef Q1F_MINB
#define Q1F_MINB 2  // resident CTAs per SM of the fused profile + compress kernel (128 registers, no spills: A/B 112.9 -> 86.4 us at 3 CTAs / 80 registers)
#endif
// Stage-1 destination of the payload byte at flat offset b: the local payload, or (peer
// exchange) the owner's receive window, slot `me` (owner o's window holds W slots of its
// shard size, R13) -- records never straddle a shard bound.
__device__ __forceinline__ uint8_t* stage1_dst(uint8_t* payload, const P2PDev* __restrict__ p2p, int64_t b) {
  if (!p2p) return payload + b;
  int o = 0;
  while (o + 1 < p2p->W && b >= p2p->bb[o + 1]) ++o;
  return p2p->recv[o] + (int64_t)p2p->me * (p2p->bb[o + 1] - p2p->bb[o]) + (b - p2p->bb[o]);
}

template <int KT, int FUSE>
__global__ void __launch_bounds__(Q1_THREADS, FUSE ? Q1F_MINB : Q1_MINB)
k_qprofile_q(const float* __restrict__ g, const float* e, const QInfo* __restrict__ qinfo, int nqc,
             unsigned* __restrict__ ticket, const CandS cs, int K, const PhiloxRK rk, uint32_t rankfield,
             uint32_t step, int ptr_aligned, double* __restrict__ partial, const QFuse fz) {
  extern __shared__ __align__(128) unsigned char qsm[];
  __shared__ __align__(8) uint64_t bars[Q1_WARPS][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane >> 3, l8 = lane & 7;
  // stage b of this warp: g at qsm + (2 warp + b) 4096 bytes, e 2048 bytes after it
  auto stage_g = [&](int b) { return reinterpret_cast<float*>(qsm + (size_t)(warp * Q1_STAGES + b) * 4096); };
  // Work hand-out: the quads are split into QP_NPART contiguous parts, each with its own
  // ticket counter (one hot address would serialise ~50K atomics in one L2 slice);
  // a warp starts on part (global warp id mod QP_NPART) and moves on when its part is
  // exhausted.  Grabs are split: lane 0 issues the atomic, the broadcast (which waits
  // for it) happens one quad later, so the atomic's latency hides behind a quad.
  const int gw = blockIdx.x * Q1_WARPS + warp;
  int part = gw % QP_NPART;
  auto plo = [&](int p) -> int { return (int)(((int64_t)nqc * p) / QP_NPART); };
  auto grab_issue = [&]() -> unsigned {
    unsigned v = 0;
    if (lane == 0) v = atomicAdd(&ticket[part * 64], 1u);
    return v;
  };
  auto resolve = [&](unsigned v) -> int {
    int q = plo(part) + (int)__shfl_sync(LG_FULL, v, 0);
    while (q >= plo(part + 1)) {
      // part exhausted: lanes 0..15 read the 16 counters at once (one L2 round trip
      // instead of one synchronous atomic per part) and the warp moves to the next part
      // in rotation order that still has quads; none left -> done
      bool left = false;
      if (lane < QP_NPART) left = plo(lane) + (int)__ldcg(&ticket[lane * 64]) < plo(lane + 1);
      const unsigned m = __ballot_sync(LG_FULL, left) & ((1u << QP_NPART) - 1u);
      if (!m) return nqc;
      const unsigned rot = ((m >> (part + 1)) | (m << (QP_NPART - 1 - part))) & ((1u << QP_NPART) - 1u);
      part = (part + __ffs(rot)) % QP_NPART;
      q = plo(part) + (int)__shfl_sync(LG_FULL, grab_issue(), 0);
    }
    return q;
  };
  auto finish = [&]() {  // after this warp found every part exhausted
#if Q1_TRIGGER
    pdl_trigger();  // K1b may be scheduled now (it still waits for this grid's completion)
#endif
    if (lane == 0 && atomicAdd(&ticket[QT_ARR * 64], 1u) == gridDim.x * Q1_WARPS - 1u) {
      for (int p2 = 0; p2 <= QT_ARR; ++p2) atomicExch(&ticket[p2 * 64], 0u);
    }
  };
  // Quad descriptors travel through a 3-slot shared ring per warp (c, nA, nB), filled by
  // lane 0 with cp.async (one commit group per descriptor), so no register holds a
  // descriptor load in flight across the compute (that pushed K1 past its register
  // budget: a spill store that waited on the load every quad).
  __shared__ __align__(16) QInfo qis[Q1_WARPS][3];
  auto info_async = [&](int ci, int slot) {
    if (lane == 0) {
      if (ci < nqc)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sm_addr(&qis[warp][slot])), "l"(qinfo + ci)
                     : "memory");
      else
        qis[warp][slot] = QInfo{0, 0u, 0};
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };
  auto info_wait1 = [&]() {  // all but the newest descriptor landed
    if (lane == 0) asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
  };
  // g / e (and the ticket reset) of the preceding kernels; the fused kernel launched
  // concurrently with a solve it does not read (LGRECO_PC_CONCURRENT) skips the wait
  if (!(FUSE && fz.nowait)) pdl_wait();
  float bad = 0.f;  // FUSE: NaN once a non-finite input was seen (K5's rule)
  // FUSE: the plan staged in shared memory (int8; 127 = outside [-2, K): flagged below)
  __shared__ int8_t s_ch[FUSE ? QF_LCACHE : 1];
  if constexpr (FUSE) {
    const int nc = min(fz.L, QF_LCACHE);
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      const int v = __ldg(fz.choice + i);
      s_ch[i] = (int8_t)((v >= LGRECO_CHOICE_SKIP && v < K) ? v : 127);
    }
    __syncthreads();
  }
  if constexpr (FUSE) {
    // the lossless layers (few, small): x copied to the output, EF zeroed (K5's raw path)
    for (int rc = gw; rc < fz.nraw; rc += gridDim.x * Q1_WARPS) {
      const ProfChunk ch = fz.raw[rc];
      if (__ldg(fz.choice + ch.layer) == LGRECO_CHOICE_SKIP) continue;
      const DevLayer ly = fz.layers[ch.layer];
      const int64_t i_beg = ch.first * (int64_t)fz.B;
      const int64_t i_end = min(ly.numel, (ch.first + ch.nbk) * (int64_t)fz.B);
      for (int64_t i = i_beg + lane; i < i_end; i += 32) {
        const float xv = canon(__ldg(g + ly.offset + i), e ? e[ly.offset + i] : 0.f);
        bad = __fadd_rn(bad, __fmul_rn(xv, 0.f));
        if (FUSE == 1) fz.out[ly.offset + i] = xv;
        else *reinterpret_cast<float*>(stage1_dst(nullptr, fz.p2p, fz.plan[ch.layer].pay_off + 4 * i)) = xv;  // raw record
        if (fz.ef) fz.ef[ly.offset + i] = 0.f;
      }
    }
  }
  auto fin_flag = [&]() {
    if constexpr (FUSE) {
      if (!isfinite(bad)) atomicOr(fz.flag, 1u);
    }
  };
  int c = resolve(grab_issue());
  if (c >= nqc) { fin_flag(); finish(); return; }
  if (lane == 0) {
    bar_init(&bars[warp][0], 1);
    bar_init(&bars[warp][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const bool pal = ptr_aligned != 0;
  const uint32_t tx = e ? 4096u : 2048u;
  const uint32_t a_bar = sm_addr(&bars[warp][0]);                      // stage b: + 8 b
  const uint32_t a_stage = sm_addr(qsm + (size_t)warp * Q1_STAGES * 4096);  // stage b: + 4096 b
  float gs = 1.f, gs2 = 1.f;  // s of candidates l8 and l8 + 8 (select chain: no local copy of cs)
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    if (j < K && j == l8) gs = cs.s[j];
    if (j < K && j == l8 + 8) gs2 = cs.s[j];
  }
  // bulk copies of quad `in` into stage b (lane 0) when regular: aligned, 4 full buckets
  auto issue = [&](const QInfo& in, int b) -> bool {
    if (!(pal && (in.elem0 & 3) == 0 && qi_nvalid(in) == 512)) return false;
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of the stage
      bar_expect_tx_a(a_bar + 8 * b, tx);
      bulk_g2s_a(a_stage + 4096 * b, g + in.elem0, 2048u, a_bar + 8 * b);
      if (e) bulk_g2s_a(a_stage + 4096 * b + 2048, e + in.elem0, 2048u, a_bar + 8 * b);
    }
    return true;
  };
  // queue: c (computing), nA (its quad prefetched during c), nB (info load in flight)
  int nA = resolve(grab_issue());
  bool failed = nA >= nqc;
  int nB = nqc;
  if (!failed) { nB = resolve(grab_issue()); failed = nB >= nqc; }
  int r = 0;  // ring slot of c; nA at r+1, nB at r+2 (mod 3)
  info_async(c, 0);
  info_async(nA, 1);
  info_async(nB, 2);
  if (lane == 0) asm volatile("cp.async.wait_group 2;" ::: "memory");
  __syncwarp();
  QInfo ic = qis[warp][0];
  uint32_t phase = 0u;  // bit b: parity of stage b's next completion
  int b = 0;
  bool inflight = issue(ic, 0);
  double acc[KT];
#pragma unroll
  for (int j = 0; j < KT; ++j) acc[j] = 0.0;

  for (;;) {
    unsigned raw = 0;
    const bool pend = !failed;
    if (pend) raw = grab_issue();
    {
      const bool cur_regular = inflight;
      // prefetch quad nA into the other stage (its previous contents were consumed in
      // the previous iteration; __syncwarp orders those reads before the copy)
      info_wait1();  // nA's descriptor (and c's) landed; also orders the stage reads
      const int ra = (r == 2) ? 0 : r + 1;
      // two stages: prefetch quad nA into the other stage now; one stage: after the
      // current quad has been read into registers (below)
      bool next_inflight = (Q1_STAGES == 2 && nA < nqc) ? issue(qis[warp][ra], b ^ 1) : false;
      const int nvalid = qi_nvalid(ic);
      const bool valid = grp * 128 < nvalid;
      int jc = 0;  // FUSE: the layer's planned candidate
      if constexpr (FUSE) {
        const int lay = qi_layer(ic);
        jc = lay < QF_LCACHE ? (int)s_ch[lay] : __ldg(fz.choice + lay);
      }
      float x[16];
      if (cur_regular) {
        bar_wait_a(a_bar + 8 * b, (phase >> b) & 1u);
        phase ^= 1u << b;
        const float* sg = stage_g(b) + grp * 128 + 4 * l8;
        const float* se = sg + 512;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 a = *reinterpret_cast<const float4*>(sg + 32 * i);
          if (e) {
            const float4 f = *reinterpret_cast<const float4*>(se + 32 * i);
            f2_t x01 = f2add(f2pk(a.x, a.y), f2pk(f.x, f.y)), x23 = f2add(f2pk(a.z, a.w), f2pk(f.z, f.w));
            if (FUSE) { x01 = f2add(x01, f2pk(0.f, 0.f)); x23 = f2add(x23, f2pk(0.f, 0.f)); }  // canon (R2): e' = x - dec
            f2up(x01, x[4 * i], x[4 * i + 1]);
            f2up(x23, x[4 * i + 2], x[4 * i + 3]);
          } else if (FUSE) {
            f2up(f2add(f2pk(a.x, a.y), f2pk(0.f, 0.f)), x[4 * i], x[4 * i + 1]);
            f2up(f2add(f2pk(a.z, a.w), f2pk(0.f, 0.f)), x[4 * i + 2], x[4 * i + 3]);
          } else {
            x[4 * i] = a.x; x[4 * i + 1] = a.y; x[4 * i + 2] = a.z; x[4 * i + 3] = a.w;
          }
        }
      } else {
        // masked direct loads: element 32i + 4*l8 + s of bucket grp of the quad
        // (offsets against lim = nvalid - lane base: immediate compares, nothing to hoist
        // into the regular quads' path)
        const int lim = nvalid - (grp * 128 + 4 * l8);
        const float* gl = g + ic.elem0 + grp * 128 + 4 * l8;
        const float* el = e ? e + ic.elem0 + grp * 128 + 4 * l8 : nullptr;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2) {
            const bool ok = 32 * i + s2 < lim;
            float v = 0.f;
            if (ok) {
              v = __ldg(gl + 32 * i + s2);
              if (el) v = __fadd_rn(v, FUSE ? el[32 * i + s2] : __ldg(el + 32 * i + s2));
              if (FUSE) v = __fadd_rn(v, 0.f);
            }
            x[4 * i + s2] = v;
          }
        }
      }
      if (Q1_STAGES == 1 && nA < nqc) {  // the stage's contents are in registers now
        __syncwarp();
        next_inflight = issue(qis[warp][ra], 0);
      }
      // (the +0 of canon() only turns -0 into +0, which changes no error: omitted here)
      float mn, mx;
      if (cur_regular) {
        mn = fmin_nan(x[0], x[1]); mx = fmax_nan(x[0], x[1]);
#pragma unroll
        for (int s2 = 2; s2 < 16; s2 += 2) { mn = fmin3_nan(mn, x[s2], x[s2 + 1]); mx = fmax3_nan(mx, x[s2], x[s2 + 1]); }
      } else {
        mn = INFINITY; mx = -INFINITY;
        const int lim = nvalid - (grp * 128 + 4 * l8);
#pragma unroll
        for (int s2 = 0; s2 < 16; ++s2) {
          if (32 * (s2 >> 2) + (s2 & 3) < lim) { mn = fmin_nan(mn, x[s2]); mx = fmax_nan(mx, x[s2]); }
        }
      }
#pragma unroll
      for (int o = 4; o; o >>= 1) {
        mn = fmin_nan(mn, __shfl_xor_sync(LG_FULL, mn, o));
        mx = fmax_nan(mx, __shfl_xor_sync(LG_FULL, mx, o));
      }
      if (!cur_regular) {
        const int lim = nvalid - (grp * 128 + 4 * l8);
#pragma unroll
        for (int s2 = 0; s2 < 16; ++s2) {
          if (!(32 * (s2 >> 2) + (s2 & 3) < lim)) x[s2] = mn;  // invalid -> t = 0, q = 0, d = 0
        }
      }
      float my_inv, my_unit, my_inv2 = 0.f, my_unit2 = 0.f;
      qparams(mn, mx, gs, my_inv, my_unit);
      if (KT > 8) qparams(mn, mx, gs2, my_inv2, my_unit2);
      float inv[KT], unit[KT];
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        inv[j] = __shfl_sync(LG_FULL, j < 8 ? my_inv : my_inv2, (lane & ~7) + (j & 7));
        unit[j] = __shfl_sync(LG_FULL, j < 8 ? my_unit : my_unit2, (lane & ~7) + (j & 7));
      }
      const uint32_t c0 = (ic.gb0 + (uint32_t)grp) * 32u + (uint32_t)l8;
      float S;
      double S2inv;
      const bool small = bucket_scale(mn, mx, S, S2inv);
      float a2[KT];
      if constexpr (FUSE) {
        FuseW fw;
        bool wr = valid && jc != LGRECO_CHOICE_SKIP;
        if (jc != LGRECO_CHOICE_SKIP && (jc < 0 || jc >= K)) {
          if (lane == 0) atomicOr(fz.flag, 2u);
          jc = 0;
        }
        if (!wr) jc = 0;
        const int src = (lane & ~7) + (jc & 7);
        fw.invc = __shfl_sync(LG_FULL, jc < 8 ? my_inv : my_inv2, src);
        fw.unitc = __shfl_sync(LG_FULL, jc < 8 ? my_unit : my_unit2, src);
        fw.ebase = ic.elem0 + grp * 128 + 4 * l8;
        fw.lim = nvalid - (grp * 128 + 4 * l8);
        fw.vec = cur_regular;
        fw.wr = wr;
        if (valid) bad = __fadd_rn(bad, __fmul_rn(__fsub_rn(mx, mn), 0.f));
        uint32_t codes[4] = {0u, 0u, 0u, 0u};
        if (__any_sync(LG_FULL, small))
          prof_cand16x2<KT, true, FUSE>(x, mn, c0, rankfield, step, rk, inv, unit, cs, S, a2, fw, fz.out, fz.ef, codes);
        else
          prof_cand16x2<KT, false, FUSE>(x, mn, c0, rankfield, step, rk, inv, unit, cs, 1.f, a2, fw, fz.out, fz.ef,
                                         codes);
        if constexpr (FUSE == 2) {
          // W > 1: the stage-1 record of bucket grp (R7) straight into its owner's window.
          // Word (p, s) holds bit p of the code of element 4l + s in bit l = 8i + l8 (lane
          // (grp, l8), sub-block i): four warp ballots per (p, s), byte grp of each.
          if (__any_sync(LG_FULL, wr)) {
            const int lay = qi_layer(ic);
            const DevPlan pl = fz.plan[lay];
            const int64_t jb = (ic.elem0 - fz.layers[lay].offset) / 128 + grp;
            uint32_t* rec = reinterpret_cast<uint32_t*>(
                stage1_dst(nullptr, fz.p2p, pl.pay_off + jb * (int64_t)pl.rec_bytes));
            const uint32_t sel = (uint32_t)grp | ((4u + (uint32_t)grp) << 4);
            for (int p = 0; p < pl.bits; ++p) {
#pragma unroll
              for (int s2 = 0; s2 < 4; ++s2) {
                const int sh = 8 * s2 + p;
                const uint32_t b0 = __ballot_sync(LG_FULL, (codes[0] >> sh) & 1u);
                const uint32_t b1 = __ballot_sync(LG_FULL, (codes[1] >> sh) & 1u);
                const uint32_t b2 = __ballot_sync(LG_FULL, (codes[2] >> sh) & 1u);
                const uint32_t b3 = __ballot_sync(LG_FULL, (codes[3] >> sh) & 1u);
                const uint32_t word = __byte_perm(__byte_perm(b0, b1, sel), __byte_perm(b2, b3, sel), 0x5410);
                if (wr && l8 == ((4 * p + s2) & 7)) rec[4 * p + s2] = word;
              }
            }
            if (wr && l8 == 0) *reinterpret_cast<float2*>(rec + 4 * pl.bits) = make_float2(mn, fw.unitc);
          }
        }
      } else {
#if QP_F32X2
      if (__any_sync(LG_FULL, small)) prof_cand16x2<KT, true>(x, mn, c0, rankfield, step, rk, inv, unit, cs, S, a2);
      else prof_cand16x2<KT, false>(x, mn, c0, rankfield, step, rk, inv, unit, cs, 1.f, a2);
#else
      if (__any_sync(LG_FULL, small)) prof_cand16<KT, true>(x, mn, c0, rankfield, step, k0, k1, inv, unit, cs, S, a2);
      else prof_cand16<KT, false>(x, mn, c0, rankfield, step, k0, k1, inv, unit, cs, 1.f, a2);
#endif
      }
      if (KT <= 8) {
        // quad row, fixed order: transpose-reduce the 8 lanes of each bucket in fp32
        // (after the xor-4/2/1 halvings lane l8 holds candidate l8's bucket SSE, from
        // 128 fp32 squares), then x 2^-2k and the 4 buckets in fp64 (xor 8, 16)
        float v8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v8[j] = (j < KT) ? a2[j] : 0.f;
#pragma unroll
        for (int h = 4; h >= 1; h >>= 1) {
          const bool up = (lane & h) != 0;
#pragma unroll
          for (int i = 0; i < h; ++i) {
            const float send = up ? v8[i] : v8[i + h];
            const float keep = up ? v8[i + h] : v8[i];
            v8[i] = __fadd_rn(keep, __shfl_xor_sync(LG_FULL, send, h));
          }
        }
        double t = valid ? __dmul_rn((double)v8[0], S2inv) : 0.0;
        t = __dadd_rn(t, __shfl_xor_sync(LG_FULL, t, 8));
        t = __dadd_rn(t, __shfl_xor_sync(LG_FULL, t, 16));
        if (lane < K) partial[(int64_t)c * K + lane] = t;
      } else if (valid) {
#pragma unroll
        for (int j = 0; j < KT; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn((double)a2[j], S2inv));
      }
      inflight = next_inflight;
      if (Q1_STAGES == 2) b ^= 1;
    }
    // chunk done (KT > 8): fixed-order warp reduction into its slot
    if (KT > 8) {
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        if (j < K) {
          const double v = warp_sum_d(acc[j]);
          if (lane == 0) partial[(int64_t)c * K + j] = v;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < KT; ++j) acc[j] = 0.0;
    if (nA >= nqc) break;
    c = nA;
    nA = nB;
    const int r_old = r;  // c's slot, read (ic) before the shuffles above: free
    r = (r == 2) ? 0 : r + 1;
    ic = qis[warp][r];    // landed: waited for at the top of this iteration
    if (pend) { nB = resolve(raw); failed = nB >= nqc; }
    else nB = nqc;
    info_async(nB, r_old);
  }
  fin_flag();
  finish();
}

// K1b: per layer, fixed-order sum of its quads' partial rows, sqrt.  One CTA per segment
// of <= QR_ROWS rows of one layer (layers without rows get one empty segment): thread t
// loads row seg0 + t (K contiguous doubles), a fixed shared-memory tree per candidate
// gives the segment sum; the layer's last segment to finish (counter per layer, reset
// by that CTA) adds the segment sums in segment order and writes err/bits.
__global__ void __launch_bounds__(QR_ROWS)
k_qprofile_reduce(const DevLayer* __restrict__ layers, const QSeg* __restrict__ segs, const int32_t* __restrict__ lseg0,
                  const double* __restrict__ partial, double* __restrict__ segsum, unsigned* __restrict__ ldone,
                  const int32_t* __restrict__ params, int K, int B, double* __restrict__ err, int64_t* __restrict__ bits) {
  __shared__ double sm[16][QR_ROWS / 32];
  __shared__ bool s_last;
  pdl_wait();  // K1's partial rows
  const QSeg sg = segs[blockIdx.x];
  const int l = sg.layer, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const DevLayer ly = layers[l];
  const double* row = partial + (int64_t)(sg.row0 + t) * K;
  double v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = (j < K && t < sg.nrows) ? __ldg(row + j) : 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < K) {
      const double w = warp_sum_d(v[j]);  // fixed xor tree
      if (lane == 0) sm[j][warp] = w;
    }
  }
  __syncthreads();
  if (t < K) {
    double s2 = 0.0;
#pragma unroll
    for (int w = 0; w < QR_ROWS / 32; ++w) s2 += sm[t][w];
    segsum[(int64_t)blockIdx.x * K + t] = s2;
  }
  __syncthreads();
  if (t == 0) {
    __threadfence();
    const int s0 = lseg0[l], s1 = lseg0[l + 1];
    s_last = atomicAdd(&ldone[l], 1u) == (unsigned)(s1 - s0 - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int s0 = lseg0[l], s1 = lseg0[l + 1];
  const int64_t nb = (ly.numel + B - 1) / B;
  // the layer's segment sums in segment order: staged a chunk at a time (one L2 round
  // trip for up to QR_ROWS / K segments, the rows of consecutive segments being
  // contiguous) and added in order from shared memory
  __shared__ double sbuf[QR_ROWS];
  const int chunk = QR_ROWS / K;
  double s = 0.0;
  for (int q0 = s0; q0 < s1; q0 += chunk) {
    const int nq = min(chunk, s1 - q0);
    if (t < nq * K) sbuf[t] = __ldcg(segsum + (int64_t)q0 * K + t);
    __syncthreads();
    if (t < K)
      for (int i = 0; i < nq; ++i) s += sbuf[i * K + t];
    __syncthreads();
  }
  if (t < K) {
    if (ly.compress) {
      err[(int64_t)l * K + t] = sqrt(s);
      bits[(int64_t)l * K + t] = nb * ((int64_t)B * params[t] + 64);
    } else {
      err[(int64_t)l * K + t] = 0.0;
      bits[(int64_t)l * K + t] = 32 * ly.numel;
    }
  }
  if (t == 0) ldone[l] = 0u;  // stream-ordered reuse by the next launch
}

// Per-layer reduction of the B > 128 kernel's chunk partials (k_qprofile).
__global__ void __launch_bounds__(256)
k_qprofile_reduce_chunks(const DevLayer* __restrict__ layers, const int32_t* __restrict__ layer_chunk0,
                         const double* __restrict__ partial, const int32_t* __restrict__ params, int K, int B,
                         double* __restrict__ err, int64_t* __restrict__ bits) {
  __shared__ double sm[256];
  const int l = blockIdx.x;
  const DevLayer ly = layers[l];
  const int c0 = layer_chunk0[l], c1 = layer_chunk0[l + 1];
  const int64_t nb = (ly.numel + B - 1) / B;
  for (int j = 0; j < K; ++j) {
    double s = 0.0;
    for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) s += partial[(int64_t)c * K + j];
    sm[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
      if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      if (ly.compress) {
        err[(int64_t)l * K + j] = sqrt(sm[0]);
        bits[(int64_t)l * K + j] = nb * ((int64_t)B * params[j] + 64);
      } else {
        err[(int64_t)l * K + j] = 0.0;
        bits[(int64_t)l * K + j] = 32 * ly.numel;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// bit-plane packing / unpacking (R7)
// ---------------------------------------------------------------------------
// Codes q[4] of sub-block t: word (t*b+p)*4+s gets bit p of code(128t+4l+s) in bit l.
__device__ __forceinline__ void pack_planes(uint32_t* __restrict__ words, int t, int b, const uint32_t* q,
                                            int lane) {
  for (int p = 0; p < b; ++p) {
    const uint32_t w0 = __ballot_sync(LG_FULL, (q[0] >> p) & 1u);
    const uint32_t w1 = __ballot_sync(LG_FULL, (q[1] >> p) & 1u);
    const uint32_t w2 = __ballot_sync(LG_FULL, (q[2] >> p) & 1u);
    const uint32_t w3 = __ballot_sync(LG_FULL, (q[3] >> p) & 1u);
    if (lane == 0) {
      uint2* dst = reinterpret_cast<uint2*>(words + (t * b + p) * 4);
      dst[0] = make_uint2(w0, w1);
      dst[1] = make_uint2(w2, w3);
    }
  }
}

// Decode sub-block t of a record with b bits -> dec[4] of this lane.
__device__ __forceinline__ void decode_sub(const uint8_t* __restrict__ rec, int t, int b, int M, int lane,
                                           float* dec) {
  const uint32_t* words = reinterpret_cast<const uint32_t*>(rec);
  const float2 mu = __ldg(reinterpret_cast<const float2*>(rec + 16 * b * M));
  uint32_t q0 = 0, q1 = 0, q2 = 0, q3 = 0;
  for (int p = 0; p < b; ++p) {
    const uint2 a = __ldg(reinterpret_cast<const uint2*>(words + (t * b + p) * 4));
    const uint2 c = __ldg(reinterpret_cast<const uint2*>(words + (t * b + p) * 4 + 2));
    q0 |= ((a.x >> lane) & 1u) << p;
    q1 |= ((a.y >> lane) & 1u) << p;
    q2 |= ((c.x >> lane) & 1u) << p;
    q3 |= ((c.y >> lane) & 1u) << p;
  }
  dec[0] = __fmaf_rn((float)q0, mu.y, mu.x);
  dec[1] = __fmaf_rn((float)q1, mu.y, mu.x);
  dec[2] = __fmaf_rn((float)q2, mu.y, mu.x);
  dec[3] = __fmaf_rn((float)q3, mu.y, mu.x);
}

// ---------------------------------------------------------------------------
// K5 stage-1 pack + EF (+ fused decode for W == 1)
// ---------------------------------------------------------------------------
// Quantise/pack/EF of one full aligned bucket (fast path); returns NaN-flag input.
__device__ __forceinline__ void pack_bucket_fast(const X4& xs, int b, int64_t gb, uint32_t rankfield,
                                                 uint32_t step, uint32_t k0, uint32_t k1, int lane,
                                                 uint8_t* __restrict__ rec, float* __restrict__ ef,
                                                 float* __restrict__ dec_out, int64_t base, float& bad) {
  const float s_b = (float)((1u << b) - 1u);
  float mn = fmin_nan(fmin_nan(xs.v[0], xs.v[1]), fmin_nan(xs.v[2], xs.v[3]));
  float mx = fmax_nan(fmax_nan(xs.v[0], xs.v[1]), fmax_nan(xs.v[2], xs.v[3]));
  warp_minmax_nan(mn, mx);
  float inv, unit;
  qparams(mn, mx, s_b, inv, unit);
  bad = __fadd_rn(bad, __fmul_rn(__fsub_rn(mx, mn), 0.f));  // NaN / inf range -> NaN
  float u[4];
  uniforms4((uint32_t)(gb * 32 + lane), rankfield, step, 0u, k0, k1, u);
  uint32_t q[4];
  float dec[4], en[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const float qf = qcode(__fsub_rn(xs.v[s], mn), inv, u[s], s_b);
    q[s] = (uint32_t)qf;
    dec[s] = __fmaf_rn(qf, unit, mn);
    en[s] = __fsub_rn(xs.v[s], dec[s]);
  }
  if (rec) {
    pack_planes(reinterpret_cast<uint32_t*>(rec), 0, b, q, lane);
    if (lane == 0) *reinterpret_cast<float2*>(rec + 16 * b) = make_float2(mn, unit);
  }
  if (ef) *reinterpret_cast<float4*>(ef + base) = make_float4(en[0], en[1], en[2], en[3]);
  if (dec_out) *reinterpret_cast<float4*>(dec_out + base) = make_float4(dec[0], dec[1], dec[2], dec[3]);
}


__global__ void __launch_bounds__(QP_THREADS)
k_qpack(const float* __restrict__ g, float* __restrict__ ef, uint8_t* __restrict__ payload,
        float* __restrict__ dec_out, const DevLayer* __restrict__ layers, const DevPlan* __restrict__ plan,
        const ProfChunk* __restrict__ chunks, int B, uint32_t k0, uint32_t k1, uint32_t rankfield,
        uint32_t step, unsigned* __restrict__ flag, const P2PDev* __restrict__ p2p,
        const int32_t* __restrict__ choice, const int32_t* __restrict__ params, int K, int l2pf) {
  const ProfChunk ch = chunks[blockIdx.x];  // (ctx tables: written at ctx creation)
  const DevLayer ly = layers[ch.layer];
  if (l2pf && threadIdx.x == 0) {
    // CTAs scheduled while the solve still runs (it triggers its dependents early) pull
    // their chunk of g and EF into L2 before waiting for the plan: HBM is idle during the
    // solve.  A prefetch is a hint with no visibility effect (L2 is the coherence point).
    const int64_t i0 = ly.offset + ch.first * (int64_t)B;
    const int64_t i1 = ly.offset + min(ly.numel, (ch.first + ch.nbk) * (int64_t)B);
    const int64_t a0 = (i0 + 3) & ~(int64_t)3, nb = ((i1 - a0) * 4) & ~(int64_t)15;
    if (nb >= 16 && (((uintptr_t)(g + a0) | (uintptr_t)(ef ? ef + a0 : g)) & 15) == 0) {
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g + a0), "r"((uint32_t)nb) : "memory");
      if (ef) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ef + a0), "r"((uint32_t)nb) : "memory");
    }
  }
  pdl_wait();  // the plan (k_plan_qsgd_dev, or the solve's choice) and the EF of the previous step
  DevPlan pl;
  if (choice) {  // W = 1: the bits straight from the device choice (k_plan_qsgd_dev's rule)
    int bits = 0;
    if (choice[ch.layer] == LGRECO_CHOICE_SKIP) return;  // another family's layer (NEXT-4): untouched
    if (ly.compress) {
      int c = choice[ch.layer];
      if (c == LGRECO_CHOICE_SKIP) return;  // another family's layer (NEXT-4): untouched
      if (c < 0 || c >= K) {
        if (threadIdx.x == 0) atomicOr(flag, 2u);
        c = 0;
      }
      bits = params[c];
    }
    pl = DevPlan{0, bits, 0};
  } else {
    pl = plan[ch.layer];
    if (pl.bits < 0) return;  // another family's layer (NEXT-4): untouched, no records
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int M = B >> 7;
  const bool aligned = (ly.offset & 3) == 0;
  float bad = 0.f;
  if (pl.bits == 0) {
    // lossless layer: raw x records, e' = 0 (R14, R15)
    const bool rawp = payload != nullptr || p2p != nullptr;
    const int64_t i_beg = ch.first * (int64_t)B;
    const int64_t i_end = min(ly.numel, (ch.first + ch.nbk) * (int64_t)B);
    for (int64_t i = i_beg + threadIdx.x; i < i_end; i += blockDim.x) {
      const float x = canon(__ldg(g + ly.offset + i), ef ? ef[ly.offset + i] : 0.f);
      bad = __fadd_rn(bad, __fmul_rn(x, 0.f));
      if (rawp) *reinterpret_cast<float*>(stage1_dst(payload, p2p, pl.pay_off + 4 * i)) = x;
      if (dec_out) dec_out[ly.offset + i] = x;
      if (ef) ef[ly.offset + i] = 0.f;
    }
    if (!isfinite(bad)) atomicOr(flag, 1u);
    return;
  }
  const int b = pl.bits;
  const float s_b = (float)((1u << b) - 1u);
  const bool fast_layer = aligned && B == 128;
  int bi = warp;
  // ---- fast path, QK_UNROLL buckets per iteration (all loads issued first) for
  //      memory-level parallelism
  if (fast_layer) {
    constexpr int U = QK_UNROLL;
    for (; bi + (U - 1) * QP_WARPS < ch.nbk; bi += U * QP_WARPS) {
      const int64_t jb0 = ch.first + bi;
      if ((jb0 + (U - 1) * QP_WARPS + 1) * 128 > ly.numel) break;  // last bucket not full: loop below
      X4 xs[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t base = ly.offset + (jb0 + u * QP_WARPS) * 128 + 4 * lane;
        xs[u] = canon4(ld4(g + base), ef ? ld4(ef + base) : make_float4(0.f, 0.f, 0.f, 0.f));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t jb = jb0 + u * QP_WARPS;
        const int64_t base = ly.offset + jb * 128 + 4 * lane;
        pack_bucket_fast(xs[u], b, ly.bucket0 + jb, rankfield, step, k0, k1, lane,
                         (payload || p2p) ? stage1_dst(payload, p2p, pl.pay_off + jb * (int64_t)pl.rec_bytes)
                                          : nullptr,
                         ef, dec_out,
                         base, bad);
      }
    }
  }
  for (; bi < ch.nbk; bi += QP_WARPS) {
    const int64_t jb = ch.first + bi;
    const int64_t gb = ly.bucket0 + jb;
    const int64_t e0 = jb * (int64_t)B;
    uint8_t* rec = (payload || p2p) ? stage1_dst(payload, p2p, pl.pay_off + jb * (int64_t)pl.rec_bytes) : nullptr;
    if (fast_layer && e0 + 128 <= ly.numel) {
      const int64_t base = ly.offset + e0 + 4 * lane;
      const X4 xs = canon4(ld4(g + base), ef ? ld4(ef + base) : make_float4(0.f, 0.f, 0.f, 0.f));
      pack_bucket_fast(xs, b, gb, rankfield, step, k0, k1, lane, rec, ef, dec_out, base, bad);
      continue;
    }
    // ---- generic path
    float mn = INFINITY, mx = -INFINITY;
    X4 xs;
    for (int t = 0; t < M; ++t) {
      const int64_t i0 = e0 + 128 * t + 4 * lane;
      const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
      xs = load_x4(g, ef, ly.offset + i0, nv, aligned);
#pragma unroll
      for (int s = 0; s < 4; ++s)
        if (s < nv) { mn = fmin_nan(mn, xs.v[s]); mx = fmax_nan(mx, xs.v[s]); }
    }
    warp_minmax_nan(mn, mx);
    float inv, unit;
    qparams(mn, mx, s_b, inv, unit);
    bad = __fadd_rn(bad, __fmul_rn(__fsub_rn(mx, mn), 0.f));
    for (int t = 0; t < M; ++t) {
      const int64_t i0 = e0 + 128 * t + 4 * lane;
      const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
      if (M > 1) xs = load_x4(g, ef, ly.offset + i0, nv, aligned);
      float u[4];
      uniforms4((uint32_t)(gb * (B >> 2) + 32 * t + lane), rankfield, step, 0u, k0, k1, u);
      uint32_t q[4];
      float dec[4], en[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const float x = (s < nv) ? xs.v[s] : mn;
        const float qf = qcode(__fsub_rn(x, mn), inv, u[s], s_b);
        q[s] = (s < nv) ? (uint32_t)qf : 0u;
        dec[s] = __fmaf_rn(qf, unit, mn);
        en[s] = __fsub_rn(x, dec[s]);
      }
      if (rec) pack_planes(reinterpret_cast<uint32_t*>(rec), t, b, q, lane);
      if (nv > 0) {
        if (ef) store_x4(ef, ly.offset + i0, nv, aligned, en);
        if (dec_out) store_x4(dec_out, ly.offset + i0, nv, aligned, dec);
      }
    }
    if (rec && lane == 0) *reinterpret_cast<float2*>(rec + 16 * b * M) = make_float2(mn, unit);
  }
  if (!isfinite(bad)) atomicOr(flag, 1u);
}

// ---------------------------------------------------------------------------
// K9 decode a full payload -> out
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(QP_THREADS)
k_qunpack(const uint8_t* __restrict__ payload, float* __restrict__ out, const DevLayer* __restrict__ layers,
          const DevPlan* __restrict__ plan, const ProfChunk* __restrict__ chunks, int B) {
  const ProfChunk ch = chunks[blockIdx.x];
  const DevLayer ly = layers[ch.layer];
  const DevPlan pl = plan[ch.layer];
  if (pl.bits < 0) return;  // another family's layer (NEXT-4): output untouched
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int M = B >> 7;
  const bool aligned = (ly.offset & 3) == 0;
  if (pl.bits == 0) {
    const float* raw = reinterpret_cast<const float*>(payload + pl.pay_off);
    const int64_t i_beg = ch.first * (int64_t)B;
    const int64_t i_end = min(ly.numel, (ch.first + ch.nbk) * (int64_t)B);
    for (int64_t i = i_beg + threadIdx.x; i < i_end; i += blockDim.x) out[ly.offset + i] = __ldg(raw + i);
    return;
  }
  for (int bi = warp; bi < ch.nbk; bi += QP_WARPS) {
    const int64_t jb = ch.first + bi;
    const int64_t e0 = jb * (int64_t)B;
    const uint8_t* rec = payload + pl.pay_off + jb * (int64_t)pl.rec_bytes;
    for (int t = 0; t < M; ++t) {
      const int64_t i0 = e0 + 128 * t + 4 * lane;
      const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
      float dec[4];
      decode_sub(rec, t, pl.bits, M, lane, dec);
      if (nv > 0) store_x4(out, ly.offset + i0, nv, aligned, dec);
    }
  }
}

// ---------------------------------------------------------------------------
// K8 owner reduce: records [r0, r1); recv = W x shard bytes (rank-major)
// ---------------------------------------------------------------------------
// Stage-2 store: the local payload and, over peer memory, every peer's stage-2 payload
// at the same offset (the owner's shard reaches all ranks as it is produced).
template <typename T>
__device__ __forceinline__ void st2(uint8_t* stage2, const P2PDev* __restrict__ p2p, int64_t off, T v) {
  *reinterpret_cast<T*>(stage2 + off) = v;
  if (p2p)
    for (int o = 0; o < p2p->W; ++o)
      if (o != p2p->me) *reinterpret_cast<T*>(p2p->s2[o] + off) = v;
}

// pack_planes into the stage-2 payload (and the peers') at byte offset roff
__device__ __forceinline__ void pack_planes2(uint8_t* stage2, const P2PDev* __restrict__ p2p, int64_t roff, int t,
                                             int b, const uint32_t* q, int lane) {
  for (int p = 0; p < b; ++p) {
    const uint32_t w0 = __ballot_sync(LG_FULL, (q[0] >> p) & 1u);
    const uint32_t w1 = __ballot_sync(LG_FULL, (q[1] >> p) & 1u);
    const uint32_t w2 = __ballot_sync(LG_FULL, (q[2] >> p) & 1u);
    const uint32_t w3 = __ballot_sync(LG_FULL, (q[3] >> p) & 1u);
    if (lane == 0) {  // (records are 8-byte aligned: two 8-byte stores)
      st2(stage2, p2p, roff + 4 * (int64_t)(t * b + p) * 4, make_uint2(w0, w1));
      st2(stage2, p2p, roff + 4 * (int64_t)(t * b + p) * 4 + 8, make_uint2(w2, w3));
    }
  }
}

__global__ void __launch_bounds__(QP_THREADS)
k_qreduce(const uint8_t* __restrict__ recv, int64_t shard_bytes, int64_t byte0, uint8_t* __restrict__ stage2,
          const DevLayer* __restrict__ layers, const DevPlan* __restrict__ plan, const int64_t* __restrict__ bucket0,
          int L, int64_t r0, int64_t r1, int B, int W, uint32_t k0, uint32_t k1, uint32_t step, int rec_per_warp,
          const P2PDev* __restrict__ p2p, int device_bounds) {
  extern __shared__ int64_t sb0[];
  for (int i = threadIdx.x; i <= L; i += blockDim.x) sb0[i] = bucket0[i];
  if (p2p && device_bounds) {  // this rank's shard from the device-side layout
    const int me = p2p->me;
    r0 = p2p->rb[me]; r1 = p2p->rb[me + 1];
    byte0 = p2p->bb[me]; shard_bytes = p2p->bb[me + 1] - p2p->bb[me];
  }
  const P2PDev* p2p_out = p2p;  // stage-2 records also stored into every peer's payload
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int M = B >> 7;
  const float invW = __fdiv_rn(1.0f, (float)W);
  for (int64_t wbase = r0 + ((int64_t)blockIdx.x * QP_WARPS + warp) * rec_per_warp; wbase < r1;
       wbase += (int64_t)gridDim.x * QP_WARPS * rec_per_warp)
  for (int ri = 0; ri < rec_per_warp; ++ri) {
    const int64_t gb = wbase + ri;
    if (gb >= r1) break;
    const int l = find_layer(sb0, L, gb);
    const DevLayer ly = layers[l];
    const DevPlan pl = plan[l];
    if (pl.bits < 0) continue;  // another family's layer (NEXT-4): no records
    const int64_t jb = gb - ly.bucket0;
    const int64_t e0 = jb * (int64_t)B;
    if (pl.bits == 0) {
      const int64_t roff = pl.pay_off + e0 * 4;
      for (int t = 0; t < M; ++t) {
        const int64_t i0 = e0 + 128 * t + 4 * lane;
        const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
        for (int s = 0; s < nv; ++s) {
          const int64_t bo = roff + 4 * (128 * t + 4 * lane + s) - byte0;
          float a = 0.f;
          for (int w = 0; w < W; ++w) {
            const float v = __ldg(reinterpret_cast<const float*>(recv + w * shard_bytes + bo));
            a = (w == 0) ? v : __fadd_rn(a, v);
          }
          st2(stage2, p2p_out, roff + 4 * (128 * t + 4 * lane + s), __fmul_rn(a, invW));
        }
      }
      continue;
    }
    const int b = pl.bits;
    const float s_b = (float)((1u << b) - 1u);
    const int64_t roff = pl.pay_off + jb * (int64_t)pl.rec_bytes;
    float mn = INFINITY, mx = -INFINITY;
    float m4[4];
    for (int pass = 0; pass < 2; ++pass) {
      float inv = 0.f, unit = 0.f;
      if (pass == 1) {
        warp_minmax_nan(mn, mx);
        qparams(mn, mx, s_b, inv, unit);
      }
      for (int t = 0; t < M; ++t) {
        const int64_t i0 = e0 + 128 * t + 4 * lane;
        const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
        if (pass == 0 || M > 1) {
          float a[4] = {0.f, 0.f, 0.f, 0.f};
          for (int w = 0; w < W; ++w) {
            float d[4];
            decode_sub(recv + w * shard_bytes + (roff - byte0), t, b, M, lane, d);
#pragma unroll
            for (int s = 0; s < 4; ++s) a[s] = (w == 0) ? d[s] : __fadd_rn(a[s], d[s]);
          }
#pragma unroll
          for (int s = 0; s < 4; ++s) m4[s] = __fmul_rn(a[s], invW);
        }
        if (pass == 0) {
#pragma unroll
          for (int s = 0; s < 4; ++s)
            if (s < nv) { mn = fmin_nan(mn, m4[s]); mx = fmax_nan(mx, m4[s]); }
          continue;
        }
        float u[4];
        uniforms4((uint32_t)(gb * (B >> 2) + 32 * t + lane), 0xFFFFFFFFu, step, 1u, k0, k1, u);
        uint32_t q[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const float x = (s < nv) ? m4[s] : mn;
          const float qf = qcode(__fsub_rn(x, mn), inv, u[s], s_b);
          q[s] = (s < nv) ? (uint32_t)qf : 0u;
        }
        pack_planes2(stage2, p2p_out, roff, t, b, q, lane);
      }
      if (pass == 1 && lane == 0) st2(stage2, p2p_out, roff + 16 * b * M, make_float2(mn, unit));
    }
  }
}

// device-side plan for the W == 1 fused path (no payload): bits per layer from the
// device-resident choice (no host round trip)
__global__ void k_plan_qsgd_dev(const int32_t* __restrict__ choice, const int32_t* __restrict__ params, int K,
                                const DevLayer* __restrict__ layers, int L, DevPlan* __restrict__ plan,
                                unsigned* __restrict__ flag) {
  pdl_wait();  // the solve's choice
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < L; l += gridDim.x * blockDim.x) {
    int bits = 0;
    if (layers[l].compress) {
      int c = choice[l];
      if (c < 0 || c >= K) { atomicOr(flag, 2u); c = 0; }
      bits = params[c];
    }
    plan[l] = DevPlan{0, bits, 0};
  }
}

cudaError_t launch_plan_qsgd_dev(const int32_t* choice, const int32_t* params, int K, const DevLayer* layers, int L,
                                 DevPlan* plan, unsigned* flag, cudaStream_t st) {
  const cudaError_t e = launch_pdl(k_plan_qsgd_dev, dim3((L + 255) / 256), dim3(256), 0, st, choice, params, K, layers,
                                   L, plan, flag);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

__global__ void k_philox(const uint32_t* __restrict__ ctr, uint32_t k0, uint32_t k1, int64_t n,
                         uint32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const U4 r = philox10(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3], k0, k1);
  out[4 * i] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_qprofile(const QProfileArgs& a, cudaStream_t st) {
  const bool quads = a.B == 128 && a.nqwarps > 0 && a.nqchunks > 0;
  if (a.nchunks > 0) {
    if (a.ev0) cudaEventRecord(a.ev0, st);
    if (quads) {
      const size_t smem = (size_t)Q1_WARPS * Q1_STAGES * 4096;
      const int nsm = a.nqwarps / 32;  // nqwarps = SMs x 4 CTAs x 8 warps (an upper bound)
#define LG_QQ2(KT, FU)                                                                                         \
  {                                                                                                            \
    long long occm = 0;                                                                                        \
    if (!memo_get((const void*)k_qprofile_q<KT, FU>, (long long)smem, Q1_THREADS, 0, 0, &occm)) {              \
      cudaError_t e = memo_smem_attr((const void*)k_qprofile_q<KT, FU>, smem);                                 \
      if (e != cudaSuccess) return e;                                                                          \
      int o = 0;                                                                                               \
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_qprofile_q<KT, FU>, Q1_THREADS, smem) !=          \
              cudaSuccess ||                                                                                   \
          o < 1) { cudaGetLastError(); o = 1; }                                                                 \
      occm = o;                                                                                                \
      memo_put((const void*)k_qprofile_q<KT, FU>, (long long)smem, Q1_THREADS, 0, 0, occm);                    \
    }                                                                                                          \
    const int occ = (int)occm;                                                                                 \
    const int grid = std::max(1, std::min(a.nqwarps / Q1_WARPS, nsm * occ));                                    \
    const cudaError_t e2 = launch_pdl(k_qprofile_q<KT, FU>, dim3(grid), dim3(Q1_THREADS), smem, st, a.g, a.e,   \
                                      a.qinfo, a.nqchunks, a.ticket, a.cs, a.K, philox_rk(a.k0, a.k1), a.rankfield, \
                                      a.step, a.ptr_aligned, a.partial, fz);                                     \
    if (e2 != cudaSuccess) return e2;                                                                            \
  }
#define LG_QQ(KT) { if (a.fuse && a.fuse->p2p) LG_QQ2(KT, 2) else if (a.fuse) LG_QQ2(KT, 1) else LG_QQ2(KT, 0) }
      const QFuse fz = a.fuse ? *a.fuse : QFuse{};
      switch (a.K) {
        case 4: LG_QQ(4); break;
        case 5: LG_QQ(5); break;
        case 6: LG_QQ(6); break;
        case 7: LG_QQ(7); break;
        case 8: LG_QQ(8); break;
        default:
          if (a.K < 4) LG_QQ(4) else LG_QQ(16)
      }
#undef LG_QQ
#undef LG_QQ2
    } else {
#define LG_QP(KT)                                                                          \
  k_qprofile<KT><<<a.nchunks, QP_THREADS, 0, st>>>(a.g, a.e, a.layers, a.chunks, a.B, a.cs, a.K, \
                                                    a.k0, a.k1, a.rankfield, a.step, a.partial)
      switch (a.K) {
        case 4: LG_QP(4); break;
        case 5: LG_QP(5); break;
        case 6: LG_QP(6); break;
        case 7: LG_QP(7); break;
        case 8: LG_QP(8); break;
        default:
          if (a.K < 4) LG_QP(4);
          else LG_QP(16);
      }
#undef LG_QP
    }
    if (a.ev1) cudaEventRecord(a.ev1, st);
  }
  if (quads) {
    // PDL: its CTAs take the SMs K1's CTAs release and wait in-kernel for K1's completion
    const cudaError_t e = launch_pdl(k_qprofile_reduce, dim3(a.nseg), dim3(QR_ROWS), 0, st, a.layers, a.segs, a.lseg0,
                                     a.partial, a.segsum, a.ldone, a.params, a.K, a.B, a.err, a.bits);
    if (e != cudaSuccess) return e;
  }
  else
    k_qprofile_reduce_chunks<<<a.L, 256, 0, st>>>(a.layers, a.layer_chunk0, a.partial, a.params, a.K, a.B, a.err,
                                                  a.bits);
  return cudaGetLastError();
}

// K5's L2 prefetch before its plan wait (LGRECO_K5_PREFETCH=0 disables it, for A/B)
static int k5_l2_prefetch() {
  static const int v = [] {
    const char* s = getenv("LGRECO_K5_PREFETCH");
    return (s && s[0] == '0') ? 0 : 1;
  }();
  return v;
}

cudaError_t launch_qpack(const QPackArgs& a, cudaStream_t st) {
  if (a.nchunks == 0) return cudaSuccess;
  const cudaError_t e = launch_pdl(k_qpack, dim3(a.nchunks), dim3(QP_THREADS), 0, st, a.g, a.ef, a.payload, a.dec,
                                   a.layers, a.plan, a.chunks, a.B, a.k0, a.k1, a.rankfield, a.step, a.flag, a.p2p,
                                   a.choice, a.params, a.K, k5_l2_prefetch());
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_qunpack(const QUnpackArgs& a, cudaStream_t st) {
  if (a.nchunks == 0) return cudaSuccess;
  k_qunpack<<<a.nchunks, QP_THREADS, 0, st>>>(a.payload, a.out, a.layers, a.plan, a.chunks, a.B);
  return cudaGetLastError();
}

cudaError_t launch_qreduce(const QReduceArgs& a, cudaStream_t st) {
  const int rpw = 2;
  const int64_t n = a.r1 - a.r0;
  const int grid = a.device_bounds ? a.grid : (int)((n + (int64_t)QP_WARPS * rpw - 1) / ((int64_t)QP_WARPS * rpw));
  if (grid == 0) return cudaSuccess;
  const size_t smem = sizeof(int64_t) * (a.L + 1);
  k_qreduce<<<grid, QP_THREADS, smem, st>>>(a.recv, a.shard_bytes, a.byte0, a.stage2, a.layers, a.plan, a.bucket0,
                                            a.L, a.r0, a.r1, a.B, a.W, a.k0, a.k1, a.step, rpw, a.p2p,
                                            a.device_bounds);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Peer-memory exchange (W > 1 without NCCL): K5 stores every stage-1 record straight
// into its owner's receive window (stage1_dst), k_p2p_signal publishes "my stage-s data
// for you is complete" as the epoch in word (s, me) of every peer's flags (system-scope
// fence, then a release store), k_p2p_wait spins (acquire) until all W senders'
// words hold the epoch, k_p2p_push copies this rank's stage-2 shard into every peer's
// stage-2 payload (16-byte stores over NVLink).  Kernel boundaries order the rest.
// ---------------------------------------------------------------------------
__global__ void k_p2p_signal(const P2PDev* __restrict__ p, int stage, unsigned epoch) {
  const int o = threadIdx.x;
  __threadfence_system();
  if (o < p->W) {
    unsigned* f = p->flag[o] + stage * p->W + p->me;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
  }
}

__global__ void k_p2p_wait(const unsigned* __restrict__ flags, int W, int me, int stage, unsigned epoch) {
  const int j = threadIdx.x;
  if (j < W) {
    const unsigned* f = flags + stage * W + j;
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    } while (v != epoch);
  }
  __syncthreads();
  __threadfence_system();
}

__global__ void k_p2p_push(const P2PDev* __restrict__ p, const uint8_t* __restrict__ src, int64_t b0, int64_t b1) {
  // bytes [b0, b1) (b1 < 0: this rank's shard from the device-side layout): unaligned
  // head and tail byte by byte, the 16-byte-aligned body as uint4 (the peer buffers have
  // the local buffer's alignment at every offset)
  const int W = p->W, me = p->me;
  if (b1 < 0) { b0 = p->bb[me]; b1 = p->bb[me + 1]; }
  const int64_t a0 = min(b1, (b0 + 15) & ~(int64_t)15);
  const int64_t n16 = (b1 - a0) / 16;
  const int64_t a1 = a0 + 16 * n16;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < n16; i += nth) {
    const uint4 v = *reinterpret_cast<const uint4*>(src + a0 + 16 * i);
    for (int o = 0; o < W; ++o)
      if (o != me) *reinterpret_cast<uint4*>(p->s2[o] + a0 + 16 * i) = v;
  }
  for (int64_t i = tid; i < (a0 - b0) + (b1 - a1); i += nth) {
    const int64_t k = (i < a0 - b0) ? b0 + i : a1 + (i - (a0 - b0));
    for (int o = 0; o < W; ++o)
      if (o != me) p->s2[o][k] = src[k];
  }
}

// Plan agreement over peer memory (R21): rank 0 stores its plan into word 3*8 + l of
// every peer's flag area, then releases epoch word (2, 0); the others acquire it and
// copy the plan out.
__global__ void k_p2p_plan_push(const P2PDev* __restrict__ p, const int32_t* __restrict__ choice, int L) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < L; l += gridDim.x * blockDim.x)
    for (int o = 1; o < p->W; ++o) p->flag[o][3 * P2P_MAXW + l] = (unsigned)choice[l];
}
__global__ void k_p2p_plan_pull(const unsigned* __restrict__ my_flags, int W, unsigned epoch, int32_t* choice, int L) {
  if (threadIdx.x == 0) {
    const unsigned* f = my_flags + 2 * W;  // word (2, sender 0)
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    } while (v != epoch);
  }
  __syncthreads();
  for (int l = threadIdx.x; l < L; l += blockDim.x) choice[l] = (int32_t)my_flags[3 * P2P_MAXW + l];
}
cudaError_t launch_p2p_plan(const P2PDev* p, const unsigned* my_flags, int W, int me, unsigned epoch, int32_t* choice,
                            int L, cudaStream_t st) {
  if (me == 0) {
    k_p2p_plan_push<<<std::max(1, std::min(64, (L + 255) / 256)), 256, 0, st>>>(p, choice, L);
    return launch_p2p_signal(p, 2, epoch, st);
  }
  k_p2p_plan_pull<<<1, 256, 0, st>>>(my_flags, W, epoch, choice, L);
  return cudaGetLastError();
}

// Device-side plan layout for W > 1 (R7, R13; the host's qsgd_layout + shard_bounds):
// one CTA; per-layer sizes, a sequential 16-byte-padded prefix by thread 0 (L is a few
// hundred), then thread j < W binary-searches the first record whose offset reaches
// floor(j S / W).
__global__ void k_plan_qsgd_layout(const int32_t* __restrict__ choice, const int32_t* __restrict__ params, int K,
                                   const DevLayer* __restrict__ layers, const int64_t* __restrict__ bucket0, int L,
                                   int64_t R, int B, DevPlan* __restrict__ plan, P2PDev* __restrict__ p,
                                   unsigned* __restrict__ flag) {
  pdl_wait();  // the solve's choice
  __shared__ int64_t S_sh;
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    int bits = 0;
    if (choice[l] == LGRECO_CHOICE_SKIP) {
      bits = -1;  // another family's layer (NEXT-4): no records, no bytes (R24)
    } else if (layers[l].compress) {
      int c = choice[l];
      if (c < 0 || c >= K) { atomicOr(flag, 2u); c = 0; }
      bits = params[c];
    }
    const int32_t rb = bits > 0 ? 16 * bits * (B / 128) + 8 : bits == 0 ? 4 * B : 0;
    plan[l] = DevPlan{0, bits, rb};
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t off = 0;
    for (int l = 0; l < L; ++l) {
      const int64_t nb = bucket0[l + 1] - bucket0[l];
      plan[l].pay_off = off;
      if (plan[l].bits < 0) continue;
      off += plan[l].bits > 0 ? nb * (int64_t)plan[l].rec_bytes : 4 * layers[l].numel;
      off = (off + 15) & ~(int64_t)15;
    }
    S_sh = off;
  }
  __syncthreads();
  const int64_t S = S_sh;
  const int W = p->W;
  auto rec_off = [&](int64_t r) -> int64_t {
    if (r >= R) return S;
    int lo = 0, hi = L - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (bucket0[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const DevPlan pl = plan[lo];
    const int64_t jb = r - bucket0[lo];
    return pl.pay_off + (pl.bits > 0 ? jb * (int64_t)pl.rec_bytes : pl.bits == 0 ? jb * 4 * (int64_t)B : 0);
  };
  const int j = threadIdx.x;
  if (j <= W) {
    int64_t rj = 0, bj = 0;
    if (j == W) { rj = R; bj = S; }
    else if (j > 0) {
      const int64_t target = (int64_t)(((__int128)j * S) / W);
      int64_t lo = 0, hi = R;
      while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (rec_off(mid) >= target) hi = mid; else lo = mid + 1;
      }
      rj = lo;
      bj = rec_off(lo);
    }
    p->rb[j] = rj;
    p->bb[j] = bj;
  }
}

cudaError_t launch_plan_qsgd_layout(const int32_t* choice, const int32_t* params, int K, const DevLayer* layers,
                                    const int64_t* bucket0, int L, int64_t R, int B, DevPlan* plan, P2PDev* p,
                                    unsigned* flag, cudaStream_t st) {
  return launch_pdl(k_plan_qsgd_layout, dim3(1), dim3(256), 0, st, choice, params, K, layers, bucket0, L, R, B, plan, p,
                    flag);
}

// CUDA 12 loads kernels lazily, at their first launch, and a lazy load waits for the
// device to go idle -- which never happens while a peer-memory wait kernel spins for a
// peer whose kernels are the ones being loaded (ranks on streams of one process: the
// simulated-rank tests deadlocked when run on their own).  Every kernel of the
// peer-memory step is loaded up front (cudaFuncGetAttributes forces the load).
cudaError_t preload_p2p_kernels() {
  cudaFuncAttributes fa;
  const void* fns[] = {
      (const void*)k_qpack, (const void*)k_qunpack, (const void*)k_qreduce, (const void*)k_p2p_signal,
      (const void*)k_p2p_wait, (const void*)k_p2p_push, (const void*)k_p2p_plan_push, (const void*)k_p2p_plan_pull,
      (const void*)k_plan_qsgd_layout, (const void*)k_plan_qsgd_dev, (const void*)k_qprofile_reduce,
      (const void*)k_qprofile_q<4, 2>, (const void*)k_qprofile_q<5, 2>, (const void*)k_qprofile_q<6, 2>,
      (const void*)k_qprofile_q<7, 2>, (const void*)k_qprofile_q<8, 2>, (const void*)k_qprofile_q<16, 2>,
      (const void*)k_qprofile_q<4, 0>, (const void*)k_qprofile_q<5, 0>, (const void*)k_qprofile_q<6, 0>,
      (const void*)k_qprofile_q<7, 0>, (const void*)k_qprofile_q<8, 0>, (const void*)k_qprofile_q<16, 0>};
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_p2p_signal(const P2PDev* p, int stage, unsigned epoch, cudaStream_t st) {
  k_p2p_signal<<<1, 32, 0, st>>>(p, stage, epoch);
  return cudaGetLastError();
}
cudaError_t launch_p2p_wait(const unsigned* my_flags, int W, int me, int stage, unsigned epoch, cudaStream_t st) {
  k_p2p_wait<<<1, 32, 0, st>>>(my_flags, W, me, stage, epoch);
  return cudaGetLastError();
}
cudaError_t launch_p2p_push(const P2PDev* p, const uint8_t* src, int64_t b0, int64_t b1, cudaStream_t st) {
  if (b1 >= 0 && b1 <= b0) return cudaSuccess;
  const int64_t n16 = b1 >= 0 ? (b1 - b0 + 15) / 16 : (int64_t)1184 * 256;  // device bounds: full grid
  k_p2p_push<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((n16 + 255) / 256, 1184)), 256, 0, st>>>(p, src, b0,
                                                                                                        b1);
  return cudaGetLastError();
}

cudaError_t launch_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, int64_t n, uint32_t* out,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_philox<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ctr, k0, k1, n, out);
  return cudaGetLastError();
}

}  // namespace lg
