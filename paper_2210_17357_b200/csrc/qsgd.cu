// qsgd.cu -- QSGD-style bucketed min/max stochastic quantisation on sm_100a.
//
//   K1  k_qprofile   (a2)  one HBM pass over x = g + e per bucket; per-bucket
//                          min/max by warp shuffles, then the realised squared error
//                          of EVERY candidate bit-width from the same Philox uniforms
//                          (R5, R6).  Deterministic:
//                          fixed chunk -> partial -> ordered reduce.
//   K1b k_qprofile_reduce  per-layer fixed-order fp64 sum of chunk partials, sqrt.
//   K5  k_qpack      (a8)  quantise with the chosen bits, bit-plane pack via
//                          __ballot_sync, fused error feedback e <- x - dec.
//   K8  k_qreduce    (a9)  owner shard: decode W stage-1 records, ordered fp32 sum,
//                          x fl(1/W), requantise (stream 1) and pack stage 2.
//   K9  k_qunpack    (a10) decode a payload into the fp32 mean gradient.
//
// One warp owns one bucket (record) of B = 128*m elements; lane l holds elements
// 128t + 4l .. 4l+3 of sub-block t (float4 loads when the layer is 16B aligned).
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace lg {

constexpr int QP_THREADS = 256;
constexpr int QP_WARPS = QP_THREADS / 32;

// ---------------------------------------------------------------------------
// element loads
// ---------------------------------------------------------------------------
struct X4 { float v[4]; };

// Load the 4 elements of lane `lane` in sub-block (flat base index `base`), nv valid.
__device__ __forceinline__ X4 load_x4(const float* __restrict__ g, const float* __restrict__ e,
                                      int64_t base, int nv, bool aligned) {
  X4 r;
  if (nv >= 4 && aligned) {
    float4 a = __ldg(reinterpret_cast<const float4*>(g + base));
    float4 b = e ? __ldg(reinterpret_cast<const float4*>(e + base)) : make_float4(0.f, 0.f, 0.f, 0.f);
    r.v[0] = canon(a.x, b.x); r.v[1] = canon(a.y, b.y);
    r.v[2] = canon(a.z, b.z); r.v[3] = canon(a.w, b.w);
  } else {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (s < nv) r.v[s] = canon(__ldg(g + base + s), e ? __ldg(e + base + s) : 0.f);
      else r.v[s] = 0.f;
    }
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

// Per-bucket quantiser parameters for s = 2^b - 1 (R5): inv = fl(s/range),
// unit = fl(range/s); constant (mx == mn) or !finite(inv) -> inv = 0 (q = 0).
__device__ __forceinline__ void qparams(float mn, float mx, float s, float& inv, float& unit) {
  if (mx == mn) { inv = 0.f; unit = 0.f; return; }
  const float range = __fsub_rn(mx, mn);
  inv = __fdiv_rn(s, range);
  unit = __fdiv_rn(range, s);
  if (!isfinite(inv)) inv = 0.f;
}

// Stochastic rounding of t = x - mn (R6): q = min(floor(v) + (u < frac(v)), s).
__device__ __forceinline__ float qcode(float t, float inv, float u, float s) {
  const float v = __fmul_rn(t, inv);
  const float fl = floor_pos(v);
  const float f = __fsub_rn(v, fl);
  const float q = __fadd_rn(fl, (u < f) ? 1.0f : 0.0f);
  return fminf(q, s);
}

// ---------------------------------------------------------------------------
// K1 profile
// ---------------------------------------------------------------------------
template <int KMAX, bool SINGLE>
__global__ void __launch_bounds__(QP_THREADS)
k_qprofile(const float* __restrict__ g, const float* __restrict__ e, const DevLayer* __restrict__ layers,
           const ProfChunk* __restrict__ chunks, int B, const float* __restrict__ cand_s, int K,
           uint32_t k0, uint32_t k1, uint32_t rankfield, uint32_t step, double* __restrict__ partial) {
  __shared__ double red[QP_WARPS][KMAX];
  const ProfChunk ch = chunks[blockIdx.x];
  const DevLayer ly = layers[ch.layer];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool aligned = (ly.offset & 3) == 0;
  const int M = B >> 7;

  float sj[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) sj[j] = (j < K) ? cand_s[j] : 1.f;
  const float my_s = (lane < K) ? cand_s[lane] : 1.f;
  double acc[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) acc[j] = 0.0;

  for (int bi = warp; bi < ch.nbk; bi += QP_WARPS) {
    const int64_t jb = ch.first + bi;             // bucket index within the layer
    const int64_t gb = ly.bucket0 + jb;           // global record index
    const int64_t e0 = jb * (int64_t)B;           // first element (layer-relative)
    // ---- pass 1: min / max over the bucket
    float mn = INFINITY, mx = -INFINITY;
    X4 xs;
    for (int t = 0; t < M; ++t) {
      const int64_t i0 = e0 + 128 * t + 4 * lane;
      const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
      xs = load_x4(g, e, ly.offset + i0, nv, aligned);
#pragma unroll
      for (int s = 0; s < 4; ++s)
        if (s < nv) { mn = fminf(mn, xs.v[s]); mx = fmaxf(mx, xs.v[s]); }
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    float my_inv, my_unit;
    qparams(mn, mx, my_s, my_inv, my_unit);
    // ---- pass 2: all candidates on the same uniforms
    for (int t = 0; t < M; ++t) {
      const int64_t i0 = e0 + 128 * t + 4 * lane;
      const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
      if (!SINGLE) xs = load_x4(g, e, ly.offset + i0, nv, aligned);
      const U4 r = philox10((uint32_t)(gb * (B >> 2) + 32 * t + lane), rankfield, step, 0u, k0, k1);
      const float u[4] = {word_u(r.x), word_u(r.y), word_u(r.z), word_u(r.w)};
      float tt[4], x[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        x[s] = (s < nv) ? xs.v[s] : mn;   // invalid -> x = mn -> d = 0
        tt[s] = __fsub_rn(x[s], mn);
      }
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        if (j < K) {
          const float inv = __shfl_sync(LG_FULL, my_inv, j);
          const float unit = __shfl_sync(LG_FULL, my_unit, j);
          float sse = 0.f;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const float q = qcode(tt[s], inv, u[s], sj[j]);
            const float dec = __fmaf_rn(q, unit, mn);
            const float d = __fsub_rn(x[s], dec);
            sse = __fmaf_rn(d, d, sse);
          }
          acc[j] += (double)sse;
        }
      }
    }
  }
  // ---- deterministic block reduction
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
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

// K1b: per layer, fixed-order tree over its chunks' partials.
__global__ void __launch_bounds__(256)
k_qprofile_reduce(const DevLayer* __restrict__ layers, const int32_t* __restrict__ layer_chunk0,
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
// quantise + pack one record (shared by K5 stage 1 and K8 stage 2)
// x[t][4] for sub-block t is produced by `getx(t, nv, xs)`; writes the record.
// ---------------------------------------------------------------------------
// Pack the codes q[4] of sub-block t as bit planes: word (t*b+p)*4+s, bit lane.
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

// ---------------------------------------------------------------------------
// K5 stage-1 pack + EF (+ optional fused decode for W == 1)
// ---------------------------------------------------------------------------
template <bool SINGLE>
__global__ void __launch_bounds__(QP_THREADS)
k_qpack(const float* __restrict__ g, float* __restrict__ ef, uint8_t* __restrict__ payload,
        float* __restrict__ dec_out, const DevLayer* __restrict__ layers, const DevPlan* __restrict__ plan,
        const int64_t* __restrict__ bucket0, int L, int64_t R, int B, uint32_t k0, uint32_t k1,
        uint32_t rankfield, uint32_t step, int rec_per_warp, unsigned* __restrict__ flag) {
  extern __shared__ int64_t sb0[];
  for (int i = threadIdx.x; i <= L; i += blockDim.x) sb0[i] = bucket0[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int M = B >> 7;
  const int64_t wbase = ((int64_t)blockIdx.x * QP_WARPS + warp) * rec_per_warp;
  float bad = 0.f;
  for (int ri = 0; ri < rec_per_warp; ++ri) {
    const int64_t gb = wbase + ri;
    if (gb >= R) break;
    const int l = find_layer(sb0, L, gb);
    const DevLayer ly = layers[l];
    const DevPlan pl = plan[l];
    const int64_t jb = gb - ly.bucket0;
    const int64_t e0 = jb * (int64_t)B;
    const bool aligned = (ly.offset & 3) == 0;
    if (pl.bits == 0) {
      // lossless record: raw x, e' = 0
      float* rawdst = payload ? reinterpret_cast<float*>(payload + pl.pay_off) : nullptr;
      for (int t = 0; t < M; ++t) {
        const int64_t i0 = e0 + 128 * t + 4 * lane;
        const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
        if (nv <= 0) continue;
        X4 xs = load_x4(g, ef, ly.offset + i0, nv, aligned);
#pragma unroll
        for (int s = 0; s < 4; ++s) if (s < nv) bad = __fmaf_rn(xs.v[s], 0.f, bad);
        if (rawdst) {
#pragma unroll
          for (int s = 0; s < 4; ++s) if (s < nv) rawdst[i0 + s] = xs.v[s];
        }
        if (dec_out) store_x4(dec_out, ly.offset + i0, nv, aligned, xs.v);
        if (ef) { const float z[4] = {0.f, 0.f, 0.f, 0.f}; store_x4(ef, ly.offset + i0, nv, aligned, z); }
      }
      continue;
    }
    const int b = pl.bits;
    const float s_b = (float)((1u << b) - 1u);
    float mn = INFINITY, mx = -INFINITY;
    X4 xs;
    for (int t = 0; t < M; ++t) {
      const int64_t i0 = e0 + 128 * t + 4 * lane;
      const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
      xs = load_x4(g, ef, ly.offset + i0, nv, aligned);
#pragma unroll
      for (int s = 0; s < 4; ++s)
        if (s < nv) { mn = fminf(mn, xs.v[s]); mx = fmaxf(mx, xs.v[s]); bad = __fmaf_rn(xs.v[s], 0.f, bad); }
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    float inv, unit;
    qparams(mn, mx, s_b, inv, unit);
    if (!isfinite(unit)) bad = __int_as_float(0x7fc00000);  // range overflow (R5)
    uint8_t* rec = payload ? payload + pl.pay_off + jb * (int64_t)pl.rec_bytes : nullptr;
    for (int t = 0; t < M; ++t) {
      const int64_t i0 = e0 + 128 * t + 4 * lane;
      const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
      if (!SINGLE) xs = load_x4(g, ef, ly.offset + i0, nv, aligned);
      const U4 r = philox10((uint32_t)(gb * (B >> 2) + 32 * t + lane), rankfield, step, 0u, k0, k1);
      const float u[4] = {word_u(r.x), word_u(r.y), word_u(r.z), word_u(r.w)};
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
    if (rec && lane == 0) {
      float* meta = reinterpret_cast<float*>(rec + 16 * b * M);
      meta[0] = mn;
      meta[1] = unit;
    }
  }
  if (!isfinite(bad)) atomicOr(flag, 1u);
}

// ---------------------------------------------------------------------------
// decode helpers
// ---------------------------------------------------------------------------
// Decode sub-block t of a record with b bits: codes of lane's 4 elements -> dec[4]
__device__ __forceinline__ void decode_sub(const uint8_t* __restrict__ rec, int t, int b, int M, int lane,
                                           float* dec) {
  const uint32_t* words = reinterpret_cast<const uint32_t*>(rec);
  const float mn = __ldg(reinterpret_cast<const float*>(rec + 16 * b * M));
  const float unit = __ldg(reinterpret_cast<const float*>(rec + 16 * b * M + 4));
  uint32_t q0 = 0, q1 = 0, q2 = 0, q3 = 0;
  for (int p = 0; p < b; ++p) {
    const uint2 a = __ldg(reinterpret_cast<const uint2*>(words + (t * b + p) * 4));
    const uint2 c = __ldg(reinterpret_cast<const uint2*>(words + (t * b + p) * 4 + 2));
    q0 |= ((a.x >> lane) & 1u) << p;
    q1 |= ((a.y >> lane) & 1u) << p;
    q2 |= ((c.x >> lane) & 1u) << p;
    q3 |= ((c.y >> lane) & 1u) << p;
  }
  dec[0] = __fmaf_rn((float)q0, unit, mn);
  dec[1] = __fmaf_rn((float)q1, unit, mn);
  dec[2] = __fmaf_rn((float)q2, unit, mn);
  dec[3] = __fmaf_rn((float)q3, unit, mn);
}

// ---------------------------------------------------------------------------
// K9 decode a full payload -> out
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(QP_THREADS)
k_qunpack(const uint8_t* __restrict__ payload, float* __restrict__ out, const DevLayer* __restrict__ layers,
          const DevPlan* __restrict__ plan, const int64_t* __restrict__ bucket0, int L, int64_t R, int B,
          int rec_per_warp) {
  extern __shared__ int64_t sb0[];
  for (int i = threadIdx.x; i <= L; i += blockDim.x) sb0[i] = bucket0[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int M = B >> 7;
  const int64_t wbase = ((int64_t)blockIdx.x * QP_WARPS + warp) * rec_per_warp;
  for (int ri = 0; ri < rec_per_warp; ++ri) {
    const int64_t gb = wbase + ri;
    if (gb >= R) break;
    const int l = find_layer(sb0, L, gb);
    const DevLayer ly = layers[l];
    const DevPlan pl = plan[l];
    const int64_t jb = gb - ly.bucket0;
    const int64_t e0 = jb * (int64_t)B;
    const bool aligned = (ly.offset & 3) == 0;
    for (int t = 0; t < M; ++t) {
      const int64_t i0 = e0 + 128 * t + 4 * lane;
      const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
      float dec[4];
      if (pl.bits == 0) {
        const float* raw = reinterpret_cast<const float*>(payload + pl.pay_off);
#pragma unroll
        for (int s = 0; s < 4; ++s) dec[s] = (s < nv) ? __ldg(raw + i0 + s) : 0.f;
      } else {
        decode_sub(payload + pl.pay_off + jb * (int64_t)pl.rec_bytes, t, pl.bits, M, lane, dec);
      }
      if (nv > 0) store_x4(out, ly.offset + i0, nv, aligned, dec);
    }
  }
}

// ---------------------------------------------------------------------------
// K8 owner reduce: records [r0, r1); recv = W x shard bytes (rank-major)
// ---------------------------------------------------------------------------
template <bool SINGLE>
__global__ void __launch_bounds__(QP_THREADS)
k_qreduce(const uint8_t* __restrict__ recv, int64_t shard_bytes, int64_t byte0, uint8_t* __restrict__ stage2,
          const DevLayer* __restrict__ layers, const DevPlan* __restrict__ plan, const int64_t* __restrict__ bucket0,
          int L, int64_t r0, int64_t r1, int B, int W, uint32_t k0, uint32_t k1, uint32_t step, int rec_per_warp) {
  extern __shared__ int64_t sb0[];
  for (int i = threadIdx.x; i <= L; i += blockDim.x) sb0[i] = bucket0[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int M = B >> 7;
  const float invW = __fdiv_rn(1.0f, (float)W);
  const int64_t wbase = r0 + ((int64_t)blockIdx.x * QP_WARPS + warp) * rec_per_warp;
  for (int ri = 0; ri < rec_per_warp; ++ri) {
    const int64_t gb = wbase + ri;
    if (gb >= r1) break;
    const int l = find_layer(sb0, L, gb);
    const DevLayer ly = layers[l];
    const DevPlan pl = plan[l];
    const int64_t jb = gb - ly.bucket0;
    const int64_t e0 = jb * (int64_t)B;
    if (pl.bits == 0) {
      const int64_t roff = pl.pay_off + e0 * 4;  // record byte offset
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
          *reinterpret_cast<float*>(stage2 + roff + 4 * (128 * t + 4 * lane + s)) = __fmul_rn(a, invW);
        }
      }
      continue;
    }
    const int b = pl.bits;
    const float s_b = (float)((1u << b) - 1u);
    const int64_t roff = pl.pay_off + jb * (int64_t)pl.rec_bytes;
    // pass 1: averaged values and their min / max
    float mn = INFINITY, mx = -INFINITY;
    float m4[4];
    for (int t = 0; t < M; ++t) {
      const int64_t i0 = e0 + 128 * t + 4 * lane;
      const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
      float a[4] = {0.f, 0.f, 0.f, 0.f};
      for (int w = 0; w < W; ++w) {
        float d[4];
        decode_sub(recv + w * shard_bytes + (roff - byte0), t, b, M, lane, d);
#pragma unroll
        for (int s = 0; s < 4; ++s) a[s] = (w == 0) ? d[s] : __fadd_rn(a[s], d[s]);
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        m4[s] = __fmul_rn(a[s], invW);
        if (s < nv) { mn = fminf(mn, m4[s]); mx = fmaxf(mx, m4[s]); }
      }
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    float inv, unit;
    qparams(mn, mx, s_b, inv, unit);
    uint8_t* rec = stage2 + roff;
    for (int t = 0; t < M; ++t) {
      const int64_t i0 = e0 + 128 * t + 4 * lane;
      const int nv = (int)max((int64_t)0, min((int64_t)4, ly.numel - i0));
      if (!SINGLE) {
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
      const U4 r = philox10((uint32_t)(gb * (B >> 2) + 32 * t + lane), 0xFFFFFFFFu, step, 1u, k0, k1);
      const float u[4] = {word_u(r.x), word_u(r.y), word_u(r.z), word_u(r.w)};
      uint32_t q[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const float x = (s < nv) ? m4[s] : mn;
        const float qf = qcode(__fsub_rn(x, mn), inv, u[s], s_b);
        q[s] = (s < nv) ? (uint32_t)qf : 0u;
      }
      pack_planes(reinterpret_cast<uint32_t*>(rec), t, b, q, lane);
    }
    if (lane == 0) {
      float* meta = reinterpret_cast<float*>(rec + 16 * b * M);
      meta[0] = mn;
      meta[1] = unit;
    }
  }
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
static int grid_for(int64_t R, int rpw) {
  return (int)((R + (int64_t)QP_WARPS * rpw - 1) / ((int64_t)QP_WARPS * rpw));
}

cudaError_t launch_qprofile(const QProfileArgs& a, cudaStream_t st) {
  if (a.nchunks > 0) {
    const bool single = a.B == 128;
#define LG_QP(KM)                                                                              \
  if (single)                                                                                  \
    k_qprofile<KM, true><<<a.nchunks, QP_THREADS, 0, st>>>(a.g, a.e, a.layers, a.chunks, a.B,  \
        a.cand_s, a.K, a.k0, a.k1, a.rankfield, a.step, a.partial);                            \
  else                                                                                         \
    k_qprofile<KM, false><<<a.nchunks, QP_THREADS, 0, st>>>(a.g, a.e, a.layers, a.chunks, a.B, \
        a.cand_s, a.K, a.k0, a.k1, a.rankfield, a.step, a.partial);
    if (a.K <= 4) { LG_QP(4) }
    else if (a.K <= 7) { LG_QP(7) }
    else if (a.K <= 8) { LG_QP(8) }
    else { LG_QP(16) }
#undef LG_QP
  }
  k_qprofile_reduce<<<a.L, 256, 0, st>>>(a.layers, a.layer_chunk0, a.partial, a.params, a.K, a.B, a.err, a.bits);
  return cudaGetLastError();
}

cudaError_t launch_qpack(const QPackArgs& a, cudaStream_t st) {
  const int rpw = 4;
  const int grid = grid_for(a.R, rpw);
  if (grid == 0) return cudaSuccess;
  const size_t smem = sizeof(int64_t) * (a.L + 1);
  if (a.B == 128)
    k_qpack<true><<<grid, QP_THREADS, smem, st>>>(a.g, a.ef, a.payload, a.dec, a.layers, a.plan, a.bucket0,
                                                  a.L, a.R, a.B, a.k0, a.k1, a.rankfield, a.step, rpw, a.flag);
  else
    k_qpack<false><<<grid, QP_THREADS, smem, st>>>(a.g, a.ef, a.payload, a.dec, a.layers, a.plan, a.bucket0,
                                                   a.L, a.R, a.B, a.k0, a.k1, a.rankfield, a.step, rpw, a.flag);
  return cudaGetLastError();
}

cudaError_t launch_qunpack(const QUnpackArgs& a, cudaStream_t st) {
  const int rpw = 4;
  const int grid = grid_for(a.R, rpw);
  if (grid == 0) return cudaSuccess;
  const size_t smem = sizeof(int64_t) * (a.L + 1);
  k_qunpack<<<grid, QP_THREADS, smem, st>>>(a.payload, a.out, a.layers, a.plan, a.bucket0, a.L, a.R, a.B, rpw);
  return cudaGetLastError();
}

cudaError_t launch_qreduce(const QReduceArgs& a, cudaStream_t st) {
  const int rpw = 2;
  const int grid = grid_for(a.r1 - a.r0, rpw);
  if (grid == 0) return cudaSuccess;
  const size_t smem = sizeof(int64_t) * (a.L + 1);
  if (a.B == 128)
    k_qreduce<true><<<grid, QP_THREADS, smem, st>>>(a.recv, a.shard_bytes, a.byte0, a.stage2, a.layers, a.plan,
                                                    a.bucket0, a.L, a.r0, a.r1, a.B, a.W, a.k0, a.k1, a.step, rpw);
  else
    k_qreduce<false><<<grid, QP_THREADS, smem, st>>>(a.recv, a.shard_bytes, a.byte0, a.stage2, a.layers, a.plan,
                                                     a.bucket0, a.L, a.r0, a.r1, a.B, a.W, a.k0, a.k1, a.step, rpw);
  return cudaGetLastError();
}

cudaError_t launch_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, int64_t n, uint32_t* out,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_philox<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ctr, k0, k1, n, out);
  return cudaGetLastError();
}

}  // namespace lg
