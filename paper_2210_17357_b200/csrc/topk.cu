// topk.cu -- per-layer TopK on sm_100a: exact radix select, profile and compression.
//
//   K2  profile (a3): for every layer and every density d_j, the k_j-th largest
//       |x| (31-bit IEEE key) and the exact dropped energy sum_{dropped} x^2, by a
//       three-level radix select over the key (11 + 10 + 10 bits):
//         P1 one pass: per-layer 2048-bin histogram of counts and fixed-point
//            sums of x^2 (CTA-private shared-memory histograms, integer atomics:
//            deterministic); S1 locates every k_j's level-1 bin;
//         P2 one pass: only elements of those boundary bins -> 1024-bin level-2
//            histograms; S2 refines;  P3 -> level-3 counts (exact keys); S3 gives
//            the threshold key T_j, the number of tied keys kept, and
//            SSE_j = sum over keys < T_j of x^2 + dropped ties * T_j^2.
//       Within one level-1 bin the exponent is fixed, so x^2 = M^2 2^(2E-300) is
//       summed exactly as the integer M^2 >> 16 (relative truncation <= 2^-30).
//   K6  compress (a8): the same select with the chosen density (one query per
//       layer), then an order-preserving compaction: per-chunk (>, ==) counts,
//       per-layer exclusive scan, and a write pass that keeps key > T and the first
//       r ties in index order (R9), writes (idx, val) pairs ascending, e' = x with
//       the kept entries zeroed, and (W == 1) the decoded output.
//   K10 exchange (a9-a10): all-gather the pair arrays; out = 0, then for each rank
//       in order out[idx] += val * fl(1/W) (R10); lossless layers: ordered sum.
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "memo.h"

namespace lg {

constexpr int TK_THREADS = 256;
constexpr int TK_WARPS = TK_THREADS / 32;

__device__ __forceinline__ uint32_t tkey(float x) { return __float_as_uint(x) & 0x7fffffffu; }

// integer M^2 >> 16 of a key (M = 24-bit significand with the implicit bit)
__device__ __forceinline__ unsigned long long fx_sq(uint32_t key) {
  const uint32_t E = key >> 23;
  const uint64_t M = (key & 0x7FFFFFu) | (E ? 0x800000u : 0u);
  return (unsigned long long)((M * M) >> 16);
}

// value of one fixed-point unit for a level-1 bin (exponent E = bin >> 3)
__device__ __forceinline__ double fx_scale(int bin1) {
  const int E = max(bin1 >> 3, 1);
  return ldexp(1.0, 16 + 2 * E - 300);
}

__device__ __forceinline__ double key_sq(uint32_t key) {
  const double v = (double)__uint_as_float(key);
  return v * v;
}

// iterate the elements of a chunk: calls f(i_layer_relative, x)
template <typename F>
__device__ __forceinline__ void for_chunk(const float* __restrict__ g, const float* __restrict__ e, const DevLayer& ly,
                                          const TChunk& ch, F&& f) {
  const bool aligned = ((ly.offset + ch.first) & 3) == 0;
  const int64_t end = ch.first + ch.n;
  if (aligned) {
    int64_t i = ch.first + 4 * threadIdx.x;
    for (; i + 4 <= end; i += 4 * TK_THREADS) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(g + ly.offset + i));
      const float4 b = e ? __ldg(reinterpret_cast<const float4*>(e + ly.offset + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
      f(i, canon(a.x, b.x)); f(i + 1, canon(a.y, b.y)); f(i + 2, canon(a.z, b.z)); f(i + 3, canon(a.w, b.w));
    }
    for (; i < end; ++i) f(i, canon(__ldg(g + ly.offset + i), e ? __ldg(e + ly.offset + i) : 0.f));
  } else {
    for (int64_t i = ch.first + threadIdx.x; i < end; i += TK_THREADS)
      f(i, canon(__ldg(g + ly.offset + i), e ? __ldg(e + ly.offset + i) : 0.f));
  }
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
  return __reduce_add_sync(LG_FULL, v);
}

// ---------------------------------------------------------------------------
// P1: level-1 histogram (counts + fixed-point x^2 sums), CTA-private, two copies
// ---------------------------------------------------------------------------
// Per-lane update of the CTA-private level-1 histogram: the count and, with WS, the
// fixed-point M^2 >> 16 (< 2^32) as two 16-bit halves in 32-bit counters (a copy sees
// <= TK_CHUNK/2 = 2^13 keys: each half-sum < 2^29) -- 32-bit shared atomics are ~4x
// faster than 64-bit ones here.  (Warp aggregation by match.any + redux was measured
// 4.7x slower on C3.)
template <bool WS>
__device__ __forceinline__ void h1_add(uint32_t* scnt, uint32_t* shi, uint32_t* slo, uint32_t b, uint32_t key,
                                       bool active) {
  if (!active) return;
  atomicAdd(&scnt[b], 1u);
  if (WS) {
    const uint32_t v = (uint32_t)fx_sq(key);
    atomicAdd(&shi[b], v >> 16);
    atomicAdd(&slo[b], v & 0xFFFFu);
  }
}

template <bool WS>
__global__ void __launch_bounds__(TK_THREADS)
k_tk_pass1(const float* __restrict__ g, const float* __restrict__ e, TkArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* scnt = reinterpret_cast<uint32_t*>(smem);  // [2][2048]
  uint32_t* shi = scnt + 2 * 2048;                      // [2][2048] (WS)
  uint32_t* slo = shi + 2 * 2048;                       // [2][2048] (WS)
  for (int i = threadIdx.x; i < 2 * 2048; i += TK_THREADS) { scnt[i] = 0; if (WS) { shi[i] = 0; slo[i] = 0; } }
  __syncthreads();
  const TChunk ch = a.chunks[blockIdx.x];
  const DevLayer ly = a.layers[a.clayer[ch.cidx]];
  const int cp = (threadIdx.x >> 7) & 1;
  uint32_t zc = 0, bad = 0;
  uint32_t* mc = scnt + cp * 2048;
  uint32_t* mh = shi + cp * 2048;
  uint32_t* ml = slo + cp * 2048;
  for_chunk(g, e, ly, ch, [&](int64_t, float x) {
    const uint32_t key = tkey(x);
    if (key == 0) { ++zc; return; }
    bad |= (key >= 0x7F800000u);
    h1_add<WS>(mc, mh, ml, key >> 20, key, true);
  });
  zc = warp_sum_u32(zc);
  bad = __reduce_or_sync(LG_FULL, bad);
  if ((threadIdx.x & 31) == 0) {
    if (zc) atomicAdd(&mc[0], zc);
    if (bad) atomicOr(a.flag, 1u);
  }
  __syncthreads();
  uint32_t* gc = a.cnt1 + (int64_t)ch.cidx * 2048;
  unsigned long long* gs = a.sum1 + (int64_t)ch.cidx * 2048;
  for (int b = threadIdx.x; b < 2048; b += TK_THREADS) {
    const uint32_t c = scnt[b] + scnt[2048 + b];
    if (c) {
      atomicAdd(gc + b, c);
      if (WS) {
        const unsigned long long s2 = (((unsigned long long)shi[b] + shi[2048 + b]) << 16) +
                                      (unsigned long long)slo[b] + slo[2048 + b];
        if (s2) atomicAdd(gs + b, s2);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// S1: per layer, locate every query's level-1 bin; assign level-2 slots
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(TK_THREADS)
k_tk_select1(TkArgs a, int nq) {
  __shared__ uint32_t suf[2049];
  __shared__ double pre[2048];
  __shared__ uint32_t tot[TK_THREADS];
  __shared__ double dtot[TK_THREADS];
  __shared__ uint32_t bitmap[64];
  __shared__ uint32_t wpre[65];
  const int c = blockIdx.x, tid = threadIdx.x;
  const uint32_t* cnt = a.cnt1 + (int64_t)c * 2048;
  const unsigned long long* sum = a.sum1 + (int64_t)c * 2048;
  // thread tid owns bins [8 tid, 8 tid + 8)
  uint32_t lc[8];
  double lv[8];
  uint32_t tc = 0;
  double tv = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int b = 8 * tid + i;
    lc[i] = cnt[b];
    lv[i] = (double)sum[b] * fx_scale(b);
    tc += lc[i];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) tv += lv[i];
  tot[tid] = tc;
  dtot[tid] = tv;
  if (tid < 64) bitmap[tid] = 0;
  __syncthreads();
  // inclusive scans (fixed Hillis-Steele pattern: deterministic)
  for (int o = 1; o < TK_THREADS; o <<= 1) {
    uint32_t x = 0;
    double y = 0.0;
    if (tid + o < TK_THREADS) x = tot[tid + o];   // suffix for counts
    if (tid >= o) y = dtot[tid - o];              // prefix for values
    __syncthreads();
    tot[tid] += x;
    dtot[tid] += y;
    __syncthreads();
  }
  uint32_t s = (tid + 1 < TK_THREADS) ? tot[tid + 1] : 0u;  // counts strictly above my bins
  double p = (tid > 0) ? dtot[tid - 1] : 0.0;                // values strictly below my bins
#pragma unroll
  for (int i = 7; i >= 0; --i) { s += lc[i]; suf[8 * tid + i] = s; }
#pragma unroll
  for (int i = 0; i < 8; ++i) { pre[8 * tid + i] = p; p += lv[i]; }
  if (tid == 0) suf[2048] = 0;
  __syncthreads();
  const bool nonfinite = suf[2040] != 0;  // bins 2040.. hold exponent 255 (inf / NaN)
  for (int q = tid; q < nq; q += TK_THREADS) {
    TQ& t = a.q[(int64_t)c * nq + q];
    const int64_t k = a.kq[(int64_t)c * nq + q];
    t.k = k;
    int lo = 0, hi = 2047;  // largest b with suf[b] >= k
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((int64_t)suf[mid] >= k) lo = mid; else hi = mid - 1;
    }
    t.b1 = lo;
    t.r = k - (int64_t)suf[lo + 1];
    t.below = pre[lo];
    t.bad = nonfinite;
    atomicOr(&bitmap[lo >> 5], 1u << (lo & 31));
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t acc = 0;
    for (int w = 0; w < 64; ++w) { wpre[w] = acc; acc += __popc(bitmap[w]); }
    wpre[64] = acc;
    a.n1[c] = (int32_t)acc;
  }
  __syncthreads();
  for (int b = tid; b < 2048; b += TK_THREADS)
    if (bitmap[b >> 5] & (1u << (b & 31)))
      a.sl1[(int64_t)c * nq + wpre[b >> 5] + __popc(bitmap[b >> 5] & ((1u << (b & 31)) - 1u))] = b;
  for (int q = tid; q < nq; q += TK_THREADS) {
    TQ& t = a.q[(int64_t)c * nq + q];
    const int b = t.b1;
    t.s1 = c * nq + (int)(wpre[b >> 5] + __popc(bitmap[b >> 5] & ((1u << (b & 31)) - 1u)));
  }
  // zero the level-2 histograms of the used slots
  const int n1 = (int)wpre[64];
  for (int64_t i = tid; i < (int64_t)n1 * 1024; i += TK_THREADS) {
    a.cnt2[(int64_t)c * nq * 1024 + i] = 0;
    a.sum2[(int64_t)c * nq * 1024 + i] = 0;
  }
}

// ---------------------------------------------------------------------------
// P2: level-2 histograms of the boundary level-1 bins
// ---------------------------------------------------------------------------
template <bool WS>
__global__ void __launch_bounds__(TK_THREADS)
k_tk_pass2(const float* __restrict__ g, const float* __restrict__ e, TkArgs a, int nq) {
  __shared__ uint8_t tbl[2048];
  const TChunk ch = a.chunks[blockIdx.x];
  const int c = ch.cidx;
  const DevLayer ly = a.layers[a.clayer[c]];
  for (int i = threadIdx.x; i < 2048; i += TK_THREADS) tbl[i] = 0xFF;
  __syncthreads();
  const int n1 = a.n1[c];
  for (int i = threadIdx.x; i < n1; i += TK_THREADS) tbl[a.sl1[(int64_t)c * nq + i]] = (uint8_t)i;
  __syncthreads();
  uint32_t* c2 = a.cnt2 + (int64_t)c * nq * 1024;
  unsigned long long* s2 = a.sum2 + (int64_t)c * nq * 1024;
  __shared__ int s_kn;
  if (threadIdx.x == 0) s_kn = 0;
  __syncthreads();
  uint32_t* ck = a.ckeys + (int64_t)blockIdx.x * TK_CKCAP;
  uint32_t zc = 0;
  __shared__ unsigned s_zc;
  if (threadIdx.x == 0) s_zc = 0;
  __syncthreads();
  for_chunk(g, e, ly, ch, [&](int64_t, float x) {
    const uint32_t key = tkey(x);
    const uint32_t s = tbl[key >> 20];
    if (s == 0xFF) return;
    if (key == 0) { ++zc; return; }  // zeros are counted, not compacted (pass 3 adds ckz)
    // keep the key for pass 3 (order-free counting): no re-read of the chunk there
    const int pos = atomicAdd(&s_kn, 1);
    if (pos < TK_CKCAP) ck[pos] = key;
    const int64_t idx = (int64_t)s * 1024 + ((key >> 10) & 1023u);
    atomicAdd(c2 + idx, 1u);
    if (WS) atomicAdd(s2 + idx, fx_sq(key));
  });
  zc = warp_sum_u32(zc);
  if ((threadIdx.x & 31) == 0 && zc) {
    atomicAdd(c2 + (int64_t)tbl[0] * 1024, zc);
    atomicAdd(&s_zc, zc);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a.ckn[blockIdx.x] = s_kn;  // > TK_CKCAP: pass 3 rescans the chunk
    a.ckz[blockIdx.x] = (int32_t)s_zc;
  }
}

// scan a 1024-bin count histogram from the top with one warp: returns the bin holding
// the r-th largest (1-based) and the residual rank inside it.
__device__ __forceinline__ void warp_find_from_top(const uint32_t* __restrict__ h, int64_t r, int lane, int& bin,
                                                   int64_t& rres) {
  uint32_t lc[32];
  uint32_t tot = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) { lc[i] = h[32 * lane + i]; tot += lc[i]; }
  // exclusive suffix over lanes: counts held by higher lanes
  uint32_t above = 0;
  for (int j = 31; j > 0; --j) {
    const uint32_t v = __shfl_sync(LG_FULL, tot, j);
    if (j > lane) above += v;
  }
  const bool mine = ((int64_t)above < r) && (r <= (int64_t)above + tot);
  const uint32_t who = __ballot_sync(LG_FULL, mine);
  const int src = __ffs(who) - 1;
  int b = 0;
  int64_t rr = 0;
  if (lane == src) {
    uint32_t acc = above;
    for (int i = 31; i >= 0; --i) {
      if ((int64_t)(acc + lc[i]) >= r) { b = 32 * lane + i; rr = r - (int64_t)acc; break; }
      acc += lc[i];
    }
  }
  bin = __shfl_sync(LG_FULL, b, src);
  rres = __shfl_sync(LG_FULL, rr, src);
}

// ---------------------------------------------------------------------------
// S2: refine to the level-2 sub-bin; assign level-3 slots
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(TK_THREADS)
k_tk_select2(TkArgs a, int nq) {
  // one warp per query (grid y: groups of TK_WARPS queries of layer blockIdx.x)
  const int c = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = blockIdx.y * TK_WARPS + warp; q < nq; q += gridDim.y * TK_WARPS) {
    TQ& t = a.q[(int64_t)c * nq + q];
    const uint32_t* h = a.cnt2 + (int64_t)t.s1 * 1024;
    const unsigned long long* hs = a.sum2 + (int64_t)t.s1 * 1024;
    int c2;
    int64_t r2;
    warp_find_from_top(h, t.r, lane, c2, r2);
    // values of the sub-bins strictly below c2, ascending, then a fixed tree
    double v = 0.0;
    for (int i = 0; i < 32; ++i) {
      const int sb = 32 * lane + i;
      if (sb < c2) v += (double)hs[sb];
    }
    v = warp_sum_d(v) * fx_scale(t.b1);
    if (lane == 0) { t.c2 = c2; t.r = r2; t.below += v; }
  }
}

// per layer: distinct (b1, c2) prefixes -> ranks (the level-3 histogram slots)
__global__ void __launch_bounds__(TK_THREADS)
k_tk_select2b(TkArgs a, int nq) {
  const int c = blockIdx.x;
  // distinct (b1, c2) prefixes -> ranks: bitonic sort of <= 256 prefixes in smem
  __shared__ uint32_t sp[256];
  __shared__ uint32_t sfirst[256];
  for (int i = threadIdx.x; i < 256; i += TK_THREADS)
    sp[i] = (i < nq) ? ((((uint32_t)a.q[(int64_t)c * nq + i].b1) << 10) | (uint32_t)a.q[(int64_t)c * nq + i].c2)
                     : 0xFFFFFFFFu;
  __syncthreads();
  for (int k2 = 2; k2 <= 256; k2 <<= 1)
    for (int j = k2 >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < 256; i += TK_THREADS) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k2) == 0;
          const uint32_t x = sp[i], y = sp[ixj];
          if ((x > y) == up) { sp[i] = y; sp[ixj] = x; }
        }
      }
      __syncthreads();
    }
  // rank of each distinct value = number of distinct values before it
  for (int i = threadIdx.x; i < 256; i += TK_THREADS) sfirst[i] = (i == 0 || sp[i] != sp[i - 1]) && sp[i] != 0xFFFFFFFFu;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t r = 0;
    for (int i = 0; i < 256; ++i) {
      const uint32_t f = sfirst[i];
      if (f) a.sl2[(int64_t)c * nq + r] = sp[i];
      sfirst[i] = r;  // rank of the group starting at i (valid where first)
      r += f;
    }
    a.n2[c] = (int32_t)r;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nq; q += TK_THREADS) {
    TQ& t = a.q[(int64_t)c * nq + q];
    const uint32_t p = ((uint32_t)t.b1 << 10) | (uint32_t)t.c2;
    int lo = 0, hi = 255;  // first index with sp >= p
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sp[mid] < p) lo = mid + 1; else hi = mid;
    }
    t.s2 = c * nq + (int)sfirst[lo];
  }
}

// ---------------------------------------------------------------------------
// P3: exact-key counts inside the boundary level-2 sub-bins
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(TK_THREADS)
k_tk_pass3(const float* __restrict__ g, const float* __restrict__ e, TkArgs a, int nq) {
  __shared__ uint8_t tbl[2048];
  __shared__ uint32_t pre[256];
  const TChunk ch = a.chunks[blockIdx.x];
  const int c = ch.cidx;
  const DevLayer ly = a.layers[a.clayer[c]];
  for (int i = threadIdx.x; i < 2048; i += TK_THREADS) tbl[i] = 0xFF;
  __syncthreads();
  const int n1 = a.n1[c], n2 = a.n2[c];
  for (int i = threadIdx.x; i < n1; i += TK_THREADS) tbl[a.sl1[(int64_t)c * nq + i]] = (uint8_t)i;
  for (int i = threadIdx.x; i < n2; i += TK_THREADS) pre[i] = a.sl2[(int64_t)c * nq + i];
  __syncthreads();
  uint32_t* c3 = a.cnt3 + (int64_t)c * nq * 1024;
  uint32_t zc = 0;
  auto count = [&](uint32_t key) {
    if (tbl[key >> 20] == 0xFF) return;
    const uint32_t p = key >> 10;
    int lo = 0, hi = n2 - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] < p) lo = mid + 1; else hi = mid;
    }
    if (pre[lo] != p) return;
    if (key == 0) { ++zc; return; }
    atomicAdd(c3 + (int64_t)lo * 1024 + (key & 1023u), 1u);
  };
  const int kn = a.ckn[blockIdx.x];
  if (kn <= TK_CKCAP) {  // the chunk's boundary keys, compacted by pass 2 (zeros counted there)
    const uint32_t* ck = a.ckeys + (int64_t)blockIdx.x * TK_CKCAP;
    for (int i = threadIdx.x; i < kn; i += TK_THREADS) count(ck[i]);
    if (threadIdx.x == 0) zc += (uint32_t)a.ckz[blockIdx.x];
  } else {
    for_chunk(g, e, ly, ch, [&](int64_t, float x) { count(tkey(x)); });
  }
  zc = warp_sum_u32(zc);
  if ((threadIdx.x & 31) == 0 && zc && n2 > 0 && pre[0] == 0) atomicAdd(c3, zc);
}

// ---------------------------------------------------------------------------
// S3: exact threshold, kept ties and SSE; profile output
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(TK_THREADS)
k_tk_select3(TkArgs a, int nq, double* __restrict__ err, int64_t* __restrict__ bits, int K) {
  const int c = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int l = a.clayer[c];
  for (int q = blockIdx.y * TK_WARPS + warp; q < nq; q += gridDim.y * TK_WARPS) {
    TQ& t = a.q[(int64_t)c * nq + q];
    const uint32_t* h = a.cnt3 + (int64_t)t.s2 * 1024;
    const uint32_t p = ((uint32_t)t.b1 << 10) | (uint32_t)t.c2;
    int t3;
    int64_t r3;
    warp_find_from_top(h, t.r, lane, t3, r3);
    double v = 0.0;
    for (int i = 0; i < 32; ++i) {
      const int tb = 32 * lane + i;
      if (tb < t3 && h[tb]) v += (double)h[tb] * key_sq((p << 10) | (uint32_t)tb);
    }
    v = warp_sum_d(v);
    if (lane == 0) {
      const uint32_t T = (p << 10) | (uint32_t)t3;
      const double sse = t.below + v + (double)((int64_t)h[t3] - r3) * key_sq(T);
      t.T = T;
      t.r = r3;
      t.ties = h[t3];
      t.sse = t.bad ? __longlong_as_double(0x7ff8000000000000ll) : sse;
      if (err) {
        err[(int64_t)l * K + q] = sqrt(t.sse);
        bits[(int64_t)l * K + q] = 64 * t.k;
      }
    }
  }
}

// lossless layers of the profile table: err 0, bits 32 n
__global__ void k_tk_lossless_rows(const DevLayer* __restrict__ layers, int L, int K, double* __restrict__ err,
                                   int64_t* __restrict__ bits) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)L * K; i += (int64_t)gridDim.x * blockDim.x) {
    const DevLayer ly = layers[i / K];
    if (!ly.compress) { err[i] = 0.0; bits[i] = 32 * ly.numel; }
  }
}

// ---------------------------------------------------------------------------
// K6 compaction: counts, scan, write
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(TK_THREADS)
k_tk_count(const float* __restrict__ g, const float* __restrict__ e, TkArgs a) {
  __shared__ uint32_t sg[TK_WARPS], se[TK_WARPS];
  const TChunk ch = a.chunks[blockIdx.x];
  const DevLayer ly = a.layers[a.clayer[ch.cidx]];
  const TQ qq = a.q[ch.cidx];
  const uint32_t T = qq.T;
  if (a.kq[ch.cidx] == 0 ||  // a skipped layer (NEXT-4)
      (!a.need_off && (qq.r == 0 || qq.r == qq.ties))) {  // every tie kept or none: no prefix needed
    if (threadIdx.x == 0) a.ccnt[blockIdx.x] = make_uint2(0u, 0u);
    return;
  }
  uint32_t gt = 0, eq = 0;
  for_chunk(g, e, ly, ch, [&](int64_t, float x) {
    const uint32_t key = tkey(x);
    gt += key > T;
    eq += key == T;
  });
  gt = warp_sum_u32(gt);
  eq = warp_sum_u32(eq);
  if ((threadIdx.x & 31) == 0) { sg[threadIdx.x >> 5] = gt; se[threadIdx.x >> 5] = eq; }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t G = 0, Q = 0;
    for (int w = 0; w < TK_WARPS; ++w) { G += sg[w]; Q += se[w]; }
    a.ccnt[blockIdx.x] = make_uint2(G, Q);
  }
}

// per compressed layer: exclusive scan of (gt, eq) over its chunks -> offsets
__global__ void __launch_bounds__(TK_THREADS)
k_tk_scan(TkArgs a) {
  __shared__ unsigned long long sg[TK_THREADS], se[TK_THREADS];
  const int c = blockIdx.x, tid = threadIdx.x;
  {  // no payload and a tie-trivial (or skipped) layer: its offsets are never read
    const TQ qq = a.q[c];
    if (!a.need_off && (a.kq[c] == 0 || qq.r == 0 || qq.r == qq.ties)) return;
  }
  const int c0 = a.cchunk0[c], c1 = a.cchunk0[c + 1];
  unsigned long long baseg = 0, basee = 0;
  for (int s = c0; s < c1; s += TK_THREADS) {
    const int i = s + tid;
    const uint2 v = (i < c1) ? a.ccnt[i] : make_uint2(0, 0);
    sg[tid] = v.x;
    se[tid] = v.y;
    __syncthreads();
    for (int o = 1; o < TK_THREADS; o <<= 1) {
      const unsigned long long x = tid >= o ? sg[tid - o] : 0ull, y = tid >= o ? se[tid - o] : 0ull;
      __syncthreads();
      sg[tid] += x;
      se[tid] += y;
      __syncthreads();
    }
    if (i < c1) a.coff[i] = make_ulonglong2(baseg + sg[tid] - v.x, basee + se[tid] - v.y);
    baseg += sg[TK_THREADS - 1];
    basee += se[TK_THREADS - 1];
    __syncthreads();
  }
}

// write pass: elements in index order, 4 per thread per iteration
__global__ void __launch_bounds__(TK_THREADS)
k_tk_write(const float* __restrict__ g, float* __restrict__ ef, uint8_t* __restrict__ payload,
           float* __restrict__ out, TkArgs a) {
  __shared__ uint32_t wk[TK_WARPS], we[TK_WARPS];
  const TChunk ch = a.chunks[blockIdx.x];
  const int c = ch.cidx;
  const int l = a.clayer[c];
  const DevLayer ly = a.layers[l];
  const TQ q = a.q[c];
  const uint32_t T = q.T;
  if (a.kq[c] == 0) return;  // a skipped layer (NEXT-4): EF and output untouched
  // no payload and every tie kept or none: k_tk_count / k_tk_scan skipped this layer, its
  // offsets were never written -- the tie rule needs none (r = 0: no tie, r = ties: all)
  const bool trivial = !a.need_off && (q.r == 0 || q.r == q.ties);
  const int64_t rties = trivial ? (q.r == 0 ? (int64_t)0 : INT64_MAX) : q.r;
  const ulonglong2 off = trivial ? make_ulonglong2(0ull, 0ull) : a.coff[blockIdx.x];
  uint2* pairs = payload ? reinterpret_cast<uint2*>(payload + a.tplan[l].pay_off) : nullptr;
  int64_t eq_run = (int64_t)off.y;                                       // ties before this position
  int64_t kept_run = (int64_t)off.x + min((int64_t)off.y, rties);        // kept entries before
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool aligned = ((ly.offset + ch.first) & 3) == 0;
  const int64_t end = ch.first + ch.n;
  for (int64_t base = ch.first; base < end; base += 4 * TK_THREADS) {
    const int64_t i0 = base + 4 * threadIdx.x;
    float x[4];
    int nv = (int)max((int64_t)0, min((int64_t)4, end - i0));
    if (aligned && nv == 4) {
      const float4 gv = __ldg(reinterpret_cast<const float4*>(g + ly.offset + i0));
      const float4 ev = ef ? *reinterpret_cast<const float4*>(ef + ly.offset + i0) : make_float4(0.f, 0.f, 0.f, 0.f);
      x[0] = canon(gv.x, ev.x); x[1] = canon(gv.y, ev.y); x[2] = canon(gv.z, ev.z); x[3] = canon(gv.w, ev.w);
    } else {
#pragma unroll
      for (int s = 0; s < 4; ++s)
        x[s] = (s < nv) ? canon(__ldg(g + ly.offset + i0 + s), ef ? ef[ly.offset + i0 + s] : 0.f) : 0.f;
    }
    uint32_t isgt[4], iseq[4];
    uint32_t neq = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const uint32_t key = tkey(x[s]);
      isgt[s] = (s < nv) && key > T;
      iseq[s] = (s < nv) && key == T;
      neq += iseq[s];
    }
    // exclusive prefix of ties across the block (index order)
    uint32_t ex_eq = neq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(LG_FULL, ex_eq, o);
      if (lane >= o) ex_eq += v;
    }
    if (lane == 31) we[warp] = ex_eq;
    ex_eq -= neq;
    __syncthreads();
    uint32_t wbefore_e = 0, tot_e = 0;
    for (int w = 0; w < TK_WARPS; ++w) { if (w < warp) wbefore_e += we[w]; tot_e += we[w]; }
    int64_t er = eq_run + wbefore_e + ex_eq;  // tie rank of my first element
    uint32_t kept[4];
    uint32_t nk = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      kept[s] = isgt[s] || (iseq[s] && er < rties);
      er += iseq[s];
      nk += kept[s];
    }
    uint32_t ex_k = nk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(LG_FULL, ex_k, o);
      if (lane >= o) ex_k += v;
    }
    if (lane == 31) wk[warp] = ex_k;
    ex_k -= nk;
    __syncthreads();
    uint32_t wbefore_k = 0, tot_k = 0;
    for (int w = 0; w < TK_WARPS; ++w) { if (w < warp) wbefore_k += wk[w]; tot_k += wk[w]; }
    int64_t pos = kept_run + wbefore_k + ex_k;
    float en[4], dv[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (kept[s]) {
        if (pairs) pairs[pos] = make_uint2((uint32_t)(i0 + s), __float_as_uint(x[s]));
        ++pos;
      }
      en[s] = kept[s] ? 0.f : x[s];
      dv[s] = kept[s] ? x[s] : 0.f;
    }
    if (aligned && nv == 4) {
      if (ef) *reinterpret_cast<float4*>(ef + ly.offset + i0) = make_float4(en[0], en[1], en[2], en[3]);
      if (out) *reinterpret_cast<float4*>(out + ly.offset + i0) = make_float4(dv[0], dv[1], dv[2], dv[3]);
    } else {
#pragma unroll
      for (int s = 0; s < 4; ++s)
        if (s < nv) {
          if (ef) ef[ly.offset + i0 + s] = en[s];
          if (out) out[ly.offset + i0 + s] = dv[s];
        }
    }
    eq_run += tot_e;
    kept_run += tot_k;
    __syncthreads();
  }
}

// lossless layers (any family): raw payload, e' = 0, out = x (W == 1)
__global__ void __launch_bounds__(TK_THREADS)
k_lossless_pack(const float* __restrict__ g, float* __restrict__ ef, uint8_t* __restrict__ payload,
                float* __restrict__ out, const DevLayer* __restrict__ layers, const TChunk* __restrict__ chunks,
                const TPlan* __restrict__ tplan, unsigned* __restrict__ flag, const int32_t* __restrict__ choice) {
  const TChunk ch = chunks[blockIdx.x];  // cidx = layer index here
  if (choice && choice[ch.cidx] == LGRECO_CHOICE_SKIP) return;  // another family's ctx owns it (NEXT-4)
  const DevLayer ly = layers[ch.cidx];
  float* raw = payload ? reinterpret_cast<float*>(payload + tplan[ch.cidx].pay_off) : nullptr;
  float bad = 0.f;
  for (int64_t i = ch.first + threadIdx.x; i < ch.first + ch.n; i += TK_THREADS) {
    const float x = canon(__ldg(g + ly.offset + i), ef ? ef[ly.offset + i] : 0.f);
    bad = __fadd_rn(bad, __fmul_rn(x, 0.f));
    if (raw) raw[i] = x;
    if (out) out[ly.offset + i] = x;
    if (ef) ef[ly.offset + i] = 0.f;
  }
  if (!isfinite(bad)) atomicOr(flag, 1u);
}

// ---------------------------------------------------------------------------
// K10 exchange combine
// ---------------------------------------------------------------------------
// lossless layers: out = (ordered sum over ranks of the raw payloads) * fl(1/W); compressed: 0
__global__ void __launch_bounds__(TK_THREADS)
k_tk_combine_init(const uint8_t* __restrict__ gathered, int64_t S, int W, float* __restrict__ out,
                  const DevLayer* __restrict__ layers, const TChunk* __restrict__ chunks,
                  const TPlan* __restrict__ tplan) {
  const TChunk ch = chunks[blockIdx.x];  // chunks over ALL layers, cidx = layer
  if (tplan[ch.cidx].k < 0) return;  // another family's layer (NEXT-4): output untouched
  const DevLayer ly = layers[ch.cidx];
  const float invW = __fdiv_rn(1.0f, (float)W);
  for (int64_t i = ch.first + threadIdx.x; i < ch.first + ch.n; i += TK_THREADS) {
    float v = 0.f;
    if (!ly.compress) {
      for (int w = 0; w < W; ++w) {
        const float r = __ldg(reinterpret_cast<const float*>(gathered + w * S + tplan[ch.cidx].pay_off) + i);
        v = (w == 0) ? r : __fadd_rn(v, r);
      }
      v = __fmul_rn(v, invW);
    }
    out[ly.offset + i] = v;
  }
}

// rank w's pairs: out[idx] += val * fl(1/W) (launched once per rank, in rank order)
__global__ void __launch_bounds__(TK_THREADS)
k_tk_scatter(const uint8_t* __restrict__ pay_w, int W, float* __restrict__ out, const DevLayer* __restrict__ layers,
             const int32_t* __restrict__ clayer, int nC, const int64_t* __restrict__ kpre, const TPlan* __restrict__ tplan) {
  __shared__ int64_t sk[1025];
  const int n = min(nC, 1024);
  for (int i = threadIdx.x; i <= n; i += TK_THREADS) sk[i] = kpre[i];
  __syncthreads();
  const float invW = __fdiv_rn(1.0f, (float)W);
  const int64_t total = kpre[nC];
  for (int64_t t = (int64_t)blockIdx.x * TK_THREADS + threadIdx.x; t < total; t += (int64_t)gridDim.x * TK_THREADS) {
    int lo = 0, hi = nC - 1;
    while (lo < hi) {  // largest c with kpre[c] <= t
      const int mid = (lo + hi + 1) >> 1;
      const int64_t v = mid <= n ? sk[mid] : kpre[mid];
      if (v <= t) lo = mid; else hi = mid - 1;
    }
    const int l = clayer[lo];
    const uint2 pr = __ldg(reinterpret_cast<const uint2*>(pay_w + tplan[l].pay_off) + (t - (lo <= n ? sk[lo] : kpre[lo])));
    float* o = out + layers[l].offset + pr.x;
    *o = __fadd_rn(*o, __fmul_rn(__uint_as_float(pr.y), invW));
  }
}

// device-side k per compressed layer from the device-resident choice (W == 1 path)
__global__ void k_plan_topk_dev(const int32_t* __restrict__ choice, const int32_t* __restrict__ params, int K,
                                const DevLayer* __restrict__ layers, const int32_t* __restrict__ clayer, int nC,
                                int64_t* __restrict__ kplan, unsigned* __restrict__ flag) {
  for (int ci = blockIdx.x * blockDim.x + threadIdx.x; ci < nC; ci += gridDim.x * blockDim.x) {
    const int l = clayer[ci];
    int c = choice[l];
    if (c == LGRECO_CHOICE_SKIP) { kplan[ci] = 0; continue; }  // another family's layer (NEXT-4)
    if (c < 0 || c >= K) { atomicOr(flag, 2u); c = 0; }
    const int64_t n = layers[l].numel;
    int64_t k = ((int64_t)params[c] * n + 999999) / 1000000;
    kplan[ci] = k < 1 ? 1 : (k > n ? n : k);
  }
}

cudaError_t launch_plan_topk_dev(const int32_t* choice, const int32_t* params, int K, const DevLayer* layers,
                                 const int32_t* clayer, int nC, int64_t* kplan, unsigned* flag, cudaStream_t st) {
  if (nC == 0) return cudaSuccess;
  k_plan_topk_dev<<<(nC + 255) / 256, 256, 0, st>>>(choice, params, K, layers, clayer, nC, kplan, flag);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_topk_select(const float* g, const float* e, const TkArgs& a, int nq, double* err, int64_t* bits,
                               int K, cudaStream_t st, int64_t* launches) {
  if (a.nC == 0 || a.nchunks == 0) return cudaSuccess;
  cudaError_t r = cudaMemsetAsync(a.cnt1, 0, sizeof(uint32_t) * 2048 * (size_t)a.nC, st);
  if (r == cudaSuccess && err) r = cudaMemsetAsync(a.sum1, 0, sizeof(unsigned long long) * 2048 * (size_t)a.nC, st);
  if (r != cudaSuccess) return r;
  const bool ws = err != nullptr;  // the compress select needs no energy sums
  const size_t sm1 = 2 * 2048 * (ws ? 12 : 4);
  r = memo_smem_attr((const void*)k_tk_pass1<true>, 2 * 2048 * 12);
  if (r != cudaSuccess) return r;
  if (ws) k_tk_pass1<true><<<a.nchunks, TK_THREADS, sm1, st>>>(g, e, a);
  else k_tk_pass1<false><<<a.nchunks, TK_THREADS, sm1, st>>>(g, e, a);
  k_tk_select1<<<a.nC, TK_THREADS, 0, st>>>(a, nq);
  if (ws) k_tk_pass2<true><<<a.nchunks, TK_THREADS, 0, st>>>(g, e, a, nq);
  else k_tk_pass2<false><<<a.nchunks, TK_THREADS, 0, st>>>(g, e, a, nq);
  const dim3 gq(a.nC, (nq + TK_WARPS - 1) / TK_WARPS);  // a warp per query
  k_tk_select2<<<gq, TK_THREADS, 0, st>>>(a, nq);
  k_tk_select2b<<<a.nC, TK_THREADS, 0, st>>>(a, nq);
  // level-3 histograms (every slot a layer may use: nC x nq x 1024) zeroed at full width
  r = cudaMemsetAsync(a.cnt3, 0, sizeof(uint32_t) * 1024 * (size_t)a.nC * nq, st);
  if (r != cudaSuccess) return r;
  k_tk_pass3<<<a.nchunks, TK_THREADS, 0, st>>>(g, e, a, nq);
  k_tk_select3<<<gq, TK_THREADS, 0, st>>>(a, nq, err, bits, K);
  *launches += 7;
  return cudaGetLastError();
}

cudaError_t launch_topk_lossless_rows(const DevLayer* layers, int L, int K, double* err, int64_t* bits, cudaStream_t st) {
  k_tk_lossless_rows<<<64, 256, 0, st>>>(layers, L, K, err, bits);
  return cudaGetLastError();
}

// compress queries from the preceding profile's (same x): qc[c] = qprof[c K + choice[layer]]
__global__ void k_tk_reuse(const int32_t* __restrict__ choice, int K, const int32_t* __restrict__ clayer, int nC,
                           const TQ* __restrict__ qprof, TQ* __restrict__ qc, unsigned* __restrict__ flag) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nC; c += gridDim.x * blockDim.x) {
    int j = choice[clayer[c]];
    if (j == LGRECO_CHOICE_SKIP) continue;  // (the layer's kplan is 0: count / write skip it)
    if (j < 0 || j >= K) { atomicOr(flag, 2u); j = 0; }
    qc[c] = qprof[(int64_t)c * K + j];
  }
}

cudaError_t launch_topk_reuse(const int32_t* choice, int K, const int32_t* clayer, int nC, const TQ* qprof, TQ* qc,
                              unsigned* flag, cudaStream_t st) {
  if (nC == 0) return cudaSuccess;
  k_tk_reuse<<<(nC + 255) / 256, 256, 0, st>>>(choice, K, clayer, nC, qprof, qc, flag);
  return cudaGetLastError();
}

cudaError_t launch_topk_compact(const float* g, float* ef, uint8_t* payload, float* out, const TkArgs& a,
                                cudaStream_t st) {
  if (a.nC == 0 || a.nchunks == 0) return cudaSuccess;
  k_tk_count<<<a.nchunks, TK_THREADS, 0, st>>>(g, ef, a);
  k_tk_scan<<<a.nC, TK_THREADS, 0, st>>>(a);
  k_tk_write<<<a.nchunks, TK_THREADS, 0, st>>>(g, ef, payload, out, a);
  return cudaGetLastError();
}

cudaError_t launch_lossless_pack(const float* g, float* ef, uint8_t* payload, float* out, const int32_t* choice,
                                 const DevLayer* layers,
                                 const TChunk* chunks, int nchunks, const TPlan* tplan, unsigned* flag,
                                 cudaStream_t st) {
  if (nchunks == 0) return cudaSuccess;
  k_lossless_pack<<<nchunks, TK_THREADS, 0, st>>>(g, ef, payload, out, layers, chunks, tplan, flag, choice);
  return cudaGetLastError();
}

cudaError_t launch_topk_combine(const uint8_t* gathered, int64_t S, int W, float* out, const DevLayer* layers,
                                const TChunk* all_chunks, int nall, const int32_t* clayer,
                                int nC, const int64_t* kpre, int64_t ktotal, const TPlan* tplan, cudaStream_t st,
                                int64_t* launches) {
  if (nall) k_tk_combine_init<<<nall, TK_THREADS, 0, st>>>(gathered, S, W, out, layers, all_chunks, tplan);
  *launches += nall ? 1 : 0;
  if (ktotal > 0) {
    const int grid = (int)std::min<int64_t>((ktotal + TK_THREADS - 1) / TK_THREADS, 148 * 16);
    for (int w = 0; w < W; ++w) {
      k_tk_scatter<<<grid, TK_THREADS, 0, st>>>(gathered + w * S, W, out, layers, clayer, nC, kpre, tplan);
      *launches += 1;
    }
  }
  return cudaGetLastError();
}

}  // namespace lg
