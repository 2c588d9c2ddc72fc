// psgd_tc.cu -- PowerSGD's P = M Q on the 5th-generation tensor cores (tcgen05).
//
// D[128 x N] (fp32, TMEM) += A[128 x 8] . B[8 x N] per tcgen05.mma.kind::tf32; three
// products per K-slice (3xTF32: Ah.Bh + Ah.Bl + Al.Bh, x = hi + lo, hi = x with the
// low 13 mantissa bits cleared) recover fp32-grade accuracy (plain TF32
// misses the 1e-5 parity on P by 4e-4; 3xTF32 matches fp32 at 5e-7).
//
// A = the M tile (128 rows of the layer view x 32 K-elements), staged by the CTA's
// threads from x = fl(fl(g + e) + 0) straight into the 128B-swizzled K-major canonical
// layout (8-row groups of 1024 B, 16-byte chunk c of row r at c ^ (r & 7)); B = 32
// K-elements of the r columns of Q (column-major, hence K-major too).  Two smem
// stages: the threads stage tile k+1 while the elected thread's MMAs consume tile k
// (completion tracked by tcgen05.commit -> mbarrier).  Every K tile accumulates into its
// own TMEM buffer (two, ping-pong): measured on B200, chaining hundreds of MMAs in one
// accumulator drifts by ~3e-5 relative (the in-MMA accumulation is not RN fp32), while
// a 12-MMA tile stays at ~7e-7; tile partials are added in registers in fp32 (RN) while
// the next tile's MMAs run.  tcgen05.ld 32x32b: warp w reads TMEM lanes 32w..32w+31 =
// tile rows -> column-major P.
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace lg {

constexpr int TC_M = 128;      // rows per tile (UMMA_M)
constexpr int TC_KT = 32;      // K elements per stage (one 128-byte swizzle row)
constexpr int TC_THREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// SW128 K-major smem descriptor (cute::UMMA::SmemDescriptor layout)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
  d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;              // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                        // version (sm100)
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}

// instruction descriptor: kind::tf32, D f32, A/B tf32, B K-major, A K- or MN-major, M = 128, N
__host__ __device__ constexpr uint32_t tf32_idesc(int N, bool a_mn = false) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(TC_M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

// stage one 16-byte chunk (4 floats) as hi / lo into the swizzled tiles
__device__ __forceinline__ void put_chunk(uint8_t* hi_tile, uint8_t* lo_tile, int row, int chunk, float4 v) {
  const uint32_t off = (uint32_t)row * 128u + (uint32_t)((chunk ^ (row & 7)) << 4);
  const uint32_t h0 = tf32_hi(v.x), h1 = tf32_hi(v.y), h2 = tf32_hi(v.z), h3 = tf32_hi(v.w);
  *reinterpret_cast<uint4*>(hi_tile + off) = make_uint4(h0, h1, h2, h3);
  *reinterpret_cast<uint4*>(lo_tile + off) =
      make_uint4(__float_as_uint(__fsub_rn(v.x, __uint_as_float(h0))), __float_as_uint(__fsub_rn(v.y, __uint_as_float(h1))),
                 __float_as_uint(__fsub_rn(v.z, __uint_as_float(h2))), __float_as_uint(__fsub_rn(v.w, __uint_as_float(h3))));
}

// NP: N padded to a multiple of 16 (16, 32, 64); grouped over layers.
// TRANS = false: P = M Q   -- tile = 128 rows of M, K runs over the k columns,
//                             A = M rows (K-major), B = Q columns, out P[j*m + i]
// TRANS = true:  Q = M^T P -- tile = 128 columns of M, K runs over rows [i0, i1),
//                             A = M^T, transposed while staged from M rows (K-major),
//                             B = P columns, out partial[split][j*k + c]
template <int NP, bool TRANS>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_ps_tc(const float* __restrict__ g, const float* __restrict__ e, const PLayer* __restrict__ pl,
        const PTile* __restrict__ tiles, const float* __restrict__ Bsrc, float* __restrict__ out) {
  constexpr int A_BYTES = TC_M * 128;        // 16 KB per A tile (hi or lo)
  constexpr int B_BYTES = NP * 128;          // per B tile (hi or lo)
  constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * NP < 32 ? 32 : 2 * NP;  // two accumulator buffers
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t mma_done[2];
  __shared__ uint32_t tmem_base_sh;

  const PTile tl = tiles[blockIdx.x];
  const PLayer p = pl[tl.ci];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // tile extent along the MMA M dimension, and the K range
  const int rows = TRANS ? min(TC_M, p.k - tl.c0) : min(TC_M, p.m - tl.i0);
  const int kbeg = TRANS ? tl.i0 : 0;
  const int kend = TRANS ? tl.i1 : p.k;
  const int nk = (kend - kbeg + TC_KT - 1) / TC_KT;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&mma_done[0], 1);
    mbar_init(&mma_done[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_d = tmem_base_sh;
  constexpr uint32_t idesc = tf32_idesc(NP);

  const int row = warp * 32 + lane;
  float acc[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) acc[j] = 0.f;
  // read the finished tile partial of K tile `t` (TMEM buffer t & 1) and add it (fp32 RN)
  auto drain = [&](int t) {
    mbar_wait(&mma_done[t & 1], (t >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
    for (int j0 = 0; j0 < NP; j0 += 16) {
      uint32_t v[16];
      const uint32_t taddr = tmem_d + ((uint32_t)(warp * 32) << 16) + (uint32_t)((t & 1) * NP + j0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[j0 + q] = __fadd_rn(acc[j0 + q], __uint_as_float(v[q]));
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
  };

  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt & 1;
    uint8_t* Ah = smem + s * STAGE;
    uint8_t* Al = Ah + A_BYTES;
    uint8_t* Bh = Al + A_BYTES;
    uint8_t* Bl = Bh + B_BYTES;
    const int k0 = kbeg + kt * TC_KT;
    if (!TRANS) {
      // A: 128 rows x 8 chunks; a warp covers 4 rows x 128 B per instruction (coalesced)
#pragma unroll 4
      for (int it = 0; it < TC_M * 8 / TC_THREADS; ++it) {
        const int idx = it * TC_THREADS + tid;
        const int r_ = idx >> 3, ch = idx & 7;
        const int col = k0 + ch * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r_ < rows) {
          const int64_t base = p.moff + (int64_t)(tl.i0 + r_) * p.k + col;
          if (col + 4 <= kend && ((base & 3) == 0)) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(g + base));
            const float4 b = e ? __ldg(reinterpret_cast<const float4*>(e + base)) : make_float4(0.f, 0.f, 0.f, 0.f);
            v = make_float4(canon(a.x, b.x), canon(a.y, b.y), canon(a.z, b.z), canon(a.w, b.w));
          } else {
            float t[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              t[q] = (col + q < kend) ? canon(__ldg(g + base + q), e ? __ldg(e + base + q) : 0.f) : 0.f;
            v = make_float4(t[0], t[1], t[2], t[3]);
          }
        }
        put_chunk(Ah, Al, r_, ch, v);
      }
    } else {
      // A^T: 32 K-rows (rows i of M) x 128 M-elements (columns c), MN-major:
      // offset = (c/32)*4096 + (kr/8)*1024 + (kr%8)*128 + (((c%32)/4) ^ (kr%8))*16
#pragma unroll 4
      for (int it = 0; it < TC_KT * 32 / TC_THREADS; ++it) {
        const int idx = it * TC_THREADS + tid;
        const int kr = idx >> 5, cq = idx & 31;  // K row, 16-byte chunk along c (4 columns)
        const int i = k0 + kr, c = tl.c0 + cq * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < kend) {
          const int64_t base = p.moff + (int64_t)i * p.k + c;
          if (c + 4 <= tl.c0 + rows && ((base & 3) == 0)) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(g + base));
            const float4 b = e ? __ldg(reinterpret_cast<const float4*>(e + base)) : make_float4(0.f, 0.f, 0.f, 0.f);
            v = make_float4(canon(a.x, b.x), canon(a.y, b.y), canon(a.z, b.z), canon(a.w, b.w));
          } else {
            float t[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              t[q] = (c + q < tl.c0 + rows) ? canon(__ldg(g + base + q), e ? __ldg(e + base + q) : 0.f) : 0.f;
            v = make_float4(t[0], t[1], t[2], t[3]);
          }
        }
        // transpose into the K-major A tile: A row = column c (local cq*4 + q), K = kr.
        // (tcgen05 kind::tf32 does not take an MN-major A here: measured all-zero D.)
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int arow = cq * 4 + q;
          const uint32_t off = (uint32_t)arow * 128u + (uint32_t)((((kr >> 2) ^ (arow & 7))) << 4) + (uint32_t)(kr & 3) * 4u;
          const uint32_t h = tf32_hi(vv[q]);
          *reinterpret_cast<uint32_t*>(Ah + off) = h;
          *reinterpret_cast<uint32_t*>(Al + off) = __float_as_uint(__fsub_rn(vv[q], __uint_as_float(h)));
        }
      }
    }
    // B: NP rows (columns j of Q, resp. of P) x 8 chunks along K
    {
      const int64_t bld = TRANS ? (int64_t)p.m : (int64_t)p.k;   // column length of Bsrc
      const int64_t boff = TRANS ? p.poff : p.qoff;
      for (int idx = tid; idx < NP * 8; idx += TC_THREADS) {
        const int j = idx >> 3, ch = idx & 7;
        const int col = k0 + ch * 4;
        float t[4] = {0.f, 0.f, 0.f, 0.f};
        if (j < p.r) {
#pragma unroll
          for (int q = 0; q < 4; ++q) t[q] = (col + q < kend) ? Bsrc[boff + (int64_t)j * bld + col + q] : 0.f;
        }
        put_chunk(Bh, Bl, j, ch, make_float4(t[0], t[1], t[2], t[3]));
      }
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t sAh = smem_u32(Ah), sAl = smem_u32(Al), sBh = smem_u32(Bh), sBl = smem_u32(Bl);
      const uint32_t dbuf = tmem_d + (uint32_t)(s * NP);
#pragma unroll
      for (int kk = 0; kk < TC_KT / 8; ++kk) {
        const uint32_t koff = kk * 32;  // 8 tf32 = 32 bytes along K inside the swizzle row
        const uint64_t dAh = sw128_desc(sAh + koff);
        const uint64_t dAl = sw128_desc(sAl + koff);
        mma_tf32(dbuf, dAh, sw128_desc(sBh + koff), idesc, kk > 0 ? 1u : 0u);
        mma_tf32(dbuf, dAh, sw128_desc(sBl + koff), idesc, 1u);
        mma_tf32(dbuf, dAl, sw128_desc(sBh + koff), idesc, 1u);
      }
      mma_commit(&mma_done[s]);
    }
    __syncwarp();
    // while tile kt's MMAs run: drain tile kt-1 (this also frees smem stage s^1 and
    // TMEM buffer s^1 for tile kt+1)
    if (kt >= 1) drain(kt - 1);
  }
  drain(nk - 1);
  if (row < rows) {
    if (!TRANS) {
#pragma unroll
      for (int j = 0; j < NP; ++j)
        if (j < p.r) out[p.poff + (int64_t)j * p.m + tl.i0 + row] = acc[j];
    } else {
      float* o = out + (int64_t)tl.split * p.qstride + p.qoff;
#pragma unroll
      for (int j = 0; j < NP; ++j)
        if (j < p.r) o[(int64_t)j * p.k + tl.c0 + row] = acc[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(TMEM_COLS));
}

template <int NP, bool TRANS>
static cudaError_t tc_launch(const PsArgs& a, const PTile* tiles, int ntiles, const float* B, float* out,
                             cudaStream_t st) {
  constexpr int STAGE = 2 * TC_M * 128 + 2 * NP * 128;
  const int smem = 2 * STAGE + 1024;
  cudaError_t e = cudaFuncSetAttribute(k_ps_tc<NP, TRANS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k_ps_tc<NP, TRANS><<<ntiles, TC_THREADS, smem, st>>>(a.g, a.e, a.pl, tiles, B, out);
  return cudaGetLastError();
}

cudaError_t launch_ps_mq_tc(const PsArgs& a, const PTile* tiles128, int ntiles, const float* Q, float* P,
                            cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  if (a.rmax <= 16) return tc_launch<16, false>(a, tiles128, ntiles, Q, P, st);
  if (a.rmax <= 32) return tc_launch<32, false>(a, tiles128, ntiles, Q, P, st);
  return tc_launch<64, false>(a, tiles128, ntiles, Q, P, st);
}

cudaError_t launch_ps_mtp_tc(const PsArgs& a, const PTile* ctiles128, int ntiles, const float* Ph, float* part,
                             cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  if (a.rmax <= 16) return tc_launch<16, true>(a, ctiles128, ntiles, Ph, part, st);
  if (a.rmax <= 32) return tc_launch<32, true>(a, ctiles128, ntiles, Ph, part, st);
  return tc_launch<64, true>(a, ctiles128, ntiles, Ph, part, st);
}

}  // namespace lg
