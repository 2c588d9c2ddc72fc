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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "memo.h"

namespace lg {

constexpr int TC_M = 128;      // rows per tile (UMMA_M)
constexpr int TC_KT = 32;      // K elements per stage (one 128-byte swizzle row)
constexpr int TC_THREADS = 256;  // 8 warps: warps w and w+4 share TMEM lanes 32*(w%4), split columns

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

// async global -> shared copies (LDGSTS): 16 bytes (zero-filled past src_bytes) or 4 bytes
__device__ __forceinline__ void cp16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp4(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// NP: N padded to a multiple of 16 (16, 32, 64); grouped over layers.
// TRANS = false: P = M Q   -- tile = 128 rows of M, K runs over the columns [c0, i1) of
//                             split `split` (split-K: enough CTAs to cover the SMs),
//                             A = M rows (K-major), B = Q columns,
//                             out partial[split][j*m + i] (summed by k_ps_preduce)
// TRANS = true:  Q = M^T P -- tile = 128 columns of M, K runs over rows [i0, i1),
//                             A = M^T, transposed while staged from M rows (K-major),
//                             B = P columns, out partial[split][j*k + c]
// Pipeline: the raw g, e and B slices of K tiles kt+1 .. kt+RS-1 are in flight (cp.async,
// RS-stage ring) while tile kt is converted (x = canon(g + e), hi/lo split, swizzle)
// into the A/B operand stage (kt & 1) and tile kt - 1's MMAs run.

template <int NP, bool TRANS>
struct TcSmem {
  static constexpr int RAW_X = TC_M * TC_KT * 4;     // 16 KB: 128 x 32 floats of g (or e)
  static constexpr int RAW_B = NP * TC_KT * 4;       // NP x 32 floats of Q (or P)
  static constexpr int RAW = 2 * RAW_X + RAW_B;
  static constexpr int A_BYTES = TC_M * 128;         // 16 KB per A tile (hi or lo)
  static constexpr int B_BYTES = NP * 128;           // per B tile (hi or lo)
  static constexpr int OPS = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int RS = (2 * OPS + 4 * RAW + 1024 <= 220 * 1024) ? 4 : 3;  // raw ring stages (RS-1 in flight)
  static constexpr int TOTAL = 2 * OPS + RS * RAW + 1024;
};

// Persistent: gridDim.x CTAs (<= one per SM) walk the tiles t = blockIdx.x + q*gridDim.x;
// the (tile, K tile) steps of a CTA form one continuous pipeline, so the copies of the
// next tile are in flight while the last K tiles of the current one are multiplied.
template <int NP, bool TRANS>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_ps_tc(const float* __restrict__ g, const float* __restrict__ e, const PLayer* __restrict__ pl,
        const PTile* __restrict__ tiles, int ntiles, const float* __restrict__ Bsrc, float* __restrict__ out) {
  using SM = TcSmem<NP, TRANS>;
  constexpr uint32_t TMEM_COLS = 2 * NP < 32 ? 32 : 2 * NP;  // two accumulator buffers
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  // 1024-byte aligned base, as an offset from the shared array (keeps the shared
  // address space: LDS/STS rather than generic LD/ST)
  uint8_t* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  uint8_t* raw0 = smem + 2 * SM::OPS;
  __shared__ uint64_t mma_done[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // tile geometry: rows along the MMA M dimension, K range [kbeg, kend)
  struct TileG {
    PTile tl;
    PLayer p;
    int rows, kbeg, kend, nk;
  };
  auto geo = [&](int t) {
    TileG G;
    G.tl = tiles[t];
    G.p = pl[G.tl.ci];
    G.rows = TRANS ? min(TC_M, G.p.k - G.tl.c0) : min(TC_M, G.p.m - G.tl.i0);
    G.kbeg = TRANS ? G.tl.i0 : G.tl.c0;
    G.kend = G.tl.i1;
    G.nk = (G.kend - G.kbeg + TC_KT - 1) / TC_KT;
    return G;
  };
  int nsteps = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) nsteps += geo(t).nk;

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

  constexpr int TC_RS = SM::RS;
  // issue cursor: the raw copies of step s (tile ti, K tile kti) into ring slot s % TC_RS
  int ti = blockIdx.x, kti = 0;
  TileG gi = geo(min(ti, ntiles - 1));
  auto issue = [&](int step) {
    uint8_t* rg = raw0 + (step % TC_RS) * SM::RAW;
    uint8_t* re = rg + SM::RAW_X;
    uint8_t* rb = re + SM::RAW_X;
    const PLayer& p = gi.p;
    const PTile& tl = gi.tl;
    const int k0 = gi.kbeg + kti * TC_KT, kend = gi.kend, rows = gi.rows;
    const bool a16 = ((p.moff & 3) == 0) && ((p.k & 3) == 0);
    const int64_t bld = TRANS ? (int64_t)p.m : (int64_t)p.k;  // column length of Bsrc
    const int64_t boff = TRANS ? p.poff : p.qoff;
    const bool b16 = ((boff & 3) == 0) && ((bld & 3) == 0);
    // X: 128 x 32 floats as 1024 16-byte chunks; MQ: [row][kchunk], MtP: [krow][cchunk]
#pragma unroll
    for (int it = 0; it < TC_M * TC_KT / 4 / TC_THREADS; ++it) {
      const int idx = it * TC_THREADS + tid;
      int64_t xi;  // flat element index of the chunk's first element
      int nval;    // valid elements in the chunk
      if (!TRANS) {
        const int r_ = idx >> 3, ch = idx & 7, col = k0 + ch * 4;
        nval = (r_ < rows) ? max(0, min(4, kend - col)) : 0;
        xi = p.moff + (int64_t)(tl.i0 + min(r_, rows - 1)) * p.k + col;
      } else {
        const int kr = idx >> 5, cq = idx & 31, i = k0 + kr, c = tl.c0 + cq * 4;
        nval = (i < kend) ? max(0, min(4, tl.c0 + rows - c)) : 0;
        xi = p.moff + (int64_t)min(i, kend - 1) * p.k + c;
      }
      // raw slot: MQ chunk idx; MtP chunk (kr, cq) at cq*32 + (kr ^ cq) (XOR swizzle: the
      // copies along cq and the transposing reads along kr are both conflict-free)
      const int slot = TRANS ? ((idx & 31) * 32 + ((idx >> 5) ^ (idx & 31))) : idx;
      if (a16) {
        cp16(rg + slot * 16, g + xi, 4 * nval);
        if (e) cp16(re + slot * 16, e + xi, 4 * nval);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          cp4(rg + slot * 16 + 4 * q, g + xi + (q < nval ? q : 0), q < nval ? 4 : 0);
          if (e) cp4(re + slot * 16 + 4 * q, e + xi + (q < nval ? q : 0), q < nval ? 4 : 0);
        }
      }
    }
    // B: NP columns x 32 K elements as NP*8 chunks [j][kchunk]
    for (int idx = tid; idx < NP * 8; idx += TC_THREADS) {
      const int j = idx >> 3, ch = idx & 7, col = k0 + ch * 4;
      const int nval = (j < p.r) ? max(0, min(4, kend - col)) : 0;
      const float* src = Bsrc + boff + (int64_t)min(j, p.r - 1) * bld + col;
      if (b16) {
        cp16(rb + idx * 16, src, 4 * nval);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) cp4(rb + idx * 16 + 4 * q, src + (q < nval ? q : 0), q < nval ? 4 : 0);
      }
    }
    if (++kti >= gi.nk) {
      kti = 0;
      ti += gridDim.x;
      if (ti < ntiles) gi = geo(ti);
    }
  };

  // prologue: steps 0 .. RS-2 in flight (one commit group per step, empty ones too)
#pragma unroll
  for (int s = 0; s < TC_RS - 1; ++s) {
    if (s < nsteps) issue(s);
    cp_commit();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_d = tmem_base_sh;
  constexpr uint32_t idesc = tf32_idesc(NP);

  // accumulator rows = TMEM lanes 32*(warp%4) + lane; columns [half*NP/2, half*NP/2 + NP/2)
  constexpr int NH = NP / 2;
  const int row = (warp & 3) * 32 + lane, half = warp >> 2;
  float acc[NH];
#pragma unroll
  for (int j = 0; j < NH; ++j) acc[j] = 0.f;
  // drain cursor: step s-1 belongs to tile td, K tile ktd
  int td = blockIdx.x, ktd = 0, nkd = (td < ntiles) ? geo(td).nk : 0;
  // add the finished partial of step t (TMEM buffer t & 1); at the tile's last K tile
  // write the tile's output and restart the accumulator
  auto drain = [&](int t) {
    mbar_wait(&mma_done[t & 1], (t >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
    for (int j0 = 0; j0 < NH; j0 += 8) {
      uint32_t v[8];
      const uint32_t taddr =
          tmem_d + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((t & 1) * NP + half * NH + j0);
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[j0 + q] = __fadd_rn(acc[j0 + q], __uint_as_float(v[q]));
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    if (++ktd >= nkd) {
      const TileG G = geo(td);
      if (row < G.rows) {
        if (!TRANS) {
          float* o = out + (int64_t)G.tl.split * G.p.pstride + G.p.poff;
#pragma unroll
          for (int q = 0; q < NH; ++q) {
            const int j = half * NH + q;
            if (j < G.p.r) o[(int64_t)j * G.p.m + G.tl.i0 + row] = acc[q];
          }
        } else {
          float* o = out + (int64_t)G.tl.split * G.p.qstride + G.p.qoff;
#pragma unroll
          for (int q = 0; q < NH; ++q) {
            const int j = half * NH + q;
            if (j < G.p.r) o[(int64_t)j * G.p.k + G.tl.c0 + row] = acc[q];
          }
        }
      }
#pragma unroll
      for (int j = 0; j < NH; ++j) acc[j] = 0.f;
      ktd = 0;
      td += gridDim.x;
      nkd = (td < ntiles) ? geo(td).nk : 0;
    }
  };

  for (int s = 0; s < nsteps; ++s) {
    // keep TC_RS - 1 steps in flight; wait for step s (this thread's copies), then a
    // barrier makes every thread's copies of step s visible
    if (s + TC_RS - 1 < nsteps) issue(s + TC_RS - 1);
    cp_commit();
    cp_wait<TC_RS - 1>();
    __syncthreads();
    const uint8_t* rg = raw0 + (s % TC_RS) * SM::RAW;
    const uint8_t* re = rg + SM::RAW_X;
    const uint8_t* rb = re + SM::RAW_X;
    const int sb = s & 1;
    uint8_t* Ah = smem + sb * SM::OPS;
    uint8_t* Al = Ah + SM::A_BYTES;
    uint8_t* Bh = Al + SM::A_BYTES;
    uint8_t* Bl = Bh + SM::B_BYTES;
#pragma unroll
    for (int it = 0; it < TC_M * TC_KT / 4 / TC_THREADS; ++it) {
      const int idx = it * TC_THREADS + tid;
      // MtP: lanes walk kr (K rows) for one cq, so the transposed 4-byte stores below
      // hit 32 distinct banks
      const int kr = idx & 31, cq = idx >> 5;
      const int slot = TRANS ? (cq * 32 + (kr ^ cq)) : idx;
      const float4 a = *reinterpret_cast<const float4*>(rg + slot * 16);
      const float4 b = e ? *reinterpret_cast<const float4*>(re + slot * 16) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 v = make_float4(canon(a.x, b.x), canon(a.y, b.y), canon(a.z, b.z), canon(a.w, b.w));
      if (!TRANS) {
        put_chunk(Ah, Al, idx >> 3, idx & 7, v);
      } else {
        // transpose into the K-major A tile: A row = column (local cq*4 + q), K = kr.
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
    for (int idx = tid; idx < NP * 8; idx += TC_THREADS)
      put_chunk(Bh, Bl, idx >> 3, idx & 7, *reinterpret_cast<const float4*>(rb + idx * 16));
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t sAh = smem_u32(Ah), sAl = smem_u32(Al), sBh = smem_u32(Bh), sBl = smem_u32(Bl);
      const uint32_t dbuf = tmem_d + (uint32_t)(sb * NP);
#pragma unroll
      for (int kk = 0; kk < TC_KT / 8; ++kk) {
        const uint32_t koff = kk * 32;  // 8 tf32 = 32 bytes along K inside the swizzle row
        const uint64_t dAh = sw128_desc(sAh + koff);
        const uint64_t dAl = sw128_desc(sAl + koff);
        mma_tf32(dbuf, dAh, sw128_desc(sBh + koff), idesc, kk > 0 ? 1u : 0u);
        mma_tf32(dbuf, dAh, sw128_desc(sBl + koff), idesc, 1u);
        mma_tf32(dbuf, dAl, sw128_desc(sBh + koff), idesc, 1u);
      }
      mma_commit(&mma_done[sb]);
    }
    __syncwarp();
    // while step s's MMAs run: drain step s-1 (this also frees operand stage s^1 and
    // TMEM buffer s^1 for step s+1)
    if (s >= 1) drain(s - 1);
  }
  cp_wait<0>();
  if (nsteps > 0) drain(nsteps - 1);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(TMEM_COLS));
}

// ---------------------------------------------------------------------------
// Warp-specialised variant (round 2): the same math per K step (3xTF32, a fresh TMEM
// accumulator per step added in fp32 registers), the roles decoupled by mbarriers so the
// conversion of step s+1, the MMAs of step s and the drain of step s-1 overlap:
//   warps 0-15  convert the raw ring (RS slots) into NOS operand stages; they also fill the
//               raw ring with 4-byte cp.async for layers TMA cannot address
//   warp 16     lane 0 issues the MMAs (waits op_full, tm_empty; commits mma_done, op_empty)
//   warps 17-20 drain TMEM (lane quarter warp % 4), add, write the tile at its last K step
//   warp 21     lane 0 fills the raw ring by 2-D TMA (per-layer tensor maps, SWIZZLE_128B)
// ---------------------------------------------------------------------------
constexpr int TC2_CONV = 512;  // converter threads (warps 0-15)
constexpr int TC2_THREADS = TC2_CONV + 32 + 128 + 32;  // + MMA warp, 4 drain warps, the TMA producer warp
constexpr int TC2_NOS = 2;
constexpr int TC2_NTM = 4;
// raw tiles as TMA lands them: MQ 128 rows x 32 floats (128 B rows, dense); M^T P four
// 32 x 32 boxes (K-rows x columns) in the 128-byte swizzle (16-byte chunk c of K-row r at
// c ^ (r & 7)): the transposing reads (lanes walk r) are conflict-free
__device__ __forceinline__ uint32_t tr_off(int kr, int cq) {  // byte offset of chunk (K-row kr, 4-column chunk cq)
  return (uint32_t)((cq >> 3) * 4096 + kr * 128 + (((cq & 7) ^ (kr & 7)) << 4));
}

template <int NP, bool TRANS>
struct Tc2Smem {
  static constexpr int RAW_X = TC_M * TC_KT * 4;  // one of g / e (16 KB, 1024-aligned: TMA swizzle)
  static constexpr int RAW_B = NP * TC_KT * 4;
  static constexpr int RAW = 2 * RAW_X + RAW_B;
  static constexpr int A_BYTES = TC_M * 128;
  static constexpr int B_BYTES = NP * 128;
  static constexpr int OPS = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int RS = (TC2_NOS * OPS + 4 * RAW + 1024 <= 220 * 1024) ? 4 : 3;
  static constexpr int TOTAL = TC2_NOS * OPS + RS * RAW + 1024;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void conv_sync() { asm volatile("bar.sync 1, %0;" ::"n"(TC2_CONV) : "memory"); }

template <int NP, bool TRANS>
__global__ void __launch_bounds__(TC2_THREADS, 1)
k_ps_tc2(const float* __restrict__ g, const float* __restrict__ e, const PLayer* __restrict__ pl,
         const PTile* __restrict__ tiles, int ntiles, const float* __restrict__ Bsrc, float* __restrict__ out,
         const CUtensorMap* __restrict__ maps /* [layer][3]: g, e, B; nullable */) {
  using SM = Tc2Smem<NP, TRANS>;
  constexpr uint32_t TMEM_COLS = TC2_NTM * NP < 32 ? 32 : TC2_NTM * NP;
  constexpr int TC_RS = SM::RS;
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  uint8_t* smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  uint8_t* raw0 = smem + TC2_NOS * SM::OPS;
  __shared__ uint64_t op_full[TC2_NOS], op_empty[TC2_NOS], mma_done[TC2_NTM], tm_empty[TC2_NTM];
  __shared__ uint64_t raw_full_t[4], raw_full_c[4], raw_empty[4];  // TMA fills, 4-byte-copy fills, slot released
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  struct TileG { PTile tl; PLayer p; int rows, kbeg, kend, nk; };
  auto geo = [&](int t) {
    TileG G;
    G.tl = tiles[t];
    G.p = pl[G.tl.ci];
    G.rows = TRANS ? min(TC_M, G.p.k - G.tl.c0) : min(TC_M, G.p.m - G.tl.i0);
    G.kbeg = TRANS ? G.tl.i0 : G.tl.c0;
    G.kend = G.tl.i1;
    G.nk = (G.kend - G.kbeg + TC_KT - 1) / TC_KT;
    return G;
  };
  int nsteps = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) nsteps += geo(t).nk;
  constexpr int WM = TC2_CONV / 32;  // the MMA warp; drain warps WM+1 .. WM+4; producer WM+5
  // a step's raw tile comes by TMA (one producer thread) when every operand of its layer is
  // 16-byte addressable, else by 4-byte cp.async of all converters (zero-filled)
  auto step_tma = [&](const TileG& G) -> bool {
    const int64_t bld = TRANS ? (int64_t)G.p.m : (int64_t)G.p.k;
    const int64_t boff = TRANS ? G.p.poff : G.p.qoff;
    return maps != nullptr && ((G.p.moff & 3) == 0) && ((G.p.k & 3) == 0) && ((boff & 3) == 0) && ((bld & 3) == 0) &&
           (((uintptr_t)g & 15) == 0) && (!e || ((uintptr_t)e & 15) == 0) && (((uintptr_t)Bsrc & 15) == 0);
  };
  if (warp == WM) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int b = 0; b < TC2_NOS; ++b) { mbar_init(&op_full[b], 1); mbar_init(&op_empty[b], 1); }
    for (int b = 0; b < TC2_NTM; ++b) { mbar_init(&mma_done[b], 1); mbar_init(&tm_empty[b], 4); }
    for (int b = 0; b < TC_RS; ++b) {
      mbar_init(&raw_full_t[b], 1);          // the producer's expect_tx arrival
      mbar_init(&raw_full_c[b], TC2_CONV);   // every converter's cp.async (noinc) arrival
      mbar_init(&raw_empty[b], 1);           // converter 0 after the slot was read
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_d = tmem_base_sh;
#ifdef LG_TC_TIMING
  long long tw_data = 0, tw_empty = 0, tw_conv = 0, tw_sync2 = 0, tw_full = 0, tw_tm = 0, tw_done = 0;
  long long tk0 = clock64();
#define TCT(var, stmt) do { long long _t0 = clock64(); stmt; var += clock64() - _t0; } while (0)
#else
#define TCT(var, stmt) do { stmt; } while (0)
#endif

  if (warp < WM) {
    // ---- converters: fill the raw ring with 4-byte cp.async for the steps TMA cannot
    // serve (one noinc arrival per converter on raw_full_c), convert into the operand stages
    int ti = blockIdx.x, kti = 0;
    TileG gi = geo(min(ti, ntiles - 1));
    auto issue = [&](int step) {
      const int slot = step % TC_RS;
      uint8_t* rg = raw0 + slot * SM::RAW;
      uint8_t* re = rg + SM::RAW_X;
      uint8_t* rb = re + SM::RAW_X;
      const PLayer& p = gi.p;
      const PTile& tl = gi.tl;
      const int k0 = gi.kbeg + kti * TC_KT, kv = min(TC_KT, gi.kend - k0), rows = gi.rows;
      const int64_t bld = TRANS ? (int64_t)p.m : (int64_t)p.k;
      const int64_t boff = TRANS ? p.poff : p.qoff;
      if (step_tma(gi)) {
        // (the producer warp fills this step)
      } else {
        // 4-byte copies (zero-filled past the valid range)
#pragma unroll
        for (int it = 0; it < TC_M * TC_KT / 4 / TC2_CONV; ++it) {
          const int idx = it * TC2_CONV + tid;
          int r_, c_;          // (row of the raw tile, first float of the chunk)
          int64_t xi;
          int nval;
          uint32_t dst;
          if (!TRANS) {
            r_ = idx >> 3; c_ = (idx & 7) * 4;
            nval = (r_ < rows) ? max(0, min(4, kv - c_)) : 0;
            xi = p.moff + (int64_t)(tl.i0 + min(r_, rows - 1)) * p.k + k0 + c_;
            dst = (uint32_t)(r_ * 128 + c_ * 4);
          } else {
            r_ = idx >> 5; c_ = (idx & 31) * 4;
            nval = (r_ < kv) ? max(0, min(4, rows - c_)) : 0;
            xi = p.moff + (int64_t)(k0 + min(r_, max(kv - 1, 0))) * p.k + tl.c0 + c_;
            dst = tr_off(r_, idx & 31);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            cp4(rg + dst + 4 * q, g + xi + (q < nval ? q : 0), q < nval ? 4 : 0);
            if (e) cp4(re + dst + 4 * q, e + xi + (q < nval ? q : 0), q < nval ? 4 : 0);
          }
        }
        for (int idx = tid; idx < NP * 8; idx += TC2_CONV) {
          const int j = idx >> 3, ch = idx & 7, col = k0 + ch * 4;
          const int nval = (j < p.r) ? max(0, min(4, gi.kend - col)) : 0;
          const float* src = Bsrc + boff + (int64_t)min(j, p.r - 1) * bld + col;
#pragma unroll
          for (int q = 0; q < 4; ++q) cp4(rb + idx * 16 + 4 * q, src + (q < nval ? q : 0), q < nval ? 4 : 0);
        }
        cp_arrive_noinc(&raw_full_c[slot]);
      }
      if (++kti >= gi.nk) {
        kti = 0;
        ti += gridDim.x;
        if (ti < ntiles) gi = geo(ti);
      }
    };
    // the converter's own cursor: the valid rows / K of step s (raw slots are not zero-filled
    // by the bulk path: the conversion masks)
    int tc = blockIdx.x, ktc = 0;
    TileG gc = geo(min(tc, ntiles - 1));
    uint32_t ph_t = 0u, ph_c = 0u;  // per-slot parity of the next completion of each fill barrier
#pragma unroll
    for (int s = 0; s < TC_RS - 1; ++s)
      if (s < nsteps) issue(s);
    for (int s = 0; s < nsteps; ++s) {
      if (s + TC_RS - 1 < nsteps) TCT(tw_sync2, issue(s + TC_RS - 1));
      const int slot = s % TC_RS;
      const bool viat = step_tma(gc);  // (gc: step s's geometry, below)
      {
        const uint32_t bit = 1u << slot;
        if (viat) { TCT(tw_data, mbar_wait(&raw_full_t[slot], (ph_t & bit) ? 1u : 0u)); ph_t ^= bit; }
        else { TCT(tw_data, mbar_wait(&raw_full_c[slot], (ph_c & bit) ? 1u : 0u)); ph_c ^= bit; }
      }
      const int ob = s % TC2_NOS;
      if (s >= TC2_NOS) TCT(tw_empty, mbar_wait(&op_empty[ob], ((s / TC2_NOS) - 1) & 1));  // MMAs of step s - NOS done
#ifdef LG_TC_TIMING
      const long long tc0 = clock64();
#endif
      const int k0c = gc.kbeg + ktc * TC_KT, kvc = min(TC_KT, gc.kend - k0c), rowsc = gc.rows, rc = gc.p.r;
      const uint8_t* rg = raw0 + slot * SM::RAW;
      const uint8_t* re = rg + SM::RAW_X;
      const uint8_t* rb = re + SM::RAW_X;
      uint8_t* Ah = smem + ob * SM::OPS;
      uint8_t* Al = Ah + SM::A_BYTES;
      uint8_t* Bh = Al + SM::A_BYTES;
      uint8_t* Bl = Bh + SM::B_BYTES;
#pragma unroll
      for (int it = 0; it < TC_M * TC_KT / 4 / TC2_CONV; ++it) {
        const int idx = it * TC2_CONV + tid;
        if (!TRANS) {
          const int r_ = idx >> 3, ch = idx & 7;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (r_ < rowsc) {
            const float4 a = *reinterpret_cast<const float4*>(rg + r_ * 128 + ch * 16);
            const float4 b = e ? *reinterpret_cast<const float4*>(re + r_ * 128 + ch * 16) : make_float4(0.f, 0.f, 0.f, 0.f);
            const int c0 = ch * 4;
            v = make_float4(c0 < kvc ? canon(a.x, b.x) : 0.f, c0 + 1 < kvc ? canon(a.y, b.y) : 0.f,
                            c0 + 2 < kvc ? canon(a.z, b.z) : 0.f, c0 + 3 < kvc ? canon(a.w, b.w) : 0.f);
          }
          put_chunk(Ah, Al, r_, ch, v);
        } else {
          // lanes walk the K-row kr (conflict-free: 528-byte row stride), cq = 4-column chunk
          const int kr = idx & 31, cq = idx >> 5;
          float vv[4] = {0.f, 0.f, 0.f, 0.f};
          if (kr < kvc) {
            const float4 a = *reinterpret_cast<const float4*>(rg + tr_off(kr, cq));
            const float4 b = e ? *reinterpret_cast<const float4*>(re + tr_off(kr, cq)) : make_float4(0.f, 0.f, 0.f, 0.f);
            const int c0 = cq * 4;
            vv[0] = c0 < rowsc ? canon(a.x, b.x) : 0.f;
            vv[1] = c0 + 1 < rowsc ? canon(a.y, b.y) : 0.f;
            vv[2] = c0 + 2 < rowsc ? canon(a.z, b.z) : 0.f;
            vv[3] = c0 + 3 < rowsc ? canon(a.w, b.w) : 0.f;
          }
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
      for (int idx = tid; idx < NP * 8; idx += TC2_CONV) {
        const int j = idx >> 3, ch = idx & 7, c0 = ch * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < rc) {
          const float4 a = *reinterpret_cast<const float4*>(rb + j * 128 + ch * 16);
          v = make_float4(c0 < kvc ? a.x : 0.f, c0 + 1 < kvc ? a.y : 0.f, c0 + 2 < kvc ? a.z : 0.f,
                          c0 + 3 < kvc ? a.w : 0.f);
        }
        put_chunk(Bh, Bl, j, ch, v);
      }
#ifdef LG_TC_TIMING
      tw_conv += clock64() - tc0;
#endif
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      conv_sync();  // the stage is complete, and every converter is done reading raw slot s
      if (tid == 0) {
        mbar_arrive(&op_full[ob]);
        mbar_arrive(&raw_empty[slot]);  // the producer may refill the slot
      }
      if (++ktc >= gc.nk) {
        ktc = 0;
        tc += gridDim.x;
        if (tc < ntiles) gc = geo(tc);
      }
    }
  } else if (warp == WM) {
    // ---- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tf32_idesc(NP);
      for (int s = 0; s < nsteps; ++s) {
        const int ob = s % TC2_NOS, tb = s % TC2_NTM;
        TCT(tw_full, mbar_wait(&op_full[ob], (s / TC2_NOS) & 1));
        if (s >= TC2_NTM) TCT(tw_tm, mbar_wait(&tm_empty[tb], ((s / TC2_NTM) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint8_t* Ah = smem + ob * SM::OPS;
        const uint32_t sAh = smem_u32(Ah), sAl = sAh + SM::A_BYTES, sBh = sAl + SM::A_BYTES, sBl = sBh + SM::B_BYTES;
        const uint32_t dbuf = tmem_d + (uint32_t)(tb * NP);
#pragma unroll
        for (int kk = 0; kk < TC_KT / 8; ++kk) {
          const uint32_t koff = kk * 32;
          const uint64_t dAh = sw128_desc(sAh + koff);
          const uint64_t dAl = sw128_desc(sAl + koff);
          mma_tf32(dbuf, dAh, sw128_desc(sBh + koff), idesc, kk > 0 ? 1u : 0u);
          mma_tf32(dbuf, dAh, sw128_desc(sBl + koff), idesc, 1u);
          mma_tf32(dbuf, dAl, sw128_desc(sBh + koff), idesc, 1u);
        }
        mma_commit(&mma_done[tb]);
        mma_commit(&op_empty[ob]);
      }
    }
    __syncwarp();
  } else if (warp <= WM + 4) {
    // ---- drain: TMEM lane quarter warp % 4, all NP columns of the row
    const int dq = warp & 3, row = dq * 32 + lane;
    float acc[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) acc[j] = 0.f;
    int td = blockIdx.x, ktd = 0, nkd = (td < ntiles) ? geo(td).nk : 0;
    for (int s = 0; s < nsteps; ++s) {
      const int tb = s % TC2_NTM;
      TCT(tw_done, mbar_wait(&mma_done[tb], (s / TC2_NTM) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int j0 = 0; j0 < NP; j0 += 8) {
        uint32_t v[8];
        const uint32_t taddr = tmem_d + ((uint32_t)(dq * 32) << 16) + (uint32_t)(tb * NP + j0);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[j0 + q] = __fadd_rn(acc[j0 + q], __uint_as_float(v[q]));
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tm_empty[tb]);
      if (++ktd >= nkd) {
        const TileG G = geo(td);
        if (row < G.rows) {
          if (!TRANS) {
            float* o = out + (int64_t)G.tl.split * G.p.pstride + G.p.poff;
#pragma unroll
            for (int j = 0; j < NP; ++j)
              if (j < G.p.r) o[(int64_t)j * G.p.m + G.tl.i0 + row] = acc[j];
          } else {
            float* o = out + (int64_t)G.tl.split * G.p.qstride + G.p.qoff;
#pragma unroll
            for (int j = 0; j < NP; ++j)
              if (j < G.p.r) o[(int64_t)j * G.p.k + G.tl.c0 + row] = acc[j];
          }
        }
#pragma unroll
        for (int j = 0; j < NP; ++j) acc[j] = 0.f;
        ktd = 0;
        td += gridDim.x;
        nkd = (td < ntiles) ? geo(td).nk : 0;
      }
    }
  } else if (lane == 0) {
    // ---- TMA producer: every TMA step's tiles, the slot released by the converters first
    int tp = blockIdx.x, ktp = 0;
    TileG gp = geo(min(tp, ntiles - 1));
    for (int s = 0; s < nsteps; ++s) {
      const int slot = s % TC_RS;
      if (s >= TC_RS) mbar_wait(&raw_empty[slot], ((s / TC_RS) - 1) & 1);
      if (step_tma(gp)) {
        uint8_t* rg = raw0 + slot * SM::RAW;
        uint8_t* re = rg + SM::RAW_X;
        uint8_t* rb = re + SM::RAW_X;
        const CUtensorMap* mg = maps + 3 * gp.tl.ci;
        const int k0 = gp.kbeg + ktp * TC_KT;
        const uint32_t bytes = (uint32_t)(e ? 2 : 1) * SM::RAW_X + (uint32_t)NP * TC_KT * 4u;
        mbar_arrive_tx(&raw_full_t[slot], bytes);
        if (!TRANS) {
          tma2d(rg, mg, k0, gp.tl.i0, &raw_full_t[slot]);
          if (e) tma2d(re, mg + 1, k0, gp.tl.i0, &raw_full_t[slot]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            tma2d(rg + q * 4096, mg, gp.tl.c0 + 32 * q, k0, &raw_full_t[slot]);
            if (e) tma2d(re + q * 4096, mg + 1, gp.tl.c0 + 32 * q, k0, &raw_full_t[slot]);
          }
        }
        tma2d(rb, mg + 2, k0, 0, &raw_full_t[slot]);
      }
      if (++ktp >= gp.nk) {
        ktp = 0;
        tp += gridDim.x;
        if (tp < ntiles) gp = geo(tp);
      }
    }
  }
#ifdef LG_TC_TIMING
  if (blockIdx.x == 0 && (tid == 0 || tid == TC2_CONV || tid == TC2_CONV + 32))
    printf("tc2<%d,%d> block0 tid %d steps %d total %lld | conv: data %lld empty %lld convert %lld sync2 %lld | mma: "
           "full %lld tm %lld | drain: done %lld (conv 'sync2' = issue)\n", NP, (int)TRANS, tid, nsteps, clock64() - tk0, tw_data, tw_empty,
           tw_conv, tw_sync2, tw_full, tw_tm, tw_done);
#endif
#undef TCT
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == WM)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(TMEM_COLS));
}

// cuTensorMapEncodeTiled from the driver (no link-time libcuda dependency)
static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    else
      cudaGetLastError();
  }
  return fn;
}

// The device maps of one GEMM flavour for (g, e, B): re-encoded (every layer: g, e, B) and
// copied only when the config or a pointer changed.  nullptr: TMA not available.
template <int NP, bool TRANS>
static const CUtensorMap* tc_maps(const PsArgs& a, const float* B, cudaStream_t st) {
  void* dmaps = TRANS ? a.maps_tr : a.maps_mq;
  TcMapCache* mc = TRANS ? a.mc_tr : a.mc_mq;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tma_encoder();
  if (!dmaps || !mc || !a.h_pl || !enc || getenv("LGRECO_PS_NO_TMA")) return nullptr;
  if (mc->ver == a.cfg_ver && mc->g == a.g && mc->e == a.e && mc->b == B) return static_cast<const CUtensorMap*>(dmaps);
  std::vector<CUtensorMap> h((size_t)3 * a.nC);
  memset(h.data(), 0, sizeof(CUtensorMap) * h.size());
  for (int ci = 0; ci < a.nC; ++ci) {
    const PLayer& p = a.h_pl[ci];
    const bool ok = (p.moff % 4 == 0) && (p.k % 4 == 0) && ((TRANS ? p.poff : p.qoff) % 4 == 0) &&
                    ((TRANS ? p.m : p.k) % 4 == 0);
    if (!ok) continue;  // the kernel takes 4-byte copies for this layer
    const cuuint32_t one[2] = {1, 1};
    const cuuint64_t gdim[2] = {(cuuint64_t)p.k, (cuuint64_t)p.m};
    const cuuint64_t gstr[1] = {(cuuint64_t)p.k * 4};
    const cuuint32_t gbox[2] = {(cuuint32_t)TC_KT, (cuuint32_t)(TRANS ? TC_KT : TC_M)};
    const CUtensorMapSwizzle sw = TRANS ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = enc(&h[3 * ci], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)(a.g + p.moff), gdim, gstr, gbox, one,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS && a.e)
      r = enc(&h[3 * ci + 1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)(a.e + p.moff), gdim, gstr, gbox, one,
              CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int64_t bl = TRANS ? p.m : p.k;  // B column length (K-major)
    const cuuint64_t bdim[2] = {(cuuint64_t)bl, (cuuint64_t)p.r};
    const cuuint64_t bstr[1] = {(cuuint64_t)bl * 4};
    const cuuint32_t bbox[2] = {(cuuint32_t)TC_KT, (cuuint32_t)NP};
    if (r == CUDA_SUCCESS)
      r = enc(&h[3 * ci + 2], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)(B + (TRANS ? p.poff : p.qoff)), bdim, bstr,
              bbox, one, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return nullptr;
  }
  if (cudaMemcpyAsync(dmaps, h.data(), sizeof(CUtensorMap) * h.size(), cudaMemcpyHostToDevice, st) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  mc->ver = a.cfg_ver; mc->g = a.g; mc->e = a.e; mc->b = B;
  return static_cast<const CUtensorMap*>(dmaps);
}

template <int NP, bool TRANS>
static cudaError_t tc_launch(const PsArgs& a, const PTile* tiles, int ntiles, const float* B, float* out,
                             cudaStream_t st) {
  int nsm = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (nsm <= 0) nsm = 148;
  if (!getenv("LGRECO_PS_TC1")) {  // the warp-specialised kernel (LGRECO_PS_TC1=1: the lock-step one, A/B)
    const int smem = Tc2Smem<NP, TRANS>::TOTAL;
    cudaError_t e = memo_smem_attr((const void*)k_ps_tc2<NP, TRANS>, smem);
    if (e != cudaSuccess) return e;
    const CUtensorMap* maps = tc_maps<NP, TRANS>(a, B, st);
    k_ps_tc2<NP, TRANS><<<std::min(ntiles, nsm), TC2_THREADS, smem, st>>>(a.g, a.e, a.pl, tiles, ntiles, B, out, maps);
    return cudaGetLastError();
  }
  const int smem = TcSmem<NP, TRANS>::TOTAL;
  cudaError_t e = memo_smem_attr((const void*)k_ps_tc<NP, TRANS>, smem);
  if (e != cudaSuccess) return e;
  k_ps_tc<NP, TRANS><<<std::min(ntiles, nsm), TC_THREADS, smem, st>>>(a.g, a.e, a.pl, tiles, ntiles, B, out);
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
