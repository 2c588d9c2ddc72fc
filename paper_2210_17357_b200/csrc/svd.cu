// svd.cu -- NEXT-2: low-rank errors from the singular values (PAPER.md:696-699,
// "e_r = sqrt(sum_{i > r} sigma_i^2) ... compute squared singular values once, and then
// compute all the errors").  The squared singular values of the m x k view M are the
// eigenvalues of the Gram matrix of its smaller side (n = min(m, k)): G = M M^T (m <= k)
// or M^T M.  G is formed in fp64 from x = fl(g + e) (R2) by a split-K tiled kernel
// (fixed-order split reduction: deterministic); its eigenvalues by this file's own
// symmetric eigensolver (k_sym_eigvals: Householder reduction to tridiagonal form in
// fp64, one CTA per matrix, every matrix of the table at once, then Sturm-count bisection,
// one thread per eigenvalue), and err_r^2 = sum of the n - r smallest eigenvalues (each
// clamped at 0), summed in fp64 in ascending order.
#include <math.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace lg {

constexpr int GT = 64;      // output tile (GT x GT) per CTA
constexpr int GKC = 16;     // reduction chunk staged in shared memory
constexpr int G_THREADS = 256;

// X (n x t): X[a][s] = x[off + a*k + s] (rows, m <= k) or x[off + s*k + a] (columns).
__device__ __forceinline__ double xval(const float* __restrict__ g, const float* __restrict__ e, int64_t off,
                                       int k, bool rows, int a, int64_t s) {
  const int64_t i = rows ? off + (int64_t)a * k + s : off + s * k + a;
  return (double)__fadd_rn(__fadd_rn(g[i], e ? e[i] : 0.f), 0.f);
}

// partial[split][n][n] (upper tiles, mirrored) = sum over s in the split's range.
__global__ void __launch_bounds__(G_THREADS)
k_gram64(const float* __restrict__ g, const float* __restrict__ e, int64_t off, int k, int n, int64_t t, int rows,
         int nsplit, double* __restrict__ part) {
  __shared__ double A[GKC][GT + 1], Bt[GKC][GT + 1];
  const int nt = (n + GT - 1) / GT;
  // upper-triangular tile index -> (ta, tb), ta <= tb
  int ti = blockIdx.x, ta = 0;
  while (ti >= nt - ta) { ti -= nt - ta; ++ta; }
  const int tb = ta + ti;
  const int split = blockIdx.y;
  const int64_t s0 = t * split / nsplit, s1 = t * (split + 1) / nsplit;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 outputs each
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int64_t sc = s0; sc < s1; sc += GKC) {
    for (int idx = threadIdx.x; idx < GKC * GT; idx += G_THREADS) {
      const int kk = rows ? idx % GKC : idx / GT, aa = rows ? idx / GKC : idx % GT;
      const int64_t s = sc + kk;
      const int ga = ta * GT + aa, gb = tb * GT + aa;
      A[kk][aa] = (s < s1 && ga < n) ? xval(g, e, off, k, rows, ga, s) : 0.0;
      Bt[kk][aa] = (s < s1 && gb < n) ? xval(g, e, off, k, rows, gb, s) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GKC; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { av[i] = A[kk][ty + 16 * i]; bv[i] = Bt[kk][tx + 16 * i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* P = part + (int64_t)split * n * n;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int a = ta * GT + ty + 16 * i, b = tb * GT + tx + 16 * j;
      if (a < n && b < n) { P[(int64_t)a * n + b] = acc[i][j]; P[(int64_t)b * n + a] = acc[i][j]; }
    }
}

// G = sum of the split partials in split order
__global__ void k_gram_reduce(const double* __restrict__ part, int nsplit, int64_t nn, double* __restrict__ G) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < nsplit; ++p) s += part[(int64_t)p * nn + i];
    G[i] = s;
  }
}

// ---------------------------------------------------------------------------
// Symmetric eigenvalues, one CTA per matrix (G: n x n, row-major, full storage, fp64;
// overwritten).  (1) Householder reduction to tridiagonal form, column k = 0 .. n-3
// (LAPACK dsytd2's lower variant, restated): x = G[k+1.., k] (= row k right of the
// diagonal: contiguous), beta = -sign(x0) ||x||, v = x / (x0 - beta) with v0 = 1,
// tau = (beta - x0) / beta; p = tau A v and w = p - (tau/2)(p.v) v on the trailing
// block A, then A -= v w^T + w v^T; e_k = beta, d_k = G[k][k].  Warp per row for the
// matrix-vector product, fixed-order block reductions (deterministic).  One pass over the
// trailing block per step: row k+1 is updated first, the next reflector is formed from it,
// and the other rows' rank-2 update also accumulates the next step's A v (the old
// update-then-matvec order read the block twice: C5 315 -> 269 ms).  (2) Eigenvalue i
// (ascending) of the tridiagonal (d, e) by bisection on the Sturm count (the number of
// negative q_j of q_0 = d_0 - s, q_j = d_j - s - e_{j-1}^2 / q_{j-1}) inside the
// Gershgorin interval, to the fp64 resolution of the interval.  Dynamic shared memory:
// v, w, d, e and the next step's v, p (6 n doubles).
constexpr int EIG_THREADS = 1024;
constexpr int EIG_NMAX = 4096;  // 6 n doubles of shared memory <= 192 KB

struct EigMat { int64_t goff; int32_t n, pad; };  // G at base + goff; eigenvalues at W + wout

__device__ __forceinline__ double block_sum_d(double v, double* red, int tid) {
  v = warp_sum_d(v);
  __syncthreads();  // (red reused)
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < EIG_THREADS / 32; ++w) s += red[w];  // every thread, same order
  return s;
}

__global__ void __launch_bounds__(EIG_THREADS, 1)
k_sym_eigvals(double* __restrict__ Gbase, const EigMat* __restrict__ mats, double* __restrict__ Wbase,
              const int64_t* __restrict__ woff) {
  extern __shared__ double esm[];
  __shared__ double red[EIG_THREADS / 32];
  const EigMat em = mats[blockIdx.x];
  const int n = em.n;
  double* G = Gbase + em.goff;
  double* W = Wbase + woff[blockIdx.x];
  double* v = esm;           // v_k
  double* w = esm + n;       // p_k = A_k v_k, then w_k = tau p + K v in place
  double* d = esm + 2 * n;
  double* e = esm + 3 * n;
  double* v2 = esm + 4 * n;  // v_{k+1}
  double* p2 = esm + 5 * n;  // p_{k+1}
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Householder vector of row r's tail (columns r+1 .. n-1) into vv; returns tau (0: H = I)
  auto reflector = [&](int r, double* vv) -> double {
    const int m = n - r - 1;
    const double* rr = G + (int64_t)r * n + (r + 1);
    double ss = 0.0;
    for (int j = tid; j < m; j += EIG_THREADS) { const double x = rr[j]; ss = fma(x, x, ss); }
    const double nrm2 = block_sum_d(ss, red, tid);
    const double x0 = rr[0];
    if (tid == 0) d[r] = G[(int64_t)r * n + r];
    if (nrm2 == 0.0) {
      if (tid == 0) e[r] = 0.0;
      for (int j = tid; j < m; j += EIG_THREADS) vv[j] = 0.0;
      return 0.0;
    }
    const double nrm = sqrt(nrm2);
    const double beta = x0 > 0.0 ? -nrm : nrm;
    const double sc = 1.0 / (x0 - beta);
    for (int j = tid; j < m; j += EIG_THREADS) vv[j] = j == 0 ? 1.0 : rr[j] * sc;
    if (tid == 0) e[r] = beta;
    return (beta - x0) / beta;
  };
  if (n > 2) {
    double tau = reflector(0, v);
    __syncthreads();
    // p_0 = A_0 v_0 (warp per row)
    {
      const int m = n - 1;
      for (int i = warp; i < m; i += EIG_THREADS / 32) {
        const double* ri = G + (int64_t)(1 + i) * n + 1;
        double a = 0.0;
        for (int j = lane; j < m; j += 32) a = fma(ri[j], v[j], a);
        a = warp_sum_d(a);
        if (lane == 0) w[i] = a;
      }
    }
    __syncthreads();
    for (int k = 0; k + 2 < n; ++k) {
      const int m = n - k - 1;  // trailing block rows / columns k+1 .. n-1
      // w = tau p + K v, K = -(tau / 2) (tau p . v)
      double pv = 0.0;
      for (int j = tid; j < m; j += EIG_THREADS) pv = fma(w[j], v[j], pv);
      const double kk = -0.5 * tau * tau * block_sum_d(pv, red, tid);
      for (int j = tid; j < m; j += EIG_THREADS) w[j] = fma(kk, v[j], tau * w[j]);
      __syncthreads();
      // row k+1 (the next reflector's source) updated first
      {
        double* r1 = G + (int64_t)(k + 1) * n + (k + 1);
        const double v0 = v[0], w0 = w[0];
        for (int j = tid; j < m; j += EIG_THREADS) r1[j] = r1[j] - v0 * w[j] - w0 * v[j];
      }
      __syncthreads();
      const bool more = k + 3 < n;  // another reflector follows
      double tau2 = 0.0;
      if (more) tau2 = reflector(k + 1, v2);
      __syncthreads();
      // the other rows: A -= v w^T + w v^T, and in the same pass the next step's
      // p_{k+1}[i'] = sum_{j >= k+2} A_new[i][j] v_{k+1}[j - k - 2] (i' = i - k - 2)
      for (int i = 1 + warp; i < m; i += EIG_THREADS / 32) {
        double* ri = G + (int64_t)(k + 1 + i) * n + (k + 1);
        const double vi = v[i], wi = w[i];
        double a = 0.0;
        for (int j = lane; j < m; j += 32) {
          const double x = ri[j] - vi * w[j] - wi * v[j];
          ri[j] = x;
          if (more && j >= 1) a = fma(x, v2[j - 1], a);
        }
        if (more) {
          a = warp_sum_d(a);
          if (lane == 0) p2[i - 1] = a;
        }
      }
      __syncthreads();
      if (more) {
        // swap (v, w) <- (v2, p2)
        double* t0 = v; v = v2; v2 = t0;
        double* t1 = w; w = p2; p2 = t1;
        tau = tau2;
      }
    }
  }
  if (tid == 0) {
    if (n >= 2) {
      d[n - 2] = G[(int64_t)(n - 2) * n + (n - 2)];
      e[n - 2] = G[(int64_t)(n - 1) * n + (n - 2)];
    }
    d[n - 1] = G[(int64_t)(n - 1) * n + (n - 1)];
  }
  __syncthreads();
  // Gershgorin interval of the tridiagonal (v, w: scratch from here on)
  double lo = INFINITY, hi = -INFINITY;
  for (int j = tid; j < n; j += EIG_THREADS) {
    const double r = (j > 0 ? fabs(e[j - 1]) : 0.0) + (j + 1 < n ? fabs(e[j]) : 0.0);
    lo = fmin(lo, d[j] - r);
    hi = fmax(hi, d[j] + r);
  }
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(LG_FULL, lo, o));
    hi = fmax(hi, __shfl_xor_sync(LG_FULL, hi, o));
  }
  __shared__ double red_hi[EIG_THREADS / 32];
  __syncthreads();
  if (lane == 0) { red[warp] = lo; red_hi[warp] = hi; }
  __syncthreads();
  lo = red[0]; hi = red_hi[0];
  for (int q = 1; q < EIG_THREADS / 32; ++q) { lo = fmin(lo, red[q]); hi = fmax(hi, red_hi[q]); }
  const double span = fmax(hi - lo, 1e-300);
  const double pivmin = 1e-300;  // |q| floor (a zero pivot counts as negative, LAPACK's rule)
  // the squared off-diagonals, reused by every count
  __syncthreads();
  for (int j = tid; j + 1 < n; j += EIG_THREADS) v[j] = e[j] * e[j];
  __syncthreads();
  for (int idx = tid; idx < n; idx += EIG_THREADS) {
    double a = lo - 1e-12 * span, b = hi + 1e-12 * span;  // count(a) <= idx < count(b)
    for (int it = 0; it < 128; ++it) {
      const double mid = 0.5 * (a + b);
      if (!(mid > a && mid < b)) break;  // fp64 resolution reached
      int cnt = 0;
      double q = d[0] - mid;
      if (fabs(q) < pivmin) q = -pivmin;
      cnt += q < 0.0;
      for (int j = 1; j < n; ++j) {
        q = (d[j] - mid) - v[j - 1] / q;
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
      }
      if (cnt > idx) b = mid; else a = mid;
    }
    W[idx] = 0.5 * (a + b);
  }
}

// err / bits of one matrix layer from its ascending eigenvalues W (n of them)
__global__ void k_svd_err(const double* __restrict__ W, int n, int64_t m, int64_t k, const int32_t* __restrict__ ranks,
                          int K, int layer, double* __restrict__ err, int64_t* __restrict__ bits) {
  const int c = threadIdx.x;
  if (c >= K) return;
  const int64_t r = ranks[c];
  if (r * (m + k) >= m * k) {  // lossless candidate (R11)
    err[(int64_t)layer * K + c] = 0.0;
    bits[(int64_t)layer * K + c] = 32 * m * k;
    return;
  }
  double s = 0.0;
  for (int64_t i = 0; i < (int64_t)n - r; ++i) s += fmax(W[i], 0.0);
  err[(int64_t)layer * K + c] = sqrt(s);
  bits[(int64_t)layer * K + c] = 32 * r * (m + k);
}

// every layer's row: lossless (err 0, 32 n bits) unless a matrix layer fills it later
__global__ void k_svd_rows_init(const DevLayer* __restrict__ layers, int L, int K, double* __restrict__ err,
                                int64_t* __restrict__ bits) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L * K; i += gridDim.x * blockDim.x) {
    err[i] = 0.0;
    bits[i] = 32 * layers[i / K].numel;
  }
}

// per-layer sum of squares: one CTA per layer, fixed strided order + fixed tree
__global__ void __launch_bounds__(256)
k_layer_norms(const float* __restrict__ g, const float* __restrict__ e, const DevLayer* __restrict__ layers,
              double* __restrict__ norm) {
  __shared__ double sm[256];
  const DevLayer ly = layers[blockIdx.x];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < ly.numel; i += 256) {
    const float x = __fadd_rn(__fadd_rn(g[ly.offset + i], e ? e[ly.offset + i] : 0.f), 0.f);
    s = fma((double)x, (double)x, s);
  }
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) norm[blockIdx.x] = sqrt(sm[0]);
}

}  // namespace lg

extern "C" int lgreco_layer_norms(lgreco_ctx* c, const float* d_g, const float* d_ef, double* d_norm, void* stream) {
  if (!c || !d_g || !d_norm) { lg_set_error("null argument"); return LGRECO_EINVAL; }
  if (c->L == 0) return LGRECO_OK;
  lg::k_layer_norms<<<c->L, 256, 0, (cudaStream_t)stream>>>(d_g, d_ef, c->d_layers, d_norm);
  LG_CUDA(cudaGetLastError());
  c->launches += 1;
  return LGRECO_OK;
}

struct SvdWs {
  double *part = nullptr, *G = nullptr, *W = nullptr;
  lg::EigMat* mats = nullptr;
  int64_t* woff = nullptr;
  size_t gcap = 0, wcap = 0, pcap = 0;
  int nmat = 0;
};

void svd_destroy(lgreco_ctx* c) {
  SvdWs* s = static_cast<SvdWs*>(c->svd);
  if (!s) return;
  cudaFree(s->part); cudaFree(s->G); cudaFree(s->W); cudaFree(s->mats); cudaFree(s->woff);
  delete s;
  c->svd = nullptr;
}

extern "C" int lgreco_psgd_profile_svd(lgreco_ctx* c, const float* d_g, const float* d_ef, double* d_err,
                                       int64_t* d_bits, void* stream) {
  if (!c || !d_g || !d_err || !d_bits) { lg_set_error("null argument"); return LGRECO_EINVAL; }
  if (c->family != LGRECO_POWERSGD) { lg_set_error("svd profile: PowerSGD ctx only"); return LGRECO_EUNSUPPORTED; }
  cudaStream_t st = (cudaStream_t)stream;
  const int L = c->L, K = c->K;
  // matrix layers (R11 view) with at least one lossy candidate
  std::vector<int> mats;
  int nmax = 0;
  size_t gtot = 0, wtot = 0;
  std::vector<lg::EigMat> em;
  std::vector<int64_t> wo;
  for (int l = 0; l < L; ++l) {
    const lgreco_layer& ly = c->layers[l];
    if (!ly.compress || ly.rows <= 0 || ly.cols <= 0) continue;
    const int64_t m = ly.rows, k = ly.cols;
    bool lossy = false;
    for (int j = 0; j < K; ++j) lossy |= (int64_t)c->params[j] * (m + k) < m * k;
    if (!lossy) continue;
    const int n = (int)std::min(m, k);
    if (n > lg::EIG_NMAX) {
      lg_set_error("svd profile: layer %d has min(m, k) = %d > %d", l, n, lg::EIG_NMAX);
      return LGRECO_EUNSUPPORTED;
    }
    mats.push_back(l);
    em.push_back(lg::EigMat{(int64_t)gtot, n, 0});
    wo.push_back((int64_t)wtot);
    gtot += (size_t)n * n;
    wtot += (size_t)n;
    nmax = std::max(nmax, n);
  }
  lg::k_svd_rows_init<<<64, 256, 0, st>>>(c->d_layers, L, K, d_err, d_bits);
  LG_CUDA(cudaGetLastError());
  c->launches += 1;
  if (mats.empty()) return LGRECO_OK;
  SvdWs* s = static_cast<SvdWs*>(c->svd);
  if (!s) { s = new SvdWs(); c->svd = s; }
  const int nsplit = 8;
  const size_t pneed = (size_t)nsplit * nmax * nmax;
  // (grown only between calls: the stream is synchronised before a buffer is replaced)
  if (s->gcap < gtot || s->wcap < wtot || s->pcap < pneed || s->nmat < (int)mats.size()) {
    LG_CUDA(cudaStreamSynchronize(st));
    cudaFree(s->part); cudaFree(s->G); cudaFree(s->W); cudaFree(s->mats); cudaFree(s->woff);
    s->part = s->G = s->W = nullptr; s->mats = nullptr; s->woff = nullptr;
    LG_CUDA(cudaMalloc(&s->part, sizeof(double) * pneed));
    LG_CUDA(cudaMalloc(&s->G, sizeof(double) * gtot));
    LG_CUDA(cudaMalloc(&s->W, sizeof(double) * wtot));
    LG_CUDA(cudaMalloc(&s->mats, sizeof(lg::EigMat) * mats.size()));
    LG_CUDA(cudaMalloc(&s->woff, sizeof(int64_t) * mats.size()));
    s->gcap = gtot; s->wcap = wtot; s->pcap = pneed; s->nmat = (int)mats.size();
  }
  LG_CUDA(cudaMemcpyAsync(s->mats, em.data(), sizeof(lg::EigMat) * em.size(), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(s->woff, wo.data(), sizeof(int64_t) * wo.size(), cudaMemcpyHostToDevice, st));
  // every matrix's fp64 Gram (each launch over the whole GPU), then all eigenvalues at once
  for (size_t i = 0; i < mats.size(); ++i) {
    const lgreco_layer& ly = c->layers[mats[i]];
    const int64_t m = ly.rows, k = ly.cols;
    const bool rows = m <= k;
    const int n = em[i].n;
    const int64_t t = rows ? k : m;
    const int nt = (n + lg::GT - 1) / lg::GT;
    lg::k_gram64<<<dim3(nt * (nt + 1) / 2, nsplit), lg::G_THREADS, 0, st>>>(d_g, d_ef, ly.offset, (int)k, n, t,
                                                                             rows ? 1 : 0, nsplit, s->part);
    lg::k_gram_reduce<<<std::max(1, std::min(1024, (int)(((int64_t)n * n + 255) / 256))), 256, 0, st>>>(
        s->part, nsplit, (int64_t)n * n, s->G + em[i].goff);
    LG_CUDA(cudaGetLastError());
    c->launches += 2;
  }
  const size_t esmem = sizeof(double) * 6 * (size_t)nmax;
  // (always: with the static reduction arrays, 48 KB of dynamic shared memory already
  // exceeds the default limit)
  LG_CUDA(cudaFuncSetAttribute(lg::k_sym_eigvals, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esmem));
  lg::k_sym_eigvals<<<(unsigned)mats.size(), lg::EIG_THREADS, esmem, st>>>(s->G, s->mats, s->W, s->woff);
  LG_CUDA(cudaGetLastError());
  c->launches += 1;
  for (size_t i = 0; i < mats.size(); ++i) {
    const lgreco_layer& ly = c->layers[mats[i]];
    lg::k_svd_err<<<1, std::max(32, ((K + 31) / 32) * 32), 0, st>>>(s->W + wo[i], em[i].n, ly.rows, ly.cols,
                                                                      c->d_params, K, mats[i], d_err, d_bits);
    c->launches += 1;
  }
  LG_CUDA(cudaGetLastError());
  return LGRECO_OK;
}

// NEXT-2 selector: resolved once per ctx from the layer shapes
extern "C" int lgreco_psgd_set_method(lgreco_ctx* c, int32_t method) {
  if (!c || c->family != LGRECO_POWERSGD) { lg_set_error("psgd_set_method: PowerSGD ctx only"); return LGRECO_EINVAL; }
  if (method == LGRECO_PSGD_POWER || method == LGRECO_PSGD_SVD) { c->psgd_method = method; return LGRECO_OK; }
  if (method != LGRECO_PSGD_AUTO) { lg_set_error("psgd_set_method: bad method %d", method); return LGRECO_EINVAL; }
  double t_pow = 0.0, t_svd = 0.0, nmax = 0.0;
  for (int l = 0; l < c->L; ++l) {
    const lgreco_layer& ly = c->layers[l];
    if (!ly.compress || ly.rows <= 0 || ly.cols <= 0) continue;
    const double m = ly.rows, k = ly.cols, n = std::min(m, k);
    int rmax = 0;
    for (int j = 0; j < c->K; ++j)
      if ((double)c->params[j] * (m + k) < m * k) rmax = std::max(rmax, c->params[j]);
    if (rmax == 0) continue;
    t_pow += (double)c->power_steps * m * k * rmax * 1.9e-13;
    // the fp64 Gram, then the eigensolver's HBM traffic (all matrices at once: ~8 n^3
    // bytes each at ~3.5 TB/s aggregate; measured: C2 20 ms, C5 269 ms)
    t_svd += m * k * n * 1e-13 + n * n * n * 2.2e-12;
    nmax = std::max(nmax, n);
  }
  // dependent-step latencies: n - 2 Householder steps of the largest matrix (~2 us each);
  // a chain of ~10 launches per power step (~3 us each)
  t_svd += nmax * 2e-6;
  t_pow += (double)c->power_steps * 3e-5;
  c->psgd_method = (t_svd < t_pow) ? LGRECO_PSGD_SVD : LGRECO_PSGD_POWER;
  return LGRECO_OK;
}

extern "C" int lgreco_psgd_method(lgreco_ctx* c) {
  if (!c || c->family != LGRECO_POWERSGD) { lg_set_error("psgd_method: PowerSGD ctx only"); return LGRECO_EINVAL; }
  return c->psgd_method;
}
