// svd.cu -- NEXT-2: low-rank errors from the singular values (PAPER.md:696-699,
// "e_r = sqrt(sum_{i > r} sigma_i^2) ... compute squared singular values once, and then
// compute all the errors").  The squared singular values of the m x k view M are the
// eigenvalues of the Gram matrix of its smaller side (n = min(m, k)): G = M M^T (m <= k)
// or M^T M.  G is formed in fp64 from x = fl(g + e) (R2) by a split-K tiled kernel
// (fixed-order split reduction: deterministic), its eigenvalues by cuSOLVER's symmetric
// eigensolver (dsyevd, values only -- a library primitive, not the hot path: this is the
// alternative profile method the paper suggests for large rank ranges), and
// err_r^2 = sum of the n - r smallest eigenvalues (each clamped at 0), summed in fp64 in
// ascending order.
#include <cusolverDn.h>
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
  cusolverDnHandle_t h = nullptr;
  double *part = nullptr, *G = nullptr, *W = nullptr, *work = nullptr;
  int* info = nullptr;
  int nmax = 0, lwork = 0, nsplit = 0;
};

void svd_destroy(lgreco_ctx* c) {
  SvdWs* s = static_cast<SvdWs*>(c->svd);
  if (!s) return;
  if (s->h) cusolverDnDestroy(s->h);
  cudaFree(s->part); cudaFree(s->G); cudaFree(s->W); cudaFree(s->work); cudaFree(s->info);
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
  for (int l = 0; l < L; ++l) {
    const lgreco_layer& ly = c->layers[l];
    if (!ly.compress || ly.rows <= 0 || ly.cols <= 0) continue;
    const int64_t m = ly.rows, k = ly.cols;
    bool lossy = false;
    for (int j = 0; j < K; ++j) lossy |= (int64_t)c->params[j] * (m + k) < m * k;
    if (!lossy) continue;
    mats.push_back(l);
    nmax = std::max<int>(nmax, (int)std::min(m, k));
  }
  lg::k_svd_rows_init<<<64, 256, 0, st>>>(c->d_layers, L, K, d_err, d_bits);
  LG_CUDA(cudaGetLastError());
  c->launches += 1;
  if (mats.empty()) return LGRECO_OK;
  SvdWs* s = static_cast<SvdWs*>(c->svd);
  if (!s) { s = new SvdWs(); c->svd = s; }
  const int nsplit = 8;
  if (!s->h) {
    if (cusolverDnCreate(&s->h) != CUSOLVER_STATUS_SUCCESS) { lg_set_error("cusolverDnCreate failed"); return LGRECO_ECUDA; }
  }
  if (s->nmax < nmax) {
    cudaFree(s->part); cudaFree(s->G); cudaFree(s->W); cudaFree(s->work); cudaFree(s->info);
    s->part = s->G = s->W = s->work = nullptr; s->info = nullptr;
    LG_CUDA(cudaMalloc(&s->part, sizeof(double) * (size_t)nsplit * nmax * nmax));
    LG_CUDA(cudaMalloc(&s->G, sizeof(double) * (size_t)nmax * nmax));
    LG_CUDA(cudaMalloc(&s->W, sizeof(double) * (size_t)nmax));
    LG_CUDA(cudaMalloc(&s->info, sizeof(int)));
    int lw = 0;
    if (cusolverDnDsyevd_bufferSize(s->h, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_UPPER, nmax, s->G, nmax, s->W,
                                    &lw) != CUSOLVER_STATUS_SUCCESS) { lg_set_error("syevd buffer size"); return LGRECO_ECUDA; }
    LG_CUDA(cudaMalloc(&s->work, sizeof(double) * (size_t)std::max(1, lw)));
    s->lwork = lw;
    s->nmax = nmax;
    s->nsplit = nsplit;
  }
  if (cusolverDnSetStream(s->h, st) != CUSOLVER_STATUS_SUCCESS) { lg_set_error("cusolverDnSetStream"); return LGRECO_ECUDA; }
  for (int l : mats) {
    const lgreco_layer& ly = c->layers[l];
    const int64_t m = ly.rows, k = ly.cols;
    const bool rows = m <= k;
    const int n = (int)std::min(m, k);
    const int64_t t = rows ? k : m;
    const int nt = (n + lg::GT - 1) / lg::GT;
    lg::k_gram64<<<dim3(nt * (nt + 1) / 2, nsplit), lg::G_THREADS, 0, st>>>(d_g, d_ef, ly.offset, (int)k, n, t,
                                                                             rows ? 1 : 0, nsplit, s->part);
    lg::k_gram_reduce<<<std::max(1, std::min(1024, (int)(((int64_t)n * n + 255) / 256))), 256, 0, st>>>(
        s->part, nsplit, (int64_t)n * n, s->G);
    LG_CUDA(cudaGetLastError());
    int lw = 0;
    if (cusolverDnDsyevd_bufferSize(s->h, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_UPPER, n, s->G, n, s->W, &lw) !=
            CUSOLVER_STATUS_SUCCESS || lw > s->lwork) {
      lg_set_error("syevd workspace");
      return LGRECO_ECUDA;
    }
    if (cusolverDnDsyevd(s->h, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_UPPER, n, s->G, n, s->W, s->work, s->lwork,
                         s->info) != CUSOLVER_STATUS_SUCCESS) {
      lg_set_error("cusolverDnDsyevd failed (layer %d)", l);
      return LGRECO_ECUDA;
    }
    lg::k_svd_err<<<1, std::max(32, ((K + 31) / 32) * 32), 0, st>>>(s->W, n, m, k, c->d_params, K, l, d_err,
                                                                      d_bits);
    LG_CUDA(cudaGetLastError());
    c->launches += 3;
  }
  return LGRECO_OK;
}

// NEXT-2 selector: resolved once per ctx from the layer shapes
extern "C" int lgreco_psgd_set_method(lgreco_ctx* c, int32_t method) {
  if (!c || c->family != LGRECO_POWERSGD) { lg_set_error("psgd_set_method: PowerSGD ctx only"); return LGRECO_EINVAL; }
  if (method == LGRECO_PSGD_POWER || method == LGRECO_PSGD_SVD) { c->psgd_method = method; return LGRECO_OK; }
  if (method != LGRECO_PSGD_AUTO) { lg_set_error("psgd_set_method: bad method %d", method); return LGRECO_EINVAL; }
  double t_pow = 0.0, t_svd = 0.0;
  for (int l = 0; l < c->L; ++l) {
    const lgreco_layer& ly = c->layers[l];
    if (!ly.compress || ly.rows <= 0 || ly.cols <= 0) continue;
    const double m = ly.rows, k = ly.cols, n = std::min(m, k);
    int rmax = 0;
    for (int j = 0; j < c->K; ++j)
      if ((double)c->params[j] * (m + k) < m * k) rmax = std::max(rmax, c->params[j]);
    if (rmax == 0) continue;
    t_pow += (double)c->power_steps * m * k * rmax * 1.9e-13;
    t_svd += m * k * n * 1e-13 + n * n * n * 1e-11;
  }
  c->psgd_method = (t_svd < t_pow) ? LGRECO_PSGD_SVD : LGRECO_PSGD_POWER;
  return LGRECO_OK;
}

extern "C" int lgreco_psgd_method(lgreco_ctx* c) {
  if (!c || c->family != LGRECO_POWERSGD) { lg_set_error("psgd_method: PowerSGD ctx only"); return LGRECO_EINVAL; }
  return c->psgd_method;
}
