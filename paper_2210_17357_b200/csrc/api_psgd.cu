// api_psgd.cu -- PowerSGD family behind the C ABI: context state, profile (K3),
// the one-step warm-started compression (K7) with two all-reduces, raw layers.
#include <algorithm>

#include "ctx.h"

struct Psgd {
  int nM = 0;                       // matrix layers handled by the low-rank path
  std::vector<int32_t> mlayer;      // their layer indices
  std::vector<int32_t> rprof;       // profile rank r_max per matrix layer (0: none compressible)
  std::vector<int64_t> poff, qoff, goff;  // slots sized for the largest candidate rank
  int64_t Psz = 0, Qsz = 0, Gsz = 0;
  int Rmax = 0;
  // profile launch config
  lg::PLayer* d_pl_prof = nullptr;
  lg::PTile *d_rt_prof = nullptr, *d_ct_prof = nullptr, *d_rt128_prof = nullptr, *d_ct128_prof = nullptr;
  lg::PTile* d_et_prof = nullptr;
  int n_prof = 0, nrt_prof = 0, nct_prof = 0, rmax_prof = 0, nrt128_prof = 0, nct128_prof = 0, net_prof = 0;
  int mmax_prof = 0, mmax_c = 0;
  // TMA maps of the tensor-core GEMMs (psgd_tc.cu): host layer lists, config versions,
  // device areas [prof MQ, prof M^T P, compress MQ, compress M^T P] and their caches
  std::vector<lg::PLayer> hpl_prof, hpl_c;
  uint64_t ver_c = 1;
  void* maps[4] = {nullptr, nullptr, nullptr, nullptr};
  lg::TcMapCache mcache[4];
  int32_t* d_et0_prof = nullptr;
  lg::PTile *d_gcp_prof = nullptr, *d_gcq_prof = nullptr;  // Gram row chunks (P-shaped / Q-shaped)
  int32_t *d_gcp0_prof = nullptr, *d_gcq0_prof = nullptr;
  int ngcp_prof = 0, ngcq_prof = 0;
  int32_t* d_ranks = nullptr;
  int32_t* d_ismat = nullptr;
  // compress launch config (per plan)
  std::vector<int32_t> plan_choice;
  bool plan_valid = false;
  std::vector<int32_t> cur_rank;    // rank currently held in Q_ws per matrix layer (0: none)
  lg::PLayer* d_pl_c = nullptr;
  lg::PTile *d_rt_c = nullptr, *d_ct_c = nullptr, *d_rt128_c = nullptr, *d_ct128_c = nullptr, *d_et_c = nullptr;
  int n_c = 0, nrt_c = 0, nct_c = 0, rmax_c = 0, nrt128_c = 0, nct128_c = 0, net_c = 0;
  lg::PTile* d_gcp_c = nullptr;
  int32_t* d_gcp0_c = nullptr;
  int ngcp_c = 0;
  int32_t* d_initflag = nullptr;
  bool need_init = false;
  lg::RawSeg* d_raw = nullptr;
  int nraw = 0;
  int64_t Sraw = 0;
  unsigned char* h_stage = nullptr;
  size_t stage_bytes = 0;
  cudaEvent_t evt = nullptr;
  // buffers
  float *P = nullptr, *Ph = nullptr, *Qprof = nullptr, *Qws = nullptr, *Qn = nullptr, *part = nullptr;
  float* Ppart = nullptr;  // split-K partials of M Q
  double *G = nullptr, *epart = nullptr;
  double *gpart = nullptr, *GP = nullptr, *GQ = nullptr, *dpart = nullptr;  // Gram partials, profile-error work
  int32_t* eflag = nullptr;
  int max_split = 1, max_ks = 1;
  int nb_max = 1;  // distinct candidate ranks <= 64 (error boundary slots)
  uint8_t *d_raw_pay = nullptr, *d_raw_gath = nullptr;
  int64_t raw_cap = 0;
};

static bool ps_lossless(int64_t m, int64_t k, int64_t r) { return r * (m + k) >= m * k; }

static constexpr int PS_TM = 64;
static constexpr int64_t PS_SPLIT_ROWS = 256;   // M^T P: rows per split (8 K tiles per CTA)
static constexpr int64_t PS_SPLIT_COLS = 256;   // M Q: K columns per split (8 K tiles per CTA)
static constexpr int PE_ROWS = 64, PE_COLS = 256, PE_SLOTS = 64;  // element tiles (psgd.cu)
static int64_t ps_nks(int64_t k) { return std::max<int64_t>(1, (k + PS_SPLIT_COLS - 1) / PS_SPLIT_COLS); }
static int64_t ps_net(int64_t m, int64_t k) { return ((m + PE_ROWS - 1) / PE_ROWS) * ((k + PE_COLS - 1) / PE_COLS); }
static constexpr int64_t RAW_CHUNK = 16384;

// Build PLayer + tiles for the ranks `r` (per matrix layer; 0 = skip)
struct GramChunks { std::vector<lg::PTile> p, q; std::vector<int32_t> p0, q0; };
static constexpr int64_t GC_ROWS = 1024;  // rows per Gram chunk (psgd.cu k_ps_gramc)

static void ps_config(lgreco_ctx* c, const std::vector<int32_t>& r, std::vector<lg::PLayer>& pl,
                      std::vector<lg::PTile>& rt, std::vector<lg::PTile>& ct, std::vector<int32_t>& et0, int& rmax,
                      std::vector<lg::PTile>& rt128, std::vector<lg::PTile>& ct128, std::vector<lg::PTile>& et,
                      GramChunks& gc) {
  Psgd* p = c->ps;
  pl.clear(); rt.clear(); ct.clear(); et0.clear(); rt128.clear(); ct128.clear(); et.clear();
  gc.p.clear(); gc.q.clear(); gc.p0.clear(); gc.q0.clear();
  rmax = 0;
  for (int i = 0; i < p->nM; ++i) {
    if (r[i] <= 0) continue;
    const lgreco_layer& ly = c->layers[p->mlayer[i]];
    const int ci = (int)pl.size();
    const int nsplit = (int)std::max<int64_t>(1, (ly.rows + PS_SPLIT_ROWS - 1) / PS_SPLIT_ROWS);
    const int nks = (int)ps_nks(ly.cols);
    pl.push_back(lg::PLayer{ly.offset, ly.rows, ly.cols, r[i], p->mlayer[i], p->poff[i], p->qoff[i], p->goff[i],
                            p->Qsz, p->Psz, nsplit, nks});
    rmax = std::max(rmax, r[i]);
    et0.push_back((int32_t)et.size());
    for (int i0 = 0; i0 < ly.rows; i0 += PS_TM) rt.push_back(lg::PTile{ci, 0, i0, 0, 0, 0});
    for (int i0 = 0; i0 < ly.rows; i0 += 128)
      for (int s = 0; s < nks; ++s) {
        const int c0 = (int)(s * PS_SPLIT_COLS), c1 = (int)std::min<int64_t>(ly.cols, (s + 1) * PS_SPLIT_COLS);
        rt128.push_back(lg::PTile{ci, s, i0, c1, c0, 0});
      }
    for (int s = 0; s < nsplit; ++s) {
      const int i0 = (int)(s * PS_SPLIT_ROWS), i1 = (int)std::min<int64_t>(ly.rows, (s + 1) * PS_SPLIT_ROWS);
      for (int c0 = 0; c0 < ly.cols; c0 += PS_TM) ct.push_back(lg::PTile{ci, s, i0, i1, c0, 0});
      for (int c0 = 0; c0 < ly.cols; c0 += 128) ct128.push_back(lg::PTile{ci, s, i0, i1, c0, 0});
    }
    for (int i0 = 0; i0 < ly.rows; i0 += PE_ROWS)
      for (int c0 = 0; c0 < ly.cols; c0 += PE_COLS) et.push_back(lg::PTile{ci, 0, i0, 0, c0, 0});
  }
  // Gram row chunks: shorter for small ranks (more CTAs; the r^2 partial per chunk stays small)
  const int64_t gcr = rmax <= 16 ? 128 : rmax <= 32 ? 256 : GC_ROWS;
  for (int ci = 0; ci < (int)pl.size(); ++ci) {
    gc.p0.push_back((int32_t)gc.p.size());
    for (int64_t i0 = 0; i0 < pl[ci].m; i0 += gcr)
      gc.p.push_back(lg::PTile{ci, 0, (int)i0, (int)std::min<int64_t>(pl[ci].m, i0 + gcr), 0, 0});
    gc.q0.push_back((int32_t)gc.q.size());
    for (int64_t i0 = 0; i0 < pl[ci].k; i0 += gcr)
      gc.q.push_back(lg::PTile{ci, 0, (int)i0, (int)std::min<int64_t>(pl[ci].k, i0 + gcr), 0, 0});
  }
  et0.push_back((int32_t)et.size());
  gc.p0.push_back((int32_t)gc.p.size());
  gc.q0.push_back((int32_t)gc.q.size());
}

int psgd_init(lgreco_ctx* c, cudaStream_t st) {
  Psgd* p = new Psgd();
  c->ps = p;
  const int L = c->L, K = c->K;
  std::vector<int32_t> ismat(L, 0);
  int rcand_max = 0;
  for (int j = 0; j < K; ++j) rcand_max = std::max(rcand_max, c->params[j]);
  int64_t raw_cap = 0;
  for (int l = 0; l < L; ++l) {
    const lgreco_layer& ly = c->layers[l];
    if (ly.compress && ly.rows > 0) {
      int rp = 0, rm = 0;
      for (int j = 0; j < K; ++j)
        if (!ps_lossless(ly.rows, ly.cols, c->params[j])) rp = std::max(rp, c->params[j]);
      rm = rp;
      if (rp > 64) {
        lg_set_error("PowerSGD rank %d > 64 not supported in this build", rp);
        return LGRECO_EUNSUPPORTED;
      }
      p->mlayer.push_back(l);
      p->rprof.push_back(rp);
      p->poff.push_back(p->Psz);
      p->qoff.push_back(p->Qsz);
      p->goff.push_back(p->Gsz);
      p->Psz += (int64_t)ly.rows * rm;
      p->Qsz += (int64_t)ly.cols * rm;
      p->Gsz += (int64_t)rm * rm;
      p->Rmax = std::max(p->Rmax, rm);
      p->max_split = std::max<int>(p->max_split, (int)((ly.rows + PS_SPLIT_ROWS - 1) / PS_SPLIT_ROWS));
      p->max_ks = std::max<int>(p->max_ks, (int)ps_nks(ly.cols));
      ismat[l] = rp > 0;
    }
    raw_cap += 4 * ly.numel + 16;
  }
  p->nM = (int)p->mlayer.size();
  p->cur_rank.assign(p->nM, 0);
  {
    std::vector<int32_t> rs;
    for (int j = 0; j < K; ++j)
      if (c->params[j] >= 1 && c->params[j] <= 64) rs.push_back(c->params[j]);
    std::sort(rs.begin(), rs.end());
    p->nb_max = std::max<int>(1, (int)(std::unique(rs.begin(), rs.end()) - rs.begin()));
  }
  p->raw_cap = raw_cap;
  std::vector<lg::PLayer> pl;
  std::vector<lg::PTile> rt, ct, rt128, ct128, et;
  std::vector<int32_t> et0;
  GramChunks gcs;
  ps_config(c, p->rprof, pl, rt, ct, et0, p->rmax_prof, rt128, ct128, et, gcs);
  for (const auto& x : pl) p->mmax_prof = std::max(p->mmax_prof, (int)x.m);
  p->hpl_prof = pl;
  p->ngcp_prof = (int)gcs.p.size();
  p->ngcq_prof = (int)gcs.q.size();
  p->n_prof = (int)pl.size(); p->nrt_prof = (int)rt.size(); p->nct_prof = (int)ct.size();
  p->nrt128_prof = (int)rt128.size(); p->nct128_prof = (int)ct128.size(); p->net_prof = (int)et.size();
  // compress configs can use at most all matrix layers / tiles of the profile shapes
  size_t max_rt = 0, max_ct = 0, max_rt128 = 0, max_et = 0, max_raw = 0;
  for (int i = 0; i < p->nM; ++i) {
    const lgreco_layer& ly = c->layers[p->mlayer[i]];
    max_rt += (ly.rows + PS_TM - 1) / PS_TM;
    max_ct += (size_t)((ly.rows + PS_SPLIT_ROWS - 1) / PS_SPLIT_ROWS) * ((ly.cols + PS_TM - 1) / PS_TM);
    max_rt128 += (size_t)((ly.rows + 127) / 128) * ps_nks(ly.cols);
    max_et += (size_t)ps_net(ly.rows, ly.cols);
  }
  for (int l = 0; l < L; ++l) max_raw += (c->layers[l].numel + RAW_CHUNK - 1) / RAW_CHUNK;
  // Gram chunks of any config: at most ceil(rows / 128) per factor (the shortest chunks)
  size_t max_gc = 1, max_gq = 1;
  for (int i = 0; i < p->nM; ++i) {
    max_gc += (size_t)((c->layers[p->mlayer[i]].rows + 127) / 128);
    max_gq += (size_t)((c->layers[p->mlayer[i]].cols + 127) / 128);
  }
  p->stage_bytes = sizeof(lg::PLayer) * std::max(1, p->nM) +
                   sizeof(lg::PTile) * (max_rt + 2 * max_ct + max_rt128 + max_et + 8) +
                   sizeof(int32_t) * (2 * (size_t)std::max(1, p->nM) + 2) + sizeof(lg::RawSeg) * (max_raw + 1) + 256 +
                   sizeof(lg::PTile) * (max_gc + 1) + sizeof(int32_t) * (gcs.p0.size() + 1) + 64;
#define PS_ALLOC(ptr, bytes)                                                                \
  if (cudaMalloc((void**)&(ptr), std::max<size_t>((size_t)(bytes), 16)) != cudaSuccess) {  \
    lg_set_error("cudaMalloc %zu bytes failed (psgd)", (size_t)(bytes));                    \
    return LGRECO_ENOMEM;                                                                   \
  }
  PS_ALLOC(p->d_pl_prof, sizeof(lg::PLayer) * std::max<size_t>(1, pl.size()));
  PS_ALLOC(p->d_rt_prof, sizeof(lg::PTile) * std::max<size_t>(1, rt.size()));
  PS_ALLOC(p->d_ct_prof, sizeof(lg::PTile) * std::max<size_t>(1, ct.size()));
  PS_ALLOC(p->d_rt128_prof, sizeof(lg::PTile) * std::max<size_t>(1, rt128.size()));
  PS_ALLOC(p->d_ct128_prof, sizeof(lg::PTile) * std::max<size_t>(1, ct128.size()));
  PS_ALLOC(p->d_et_prof, sizeof(lg::PTile) * std::max<size_t>(1, et.size()));
  PS_ALLOC(p->d_et0_prof, sizeof(int32_t) * et0.size());
  PS_ALLOC(p->d_ranks, sizeof(int32_t) * K);
  PS_ALLOC(p->d_ismat, sizeof(int32_t) * L);
  PS_ALLOC(p->d_pl_c, sizeof(lg::PLayer) * std::max(1, p->nM));
  PS_ALLOC(p->d_rt_c, sizeof(lg::PTile) * std::max<size_t>(1, max_rt));
  PS_ALLOC(p->d_ct_c, sizeof(lg::PTile) * std::max<size_t>(1, max_ct));
  PS_ALLOC(p->d_rt128_c, sizeof(lg::PTile) * std::max<size_t>(1, max_rt128));
  PS_ALLOC(p->d_et_c, sizeof(lg::PTile) * std::max<size_t>(1, max_et));
  PS_ALLOC(p->d_ct128_c, sizeof(lg::PTile) * std::max<size_t>(1, max_ct));
  PS_ALLOC(p->d_initflag, sizeof(int32_t) * std::max(1, p->nM));
  PS_ALLOC(p->d_raw, sizeof(lg::RawSeg) * (max_raw + 1));
  PS_ALLOC(p->P, sizeof(float) * p->Psz);
  PS_ALLOC(p->Ph, sizeof(float) * p->Psz);
  PS_ALLOC(p->Qprof, sizeof(float) * p->Qsz);
  PS_ALLOC(p->Qws, sizeof(float) * p->Qsz);
  PS_ALLOC(p->Qn, sizeof(float) * p->Qsz);
  PS_ALLOC(p->part, sizeof(float) * p->Qsz * p->max_split);
  PS_ALLOC(p->Ppart, sizeof(float) * p->Psz * p->max_ks);
  PS_ALLOC(p->G, sizeof(double) * p->Gsz);
  PS_ALLOC(p->epart, sizeof(double) * std::max<size_t>(1, et.size()) * PE_SLOTS);
  PS_ALLOC(p->gpart, sizeof(double) * 64 * 64 * std::max(max_gc, max_gq));
  PS_ALLOC(p->GP, sizeof(double) * p->Gsz);
  PS_ALLOC(p->GQ, sizeof(double) * p->Gsz);
  PS_ALLOC(p->dpart, sizeof(double) * 65 * std::max<size_t>(1, et.size()));
  PS_ALLOC(p->eflag, sizeof(int32_t) * std::max(1, p->nM));
  for (int q = 0; q < 4; ++q) PS_ALLOC(p->maps[q], (size_t)128 * 3 * std::max(1, p->nM));  // CUtensorMap = 128 B
  PS_ALLOC(p->d_gcp_prof, sizeof(lg::PTile) * std::max<size_t>(1, gcs.p.size()));
  PS_ALLOC(p->d_gcq_prof, sizeof(lg::PTile) * std::max<size_t>(1, gcs.q.size()));
  PS_ALLOC(p->d_gcp0_prof, sizeof(int32_t) * gcs.p0.size());
  PS_ALLOC(p->d_gcq0_prof, sizeof(int32_t) * gcs.q0.size());
  PS_ALLOC(p->d_gcp_c, sizeof(lg::PTile) * max_gc);
  PS_ALLOC(p->d_gcp0_c, sizeof(int32_t) * gcs.p0.size());
  if (K > 128) { lg_set_error("PowerSGD: at most 128 candidate ranks"); return LGRECO_EINVAL; }
  if (c->world > 1) {
    PS_ALLOC(p->d_raw_pay, raw_cap);
    PS_ALLOC(p->d_raw_gath, raw_cap * c->world);
  }
#undef PS_ALLOC
  if (cudaMallocHost((void**)&p->h_stage, p->stage_bytes) != cudaSuccess) return LGRECO_ENOMEM;
  LG_CUDA(cudaEventCreateWithFlags(&p->evt, cudaEventDisableTiming));
  if (!pl.empty()) LG_CUDA(cudaMemcpyAsync(p->d_pl_prof, pl.data(), sizeof(lg::PLayer) * pl.size(), cudaMemcpyHostToDevice, st));
  if (!rt.empty()) LG_CUDA(cudaMemcpyAsync(p->d_rt_prof, rt.data(), sizeof(lg::PTile) * rt.size(), cudaMemcpyHostToDevice, st));
  if (!ct.empty()) LG_CUDA(cudaMemcpyAsync(p->d_ct_prof, ct.data(), sizeof(lg::PTile) * ct.size(), cudaMemcpyHostToDevice, st));
  if (!rt128.empty())
    LG_CUDA(cudaMemcpyAsync(p->d_rt128_prof, rt128.data(), sizeof(lg::PTile) * rt128.size(), cudaMemcpyHostToDevice, st));
  if (!ct128.empty())
    LG_CUDA(cudaMemcpyAsync(p->d_ct128_prof, ct128.data(), sizeof(lg::PTile) * ct128.size(), cudaMemcpyHostToDevice, st));
  if (!et.empty()) LG_CUDA(cudaMemcpyAsync(p->d_et_prof, et.data(), sizeof(lg::PTile) * et.size(), cudaMemcpyHostToDevice, st));
  if (!gcs.p.empty())
    LG_CUDA(cudaMemcpyAsync(p->d_gcp_prof, gcs.p.data(), sizeof(lg::PTile) * gcs.p.size(), cudaMemcpyHostToDevice, st));
  if (!gcs.q.empty())
    LG_CUDA(cudaMemcpyAsync(p->d_gcq_prof, gcs.q.data(), sizeof(lg::PTile) * gcs.q.size(), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(p->d_gcp0_prof, gcs.p0.data(), sizeof(int32_t) * gcs.p0.size(), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(p->d_gcq0_prof, gcs.q0.data(), sizeof(int32_t) * gcs.q0.size(), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(p->d_et0_prof, et0.data(), sizeof(int32_t) * et0.size(), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(p->d_ranks, c->params.data(), sizeof(int32_t) * K, cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(p->d_ismat, ismat.data(), sizeof(int32_t) * L, cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaStreamSynchronize(st));
  return LGRECO_OK;
}

void psgd_destroy(lgreco_ctx* c) {
  Psgd* p = c->ps;
  if (!p) return;
  cudaFree(p->d_pl_prof); cudaFree(p->d_rt_prof); cudaFree(p->d_ct_prof); cudaFree(p->d_et_prof);
  cudaFree(p->d_et0_prof); cudaFree(p->d_et_c); cudaFree(p->Ppart); cudaFree(p->epart);
  cudaFree(p->d_rt128_prof); cudaFree(p->d_ct128_prof); cudaFree(p->d_rt128_c); cudaFree(p->d_ct128_c);
  cudaFree(p->d_ranks); cudaFree(p->d_ismat); cudaFree(p->d_pl_c); cudaFree(p->d_rt_c); cudaFree(p->d_ct_c);
  cudaFree(p->d_initflag); cudaFree(p->d_raw); cudaFree(p->P); cudaFree(p->Ph); cudaFree(p->Qprof);
  cudaFree(p->Qws); cudaFree(p->Qn); cudaFree(p->part); cudaFree(p->G);
  cudaFree(p->d_raw_pay); cudaFree(p->d_raw_gath);
  cudaFree(p->gpart); cudaFree(p->GP); cudaFree(p->GQ); cudaFree(p->dpart); cudaFree(p->eflag);
  cudaFree(p->d_gcp_prof); cudaFree(p->d_gcq_prof); cudaFree(p->d_gcp0_prof); cudaFree(p->d_gcq0_prof);
  cudaFree(p->d_gcp_c); cudaFree(p->d_gcp0_c);
  for (int q = 0; q < 4; ++q) cudaFree(p->maps[q]);
  if (p->h_stage) cudaFreeHost(p->h_stage);
  if (p->evt) cudaEventDestroy(p->evt);
  delete p;
  c->ps = nullptr;
}

static lg::PsArgs ps_args_prof(lgreco_ctx* c, const float* g, const float* e) {
  Psgd* p = c->ps;
  lg::PsArgs a{g, e, p->d_pl_prof, p->n_prof, p->d_rt_prof, p->nrt_prof, p->d_ct_prof, p->nct_prof, p->rmax_prof,
               p->d_rt128_prof, p->nrt128_prof, p->d_ct128_prof, p->nct128_prof,
               p->d_et_prof, p->net_prof, p->d_et0_prof};
  a.gcp = p->d_gcp_prof; a.n_gcp = p->ngcp_prof; a.gcp0 = p->d_gcp0_prof;
  a.gcq = p->d_gcq_prof; a.n_gcq = p->ngcq_prof; a.gcq0 = p->d_gcq0_prof;
  a.gpart = p->gpart;
  a.mmax = p->mmax_prof;
  a.h_pl = p->hpl_prof.data(); a.cfg_ver = 0;
  a.maps_mq = p->maps[0]; a.maps_tr = p->maps[1]; a.mc_mq = &p->mcache[0]; a.mc_tr = &p->mcache[1];
  return a;
}
static lg::PsArgs ps_args_c(lgreco_ctx* c, const float* g, const float* e) {
  Psgd* p = c->ps;
  lg::PsArgs a{g, e, p->d_pl_c, p->n_c, p->d_rt_c, p->nrt_c, p->d_ct_c, p->nct_c, p->rmax_c,
               p->d_rt128_c, p->nrt128_c, p->d_ct128_c, p->nct128_c, p->d_et_c, p->net_c, nullptr};
  a.gcp = p->d_gcp_c; a.n_gcp = p->ngcp_c; a.gcp0 = p->d_gcp0_c;
  a.gpart = p->gpart;
  a.mmax = p->mmax_c;
  a.h_pl = p->hpl_c.data(); a.cfg_ver = p->ver_c;
  a.maps_mq = p->maps[2]; a.maps_tr = p->maps[3]; a.mc_mq = &p->mcache[2]; a.mc_tr = &p->mcache[3];
  return a;
}

int psgd_profile(lgreco_ctx* c, const float* g, const float* e, uint64_t step, double* err, int64_t* bits,
                 cudaStream_t st) {
  Psgd* p = c->ps;
  LG_LAUNCH(c, lg::launch_ps_lossless_rows(c->d_layers, c->L, c->K, p->d_ismat, err, bits, st));
  c->launches += 1;
  if (p->n_prof == 0) return LGRECO_OK;
  const lg::PsArgs a = ps_args_prof(c, g, e);
  const uint32_t k0 = (uint32_t)c->seed, k1 = (uint32_t)(c->seed >> 32);
  LG_LAUNCH(c, lg::launch_ps_initq(a, p->Qprof, k0, k1, (uint32_t)step, nullptr, st));
  c->launches += 1;
  for (int s = 0; s < c->power_steps; ++s) {
    LG_LAUNCH(c, lg::launch_ps_mq(a, p->Qprof, p->P, p->Ppart, st));
    LG_LAUNCH(c, lg::launch_ps_orth(a, p->P, 1.0f, p->G, p->Ph, st));
    LG_LAUNCH(c, lg::launch_ps_mtp(a, p->Ph, p->part, p->Qprof, 1.0f, st));
    c->launches += 12;  // mq 2 + orth 8 (gram 2 x 2) + mtp 2
  }
  const lg::PsErrBufs w{p->dpart, p->GP, p->GQ, p->eflag};
  LG_LAUNCH(c, lg::launch_ps_err(a, p->Ph, p->Qprof, p->d_ranks, c->K, p->nb_max, err, bits, p->epart, w, st));
  c->launches += 8;  // gram 2 x 2 + edot + err_exp + (flagged) err_cols + err_final
  return LGRECO_OK;
}

// plan: chosen ranks -> compress config, raw segments; re-init Q_ws where the rank changed
static int psgd_set_plan(lgreco_ctx* c, const int32_t* choice, cudaStream_t st) {
  Psgd* p = c->ps;
  std::vector<int32_t> chv(choice, choice + c->L);
  for (int l = 0; l < c->L; ++l)
    if (!c->layers[l].compress) chv[l] = -1;
  if (p->plan_valid && chv == p->plan_choice) return LGRECO_OK;
  std::vector<int32_t> r(p->nM, 0), initf(std::max(1, p->nM), 0);
  std::vector<char> raw(c->L, 1);
  for (int l = 0; l < c->L; ++l)  // another family's layers (NEXT-4): neither low-rank nor raw
    if (choice[l] == LGRECO_CHOICE_SKIP) raw[l] = 0;
  for (int i = 0; i < p->nM; ++i) {
    const int l = p->mlayer[i];
    const int j = choice[l];
    if (j == LGRECO_CHOICE_SKIP) continue;
    if (j < 0 || j >= c->K) {
      lg_set_error("choice[%d]=%d out of range [0,%d)", l, j, c->K);
      return LGRECO_EINVAL;
    }
    const int rk = c->params[j];
    if (!ps_lossless(c->layers[l].rows, c->layers[l].cols, rk)) {
      r[i] = rk;
      raw[l] = 0;
    }
  }
  for (int l = 0; l < c->L; ++l)
    if (c->layers[l].compress && c->layers[l].rows <= 0 && choice[l] != LGRECO_CHOICE_SKIP &&
        (choice[l] < 0 || choice[l] >= c->K)) {
      lg_set_error("choice[%d]=%d out of range [0,%d)", l, choice[l], c->K);
      return LGRECO_EINVAL;
    }
  std::vector<lg::PLayer> pl;
  std::vector<lg::PTile> rt, ct, rt128, ct128, et;
  std::vector<int32_t> et0;
  int rmax = 0;
  GramChunks gcs;
  ps_config(c, r, pl, rt, ct, et0, rmax, rt128, ct128, et, gcs);
  int mmax = 0;
  for (const auto& x : pl) mmax = std::max(mmax, (int)x.m);
  // init flags follow the compress config order (layers with r > 0)
  int ci = 0;
  bool any_init = false;
  for (int i = 0; i < p->nM; ++i) {
    if (r[i] <= 0) { p->cur_rank[i] = 0; continue; }
    initf[ci] = (p->cur_rank[i] != r[i]);
    any_init |= initf[ci] != 0;
    p->cur_rank[i] = r[i];
    ++ci;
  }
  std::vector<lg::RawSeg> segs;
  int64_t off = 0;
  for (int l = 0; l < c->L; ++l) {
    if (!raw[l]) continue;
    const lgreco_layer& ly = c->layers[l];
    for (int64_t f = 0; f < ly.numel; f += RAW_CHUNK)
      segs.push_back(lg::RawSeg{ly.offset + f, std::min(RAW_CHUNK, ly.numel - f), off + 4 * f});
    off += 4 * ly.numel;
    off = (off + 15) & ~(int64_t)15;
  }
  LG_CUDA(cudaEventSynchronize(p->evt));
  unsigned char* h = p->h_stage;
  size_t o = 0;
  auto put = [&](const void* src, size_t n) { memcpy(h + o, src, n); size_t at = o; o += (n + 15) & ~(size_t)15; return at; };
  const size_t o_pl = put(pl.data(), sizeof(lg::PLayer) * pl.size());
  const size_t o_rt = put(rt.data(), sizeof(lg::PTile) * rt.size());
  const size_t o_ct = put(ct.data(), sizeof(lg::PTile) * ct.size());
  const size_t o_rt2 = put(rt128.data(), sizeof(lg::PTile) * rt128.size());
  const size_t o_ct2 = put(ct128.data(), sizeof(lg::PTile) * ct128.size());
  const size_t o_et = put(et.data(), sizeof(lg::PTile) * et.size());
  const size_t o_if = put(initf.data(), sizeof(int32_t) * initf.size());
  const size_t o_sg = put(segs.data(), sizeof(lg::RawSeg) * segs.size());
  const size_t o_gc = put(gcs.p.data(), sizeof(lg::PTile) * gcs.p.size());
  const size_t o_gc0 = put(gcs.p0.data(), sizeof(int32_t) * gcs.p0.size());
  if (!gcs.p.empty())
    LG_CUDA(cudaMemcpyAsync(p->d_gcp_c, h + o_gc, sizeof(lg::PTile) * gcs.p.size(), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(p->d_gcp0_c, h + o_gc0, sizeof(int32_t) * gcs.p0.size(), cudaMemcpyHostToDevice, st));
  if (!pl.empty()) LG_CUDA(cudaMemcpyAsync(p->d_pl_c, h + o_pl, sizeof(lg::PLayer) * pl.size(), cudaMemcpyHostToDevice, st));
  if (!rt.empty()) LG_CUDA(cudaMemcpyAsync(p->d_rt_c, h + o_rt, sizeof(lg::PTile) * rt.size(), cudaMemcpyHostToDevice, st));
  if (!ct.empty()) LG_CUDA(cudaMemcpyAsync(p->d_ct_c, h + o_ct, sizeof(lg::PTile) * ct.size(), cudaMemcpyHostToDevice, st));
  if (!rt128.empty())
    LG_CUDA(cudaMemcpyAsync(p->d_rt128_c, h + o_rt2, sizeof(lg::PTile) * rt128.size(), cudaMemcpyHostToDevice, st));
  if (!ct128.empty())
    LG_CUDA(cudaMemcpyAsync(p->d_ct128_c, h + o_ct2, sizeof(lg::PTile) * ct128.size(), cudaMemcpyHostToDevice, st));
  if (!et.empty()) LG_CUDA(cudaMemcpyAsync(p->d_et_c, h + o_et, sizeof(lg::PTile) * et.size(), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(p->d_initflag, h + o_if, sizeof(int32_t) * initf.size(), cudaMemcpyHostToDevice, st));
  if (!segs.empty()) LG_CUDA(cudaMemcpyAsync(p->d_raw, h + o_sg, sizeof(lg::RawSeg) * segs.size(), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaEventRecord(p->evt, st));
  p->n_c = (int)pl.size(); p->nrt_c = (int)rt.size(); p->nct_c = (int)ct.size(); p->rmax_c = rmax;
  p->nrt128_c = (int)rt128.size(); p->nct128_c = (int)ct128.size(); p->net_c = (int)et.size();
  p->ngcp_c = (int)gcs.p.size();
  p->mmax_c = mmax;
  p->hpl_c = pl;
  ++p->ver_c;
  p->nraw = (int)segs.size();
  p->Sraw = off;
  p->need_init = any_init;
  p->plan_choice = chv;
  p->plan_valid = true;
  return LGRECO_OK;
}

int64_t psgd_payload_bytes(lgreco_ctx* c, const int32_t* choice) {
  // raw (uncompressed) bytes of the plan; the low-rank factors travel through the all-reduces
  int64_t off = 0;
  for (int l = 0; l < c->L; ++l) {
    const lgreco_layer& ly = c->layers[l];
    bool raw = true;
    if (choice[l] == LGRECO_CHOICE_SKIP) continue;  // another family's layer
    if (ly.compress && ly.rows > 0) {
      const int j = choice[l];
      if (j < 0 || j >= c->K) return LGRECO_EINVAL;
      raw = ps_lossless(ly.rows, ly.cols, c->params[j]);
    }
    if (!raw) continue;
    off += 4 * ly.numel;
    off = (off + 15) & ~(int64_t)15;
  }
  return off;
}

// stage 1: P_w = M_w Q_ws into d_P (nullable: internal), with Q_ws (re)initialised where needed
int psgd_p(lgreco_ctx* c, const int32_t* choice, const float* g, const float* e, float* d_P, uint64_t step,
           cudaStream_t st) {
  Psgd* p = c->ps;
  LG_TRY(psgd_set_plan(c, choice, st));
  const lg::PsArgs a = ps_args_c(c, g, e);
  if (p->need_init) {
    const uint32_t k0 = (uint32_t)c->seed, k1 = (uint32_t)(c->seed >> 32);
    LG_LAUNCH(c, lg::launch_ps_initq(a, p->Qws, k0, k1, (uint32_t)step, p->d_initflag, st));
    c->launches += 1;
    p->need_init = false;
  }
  LG_LAUNCH(c, lg::launch_ps_mq(a, p->Qws, d_P ? d_P : p->P, p->Ppart, st));
  c->launches += 2;
  return LGRECO_OK;
}

// stage 2: Phat = orth(Psum / W); Q_w = M_w^T Phat into d_Q (Qws when d_Q == Qws)
int psgd_q(lgreco_ctx* c, const int32_t* choice, const float* g, const float* e, const float* d_Psum, int W,
           float* d_Q, cudaStream_t st) {
  Psgd* p = c->ps;
  LG_TRY(psgd_set_plan(c, choice, st));
  const lg::PsArgs a = ps_args_c(c, g, e);
  const float invW = 1.0f / (float)W;
  LG_LAUNCH(c, lg::launch_ps_orth(a, d_Psum ? d_Psum : p->P, invW, p->G, p->Ph, st));
  LG_LAUNCH(c, lg::launch_ps_mtp(a, p->Ph, p->part, d_Q ? d_Q : p->Qn, 1.0f, st));
  c->launches += 8;  // orth 6 + mtp 2
  return LGRECO_OK;
}

// stage 3: Q_ws = Qsum / W; out = Phat Q_ws^T; e = x - out
int psgd_out(lgreco_ctx* c, const int32_t* choice, const float* g, float* ef, const float* d_Qsum, int W, float* out,
             cudaStream_t st) {
  Psgd* p = c->ps;
  LG_TRY(psgd_set_plan(c, choice, st));
  const lg::PsArgs a = ps_args_c(c, g, ef);
  if (d_Qsum && d_Qsum != p->Qws) {
    LG_LAUNCH(c, lg::launch_ps_mtp_scale(a, d_Qsum, p->Qws, 1.0f / (float)W, st));
    c->launches += 1;
  }
  LG_LAUNCH(c, lg::launch_ps_out(a, ef, out, p->Ph, p->Qws, st));
  c->launches += 1;
  return LGRECO_OK;
}

int psgd_raw_pack(lgreco_ctx* c, const int32_t* choice, const float* g, float* ef, uint8_t* payload, float* out,
                  cudaStream_t st) {
  Psgd* p = c->ps;
  LG_TRY(psgd_set_plan(c, choice, st));
  LG_LAUNCH(c, lg::launch_ps_raw_pack(g, ef, payload, out, p->d_raw, p->nraw, c->d_flag, st));
  c->launches += p->nraw > 0;
  return LGRECO_OK;
}

int psgd_raw_combine(lgreco_ctx* c, const int32_t* choice, int W, const uint8_t* gathered, float* out, cudaStream_t st) {
  Psgd* p = c->ps;
  LG_TRY(psgd_set_plan(c, choice, st));
  LG_LAUNCH(c, lg::launch_ps_raw_mean(gathered, p->Sraw, W, out, p->d_raw, p->nraw, st));
  c->launches += p->nraw > 0;
  return LGRECO_OK;
}

int psgd_compress_allreduce(lgreco_ctx* c, const int32_t* choice, const float* g, float* ef, float* out,
                            uint64_t step, cudaStream_t st) {
  Psgd* p = c->ps;
  const int W = c->world;
  if (W == 1) {
    LG_TRY(psgd_p(c, choice, g, ef, nullptr, step, st));
    LG_TRY(psgd_q(c, choice, g, ef, nullptr, 1, p->Qws, st));
    LG_TRY(psgd_out(c, choice, g, ef, nullptr, 1, out, st));
    return psgd_raw_pack(c, choice, g, ef, nullptr, out, st);
  }
  LG_TRY(psgd_p(c, choice, g, ef, p->P, step, st));
  if (p->Psz) LG_NCCL(ncclAllReduce(p->P, p->P, (size_t)p->Psz, ncclFloat, ncclSum, c->comm, st));
  LG_TRY(psgd_q(c, choice, g, ef, p->P, W, p->Qn, st));
  if (p->Qsz) LG_NCCL(ncclAllReduce(p->Qn, p->Qn, (size_t)p->Qsz, ncclFloat, ncclSum, c->comm, st));
  LG_TRY(psgd_out(c, choice, g, ef, p->Qn, W, out, st));
  LG_TRY(psgd_raw_pack(c, choice, g, ef, p->d_raw_pay, nullptr, st));
  if (p->Sraw) LG_NCCL(ncclAllGather(p->d_raw_pay, p->d_raw_gath, (size_t)p->Sraw, ncclUint8, c->comm, st));
  return psgd_raw_combine(c, choice, W, p->d_raw_gath, out, st);
}

float* psgd_internal_P(lgreco_ctx* c) { return c->ps ? c->ps->P : nullptr; }
int64_t psgd_sizes(lgreco_ctx* c, int which) { return !c->ps ? 0 : which == 0 ? c->ps->Psz : c->ps->Qsz; }

// The ctx's current factors: Phat (orthonormalised mean P of the last stage 2) and the
// warm-start Q (the mean Q of the last stage 3), in the P / Q slot layout.
int psgd_factors(lgreco_ctx* c, float* d_Phat, float* d_Q, cudaStream_t st) {
  Psgd* p = c->ps;
  if (d_Phat && p->Psz) LG_CUDA(cudaMemcpyAsync(d_Phat, p->Ph, sizeof(float) * p->Psz, cudaMemcpyDeviceToDevice, st));
  if (d_Q && p->Qsz) LG_CUDA(cudaMemcpyAsync(d_Q, p->Qws, sizeof(float) * p->Qsz, cudaMemcpyDeviceToDevice, st));
  return LGRECO_OK;
}

// Debug / unit-test entry: P = M Q on the tcgen05 path for one matrix (M = canon(g + e),
// m x k row-major; Q k x r column-major; P m x r column-major).  Allocates its tiny
// descriptor arrays (debug only).
extern "C" int lgreco_debug_tc_mq(const float* d_g, const float* d_e, int64_t m, int32_t k, const float* d_Q, int32_t r,
                                  float* d_P, void* stream) {
  if (!d_g || !d_Q || !d_P || m <= 0 || k <= 0 || r < 1 || r > 64 || m > 0x7fffffff) return LGRECO_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  lg::PLayer pl{0, (int32_t)m, k, r, 0, 0, 0, 0, (int64_t)k * r, m * r, 1, 1};
  std::vector<lg::PTile> tiles;  // one K split: P written directly
  for (int64_t i0 = 0; i0 < m; i0 += 128) tiles.push_back(lg::PTile{0, 0, (int32_t)i0, k, 0, 0});
  lg::PLayer* d_pl = nullptr;
  lg::PTile* d_t = nullptr;
  LG_CUDA(cudaMalloc(&d_pl, sizeof(pl)));
  LG_CUDA(cudaMalloc(&d_t, sizeof(lg::PTile) * tiles.size()));
  LG_CUDA(cudaMemcpyAsync(d_pl, &pl, sizeof(pl), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(d_t, tiles.data(), sizeof(lg::PTile) * tiles.size(), cudaMemcpyHostToDevice, st));
  lg::PsArgs a{d_g, d_e, d_pl, 1, nullptr, 0, nullptr, 0, r, nullptr, 0, nullptr, 0, nullptr, 0, nullptr};
  cudaError_t e = lg::launch_ps_mq_tc(a, d_t, (int)tiles.size(), d_Q, d_P, st);
  cudaError_t e2 = cudaStreamSynchronize(st);
  cudaFree(d_pl);
  cudaFree(d_t);
  if (e != cudaSuccess || e2 != cudaSuccess) {
    lg_set_error("tc_mq: %s / %s", cudaGetErrorString(e), cudaGetErrorString(e2));
    return LGRECO_ECUDA;
  }
  return LGRECO_OK;
}

// Debug / unit-test entry: Q = M^T P on the tcgen05 path for one matrix (one row split):
// M = canon(g + e) m x k row-major, P m x r column-major, Q k x r column-major.
extern "C" int lgreco_debug_tc_mtp(const float* d_g, const float* d_e, int64_t m, int32_t k, const float* d_P, int32_t r,
                                   float* d_Q, void* stream) {
  if (!d_g || !d_P || !d_Q || m <= 0 || k <= 0 || r < 1 || r > 64 || m > 0x7fffffff) return LGRECO_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  lg::PLayer pl{0, (int32_t)m, k, r, 0, 0, 0, 0, (int64_t)k * r, m * r, 1, 1};
  std::vector<lg::PTile> tiles;
  for (int c0 = 0; c0 < k; c0 += 128) tiles.push_back(lg::PTile{0, 0, 0, (int32_t)m, c0, 0});
  lg::PLayer* d_pl = nullptr;
  lg::PTile* d_t = nullptr;
  LG_CUDA(cudaMalloc(&d_pl, sizeof(pl)));
  LG_CUDA(cudaMalloc(&d_t, sizeof(lg::PTile) * tiles.size()));
  LG_CUDA(cudaMemcpyAsync(d_pl, &pl, sizeof(pl), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(d_t, tiles.data(), sizeof(lg::PTile) * tiles.size(), cudaMemcpyHostToDevice, st));
  lg::PsArgs a{d_g, d_e, d_pl, 1, nullptr, 0, nullptr, 0, r, nullptr, 0, nullptr, 0, nullptr, 0, nullptr};
  cudaError_t e = lg::launch_ps_mtp_tc(a, d_t, (int)tiles.size(), d_P, d_Q, st);
  cudaError_t e2 = cudaStreamSynchronize(st);
  cudaFree(d_pl);
  cudaFree(d_t);
  if (e != cudaSuccess || e2 != cudaSuccess) {
    lg_set_error("tc_mtp: %s / %s", cudaGetErrorString(e), cudaGetErrorString(e2));
    return LGRECO_ECUDA;
  }
  return LGRECO_OK;
}
