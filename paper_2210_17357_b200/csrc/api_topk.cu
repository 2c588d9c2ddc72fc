// api_topk.cu -- TopK family behind the C ABI: context state, plan layout,
// profile (K2), compress (K6) and the all-gather exchange (K10).
#include <algorithm>

#include "ctx.h"

struct Topk {
  int nC = 0;
  std::vector<int32_t> clayer;
  int32_t* d_clayer = nullptr;
  lg::TChunk *d_chunks = nullptr, *d_chunks_ll = nullptr, *d_chunks_all = nullptr;
  int n_chunks = 0, n_ll = 0, n_all = 0;
  int32_t* d_cchunk0 = nullptr;
  uint32_t *cnt1 = nullptr, *cnt2 = nullptr, *cnt3 = nullptr;
  unsigned long long *sum1 = nullptr, *sum2 = nullptr;
  int32_t *n1 = nullptr, *n2 = nullptr, *sl1 = nullptr;
  uint32_t* sl2 = nullptr;
  lg::TQ* q = nullptr;
  int64_t *d_kprof = nullptr, *d_kplan = nullptr, *d_kpre = nullptr;
  uint2* ccnt = nullptr;
  ulonglong2* coff = nullptr;
  uint32_t* ckeys = nullptr;
  int32_t* ckn = nullptr;
  int32_t* ckz = nullptr;
  lg::TPlan* d_tplan = nullptr;
  // plan cache + pinned staging [TPlan L | kplan nC | kpre nC+1]
  std::vector<int32_t> plan_choice;
  bool plan_valid = false;
  int64_t S = 0, ktotal = 0;
  unsigned char* h_stage = nullptr;
  cudaEvent_t evt = nullptr;
  uint8_t *d_pay = nullptr, *d_gath = nullptr;
  int64_t pay_cap = 0;
  // the preceding profile's per-(layer, density) thresholds, reusable by a compress of
  // the same x (same g / e pointers and step; the compress rewrites e, so one use)
  lg::TQ* qc = nullptr;           // compress queries taken from the profile's
  int32_t* d_choice = nullptr;    // the host plan's choice, uploaded with the plan
  const void* prof_g = nullptr;
  const void* prof_e = nullptr;
  uint64_t prof_step = 0;
  bool prof_valid = false;
};

static int64_t topk_k(int64_t n, int32_t ppm) {
  int64_t k = ((int64_t)ppm * n + 999999) / 1000000;
  return std::max<int64_t>(1, std::min<int64_t>(k, n));
}

static constexpr int64_t TK_CHUNK = 16384;

static lg::TkArgs tk_args(lgreco_ctx* c, const int64_t* kq) {
  Topk* t = c->tk;
  lg::TkArgs a{};
  a.layers = c->d_layers; a.clayer = t->d_clayer; a.nC = t->nC;
  a.chunks = t->d_chunks; a.nchunks = t->n_chunks; a.cchunk0 = t->d_cchunk0;
  a.cnt1 = t->cnt1; a.sum1 = t->sum1; a.cnt2 = t->cnt2; a.sum2 = t->sum2; a.cnt3 = t->cnt3;
  a.n1 = t->n1; a.n2 = t->n2; a.sl1 = t->sl1; a.sl2 = t->sl2;
  a.q = t->q; a.kq = kq; a.ccnt = t->ccnt; a.coff = t->coff; a.tplan = t->d_tplan; a.flag = c->d_flag;
  a.ckeys = t->ckeys; a.ckn = t->ckn; a.ckz = t->ckz;
  return a;
}

int topk_init(lgreco_ctx* c, cudaStream_t st) {
  Topk* t = new Topk();
  c->tk = t;
  const int L = c->L, K = c->K;
  std::vector<lg::TChunk> ch, ll, all;
  std::vector<int32_t> cc0;
  int32_t maxppm = 0;
  for (int j = 0; j < K; ++j) maxppm = std::max(maxppm, c->params[j]);
  int64_t cap = 0;
  for (int l = 0; l < L; ++l) {
    const lgreco_layer& ly = c->layers[l];
    for (int64_t f = 0; f < ly.numel; f += TK_CHUNK)
      all.push_back(lg::TChunk{l, (int32_t)std::min(TK_CHUNK, ly.numel - f), f});
    if (ly.compress) {
      const int ci = (int)t->clayer.size();
      t->clayer.push_back(l);
      cc0.push_back((int32_t)ch.size());
      for (int64_t f = 0; f < ly.numel; f += TK_CHUNK)
        ch.push_back(lg::TChunk{ci, (int32_t)std::min(TK_CHUNK, ly.numel - f), f});
      cap += 8 * topk_k(ly.numel, maxppm) + 16;
    } else {
      for (int64_t f = 0; f < ly.numel; f += TK_CHUNK)
        ll.push_back(lg::TChunk{l, (int32_t)std::min(TK_CHUNK, ly.numel - f), f});
      cap += 4 * ly.numel + 16;
    }
  }
  cc0.push_back((int32_t)ch.size());
  t->nC = (int)t->clayer.size();
  t->n_chunks = (int)ch.size(); t->n_ll = (int)ll.size(); t->n_all = (int)all.size();
  t->pay_cap = cap;
  const int nC = std::max(1, t->nC);
  std::vector<int64_t> kprof((size_t)nC * K, 1);
  for (int ci = 0; ci < t->nC; ++ci)
    for (int j = 0; j < K; ++j) kprof[(size_t)ci * K + j] = topk_k(c->layers[t->clayer[ci]].numel, c->params[j]);
#define TK_ALLOC(ptr, bytes)                                                                 \
  if (cudaMalloc((void**)&(ptr), std::max<size_t>((size_t)(bytes), 16)) != cudaSuccess) {   \
    lg_set_error("cudaMalloc %zu bytes failed (topk)", (size_t)(bytes));                     \
    return LGRECO_ENOMEM;                                                                    \
  }
  TK_ALLOC(t->d_clayer, sizeof(int32_t) * nC);
  TK_ALLOC(t->d_chunks, sizeof(lg::TChunk) * std::max<size_t>(1, ch.size()));
  TK_ALLOC(t->d_chunks_ll, sizeof(lg::TChunk) * std::max<size_t>(1, ll.size()));
  TK_ALLOC(t->d_chunks_all, sizeof(lg::TChunk) * std::max<size_t>(1, all.size()));
  TK_ALLOC(t->d_cchunk0, sizeof(int32_t) * (nC + 1));
  TK_ALLOC(t->cnt1, sizeof(uint32_t) * 2048 * nC);
  TK_ALLOC(t->sum1, sizeof(unsigned long long) * 2048 * nC);
  TK_ALLOC(t->cnt2, sizeof(uint32_t) * 1024 * (size_t)nC * K);
  TK_ALLOC(t->sum2, sizeof(unsigned long long) * 1024 * (size_t)nC * K);
  TK_ALLOC(t->cnt3, sizeof(uint32_t) * 1024 * (size_t)nC * K);
  TK_ALLOC(t->n1, sizeof(int32_t) * nC);
  TK_ALLOC(t->n2, sizeof(int32_t) * nC);
  TK_ALLOC(t->sl1, sizeof(int32_t) * (size_t)nC * K);
  TK_ALLOC(t->sl2, sizeof(uint32_t) * (size_t)nC * K);
  TK_ALLOC(t->q, sizeof(lg::TQ) * (size_t)nC * K);
  TK_ALLOC(t->d_kprof, sizeof(int64_t) * (size_t)nC * K);
  TK_ALLOC(t->d_kplan, sizeof(int64_t) * nC);
  TK_ALLOC(t->d_kpre, sizeof(int64_t) * (nC + 1));
  TK_ALLOC(t->ccnt, sizeof(uint2) * std::max<size_t>(1, ch.size()));
  TK_ALLOC(t->coff, sizeof(ulonglong2) * std::max<size_t>(1, ch.size()));
  TK_ALLOC(t->ckeys, sizeof(uint32_t) * lg::TK_CKCAP * std::max<size_t>(1, ch.size()));
  TK_ALLOC(t->ckn, sizeof(int32_t) * std::max<size_t>(1, ch.size()));
  TK_ALLOC(t->ckz, sizeof(int32_t) * std::max<size_t>(1, ch.size()));
  TK_ALLOC(t->d_tplan, sizeof(lg::TPlan) * L);
  TK_ALLOC(t->qc, sizeof(lg::TQ) * nC);
  TK_ALLOC(t->d_choice, sizeof(int32_t) * L);
  if (c->world > 1) {
    TK_ALLOC(t->d_pay, cap);
    TK_ALLOC(t->d_gath, cap * c->world);
  }
#undef TK_ALLOC
  if (cudaMallocHost((void**)&t->h_stage, sizeof(lg::TPlan) * L + sizeof(int64_t) * (2 * nC + 1) +
                                              sizeof(int32_t) * L) != cudaSuccess)
    return LGRECO_ENOMEM;
  LG_CUDA(cudaEventCreateWithFlags(&t->evt, cudaEventDisableTiming));
  LG_CUDA(cudaMemcpyAsync(t->d_clayer, t->clayer.data(), sizeof(int32_t) * t->nC, cudaMemcpyHostToDevice, st));
  if (!ch.empty()) LG_CUDA(cudaMemcpyAsync(t->d_chunks, ch.data(), sizeof(lg::TChunk) * ch.size(), cudaMemcpyHostToDevice, st));
  if (!ll.empty()) LG_CUDA(cudaMemcpyAsync(t->d_chunks_ll, ll.data(), sizeof(lg::TChunk) * ll.size(), cudaMemcpyHostToDevice, st));
  if (!all.empty()) LG_CUDA(cudaMemcpyAsync(t->d_chunks_all, all.data(), sizeof(lg::TChunk) * all.size(), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(t->d_cchunk0, cc0.data(), sizeof(int32_t) * cc0.size(), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaMemcpyAsync(t->d_kprof, kprof.data(), sizeof(int64_t) * kprof.size(), cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaStreamSynchronize(st));
  return LGRECO_OK;
}

void topk_destroy(lgreco_ctx* c) {
  Topk* t = c->tk;
  if (!t) return;
  cudaFree(t->d_clayer); cudaFree(t->d_chunks); cudaFree(t->d_chunks_ll); cudaFree(t->d_chunks_all);
  cudaFree(t->d_cchunk0); cudaFree(t->cnt1); cudaFree(t->sum1); cudaFree(t->cnt2); cudaFree(t->sum2);
  cudaFree(t->cnt3); cudaFree(t->n1); cudaFree(t->n2); cudaFree(t->sl1); cudaFree(t->sl2); cudaFree(t->q);
  cudaFree(t->d_kprof); cudaFree(t->d_kplan); cudaFree(t->d_kpre); cudaFree(t->ccnt); cudaFree(t->coff);
  cudaFree(t->d_tplan); cudaFree(t->d_pay); cudaFree(t->d_gath); cudaFree(t->ckeys); cudaFree(t->ckn); cudaFree(t->ckz);
  cudaFree(t->qc); cudaFree(t->d_choice);
  if (t->h_stage) cudaFreeHost(t->h_stage);
  if (t->evt) cudaEventDestroy(t->evt);
  delete t;
  c->tk = nullptr;
}

// Host layout of a TopK plan: per layer (payload offset, k); 16-byte aligned blocks (R9).
static int topk_layout(lgreco_ctx* c, const int32_t* choice, std::vector<lg::TPlan>& plan, std::vector<int64_t>& kplan,
                       std::vector<int64_t>& kpre, int64_t& S) {
  Topk* t = c->tk;
  plan.assign(c->L, lg::TPlan{0, 0});
  kplan.assign(std::max(1, t->nC), 0);
  kpre.assign(t->nC + 1, 0);
  int64_t off = 0;
  int ci = 0;
  for (int l = 0; l < c->L; ++l) {
    const lgreco_layer& ly = c->layers[l];
    plan[l].pay_off = off;
    if (choice[l] == LGRECO_CHOICE_SKIP) {
      // another family's layer (NEXT-4, R24): no pairs, no bytes; k = -1 marks it for the
      // combine, which leaves its output untouched
      plan[l].k = -1;
      if (ly.compress) kpre[ci + 1] = kpre[ci], kplan[ci++] = 0;
      continue;
    }
    if (ly.compress) {
      const int j = choice[l];
      if (j < 0 || j >= c->K) {
        lg_set_error("choice[%d]=%d out of range [0,%d)", l, j, c->K);
        return LGRECO_EINVAL;
      }
      const int64_t k = topk_k(ly.numel, c->params[j]);
      plan[l].k = k;
      kplan[ci] = k;
      kpre[ci + 1] = kpre[ci] + k;
      ++ci;
      off += 8 * k;
    } else {
      off += 4 * ly.numel;
    }
    off = (off + 15) & ~(int64_t)15;
  }
  S = off;
  return LGRECO_OK;
}

static int topk_set_plan(lgreco_ctx* c, const int32_t* choice, cudaStream_t st) {
  Topk* t = c->tk;
  std::vector<int32_t> chv(choice, choice + c->L);
  for (int l = 0; l < c->L; ++l)
    if (!c->layers[l].compress && chv[l] != LGRECO_CHOICE_SKIP) chv[l] = -1;
  if (t->plan_valid && chv == t->plan_choice) return LGRECO_OK;
  std::vector<lg::TPlan> plan;
  std::vector<int64_t> kplan, kpre;
  int64_t S = 0;
  LG_TRY(topk_layout(c, choice, plan, kplan, kpre, S));
  LG_CUDA(cudaEventSynchronize(t->evt));
  unsigned char* p = t->h_stage;
  memcpy(p, plan.data(), sizeof(lg::TPlan) * c->L);
  memcpy(p + sizeof(lg::TPlan) * c->L, kplan.data(), sizeof(int64_t) * kplan.size());
  memcpy(p + sizeof(lg::TPlan) * c->L + sizeof(int64_t) * kplan.size(), kpre.data(), sizeof(int64_t) * kpre.size());
  LG_CUDA(cudaMemcpyAsync(t->d_tplan, p, sizeof(lg::TPlan) * c->L, cudaMemcpyHostToDevice, st));
  int32_t* hc = reinterpret_cast<int32_t*>(p + sizeof(lg::TPlan) * c->L + sizeof(int64_t) * (kplan.size() + kpre.size()));
  memcpy(hc, chv.data(), sizeof(int32_t) * c->L);
  LG_CUDA(cudaMemcpyAsync(t->d_choice, hc, sizeof(int32_t) * c->L, cudaMemcpyHostToDevice, st));
  if (t->nC) {
    LG_CUDA(cudaMemcpyAsync(t->d_kplan, p + sizeof(lg::TPlan) * c->L, sizeof(int64_t) * t->nC, cudaMemcpyHostToDevice, st));
    LG_CUDA(cudaMemcpyAsync(t->d_kpre, p + sizeof(lg::TPlan) * c->L + sizeof(int64_t) * kplan.size(),
                            sizeof(int64_t) * (t->nC + 1), cudaMemcpyHostToDevice, st));
  }
  LG_CUDA(cudaEventRecord(t->evt, st));
  t->S = S;
  t->ktotal = kpre[t->nC];
  t->plan_choice = chv;
  t->plan_valid = true;
  return LGRECO_OK;
}

int64_t topk_payload_bytes(lgreco_ctx* c, const int32_t* choice) {
  std::vector<lg::TPlan> plan;
  std::vector<int64_t> kplan, kpre;
  int64_t S = 0;
  const int s = topk_layout(c, choice, plan, kplan, kpre, S);
  return s == LGRECO_OK ? S : s;
}

int topk_profile(lgreco_ctx* c, const float* g, const float* e, uint64_t step, double* err, int64_t* bits,
                 cudaStream_t st) {
  Topk* t = c->tk;
  const lg::TkArgs a = tk_args(c, t->d_kprof);
  LG_LAUNCH(c, lg::launch_topk_lossless_rows(c->d_layers, c->L, c->K, err, bits, st));
  c->launches += 1;
  if (t->nC) LG_LAUNCH(c, lg::launch_topk_select(g, e, a, c->K, err, bits, c->K, st, &c->launches));
  t->prof_g = g;
  t->prof_e = e;
  t->prof_step = step;
  t->prof_valid = true;
  return LGRECO_OK;
}

// The compress's per-layer queries: taken from the preceding profile when it ran on the
// same x (same g / e pointers and step: the caller contract of the per-step pipeline,
// as for QSGD's common random numbers), else a fresh one-query select.  d_choice: the
// plan on the device.
static int topk_queries(lgreco_ctx* c, const int32_t* d_choice, const float* g, const float* ef, uint64_t step,
                        lg::TkArgs& a, cudaStream_t st) {
  Topk* t = c->tk;
  const bool reuse = t->prof_valid && t->prof_g == g && t->prof_e == ef && t->prof_step == step &&
                     step != ~0ull && !getenv("LGRECO_TOPK_NO_REUSE");
  t->prof_valid = false;  // this compress rewrites e
  if (reuse) {
    LG_LAUNCH(c, lg::launch_topk_reuse(d_choice, c->K, t->d_clayer, t->nC, t->q, t->qc, c->d_flag, st));
    a.q = t->qc;
    c->launches += 1;
  } else {
    LG_LAUNCH(c, lg::launch_topk_select(g, ef, a, 1, nullptr, nullptr, 1, st, &c->launches));
  }
  return LGRECO_OK;
}

int topk_pack(lgreco_ctx* c, const int32_t* choice, const float* g, float* ef, uint8_t* payload, float* out,
              uint64_t step, cudaStream_t st) {
  Topk* t = c->tk;
  LG_TRY(topk_set_plan(c, choice, st));
  lg::TkArgs a = tk_args(c, t->d_kplan);
  a.need_off = payload != nullptr;
  if (t->nC) {
    LG_TRY(topk_queries(c, t->d_choice, g, ef, step, a, st));
    LG_LAUNCH(c, lg::launch_topk_compact(g, ef, payload, out, a, st));
    c->launches += 3;
  }
  if (t->n_ll) {
    LG_LAUNCH(c, lg::launch_lossless_pack(g, ef, payload, out, t->d_choice, c->d_layers, t->d_chunks_ll, t->n_ll, t->d_tplan,
                                          c->d_flag, st));
    c->launches += 1;
  }
  return LGRECO_OK;
}

int topk_combine(lgreco_ctx* c, const int32_t* choice, int W, const uint8_t* gathered, float* out, cudaStream_t st) {
  Topk* t = c->tk;
  LG_TRY(topk_set_plan(c, choice, st));
  LG_LAUNCH(c, lg::launch_topk_combine(gathered, t->S, W, out, c->d_layers, t->d_chunks_all, t->n_all, t->d_clayer,
                                       t->nC, t->d_kpre, t->ktotal, t->d_tplan, st, &c->launches));
  return LGRECO_OK;
}

int topk_compress_allreduce(lgreco_ctx* c, const int32_t* choice, const float* g, float* ef, float* out,
                            uint64_t step, cudaStream_t st) {
  Topk* t = c->tk;
  if (c->world == 1) return topk_pack(c, choice, g, ef, nullptr, out, step, st);  // W = 1: fused decode
  LG_TRY(topk_pack(c, choice, g, ef, t->d_pay, nullptr, step, st));
  LG_NCCL(ncclAllGather(t->d_pay, t->d_gath, (size_t)t->S, ncclUint8, c->comm, st));
  return topk_combine(c, choice, c->world, t->d_gath, out, st);
}

// W == 1 fused TopK compress with the plan read on the device (no host round trip).
int topk_compress_dev(lgreco_ctx* c, const int32_t* d_choice, const float* g, float* ef, float* out, uint64_t step,
                      cudaStream_t st) {
  Topk* t = c->tk;
  LG_LAUNCH(c, lg::launch_plan_topk_dev(d_choice, c->d_params, c->K, c->d_layers, t->d_clayer, t->nC, t->d_kplan,
                                        c->d_flag, st));
  t->plan_valid = false;  // d_kplan now holds a device-chosen plan
  lg::TkArgs a = tk_args(c, t->d_kplan);
  a.need_off = 0;  // no payload at W = 1
  c->launches += 1;
  if (t->nC) {
    LG_TRY(topk_queries(c, d_choice, g, ef, step, a, st));
    LG_LAUNCH(c, lg::launch_topk_compact(g, ef, nullptr, out, a, st));
    c->launches += 3;
  }
  if (t->n_ll) {
    LG_LAUNCH(c, lg::launch_lossless_pack(g, ef, nullptr, out, d_choice, c->d_layers, t->d_chunks_ll, t->n_ll, t->d_tplan,
                                          c->d_flag, st));
    c->launches += 1;
  }
  return LGRECO_OK;
}
