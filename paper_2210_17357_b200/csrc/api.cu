// api.cu -- the C ABI declared in include/lgreco.h: context, plan layout,
// dispatch of the kernels and the NCCL exchange (one process per GPU).
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>

#include "ctx.h"

static thread_local char g_err[1024] = "";

void lg_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" {

const char* lgreco_last_error(void) { return g_err; }
int32_t lgreco_version(void) { return 1; }

int lgreco_nccl_unique_id(void* h_out) {
  ncclUniqueId id;
  LG_NCCL(ncclGetUniqueId(&id));
  memcpy(h_out, &id, sizeof(id));
  return LGRECO_OK;
}

}  // extern "C"

static int64_t max_param(const lgreco_ctx* c) {
  int64_t m = 0;
  for (int32_t p : c->params) m = std::max<int64_t>(m, p);
  return m;
}

static int64_t rec_bytes_full(int bits, int B) { return bits > 0 ? (int64_t)16 * bits * (B / 128) + 8 : (int64_t)4 * B; }

// Host layout of plan `choice` (QSGD): per-layer DevPlan, total bytes S (R7).
static int qsgd_layout(const lgreco_ctx* c, const int32_t* choice, std::vector<lg::DevPlan>& plan, int64_t& S) {
  plan.resize(c->L);
  int64_t off = 0;
  for (int l = 0; l < c->L; ++l) {
    const lgreco_layer& ly = c->layers[l];
    int bits = 0;
    if (choice[l] == LGRECO_CHOICE_SKIP) {
      // another family's layer (NEXT-4, R24): no records and no bytes in this ctx's payload
      plan[l].pay_off = off;
      plan[l].bits = -1;
      plan[l].rec_bytes = 0;
      continue;
    }
    if (ly.compress) {
      const int ci = choice[l];
      if (ci < 0 || ci >= c->K) {
        lg_set_error("choice[%d]=%d out of range [0,%d)", l, ci, c->K);
        return LGRECO_EINVAL;
      }
      bits = c->params[ci];
    }
    const int64_t nb = c->bucket0[l + 1] - c->bucket0[l];
    plan[l].pay_off = off;
    plan[l].bits = bits;
    plan[l].rec_bytes = (int32_t)rec_bytes_full(bits, c->B);
    off += bits > 0 ? nb * rec_bytes_full(bits, c->B) : 4 * ly.numel;
    off = (off + 15) & ~(int64_t)15;  // every layer's records start 16-byte aligned (R7)
  }
  S = off;
  return LGRECO_OK;
}

// byte offset of record r under plan
static int64_t rec_off(const lgreco_ctx* c, const std::vector<lg::DevPlan>& plan, int64_t r, int64_t S) {
  if (r >= c->R) return S;
  const int l = (int)(std::upper_bound(c->bucket0.begin(), c->bucket0.begin() + c->L, r) - c->bucket0.begin()) - 1;
  const int64_t jb = r - c->bucket0[l];
  if (plan[l].bits < 0) return plan[l].pay_off;  // (a skipped layer has no bytes)
  return plan[l].pay_off + (plan[l].bits > 0 ? jb * (int64_t)plan[l].rec_bytes : jb * 4 * (int64_t)c->B);
}

static void shard_bounds(const lgreco_ctx* c, const std::vector<lg::DevPlan>& plan, int64_t S, int W,
                         std::vector<int64_t>& rb, std::vector<int64_t>& bb) {
  rb.assign(W + 1, 0);
  bb.assign(W + 1, 0);
  for (int j = 1; j < W; ++j) {
    const int64_t target = (int64_t)((__int128)j * S / W);
    int64_t lo = 0, hi = c->R;  // first r with off(r) >= target
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (rec_off(c, plan, mid, S) >= target) hi = mid; else lo = mid + 1;
    }
    rb[j] = lo;
    bb[j] = rec_off(c, plan, lo, S);
  }
  rb[W] = c->R;
  bb[W] = S;
}

// Upload the plan if it changed (pinned staging guarded by an event).
static int set_plan(lgreco_ctx* c, const int32_t* choice, cudaStream_t st) {
  std::vector<int32_t> ch(choice, choice + c->L);
  for (int l = 0; l < c->L; ++l)
    if (!c->layers[l].compress && ch[l] != LGRECO_CHOICE_SKIP) ch[l] = -1;
  if (c->plan_valid && ch == c->plan_choice) return LGRECO_OK;
  std::vector<lg::DevPlan> plan;
  int64_t S = 0;
  LG_TRY(qsgd_layout(c, choice, plan, S));
  LG_CUDA(cudaEventSynchronize(c->plan_evt));
  memcpy(c->h_plan_pinned, plan.data(), sizeof(lg::DevPlan) * c->L);
  LG_CUDA(cudaMemcpyAsync(c->d_plan, c->h_plan_pinned, sizeof(lg::DevPlan) * c->L, cudaMemcpyHostToDevice, st));
  LG_CUDA(cudaEventRecord(c->plan_evt, st));
  c->h_plan_v = plan;
  c->S = S;
  shard_bounds(c, plan, S, c->world, c->rec_bounds, c->byte_bounds);
  c->plan_choice = ch;
  c->plan_valid = true;
  return LGRECO_OK;
}

static void key_of(const lgreco_ctx* c, uint32_t& k0, uint32_t& k1) {
  k0 = (uint32_t)c->seed;
  k1 = (uint32_t)(c->seed >> 32);
}

extern "C" {

int lgreco_ctx_create(lgreco_ctx** out, const lgreco_layer* layers, int32_t L, const lgreco_candidates* cand,
                      int32_t rank, int32_t world, const void* nccl_unique_id, void* stream) {
  if (!out || !layers || L <= 0 || !cand || !cand->params) { lg_set_error("null argument or L <= 0"); return LGRECO_EINVAL; }
  if (L >= lg::QI_MAX_LAYERS) { lg_set_error("L = %d: at most %d layers", L, lg::QI_MAX_LAYERS - 1); return LGRECO_EINVAL; }
  if (world < 1 || rank < 0 || rank >= world) { lg_set_error("bad rank/world %d/%d", rank, world); return LGRECO_EINVAL; }
  if (cand->K <= 0 || cand->K > 255) { lg_set_error("K=%d out of range", cand->K); return LGRECO_EINVAL; }
  if (cand->family != LGRECO_QSGD && cand->family != LGRECO_TOPK && cand->family != LGRECO_POWERSGD) {
    lg_set_error("unknown family %d", cand->family);
    return LGRECO_EINVAL;
  }
  for (int j = 0; j < cand->K; ++j) {
    const int p = cand->params[j];
    if ((cand->family == LGRECO_QSGD && (p < 1 || p > 16)) || (cand->family == LGRECO_TOPK && (p < 1 || p > 1000000)) ||
        (cand->family == LGRECO_POWERSGD && p < 1)) {
      lg_set_error("candidate %d parameter %d invalid for family %d", j, p, cand->family);
      return LGRECO_EINVAL;
    }
  }
  if (cand->family == LGRECO_QSGD && (cand->K > 16 || cand->qbucket < 128 || cand->qbucket % 128 || cand->qbucket > 8192)) {
    lg_set_error("QSGD needs K <= 16 and bucket a multiple of 128 in [128, 8192]");
    return LGRECO_EINVAL;
  }
  int64_t end = 0;
  for (int l = 0; l < L; ++l) {
    const lgreco_layer& ly = layers[l];
    if (ly.numel < 1 || ly.offset < end || (ly.rows > 0 && (int64_t)ly.rows * ly.cols != ly.numel) || ly.rows < 0) {
      lg_set_error("layer %d invalid (offset %lld numel %lld rows %d cols %d)", l, (long long)ly.offset,
                   (long long)ly.numel, ly.rows, ly.cols);
      return LGRECO_EINVAL;
    }
    end = ly.offset + ly.numel;
  }
  cudaStream_t st = (cudaStream_t)stream;
  lgreco_ctx* c = new lgreco_ctx();
  c->L = L; c->rank = rank; c->world = world;
  c->family = cand->family; c->K = cand->K; c->power_steps = cand->power_steps;
  c->B = cand->family == LGRECO_QSGD ? cand->qbucket : 128;  // bucket tables only used by QSGD
  c->seed = cand->seed;
  c->layers.assign(layers, layers + L);
  c->params.assign(cand->params, cand->params + cand->K);
  c->N = end;
  c->bucket0.resize(L + 1);
  std::vector<lg::DevLayer> dl(L);
  std::vector<lg::ProfChunk> chunks, chunks_all, chunks_raw;
  std::vector<int32_t> lc0(L + 1);
  const int CB = 64;  // buckets per profile chunk
  int64_t gb = 0;
  for (int l = 0; l < L; ++l) {
    const int64_t nb = (layers[l].numel + c->B - 1) / c->B;
    c->bucket0[l] = gb;
    dl[l] = lg::DevLayer{layers[l].offset, layers[l].numel, gb, layers[l].rows, layers[l].cols, layers[l].compress, 0};
    lc0[l] = (int32_t)chunks.size();
    for (int64_t j = 0; j < nb; j += CB) {
      const lg::ProfChunk ch{l, (int32_t)std::min<int64_t>(CB, nb - j), j};
      if (layers[l].compress) chunks.push_back(ch);
      else chunks_raw.push_back(ch);
      chunks_all.push_back(ch);
    }
    gb += nb;
  }
  c->bucket0[L] = gb;
  lc0[L] = (int32_t)chunks.size();
  c->R = gb;
  c->nchunks = (int)chunks.size();
  c->nchunks_all = (int)chunks_all.size();
  c->nchunks_raw = (int)chunks_raw.size();
  // K1 (B = 128): chunks of <= 4 buckets (one quad) of the compressed layers, handed
  // out to the resident warps (occupancy x SMs CTAs of 8 warps) by a ticket counter: the
  // fine grain keeps every warp busy to the end (a quad is ~1/14 of a warp's share)
  std::vector<lg::QInfo> qchunks;
  std::vector<int32_t> lqc0(L + 1, 0);
  std::vector<lg::QSeg> qsegs;
  std::vector<int32_t> lqs0(L + 1, 0);
  if (c->B == 128) {
    for (int l = 0; l < L; ++l) {
      lqc0[l] = (int32_t)qchunks.size();
      if (!layers[l].compress) continue;
      const int64_t nb = (layers[l].numel + 127) / 128;
      for (int64_t j = 0; j < nb; j += 4)
        qchunks.push_back(lg::QInfo{layers[l].offset + 128 * j, (uint32_t)(c->bucket0[l] + j),
                                    (int32_t)std::min<int64_t>(512, layers[l].numel - 128 * j) | (l << 10)});
    }
    lqc0[L] = (int32_t)qchunks.size();
    for (int l = 0; l < L; ++l) {
      lqs0[l] = (int32_t)qsegs.size();
      const int r0 = lqc0[l], r1 = lqc0[l + 1];
      if (r1 == r0) qsegs.push_back(lg::QSeg{l, r0, 0, 0});
      for (int r = r0; r < r1; r += 256) qsegs.push_back(lg::QSeg{l, r, std::min(256, r1 - r), 0});
    }
    lqs0[L] = (int32_t)qsegs.size();
    c->nqseg = (int)qsegs.size();
    int nsm = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    c->nqwarps = nsm * 4 * 8;  // upper bound; the launcher sizes the grid by the kernel's occupancy
    c->nqchunks = (int)qchunks.size();
  }
  std::vector<float> cs(c->K);
  for (int j = 0; j < c->K; ++j) cs[j] = c->family == LGRECO_QSGD ? (float)((1u << c->params[j]) - 1u) : 0.f;
  for (int j = 0; j < c->K && j < 16; ++j) c->cs.s[j] = cs[j];
  // max payload over all plans: every compressed layer at the largest candidate
  const int bmax = c->family == LGRECO_QSGD ? (int)max_param(c) : 0;
  int64_t cap = 0;
  for (int l = 0; l < L; ++l)
    cap += (layers[l].compress ? (c->bucket0[l + 1] - c->bucket0[l]) * rec_bytes_full(bmax, c->B) : 4 * layers[l].numel) + 16;
  c->pay_cap = cap;
  auto fail = [&](int s) { lgreco_ctx_destroy(c); return s; };
#define LG_ALLOC(ptr, bytes)                                                   \
  if (cudaMalloc((void**)&(ptr), std::max<size_t>((size_t)(bytes), 16)) != cudaSuccess) { \
    lg_set_error("cudaMalloc %zu bytes failed", (size_t)(bytes));               \
    return fail(LGRECO_ENOMEM);                                                \
  }
  LG_ALLOC(c->d_layers, sizeof(lg::DevLayer) * L);
  LG_ALLOC(c->d_bucket0, sizeof(int64_t) * (L + 1));
  LG_ALLOC(c->d_cand_s, sizeof(float) * c->K);
  LG_ALLOC(c->d_params, sizeof(int32_t) * c->K);
  LG_ALLOC(c->d_chunks, sizeof(lg::ProfChunk) * std::max(1, c->nchunks));
  LG_ALLOC(c->d_chunks_all, sizeof(lg::ProfChunk) * std::max(1, c->nchunks_all));
  LG_ALLOC(c->d_layer_chunk0, sizeof(int32_t) * (L + 1));
  LG_ALLOC(c->d_chunks_raw, sizeof(lg::ProfChunk) * std::max(1, c->nchunks_raw));
  LG_ALLOC(c->d_partial, sizeof(double) * (size_t)std::max(1, std::max(c->nchunks, c->nqchunks)) * c->K);
  LG_ALLOC(c->d_qinfo, sizeof(lg::QInfo) * std::max(1, c->nqchunks));
  LG_ALLOC(c->d_layer_qchunk0, sizeof(int32_t) * (L + 1));
  LG_ALLOC(c->d_ticket, lg::QT_WORDS * sizeof(unsigned));
  LG_ALLOC(c->d_qseg, sizeof(lg::QSeg) * std::max(1, c->nqseg));
  LG_ALLOC(c->d_lqseg0, sizeof(int32_t) * (L + 1));
  LG_ALLOC(c->d_segsum, sizeof(double) * std::max(1, c->nqseg) * c->K);
  LG_ALLOC(c->d_ldone, sizeof(unsigned) * L);
  LG_ALLOC(c->d_flag, sizeof(unsigned));
  LG_ALLOC(c->d_plan, sizeof(lg::DevPlan) * L);
  if (world > 1 && c->family == LGRECO_QSGD) {
    LG_ALLOC(c->d_pay1, cap);
    LG_ALLOC(c->d_recv, cap + (int64_t)world * 4 * 8192 * 4);
    LG_ALLOC(c->d_pay2, cap);
  }
#undef LG_ALLOC
  if (cudaMallocHost((void**)&c->h_plan_pinned, sizeof(lg::DevPlan) * L) != cudaSuccess) return fail(LGRECO_ENOMEM);
  if (cudaMallocHost((void**)&c->h_choice_pinned, sizeof(int32_t) * L) != cudaSuccess) return fail(LGRECO_ENOMEM);
  if (cudaEventCreateWithFlags(&c->plan_evt, cudaEventDisableTiming) != cudaSuccess) return fail(LGRECO_ECUDA);
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->d_layers, dl.data(), sizeof(lg::DevLayer) * L, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->d_bucket0, c->bucket0.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->d_cand_s, cs.data(), sizeof(float) * c->K, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->d_params, c->params.data(), sizeof(int32_t) * c->K, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && c->nchunks)
    e = cudaMemcpyAsync(c->d_chunks, chunks.data(), sizeof(lg::ProfChunk) * c->nchunks, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && c->nchunks_all)
    e = cudaMemcpyAsync(c->d_chunks_all, chunks_all.data(), sizeof(lg::ProfChunk) * c->nchunks_all,
                        cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->d_layer_chunk0, lc0.data(), sizeof(int32_t) * (L + 1), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && c->nchunks_raw)
    e = cudaMemcpyAsync(c->d_chunks_raw, chunks_raw.data(), sizeof(lg::ProfChunk) * c->nchunks_raw,
                        cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && c->nqchunks)
    e = cudaMemcpyAsync(c->d_qinfo, qchunks.data(), sizeof(lg::QInfo) * c->nqchunks, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->d_layer_qchunk0, lqc0.data(), sizeof(int32_t) * (L + 1), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->d_ticket, 0, lg::QT_WORDS * sizeof(unsigned), st);
  if (e == cudaSuccess && c->nqseg)
    e = cudaMemcpyAsync(c->d_qseg, qsegs.data(), sizeof(lg::QSeg) * c->nqseg, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->d_lqseg0, lqs0.data(), sizeof(int32_t) * (L + 1), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->d_ldone, 0, sizeof(unsigned) * L, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->d_flag, 0, sizeof(unsigned), st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    lg_set_error("ctx upload: %s", cudaGetErrorString(e));
    return fail(LGRECO_ECUDA);
  }
  if (c->family == LGRECO_TOPK) {
    const int s = topk_init(c, st);
    if (s != LGRECO_OK) return fail(s);
  }
  if (c->family == LGRECO_POWERSGD) {
    if (c->power_steps < 1) { lg_set_error("power_steps must be >= 1"); return fail(LGRECO_EINVAL); }
    const int s = psgd_init(c, st);
    if (s != LGRECO_OK) return fail(s);
  }
  if (world > 1 && world <= lg::P2P_MAXW && c->family == LGRECO_QSGD) {
    const size_t fbytes = sizeof(unsigned) * (3 * lg::P2P_MAXW + (size_t)L);
    if (cudaMalloc((void**)&c->d_flags, fbytes) != cudaSuccess || cudaMemset(c->d_flags, 0, fbytes) != cudaSuccess ||
        cudaMalloc((void**)&c->d_p2p, sizeof(lg::P2PDev)) != cudaSuccess) {
      lg_set_error("p2p buffers");
      return fail(LGRECO_ENOMEM);
    }
  }
  if (world > 1 && !nccl_unique_id && c->family != LGRECO_QSGD) {
    lg_set_error("world > 1 needs an ncclUniqueId (the peer-memory exchange is QSGD only)");
    return fail(LGRECO_EINVAL);
  }
  if (world > 1 && nccl_unique_id) {  // (without an id: QSGD over peer memory, lgreco_p2p_*)
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
      lg_set_error("ncclCommInitRank: %s", ncclGetErrorString(r));
      c->comm = nullptr;
      return fail(LGRECO_ENCCL);
    }
  }
  *out = c;
  return LGRECO_OK;
}

void lgreco_ctx_destroy(lgreco_ctx* c) {
  if (c) svd_destroy(c);
  if (c) {
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    cudaFree(c->d_flags);
    cudaFree(c->d_p2p);
  }
  if (!c) return;
  topk_destroy(c);
  psgd_destroy(c);
  if (c->comm) ncclCommDestroy(c->comm);
  cudaFree(c->d_layers); cudaFree(c->d_bucket0); cudaFree(c->d_cand_s); cudaFree(c->d_params);
  cudaFree(c->d_chunks); cudaFree(c->d_chunks_all); cudaFree(c->d_chunks_raw); cudaFree(c->d_layer_chunk0); cudaFree(c->d_partial);
  cudaFree(c->d_qinfo); cudaFree(c->d_layer_qchunk0); cudaFree(c->d_ticket);
  cudaFree(c->d_qseg); cudaFree(c->d_lqseg0); cudaFree(c->d_segsum); cudaFree(c->d_ldone); cudaFree(c->d_flag);
  cudaFree(c->d_plan); cudaFree(c->d_pay1); cudaFree(c->d_recv); cudaFree(c->d_pay2);
  if (c->h_plan_pinned) cudaFreeHost(c->h_plan_pinned);
  if (c->h_choice_pinned) cudaFreeHost(c->h_choice_pinned);
  if (c->plan_evt) cudaEventDestroy(c->plan_evt);
  delete c;
}

int lgreco_ctx_check(lgreco_ctx* c, void* stream) {
  if (!c) return LGRECO_EINVAL;
  unsigned f = 0;
  LG_CUDA(cudaMemcpyAsync(&f, c->d_flag, sizeof(unsigned), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  LG_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (f) {
    LG_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(unsigned), (cudaStream_t)stream));
    if (f & 2u) {
      lg_set_error("device plan: choice outside [0, K) for a compressed layer");
      return LGRECO_EINVAL;
    }
    lg_set_error("non-finite gradient value seen");
    return LGRECO_ENONFINITE;
  }
  return LGRECO_OK;
}

int64_t lgreco_ctx_launches(lgreco_ctx* c) { return c ? c->launches : -1; }

int lgreco_ctx_timing(lgreco_ctx* c, int32_t enable) {
  if (!c) { lg_set_error("null ctx"); return LGRECO_EINVAL; }
  c->timing = enable != 0;
  return LGRECO_OK;
}

int lgreco_ctx_kernel_ms(lgreco_ctx* c, double* total_ms, int64_t* count) {
  if (!c || !total_ms || !count) { lg_set_error("null argument"); return LGRECO_EINVAL; }
  double t = 0.0;
  int rc = LGRECO_OK;
  for (auto& pr : c->tev) {
    float ms = 0.f;
    if (cudaEventSynchronize(pr.second) != cudaSuccess || cudaEventElapsedTime(&ms, pr.first, pr.second) != cudaSuccess) {
      lg_set_error("kernel timing event: %s", cudaGetErrorString(cudaGetLastError()));
      rc = LGRECO_ECUDA;
    }
    t += ms;
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  *total_ms = t;
  *count = (int64_t)c->tev.size();
  c->tev.clear();
  return rc;
}

// Base pointers of the fp32 gradient-sized buffers must be 16-byte aligned for the
// 128-bit (and bulk-copy) paths of every kernel except the QSGD profile (which falls
// back to masked loads).  Argument error otherwise (include/lgreco.h).
static int check_align16(const char* what, const void* a, const void* b = nullptr, const void* d = nullptr) {
  const uintptr_t m = reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(d);
  if (m & 15) {
    lg_set_error("%s: gradient / EF / output base pointers must be 16-byte aligned", what);
    return LGRECO_EINVAL;
  }
  return LGRECO_OK;
}

int lgreco_profile(lgreco_ctx* c, const float* d_g, const float* d_ef, uint64_t step, double* d_err,
                   int64_t* d_bits, void* stream) {
  if (!c || !d_g || !d_err || !d_bits) { lg_set_error("null argument"); return LGRECO_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t k0, k1;
  key_of(c, k0, k1);
  if (c->family == LGRECO_QSGD) {
    lg::QProfileArgs a{d_g, d_ef, c->d_layers, c->L, c->d_chunks, c->nchunks, c->d_layer_chunk0,
                       c->B, c->cs, c->d_params, c->K, k0, k1, (uint32_t)c->rank, (uint32_t)step,
                       c->d_partial, d_err, d_bits};
    a.qinfo = c->d_qinfo; a.nqchunks = c->nqchunks; a.layer_qchunk0 = c->d_layer_qchunk0;
    a.nqwarps = c->nqwarps; a.ticket = c->d_ticket;
    a.segs = c->d_qseg; a.nseg = c->nqseg; a.lseg0 = c->d_lqseg0; a.segsum = c->d_segsum; a.ldone = c->d_ldone;
    a.ptr_aligned = ((reinterpret_cast<uintptr_t>(d_g) | reinterpret_cast<uintptr_t>(d_ef)) & 15) == 0;
    if (c->timing && c->nchunks > 0) {
      cudaEvent_t e0, e1;
      LG_CUDA(cudaEventCreate(&e0));
      LG_CUDA(cudaEventCreate(&e1));
      c->tev.emplace_back(e0, e1);
      a.ev0 = e0;
      a.ev1 = e1;
    }
    LG_LAUNCH(c, lg::launch_qprofile(a, st));
    c->launches += (c->nchunks > 0) + 1;
    return LGRECO_OK;
  }
  LG_TRY(check_align16("profile", d_g, d_ef));  // (QSGD above handles any 4-byte alignment)
  if (c->family == LGRECO_TOPK) return topk_profile(c, d_g, d_ef, step, d_err, d_bits, st);
  if (c->family == LGRECO_POWERSGD) {
    if (c->psgd_method == LGRECO_PSGD_SVD) return lgreco_psgd_profile_svd(c, d_g, d_ef, d_err, d_bits, stream);
    return psgd_profile(c, d_g, d_ef, step, d_err, d_bits, st);
  }
  lg_set_error("profile: family %d unsupported", c->family);
  return LGRECO_EUNSUPPORTED;
}

int lgreco_weight_costs(const int64_t* d_bits, const int64_t* d_weight, int32_t L, int32_t K, int64_t* d_out,
                        void* stream) {
  if (!d_bits || !d_weight || !d_out || L < 0 || K <= 0) { lg_set_error("weight_costs: bad argument"); return LGRECO_EINVAL; }
  LG_CUDA(lg::launch_weight_costs(d_bits, d_weight, L, K, d_out, (cudaStream_t)stream));
  return LGRECO_OK;
}

size_t lgreco_solve_workspace_bytes(int32_t L, int32_t K, int32_t D) {
  if (L < 0 || K <= 0 || D <= 0) return 0;
  return lg::solve_workspace_bytes(L, K, D);
}

static bool host_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

// Host mode of lgreco_solve: the tables and outputs in host memory are staged through
// device scratch around the same kernels, and the call returns after the results are back.
static int solve_host(const double* h_err, const int64_t* h_bits, int32_t L, int32_t K, const int32_t* h_def,
                      const int32_t* h_comp, int32_t D, uint32_t flags, int32_t* h_choice, lgreco_solve_info* h_info,
                      cudaStream_t st) {
  const size_t ws = lg::solve_workspace_bytes(L, K, D);
  const size_t n = (size_t)L * K;
  const size_t bytes = n * 8 * 2 + (size_t)L * 4 * 3 + sizeof(lgreco_solve_info) + 64 + ws + 256;
  uint8_t* d = nullptr;
  if (cudaMallocAsync((void**)&d, bytes, st) != cudaSuccess) { lg_set_error("solve host mode: allocation"); return LGRECO_ENOMEM; }
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  uint8_t* q = d;
  double* e = reinterpret_cast<double*>(q); q += al(n * 8);
  int64_t* b = reinterpret_cast<int64_t*>(q); q += al(n * 8);
  int32_t* df = reinterpret_cast<int32_t*>(q); q += al((size_t)L * 4);
  int32_t* cp = h_comp ? reinterpret_cast<int32_t*>(q) : nullptr; q += al((size_t)L * 4);
  int32_t* ch = reinterpret_cast<int32_t*>(q); q += al((size_t)L * 4);
  lgreco_solve_info* inf = reinterpret_cast<lgreco_solve_info*>(q); q += al(sizeof(lgreco_solve_info));
  cudaError_t ce = cudaSuccess;
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(e, h_err, n * 8, cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(b, h_bits, n * 8, cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(df, h_def, (size_t)L * 4, cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess && cp) ce = cudaMemcpyAsync(cp, h_comp, (size_t)L * 4, cudaMemcpyHostToDevice, st);
  lg::SolveArgs a{e, b, L, K, df, cp, D, flags, ch, inf, nullptr, nullptr};
  if (ce == cudaSuccess) ce = lg::launch_solve(a, q, st);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(h_choice, ch, (size_t)L * 4, cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(h_info, inf, sizeof(lgreco_solve_info), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) { lg_set_error("solve host mode: %s", cudaGetErrorString(ce)); return LGRECO_ECUDA; }
  return LGRECO_OK;
}

int lgreco_solve(const double* d_err, const int64_t* d_bits, int32_t L, int32_t K, const int32_t* d_default_idx,
                 const int32_t* d_compress, int32_t D, uint32_t flags, int32_t* d_choice, lgreco_solve_info* d_info,
                 void* d_ws, size_t ws_bytes, void* stream) {
  if (L <= 0 || K <= 0 || K > 255 || D <= 0) { lg_set_error("bad L/K/D %d/%d/%d", L, K, D); return LGRECO_EINVAL; }
  if (!d_err || !d_bits || !d_default_idx || !d_choice || !d_info) { lg_set_error("null argument"); return LGRECO_EINVAL; }
  {
    const bool h[5] = {host_ptr(d_err), host_ptr(d_bits), host_ptr(d_default_idx), host_ptr(d_choice), host_ptr(d_info)};
    const bool hc = d_compress ? host_ptr(d_compress) : h[0];
    if (h[0] || h[1] || h[2] || h[3] || h[4] || hc) {
      if (!(h[0] && h[1] && h[2] && h[3] && h[4] && hc)) {
        lg_set_error("solve: tables and outputs must be all host or all device pointers");
        return LGRECO_EINVAL;
      }
      return solve_host(d_err, d_bits, L, K, d_default_idx, d_compress, D, flags, d_choice, d_info, (cudaStream_t)stream);
    }
  }
  if (!d_ws) { lg_set_error("null workspace (device mode)"); return LGRECO_EINVAL; }
  if (ws_bytes < lg::solve_workspace_bytes(L, K, D)) { lg_set_error("workspace too small"); return LGRECO_EINVAL; }
  lg::SolveArgs a{d_err, d_bits, L, K, d_default_idx, d_compress, D, flags, d_choice, d_info, nullptr, nullptr};
  cudaError_t e = lg::launch_solve(a, d_ws, (cudaStream_t)stream);
  if (e != cudaSuccess) { lg_set_error("solve launch: %s", cudaGetErrorString(e)); return LGRECO_ECUDA; }
  return LGRECO_OK;
}

int lgreco_plan_broadcast(lgreco_ctx* c, int32_t* d_choice, void* stream) {
  if (!c || !d_choice) return LGRECO_EINVAL;
  if (c->world == 1) return LGRECO_OK;
  if (c->p2p) {  // over peer memory (rank 0 pushes, the others acquire)
    LG_CUDA(lg::launch_p2p_plan(c->d_p2p, c->d_flags, c->world, c->rank, ++c->plan_epoch, d_choice, c->L,
                                (cudaStream_t)stream));
    return LGRECO_OK;
  }
  if (!c->comm) { lg_set_error("plan_broadcast: no NCCL communicator and no peers"); return LGRECO_EINVAL; }
  LG_NCCL(ncclBroadcast(d_choice, d_choice, (size_t)c->L, ncclInt32, 0, c->comm, (cudaStream_t)stream));
  return LGRECO_OK;
}

int64_t lgreco_payload_bytes(lgreco_ctx* c, const int32_t* h_choice) {
  if (!c || !h_choice) return LGRECO_EINVAL;
  if (c->family == LGRECO_TOPK) return topk_payload_bytes(c, h_choice);
  if (c->family == LGRECO_POWERSGD) return psgd_payload_bytes(c, h_choice);
  std::vector<lg::DevPlan> plan;
  int64_t S = 0;
  int s = qsgd_layout(c, h_choice, plan, S);
  return s == LGRECO_OK ? S : s;
}

int lgreco_shard_bounds(lgreco_ctx* c, const int32_t* h_choice, int32_t W, int64_t* h_rb, int64_t* h_bb) {
  if (!c || !h_choice || W < 1 || !h_rb || !h_bb) return LGRECO_EINVAL;
  std::vector<lg::DevPlan> plan;
  int64_t S = 0;
  LG_TRY(qsgd_layout(c, h_choice, plan, S));
  std::vector<int64_t> rb, bb;
  shard_bounds(c, plan, S, W, rb, bb);
  memcpy(h_rb, rb.data(), sizeof(int64_t) * (W + 1));
  memcpy(h_bb, bb.data(), sizeof(int64_t) * (W + 1));
  return LGRECO_OK;
}


int lgreco_qsgd_pack(lgreco_ctx* c, const int32_t* h_choice, const float* d_g, float* d_ef, uint8_t* d_payload,
                     float* d_dec, uint32_t rank, uint64_t step, void* stream) {
  if (!c || !h_choice || !d_g) return LGRECO_EINVAL;
  if (c->family != LGRECO_QSGD) return LGRECO_EUNSUPPORTED;
  LG_TRY(check_align16("qsgd_pack", d_g, d_ef, d_dec));
  cudaStream_t st = (cudaStream_t)stream;
  LG_TRY(set_plan(c, h_choice, st));
  uint32_t k0, k1;
  key_of(c, k0, k1);
  lg::QPackArgs a{d_g, d_ef, d_payload, d_dec, c->d_layers, c->d_plan, c->d_chunks_all, c->nchunks_all, c->B,
                  k0, k1, rank, (uint32_t)step, c->d_flag};
  LG_LAUNCH(c, lg::launch_qpack(a, st));
  c->launches += 1;
  return LGRECO_OK;
}

int lgreco_qsgd_reduce(lgreco_ctx* c, const int32_t* h_choice, int32_t W, int64_t r0, int64_t r1,
                       const uint8_t* d_recv, uint8_t* d_stage2, uint64_t step, void* stream) {
  if (!c || !h_choice || W < 1 || r0 < 0 || r1 < r0 || r1 > c->R) return LGRECO_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  LG_TRY(set_plan(c, h_choice, st));
  const int64_t b0 = rec_off(c, c->h_plan_v, r0, c->S), b1 = rec_off(c, c->h_plan_v, r1, c->S);
  uint32_t k0, k1;
  key_of(c, k0, k1);
  lg::QReduceArgs a{d_recv, b1 - b0, b0, d_stage2, c->d_layers, c->d_plan, c->d_bucket0, c->L, r0, r1,
                    c->B, W, k0, k1, (uint32_t)step};
  LG_LAUNCH(c, lg::launch_qreduce(a, st));
  c->launches += 1;
  return LGRECO_OK;
}

int lgreco_qsgd_unpack(lgreco_ctx* c, const int32_t* h_choice, const uint8_t* d_payload, float* d_out, void* stream) {
  if (!c || !h_choice || !d_payload || !d_out) return LGRECO_EINVAL;
  LG_TRY(check_align16("qsgd_unpack", d_out));
  cudaStream_t st = (cudaStream_t)stream;
  LG_TRY(set_plan(c, h_choice, st));
  lg::QUnpackArgs a{d_payload, d_out, c->d_layers, c->d_plan, c->d_chunks_all, c->nchunks_all, c->B};
  LG_LAUNCH(c, lg::launch_qunpack(a, st));
  c->launches += 1;
  return LGRECO_OK;
}

int lgreco_compress_allreduce(lgreco_ctx* c, const int32_t* h_choice, const float* d_g, float* d_ef, float* d_out,
                              uint64_t step, void* stream) {
  if (!c || !h_choice || !d_g || !d_out) { lg_set_error("null argument"); return LGRECO_EINVAL; }
  LG_TRY(check_align16("compress_allreduce", d_g, d_ef, d_out));
  cudaStream_t st = (cudaStream_t)stream;
  if (c->family == LGRECO_TOPK) return topk_compress_allreduce(c, h_choice, d_g, d_ef, d_out, step, st);
  if (c->family == LGRECO_POWERSGD) return psgd_compress_allreduce(c, h_choice, d_g, d_ef, d_out, step, st);
  if (c->family != LGRECO_QSGD) { lg_set_error("family unsupported"); return LGRECO_EUNSUPPORTED; }
  if (c->world == 1)  // stage 2 skipped (R13): fused pack + EF + decode, nothing leaves the GPU
    return lgreco_qsgd_pack(c, h_choice, d_g, d_ef, nullptr, d_out, 0u, step, stream);
  if (c->p2p) {
    for (int sg = 1; sg <= 3; ++sg) LG_TRY(lgreco_p2p_stage(c, h_choice, d_g, d_ef, d_out, step, sg, stream));
    return LGRECO_OK;
  }
  if (!c->comm) { lg_set_error("world > 1: neither an NCCL communicator nor peer buffers (lgreco_p2p_open)"); return LGRECO_EINVAL; }
  LG_TRY(lgreco_qsgd_pack(c, h_choice, d_g, d_ef, c->d_pay1, nullptr, (uint32_t)c->rank, step, stream));
  const int W = c->world, me = c->rank;
  const int64_t mine = c->byte_bounds[me + 1] - c->byte_bounds[me];
  // all-to-all of stage-1 shards: shard j -> rank j (the reduce-scatter pattern)
  LG_NCCL(ncclGroupStart());
  for (int j = 0; j < W; ++j) {
    const int64_t bj = c->byte_bounds[j + 1] - c->byte_bounds[j];
    if (bj > 0) LG_NCCL(ncclSend(c->d_pay1 + c->byte_bounds[j], (size_t)bj, ncclUint8, j, c->comm, st));
    if (mine > 0) LG_NCCL(ncclRecv(c->d_recv + (int64_t)j * mine, (size_t)mine, ncclUint8, j, c->comm, st));
  }
  LG_NCCL(ncclGroupEnd());
  LG_TRY(lgreco_qsgd_reduce(c, h_choice, W, c->rec_bounds[me], c->rec_bounds[me + 1], c->d_recv, c->d_pay2, step, stream));
  // all-gather of the stage-2 shards (ragged: grouped send/recv)
  LG_NCCL(ncclGroupStart());
  for (int j = 0; j < W; ++j) {
    if (j == me) continue;
    const int64_t bj = c->byte_bounds[j + 1] - c->byte_bounds[j];
    if (mine > 0) LG_NCCL(ncclSend(c->d_pay2 + c->byte_bounds[me], (size_t)mine, ncclUint8, j, c->comm, st));
    if (bj > 0) LG_NCCL(ncclRecv(c->d_pay2 + c->byte_bounds[j], (size_t)bj, ncclUint8, j, c->comm, st));
  }
  LG_NCCL(ncclGroupEnd());
  return lgreco_qsgd_unpack(c, h_choice, c->d_pay2, d_out, stream);
}

// ---- peer-memory exchange (QSGD, W > 1, no NCCL on the data path) -------------------
int lgreco_p2p_local(lgreco_ctx* c, void** h_ptrs3) {
  if (!c || !h_ptrs3 || !c->d_flags || !c->d_recv || !c->d_pay2) { lg_set_error("p2p_local: QSGD ctx with world > 1 only"); return LGRECO_EINVAL; }
  h_ptrs3[0] = c->d_recv; h_ptrs3[1] = c->d_pay2; h_ptrs3[2] = c->d_flags;
  return LGRECO_OK;
}

int lgreco_p2p_set_peers(lgreco_ctx* c, void* const* h_recv, void* const* h_stage2, void* const* h_flags) {
  if (!c || !h_recv || !h_stage2 || !h_flags || !c->d_p2p || c->world > lg::P2P_MAXW) {
    lg_set_error("p2p_set_peers: bad argument");
    return LGRECO_EINVAL;
  }
  for (int j = 0; j < c->world; ++j) {
    c->h_p2p.recv[j] = static_cast<uint8_t*>(h_recv[j]);
    c->h_p2p.s2[j] = static_cast<uint8_t*>(h_stage2[j]);
    c->h_p2p.flag[j] = static_cast<unsigned*>(h_flags[j]);
  }
  c->h_p2p.W = c->world;
  c->h_p2p.me = c->rank;
  // the pointers are needed before the first exchange (plan_broadcast); the shard bounds
  // are refreshed with every plan
  LG_CUDA(cudaMemcpy(c->d_p2p, &c->h_p2p, sizeof(lg::P2PDev), cudaMemcpyHostToDevice));
  LG_CUDA(lg::preload_p2p_kernels());  // no lazy module load while a peer waits (qsgd.cu)
  c->p2p = true;
  c->plan_valid = false;  // re-upload the descriptor with the next plan
  return LGRECO_OK;
}

int lgreco_p2p_export(lgreco_ctx* c, void* h_blob) {
  void* p[3];
  LG_TRY(lgreco_p2p_local(c, p));
  if (!h_blob) return LGRECO_EINVAL;
  for (int i = 0; i < 3; ++i)
    LG_CUDA(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(h_blob) + i, p[i]));
  return LGRECO_OK;
}

int lgreco_p2p_open(lgreco_ctx* c, const void* h_blobs) {
  void* mine[3];
  LG_TRY(lgreco_p2p_local(c, mine));
  if (!h_blobs) return LGRECO_EINVAL;
  void* ptrs[3][lg::P2P_MAXW];
  const cudaIpcMemHandle_t* hs = reinterpret_cast<const cudaIpcMemHandle_t*>(h_blobs);
  for (int j = 0; j < c->world; ++j)
    for (int i = 0; i < 3; ++i) {
      if (j == c->rank) { ptrs[i][j] = mine[i]; continue; }
      void* q = nullptr;
      LG_CUDA(cudaIpcOpenMemHandle(&q, hs[3 * j + i], cudaIpcMemLazyEnablePeerAccess));
      c->ipc_opened.push_back(q);
      ptrs[i][j] = q;
    }
  return lgreco_p2p_set_peers(c, ptrs[0], ptrs[1], ptrs[2]);
}

// Stage s of the peer-memory exchange on this rank: 1 = pack + EF with every record
// stored straight into its owner's window, then signal; 2 = wait for all stage-1 data,
// owner dequantise-sum-requantise (K8), push the stage-2 shard to every peer, signal;
// 3 = wait for all stage-2 shards, decode (K9).  lgreco_compress_allreduce runs 1, 2, 3.
int lgreco_p2p_stage(lgreco_ctx* c, const int32_t* h_choice, const float* d_g, float* d_ef, float* d_out,
                     uint64_t step, int32_t stage, void* stream) {
  if (!c || !c->p2p || !h_choice || stage < 1 || stage > 3) { lg_set_error("p2p_stage: bad argument / no peers"); return LGRECO_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  const bool fresh = !c->plan_valid;
  LG_TRY(set_plan(c, h_choice, st));
  const int W = c->world, me = c->rank;
  if (fresh || stage == 1) {
    for (int j = 0; j <= W; ++j) c->h_p2p.bb[j] = c->byte_bounds[j];
    LG_CUDA(cudaMemcpyAsync(c->d_p2p, &c->h_p2p, sizeof(lg::P2PDev), cudaMemcpyHostToDevice, st));
  }
  uint32_t k0, k1;
  key_of(c, k0, k1);
  if (stage == 1) {
    ++c->epoch;
    LG_TRY(check_align16("p2p_stage", d_g, d_ef, d_out));
    lg::QPackArgs a{d_g, d_ef, nullptr, nullptr, c->d_layers, c->d_plan, c->d_chunks_all, c->nchunks_all, c->B,
                    k0, k1, (uint32_t)me, (uint32_t)step, c->d_flag};
    a.p2p = c->d_p2p;
    LG_LAUNCH(c, lg::launch_qpack(a, st));
    LG_CUDA(lg::launch_p2p_signal(c->d_p2p, 0, c->epoch, st));
    c->launches += 2;
    return LGRECO_OK;
  }
  const int64_t mine = c->byte_bounds[me + 1] - c->byte_bounds[me];
  if (stage == 2) {
    LG_CUDA(lg::launch_p2p_wait(c->d_flags, W, me, 0, c->epoch, st));
    lg::QReduceArgs r{c->d_recv, mine, c->byte_bounds[me], c->d_pay2, c->d_layers, c->d_plan, c->d_bucket0, c->L,
                      c->rec_bounds[me], c->rec_bounds[me + 1], c->B, W, k0, k1, (uint32_t)step};
    r.p2p = c->d_p2p;  // stage-2 records stored into every peer's payload as they are produced
    LG_LAUNCH(c, lg::launch_qreduce(r, st));
    LG_CUDA(lg::launch_p2p_signal(c->d_p2p, 1, c->epoch, st));
    c->launches += 3;
    return LGRECO_OK;
  }
  LG_CUDA(lg::launch_p2p_wait(c->d_flags, W, me, 1, c->epoch, st));
  c->launches += 1;
  return lgreco_qsgd_unpack(c, h_choice, c->d_pay2, d_out, stream);
}

int lgreco_compress_allreduce_dev(lgreco_ctx* c, const int32_t* d_choice, const float* d_g, float* d_ef,
                                  float* d_out, uint64_t step, void* stream) {
  if (!c || !d_choice || !d_g || !d_out) { lg_set_error("null argument"); return LGRECO_EINVAL; }
  LG_TRY(check_align16("compress_allreduce_dev", d_g, d_ef, d_out));
  cudaStream_t st = (cudaStream_t)stream;
  if (c->world == 1 && c->family == LGRECO_QSGD) {
    // W = 1: nothing leaves the GPU, the fused pass needs only the bits per layer, which
    // K5 reads from the device choice itself (one launch)
    uint32_t k0, k1;
    key_of(c, k0, k1);
    lg::QPackArgs a{d_g, d_ef, nullptr, d_out, c->d_layers, c->d_plan, c->d_chunks_all, c->nchunks_all, c->B,
                    k0, k1, 0u, (uint32_t)step, c->d_flag};
    a.choice = d_choice;
    a.params = c->d_params;
    a.K = c->K;
    LG_LAUNCH(c, lg::launch_qpack(a, st));
    c->launches += 1;
    return LGRECO_OK;
  }
  if (c->world == 1 && c->family == LGRECO_TOPK) {
    c->launches += 0;
    return topk_compress_dev(c, d_choice, d_g, d_ef, d_out, step, st);
  }
  if (c->p2p && c->family == LGRECO_QSGD) {
    // W > 1 over peer memory with the plan laid out on the device: no host round trip
    LG_CUDA(lg::launch_plan_qsgd_layout(d_choice, c->d_params, c->K, c->d_layers, c->d_bucket0, c->L, c->R, c->B,
                                        c->d_plan, c->d_p2p, c->d_flag, st));
    c->plan_valid = false;  // d_plan / d_p2p now hold a device-chosen plan
    uint32_t k0, k1;
    key_of(c, k0, k1);
    const int W = c->world, me = c->rank;
    ++c->epoch;
    lg::QPackArgs a{d_g, d_ef, nullptr, nullptr, c->d_layers, c->d_plan, c->d_chunks_all, c->nchunks_all, c->B,
                    k0, k1, (uint32_t)me, (uint32_t)step, c->d_flag};
    a.p2p = c->d_p2p;
    LG_LAUNCH(c, lg::launch_qpack(a, st));
    LG_CUDA(lg::launch_p2p_signal(c->d_p2p, 0, c->epoch, st));
    LG_CUDA(lg::launch_p2p_wait(c->d_flags, W, me, 0, c->epoch, st));
    int nsm = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    lg::QReduceArgs r{c->d_recv, 0, 0, c->d_pay2, c->d_layers, c->d_plan, c->d_bucket0, c->L, 0, 0, c->B, W, k0, k1,
                      (uint32_t)step};
    r.p2p = c->d_p2p;
    r.device_bounds = 1;
    r.grid = nsm * 4;
    LG_LAUNCH(c, lg::launch_qreduce(r, st));  // stores its stage-2 records into every peer's payload too
    LG_CUDA(lg::launch_p2p_signal(c->d_p2p, 1, c->epoch, st));
    LG_CUDA(lg::launch_p2p_wait(c->d_flags, W, me, 1, c->epoch, st));
    lg::QUnpackArgs u{c->d_pay2, d_out, c->d_layers, c->d_plan, c->d_chunks_all, c->nchunks_all, c->B};
    LG_LAUNCH(c, lg::launch_qunpack(u, st));
    c->launches += 8;
    return LGRECO_OK;
  }
  // the exchange needs host-side shard sizes: bring the plan to the host
  LG_CUDA(cudaMemcpyAsync(c->h_choice_pinned, d_choice, sizeof(int32_t) * c->L, cudaMemcpyDeviceToHost, st));
  LG_CUDA(cudaStreamSynchronize(st));
  return lgreco_compress_allreduce(c, c->h_choice_pinned, d_g, d_ef, d_out, step, stream);
}

// Fused per-step pass (the plan in force compresses the step, the
// profile of the same x feeds the next solve): K1 profiles x = g + e for every candidate
// and, from the same registers and uniforms, quantises x with the planned candidate
// (K5's arithmetic: out, e'), one read of g and e.  Any other configuration runs the two
// calls it is defined as.
int lgreco_profile_compress(lgreco_ctx* c, const int32_t* d_choice, const float* d_g, float* d_ef, float* d_out,
                            uint64_t step, double* d_err, int64_t* d_bits, uint32_t flags, void* stream) {
  if (!c || !d_choice || !d_g || !d_out || !d_err || !d_bits) { lg_set_error("null argument"); return LGRECO_EINVAL; }
  if (flags & ~(uint32_t)LGRECO_PC_CONCURRENT) { lg_set_error("profile_compress: unknown flags 0x%x", flags); return LGRECO_EINVAL; }
  LG_TRY(check_align16("profile_compress", d_g, d_ef, d_out));
  cudaStream_t st = (cudaStream_t)stream;
  const bool p2p_fused = c->family == LGRECO_QSGD && c->world > 1 && c->p2p && c->B == 128 && c->nqchunks > 0;
  // (the fused kernel stores e' unconditionally: without an EF buffer, the two calls)
  const bool fused = d_ef != nullptr &&
                     ((c->family == LGRECO_QSGD && c->world == 1 && c->B == 128 && c->nqchunks > 0) || p2p_fused);
  if (!fused) {
    LG_TRY(lgreco_profile(c, d_g, d_ef, step, d_err, d_bits, stream));
    return lgreco_compress_allreduce_dev(c, d_choice, d_g, d_ef, d_out, step, stream);
  }
  uint32_t k0, k1;
  key_of(c, k0, k1);
  lg::QProfileArgs a{d_g, d_ef, c->d_layers, c->L, c->d_chunks, c->nchunks, c->d_layer_chunk0,
                     c->B, c->cs, c->d_params, c->K, k0, k1, (uint32_t)c->rank, (uint32_t)step,
                     c->d_partial, d_err, d_bits};
  a.qinfo = c->d_qinfo; a.nqchunks = c->nqchunks; a.layer_qchunk0 = c->d_layer_qchunk0;
  a.nqwarps = c->nqwarps; a.ticket = c->d_ticket;
  a.segs = c->d_qseg; a.nseg = c->nqseg; a.lseg0 = c->d_lqseg0; a.segsum = c->d_segsum; a.ldone = c->d_ldone;
  a.ptr_aligned = 1;  // (checked above)
  const bool conc = (flags & LGRECO_PC_CONCURRENT) != 0;
  lg::QFuse fz{d_ef, d_out, d_choice, c->d_flag, c->d_chunks_raw, c->nchunks_raw, c->d_layers, c->B, conc ? 1 : 0,
                 c->L};
  if (p2p_fused) {
    // W > 1 over peer memory: the plan laid out on the device (payload offsets, shard
    // bounds), then the fused pass stores every stage-1 record straight into its owner's
    // window -- the rest is compress_allreduce_dev's peer-memory step (R13)
    LG_CUDA(lg::launch_plan_qsgd_layout(d_choice, c->d_params, c->K, c->d_layers, c->d_bucket0, c->L, c->R, c->B,
                                        c->d_plan, c->d_p2p, c->d_flag, st));
    c->plan_valid = false;  // d_plan / d_p2p now hold a device-chosen plan
    ++c->epoch;
    fz.plan = c->d_plan;
    fz.p2p = c->d_p2p;
    fz.nowait = 0;  // (the layout kernel precedes it)
  }
  a.fuse = &fz;
  if (c->timing) {
    cudaEvent_t e0, e1;
    LG_CUDA(cudaEventCreate(&e0));
    LG_CUDA(cudaEventCreate(&e1));
    c->tev.emplace_back(e0, e1);
    a.ev0 = e0;
    a.ev1 = e1;
  }
  LG_LAUNCH(c, lg::launch_qprofile(a, st));
  c->launches += 2;
  if (p2p_fused) {
    const int W = c->world, me = c->rank;
    LG_CUDA(lg::launch_p2p_signal(c->d_p2p, 0, c->epoch, st));
    LG_CUDA(lg::launch_p2p_wait(c->d_flags, W, me, 0, c->epoch, st));
    int nsm = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    lg::QReduceArgs r{c->d_recv, 0, 0, c->d_pay2, c->d_layers, c->d_plan, c->d_bucket0, c->L, 0, 0, c->B, W, k0, k1,
                      (uint32_t)step};
    r.p2p = c->d_p2p;
    r.device_bounds = 1;
    r.grid = nsm * 4;
    LG_LAUNCH(c, lg::launch_qreduce(r, st));
    LG_CUDA(lg::launch_p2p_signal(c->d_p2p, 1, c->epoch, st));
    LG_CUDA(lg::launch_p2p_wait(c->d_flags, W, me, 1, c->epoch, st));
    lg::QUnpackArgs u{c->d_pay2, d_out, c->d_layers, c->d_plan, c->d_chunks_all, c->nchunks_all, c->B};
    LG_LAUNCH(c, lg::launch_qunpack(u, st));
    c->launches += 7;
  }
  return LGRECO_OK;
}

int lgreco_topk_pack(lgreco_ctx* c, const int32_t* h_choice, const float* d_g, float* d_ef, uint8_t* d_payload,
                     float* d_out, void* stream) {
  if (!c || !h_choice || !d_g) return LGRECO_EINVAL;
  if (c->family != LGRECO_TOPK) return LGRECO_EUNSUPPORTED;
  return topk_pack(c, h_choice, d_g, d_ef, d_payload, d_out, ~0ull, (cudaStream_t)stream);  // (no step: no reuse)
}

int lgreco_topk_combine(lgreco_ctx* c, const int32_t* h_choice, int32_t W, const uint8_t* d_gathered, float* d_out,
                        void* stream) {
  if (!c || !h_choice || W < 1 || !d_gathered || !d_out) return LGRECO_EINVAL;
  if (c->family != LGRECO_TOPK) return LGRECO_EUNSUPPORTED;
  return topk_combine(c, h_choice, W, d_gathered, d_out, (cudaStream_t)stream);
}

int lgreco_psgd_sizes(lgreco_ctx* c, int64_t* h_p_elems, int64_t* h_q_elems) {
  if (!c || c->family != LGRECO_POWERSGD || !h_p_elems || !h_q_elems) return LGRECO_EINVAL;
  *h_p_elems = psgd_sizes(c, 0);
  *h_q_elems = psgd_sizes(c, 1);
  return LGRECO_OK;
}

int lgreco_psgd_factors(lgreco_ctx* c, float* d_Phat, float* d_Q, void* stream) {
  if (!c || c->family != LGRECO_POWERSGD) { lg_set_error("psgd_factors: not a PowerSGD ctx"); return LGRECO_EINVAL; }
  return psgd_factors(c, d_Phat, d_Q, (cudaStream_t)stream);
}

int lgreco_psgd_p(lgreco_ctx* c, const int32_t* h_choice, const float* d_g, const float* d_ef, float* d_P,
                  uint64_t step, void* stream) {
  if (!c || !h_choice || !d_g || !d_P || c->family != LGRECO_POWERSGD) return LGRECO_EINVAL;
  return psgd_p(c, h_choice, d_g, d_ef, d_P, step, (cudaStream_t)stream);
}

int lgreco_psgd_q(lgreco_ctx* c, const int32_t* h_choice, const float* d_g, const float* d_ef, const float* d_Psum,
                  int32_t W, float* d_Q, void* stream) {
  if (!c || !h_choice || !d_g || !d_Psum || !d_Q || W < 1 || c->family != LGRECO_POWERSGD) return LGRECO_EINVAL;
  return psgd_q(c, h_choice, d_g, d_ef, d_Psum, W, d_Q, (cudaStream_t)stream);
}

int lgreco_psgd_out(lgreco_ctx* c, const int32_t* h_choice, const float* d_g, float* d_ef, const float* d_Qsum,
                    int32_t W, float* d_out, void* stream) {
  if (!c || !h_choice || !d_g || !d_Qsum || W < 1 || c->family != LGRECO_POWERSGD) return LGRECO_EINVAL;
  return psgd_out(c, h_choice, d_g, d_ef, d_Qsum, W, d_out, (cudaStream_t)stream);
}

int lgreco_psgd_raw_pack(lgreco_ctx* c, const int32_t* h_choice, const float* d_g, float* d_ef, uint8_t* d_payload,
                         float* d_out, void* stream) {
  if (!c || !h_choice || !d_g || c->family != LGRECO_POWERSGD) return LGRECO_EINVAL;
  return psgd_raw_pack(c, h_choice, d_g, d_ef, d_payload, d_out, (cudaStream_t)stream);
}

int lgreco_psgd_raw_combine(lgreco_ctx* c, const int32_t* h_choice, int32_t W, const uint8_t* d_gathered,
                            float* d_out, void* stream) {
  if (!c || !h_choice || W < 1 || !d_gathered || !d_out || c->family != LGRECO_POWERSGD) return LGRECO_EINVAL;
  return psgd_raw_combine(c, h_choice, W, d_gathered, d_out, (cudaStream_t)stream);
}

int lgreco_plan_layout(const lgreco_layer* layers, int32_t L, const lgreco_candidates* cand, const int32_t* h_choice,
                       int32_t W, int64_t* h_S, int64_t* h_rec_bounds, int64_t* h_byte_bounds) {
  if (!layers || L <= 0 || !cand || !cand->params || !h_choice || W < 1 || !h_S) return LGRECO_EINVAL;
  lgreco_ctx c;  // host-only view: no device state is touched
  c.L = L; c.K = cand->K; c.family = cand->family;
  c.B = cand->family == LGRECO_QSGD ? cand->qbucket : 128;
  if (c.B < 128 || c.B % 128) return LGRECO_EINVAL;
  c.layers.assign(layers, layers + L);
  c.params.assign(cand->params, cand->params + cand->K);
  c.bucket0.resize(L + 1);
  int64_t gb = 0;
  for (int l = 0; l < L; ++l) { c.bucket0[l] = gb; gb += (layers[l].numel + c.B - 1) / c.B; }
  c.bucket0[L] = gb;
  c.R = gb;
  int64_t S = 0;
  if (cand->family == LGRECO_QSGD) {
    std::vector<lg::DevPlan> plan;
    LG_TRY(qsgd_layout(&c, h_choice, plan, S));
    std::vector<int64_t> rb, bb;
    shard_bounds(&c, plan, S, W, rb, bb);
    if (h_rec_bounds) memcpy(h_rec_bounds, rb.data(), sizeof(int64_t) * (W + 1));
    if (h_byte_bounds) memcpy(h_byte_bounds, bb.data(), sizeof(int64_t) * (W + 1));
  } else {
    for (int l = 0; l < L; ++l) {
      const lgreco_layer& ly = layers[l];
      int64_t bytes = 4 * ly.numel;
      if (ly.compress) {
        const int j = h_choice[l];
        if (j < 0 || j >= cand->K) return LGRECO_EINVAL;
        const int32_t prm = cand->params[j];
        if (cand->family == LGRECO_TOPK) {
          int64_t k = ((int64_t)prm * ly.numel + 999999) / 1000000;
          k = std::max<int64_t>(1, std::min<int64_t>(k, ly.numel));
          bytes = 8 * k;
        } else if (ly.rows > 0 && (int64_t)prm * (ly.rows + ly.cols) < ly.numel) {
          bytes = 0;  // low-rank factors travel through the all-reduces
        }
      }
      S += bytes;
      S = (S + 15) & ~(int64_t)15;
    }
    if (h_rec_bounds || h_byte_bounds)
      for (int j = 0; j <= W; ++j) {
        if (h_rec_bounds) h_rec_bounds[j] = 0;
        if (h_byte_bounds) h_byte_bounds[j] = j == W ? S : 0;
      }
  }
  *h_S = S;
  return LGRECO_OK;
}

int lgreco_debug_philox(const uint32_t* d_ctr, uint32_t key0, uint32_t key1, int64_t n, uint32_t* d_out, void* stream) {
  cudaError_t e = lg::launch_philox(d_ctr, key0, key1, n, d_out, (cudaStream_t)stream);
  if (e != cudaSuccess) { lg_set_error("philox: %s", cudaGetErrorString(e)); return LGRECO_ECUDA; }
  return LGRECO_OK;
}

}  // extern "C"
