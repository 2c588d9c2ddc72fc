// ctx.h -- internal definition of lgreco_ctx shared by the C-ABI translation units.
#pragma once
#include <nccl.h>
#include <string.h>

#include <vector>

#include "common.cuh"
#include "kernels.h"

#define LG_NCCL(call)                                                                   \
  do {                                                                                  \
    ncclResult_t _r = (call);                                                           \
    if (_r != ncclSuccess) {                                                            \
      lg_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, ncclGetErrorString(_r));  \
      return LGRECO_ENCCL;                                                              \
    }                                                                                   \
  } while (0)

#define LG_TRY(call)                 \
  do {                               \
    int _s = (call);                 \
    if (_s != LGRECO_OK) return _s;  \
  } while (0)

#define LG_LAUNCH(ctx, call)                                                              \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess) {                                                              \
      lg_set_error("%s:%d launch %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
      return LGRECO_ECUDA;                                                                \
    }                                                                                     \
  } while (0)

struct lgreco_ctx {
  int L = 0, rank = 0, world = 1;
  int family = 0, K = 0, B = 128, power_steps = 5;
  uint64_t seed = 0;
  std::vector<lgreco_layer> layers;
  std::vector<int32_t> params;
  std::vector<int64_t> bucket0;  // L+1
  int64_t N = 0, R = 0;
  int64_t launches = 0;
  // optional per-launch CUDA events around the family's dominant profile kernel
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;
  // device tables
  lg::DevLayer* d_layers = nullptr;
  int64_t* d_bucket0 = nullptr;
  float* d_cand_s = nullptr;
  int32_t* d_params = nullptr;
  lg::ProfChunk* d_chunks = nullptr;      // chunks of compressed layers (profile)
  int nchunks = 0;
  lg::ProfChunk* d_chunks_all = nullptr;  // chunks of every layer (pack / unpack)
  int nchunks_all = 0;
  lg::ProfChunk* d_chunks_raw = nullptr;  // chunks of the lossless layers (fused profile + compress)
  int nchunks_raw = 0;
  lg::CandS cs{};
  int32_t* d_layer_chunk0 = nullptr;
  double* d_partial = nullptr;
  // K1 at B = 128: persistent warps over 32-bucket chunks of the compressed layers
  lg::QInfo* d_qinfo = nullptr;
  int nqchunks = 0;
  int32_t* d_layer_qchunk0 = nullptr;
  int nqwarps = 0;
  unsigned* d_ticket = nullptr;
  lg::QSeg* d_qseg = nullptr;    // K1b segments (<= 256 quad rows of one layer)
  int nqseg = 0;
  int32_t* d_lqseg0 = nullptr;   // per-layer first segment [L+1]
  double* d_segsum = nullptr;    // [nqseg][K]
  unsigned* d_ldone = nullptr;   // per-layer finished-segment counters [L]
  int psgd_method = 0;           // resolved PowerSGD profile method (LGRECO_PSGD_POWER / _SVD)
  unsigned* d_flag = nullptr;
  // plan
  std::vector<int32_t> plan_choice;
  bool plan_valid = false;
  std::vector<lg::DevPlan> h_plan_v;
  lg::DevPlan* h_plan_pinned = nullptr;
  lg::DevPlan* d_plan = nullptr;
  cudaEvent_t plan_evt = nullptr;
  int64_t S = 0;
  std::vector<int64_t> rec_bounds, byte_bounds;
  // exchange buffers
  uint8_t *d_pay1 = nullptr, *d_recv = nullptr, *d_pay2 = nullptr;
  int64_t pay_cap = 0;
  ncclComm_t comm = nullptr;
  int32_t* h_choice_pinned = nullptr;  // D2H staging for lgreco_compress_allreduce_dev
  // TopK state (family == LGRECO_TOPK)
  struct Topk* tk = nullptr;
  // PowerSGD state (family == LGRECO_POWERSGD)
  struct Psgd* ps = nullptr;
  // SVD-profile workspace (svd.cu, created on first use)
  void* svd = nullptr;
  // peer-memory exchange (QSGD, W > 1): peers' buffers (IPC-opened or given), flags
  bool p2p = false;
  unsigned* d_flags = nullptr;          // this rank's flag words [3][W] (stage, sender) + plan [L]
  lg::P2PDev h_p2p{};                   // host copy (pointers + shard bounds of the plan)
  lg::P2PDev* d_p2p = nullptr;
  std::vector<void*> ipc_opened;        // to cudaIpcCloseMemHandle
  unsigned epoch = 0;
  unsigned plan_epoch = 0;
};

// family-specific parts (api_topk.cu, api_psgd.cu)
int topk_init(lgreco_ctx* c, cudaStream_t st);
void topk_destroy(lgreco_ctx* c);
int topk_profile(lgreco_ctx* c, const float* g, const float* e, uint64_t step, double* err, int64_t* bits,
                 cudaStream_t st);
int topk_pack(lgreco_ctx* c, const int32_t* choice, const float* g, float* ef, uint8_t* payload, float* out, uint64_t step,
              cudaStream_t st);
int topk_combine(lgreco_ctx* c, const int32_t* choice, int W, const uint8_t* gathered, float* out, cudaStream_t st);
int topk_compress_allreduce(lgreco_ctx* c, const int32_t* choice, const float* g, float* ef, float* out,
                            uint64_t step, cudaStream_t st);
int64_t topk_payload_bytes(lgreco_ctx* c, const int32_t* choice);
int topk_compress_dev(lgreco_ctx* c, const int32_t* d_choice, const float* g, float* ef, float* out, uint64_t step,
                      cudaStream_t st);
int psgd_init(lgreco_ctx* c, cudaStream_t st);
void psgd_destroy(lgreco_ctx* c);
int psgd_profile(lgreco_ctx* c, const float* g, const float* e, uint64_t step, double* err, int64_t* bits,
                 cudaStream_t st);
int64_t psgd_payload_bytes(lgreco_ctx* c, const int32_t* choice);
int psgd_p(lgreco_ctx* c, const int32_t* choice, const float* g, const float* e, float* d_P, uint64_t step,
           cudaStream_t st);
int psgd_q(lgreco_ctx* c, const int32_t* choice, const float* g, const float* e, const float* d_Psum, int W,
           float* d_Q, cudaStream_t st);
int psgd_out(lgreco_ctx* c, const int32_t* choice, const float* g, float* ef, const float* d_Qsum, int W, float* out,
             cudaStream_t st);
int psgd_raw_pack(lgreco_ctx* c, const int32_t* choice, const float* g, float* ef, uint8_t* payload, float* out,
                  cudaStream_t st);
int psgd_raw_combine(lgreco_ctx* c, const int32_t* choice, int W, const uint8_t* gathered, float* out, cudaStream_t st);
int psgd_compress_allreduce(lgreco_ctx* c, const int32_t* choice, const float* g, float* ef, float* out,
                            uint64_t step, cudaStream_t st);
int64_t psgd_sizes(lgreco_ctx* c, int which);
int psgd_factors(lgreco_ctx* c, float* d_Phat, float* d_Q, cudaStream_t st);
void svd_destroy(lgreco_ctx* c);


