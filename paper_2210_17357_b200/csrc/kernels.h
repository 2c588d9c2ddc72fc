// kernels.h -- internal launcher interface between the C ABI (api.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace lg {

struct ProfChunk {
  int32_t layer;  // layer index
  int32_t nbk;    // buckets in this chunk
  int64_t first;  // first bucket index within the layer
};

struct CandS { float s[16]; };

// K1 (B = 128) work unit: one quad (4 buckets of one layer): flat element offset of its
// first element, global index of its first bucket (Philox counter base, mod 2^32),
// number of valid elements (512 unless the layer ends inside the quad) in bits 0-9 of
// nv_layer and the quad's layer index in bits 10-31 (the fused profile + compress reads
// the layer's plan entry).
struct QInfo { int64_t elem0; uint32_t gb0; int32_t nv_layer; };
__host__ __device__ __forceinline__ int qi_nvalid(const QInfo& q) { return q.nv_layer & 1023; }
__host__ __device__ __forceinline__ int qi_layer(const QInfo& q) { return (int)((uint32_t)q.nv_layer >> 10); }
constexpr int QI_MAX_LAYERS = 1 << 22;
// K1b segment: <= 256 consecutive quad rows of one layer
struct QSeg { int32_t layer, row0, nrows, pad; };
  // s_j = 2^{b_j} - 1, passed by value (constant bank)

struct P2PDev;
// Fused profile + compress (lgreco_profile_compress, W = 1): besides the profile's
// partial rows, K1 quantises every quad with the layer's planned candidate and writes
// the decoded output and the new EF (K5's arithmetic), and its first warps handle the
// lossless layers' chunks (raw copy, EF zeroed).
struct QFuse {
  float* ef;                 // EF in / out (the profile's e)
  float* out;                // decoded output
  const int32_t* choice;     // plan: candidate per layer (LGRECO_CHOICE_SKIP: untouched)
  unsigned* flag;            // bit 0 non-finite input, bit 1 choice outside [0, K)
  const ProfChunk* raw; int nraw;  // chunks of the lossless layers
  const DevLayer* layers; int B;
  int nowait;                // 1: no griddepcontrol.wait (LGRECO_PC_CONCURRENT)
  int L;                     // layers (the first QF_LCACHE plan entries are staged in shared memory)
  // W > 1 (peer-memory exchange): stage-1 records (R7) stored into the owners' windows
  // instead of the decoded output; `plan` is the device layout of `choice`
  const DevPlan* plan = nullptr;
  const P2PDev* p2p = nullptr;
};
constexpr int QF_LCACHE = 4096;
// K1's ticket words (64 apart): [0, 16) the parts' quad tickets, then the finish counter
constexpr int QT_ARR = 16, QT_WORDS = 17 * 64;

struct QProfileArgs {
  const float* g; const float* e;
  const DevLayer* layers; int L;
  const ProfChunk* chunks; int nchunks; const int32_t* layer_chunk0;
  int B; CandS cs; const int32_t* params; int K;
  uint32_t k0, k1, rankfield, step;
  double* partial; double* err; int64_t* bits;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // when set: recorded around the K1 launch
  // B == 128: persistent quad kernel over 32-bucket chunks (qchunks, per-layer
  // layer_qchunk0[L+1]), nqwarps resident warps, ticket[2] zeroed counters
  const QInfo* qinfo = nullptr; int nqchunks = 0; const int32_t* layer_qchunk0 = nullptr;
  int nqwarps = 0; unsigned* ticket = nullptr; int ptr_aligned = 0;
  const QSeg* segs = nullptr; int nseg = 0; const int32_t* lseg0 = nullptr; double* segsum = nullptr;
  unsigned* ldone = nullptr;
  const QFuse* fuse = nullptr;  // non-null: the fused profile + compress kernel
};

// Peer-memory exchange (W <= 8 ranks): device pointers to every rank's stage-1 receive
// window, stage-2 payload and flag words, and the shard byte bounds of the current plan.
constexpr int P2P_MAXW = 8;
struct P2PDev {
  uint8_t* recv[P2P_MAXW];
  uint8_t* s2[P2P_MAXW];
  unsigned* flag[P2P_MAXW];   // flag[j][0..W) stage 1, [W..2W) stage 2, [2W..3W) plan (word =
                              // sender); the plan itself at words [3*P2P_MAXW, +L)
  int64_t bb[P2P_MAXW + 1];   // shard byte bounds of the current plan (R13)
  int64_t rb[P2P_MAXW + 1];   // shard record bounds
  int W, me;
};

struct QPackArgs {
  const float* g; float* ef; uint8_t* payload; float* dec;
  const DevLayer* layers; const DevPlan* plan; const ProfChunk* chunks; int nchunks; int B;
  uint32_t k0, k1, rankfield, step; unsigned* flag;
  const P2PDev* p2p = nullptr;  // non-null: records go straight to their owner's window
  // non-null (W = 1, no payload): bits per layer = params[choice[l]] read in the kernel
  // itself (no plan kernel); a choice outside [0, K) sets flag bit 2 and uses 0
  const int32_t* choice = nullptr; const int32_t* params = nullptr; int K = 0;
};

struct QUnpackArgs {
  const uint8_t* payload; float* out;
  const DevLayer* layers; const DevPlan* plan; const ProfChunk* chunks; int nchunks; int B;
};

struct QReduceArgs {
  const uint8_t* recv; int64_t shard_bytes; int64_t byte0; uint8_t* stage2;
  const DevLayer* layers; const DevPlan* plan; const int64_t* bucket0; int L;
  int64_t r0, r1; int B; int W; uint32_t k0, k1, step;
  const P2PDev* p2p = nullptr;  // non-null: stage-2 records also stored into every peer's payload
  int device_bounds = 0;        // 1: this rank's shard (r0, r1, byte0, bytes) read from p2p on the device
  int grid = 0;                 // with device_bounds: fixed grid (the shard size is not known on the host)
};

cudaError_t launch_qprofile(const QProfileArgs& a, cudaStream_t st);
cudaError_t preload_p2p_kernels();
cudaError_t launch_qpack(const QPackArgs& a, cudaStream_t st);
cudaError_t launch_qunpack(const QUnpackArgs& a, cudaStream_t st);
cudaError_t launch_qreduce(const QReduceArgs& a, cudaStream_t st);
cudaError_t launch_plan_qsgd_dev(const int32_t* choice, const int32_t* params, int K, const DevLayer* layers, int L,
                                 DevPlan* plan, unsigned* flag, cudaStream_t st);
cudaError_t launch_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, int64_t n, uint32_t* out,
                          cudaStream_t st);

// TopK (topk.cu) -----------------------------------------------------------------
struct TChunk { int32_t cidx; int32_t n; int64_t first; };  // cidx: compressed-layer (or layer) index
struct TQ {  // one radix-select query (layer, density)
  int64_t k, r;          // kept count; residual rank inside the current bin
  int32_t b1, s1, c2, s2; // level-1 bin / slot, level-2 sub-bin / slot
  uint32_t T; int32_t bad;  // threshold key; non-finite input seen
  double below, sse;     // sum x^2 strictly below the current bin; final dropped energy
  int64_t ties;          // keys equal to T in the layer (after S3)
};
struct TPlan { int64_t pay_off; int64_t k; };
struct TkArgs {
  const DevLayer* layers; const int32_t* clayer; int nC;
  const TChunk* chunks; int nchunks; const int32_t* cchunk0;
  uint32_t* cnt1; unsigned long long* sum1; uint32_t* cnt2; unsigned long long* sum2; uint32_t* cnt3;
  int32_t* n1; int32_t* n2; int32_t* sl1; uint32_t* sl2;
  TQ* q; const int64_t* kq; uint2* ccnt; ulonglong2* coff; const TPlan* tplan; unsigned* flag;
  uint32_t* ckeys; int32_t* ckn;  // per chunk: keys of its boundary level-1 bins (pass2 -> pass3), count
  int32_t* ckz;                   // per chunk: its zero keys when the zero bin is a boundary bin (not compacted)
  int need_off = 1;  // 0: no payload (W = 1 fused): chunks of layers keeping all or none of T's ties skip the count
};
cudaError_t launch_topk_reuse(const int32_t* choice, int K, const int32_t* clayer, int nC, const TQ* qprof, TQ* qc,
                              unsigned* flag, cudaStream_t st);
constexpr int TK_CKCAP = 2048;  // compacted boundary keys kept per 16384-element chunk
cudaError_t launch_topk_select(const float* g, const float* e, const TkArgs& a, int nq, double* err, int64_t* bits,
                               int K, cudaStream_t st, int64_t* launches);
cudaError_t launch_plan_topk_dev(const int32_t* choice, const int32_t* params, int K, const DevLayer* layers,
                                 const int32_t* clayer, int nC, int64_t* kplan, unsigned* flag, cudaStream_t st);
cudaError_t launch_topk_lossless_rows(const DevLayer* layers, int L, int K, double* err, int64_t* bits, cudaStream_t st);
cudaError_t launch_topk_compact(const float* g, float* ef, uint8_t* payload, float* out, const TkArgs& a,
                                cudaStream_t st);
cudaError_t launch_lossless_pack(const float* g, float* ef, uint8_t* payload, float* out, const int32_t* choice,
                                 const DevLayer* layers,
                                 const TChunk* chunks, int nchunks, const TPlan* tplan, unsigned* flag,
                                 cudaStream_t st);
cudaError_t launch_topk_combine(const uint8_t* gathered, int64_t S, int W, float* out, const DevLayer* layers,
                                const TChunk* all_chunks, int nall, const int32_t* clayer,
                                int nC, const int64_t* kpre, int64_t ktotal, const TPlan* tplan, cudaStream_t st,
                                int64_t* launches);

// PowerSGD (psgd.cu) ---------------------------------------------------------------
struct PLayer {        // one compressed matrix layer in a grouped launch
  int64_t moff;        // element offset of M (m x k row-major) in the flat gradient
  int32_t m, k, r;     // view and the rank of this launch
  int32_t layer;       // layer index in the table
  int64_t poff, qoff, goff;  // offsets into P (m x r), Q (k x r) col-major, G (r x r)
  int64_t qstride;     // elements between split partials of Q (M^T P row splits)
  int64_t pstride;     // elements between split partials of P (M Q column splits)
  int32_t nsplit;      // row splits of M^T P
  int32_t nks;         // column (K) splits of M Q
};
// tile of a grouped launch: MQ tensor-core tile (rows i0.., K columns [c0, i1), split);
// MtP tile (columns c0.., rows [i0, i1), split); row tile (i0); element tile (i0, c0)
struct PTile { int32_t ci, split, i0, i1, c0, pad; };
struct TcMapCache { uint64_t ver = ~0ull; const void* g = nullptr; const void* e = nullptr; const void* b = nullptr; };
struct RawSeg { int64_t off, n, pay_off; };            // raw (uncompressed) segment of the gradient
struct PsArgs {
  const float* g; const float* e; const PLayer* pl; int nC;
  const PTile* rtiles; int n_rtiles; const PTile* ctiles; int n_ctiles; int rmax;
  const PTile* rt128; int n_rt128; const PTile* ct128; int n_ct128;  // tensor-core tiles (128 rows / cols)
  const PTile* etiles; int n_etiles; const int32_t* etile0;           // element tiles (64 rows x 256 cols)
  // Gram row chunks (<= 1024 rows of one layer) of P-shaped / Q-shaped factors, per-layer
  // chunk ranges, and the RMAX x RMAX partial per chunk
  const PTile* gcp = nullptr; int n_gcp = 0; const int32_t* gcp0 = nullptr;
  const PTile* gcq = nullptr; int n_gcq = 0; const int32_t* gcq0 = nullptr;
  double* gpart = nullptr;
  int mmax = 0;  // the largest m of the config (the fused small-layer CholQR2 when it fits)
  // TMA tensor maps of the tensor-core GEMMs (psgd_tc.cu): the config's host layer list,
  // its version, a device area of 3 maps (g, e, B) per layer for each GEMM flavour and the
  // host cache of what the area currently encodes (nullptr: no TMA, 4-byte copies)
  const PLayer* h_pl = nullptr; uint64_t cfg_ver = 0;
  void* maps_mq = nullptr; void* maps_tr = nullptr; TcMapCache* mc_mq = nullptr; TcMapCache* mc_tr = nullptr;
};
// profile-error work buffers: d / ||M||^2 partials [etiles][RMAX+1], G_P, G_Q (per layer
// r x r at goff), the per-layer fallback flag
struct PsErrBufs { double* dpart; double* GP; double* GQ; int32_t* flag; };
cudaError_t launch_ps_gram(const PsArgs& a, const float* X, int isq, float scale, double* G, cudaStream_t st);
cudaError_t launch_ps_initq(const PsArgs& a, float* Q, uint32_t k0, uint32_t k1, uint32_t step, const int32_t* only,
                            cudaStream_t st);
cudaError_t launch_ps_mq(const PsArgs& a, const float* Q, float* P, float* Ppart, cudaStream_t st);
cudaError_t launch_ps_orth(const PsArgs& a, const float* P, float scale, double* G, float* Ph, cudaStream_t st);
cudaError_t launch_ps_mtp(const PsArgs& a, const float* Ph, float* part, float* Q, float scale, cudaStream_t st);
cudaError_t launch_ps_mq_tc(const PsArgs& a, const PTile* tiles128, int ntiles, const float* Q, float* P,
                            cudaStream_t st);
cudaError_t launch_ps_preduce(const PsArgs& a, const float* part, float* P, cudaStream_t st);
cudaError_t launch_ps_mtp_tc(const PsArgs& a, const PTile* ctiles128, int ntiles, const float* Ph, float* part,
                             cudaStream_t st);
cudaError_t launch_ps_mtp_scale(const PsArgs& a, const float* src, float* dst, float scale, cudaStream_t st);
cudaError_t launch_ps_err(const PsArgs& a, const float* Ph, const float* Q, const int32_t* ranks, int K, int nbmax,
                          double* err, int64_t* bits, double* epart, const PsErrBufs& w, cudaStream_t st);
cudaError_t launch_ps_lossless_rows(const DevLayer* layers, int L, int K, const int32_t* ismat, double* err,
                                    int64_t* bits, cudaStream_t st);
cudaError_t launch_ps_out(const PsArgs& a, float* ef, float* out, const float* Ph, const float* Q, cudaStream_t st);
cudaError_t launch_ps_raw_pack(const float* g, float* ef, uint8_t* payload, float* out, const RawSeg* segs, int nseg,
                               unsigned* flag, cudaStream_t st);
cudaError_t launch_ps_raw_mean(const uint8_t* gathered, int64_t S, int W, float* out, const RawSeg* segs, int nseg,
                               cudaStream_t st);

// peer-memory exchange helpers (qsgd.cu)
cudaError_t launch_p2p_signal(const P2PDev* p, int stage, unsigned epoch, cudaStream_t st);
cudaError_t launch_p2p_wait(const unsigned* my_flags, int W, int me, int stage, unsigned epoch, cudaStream_t st);
cudaError_t launch_p2p_push(const P2PDev* p, const uint8_t* src, int64_t b0, int64_t b1, cudaStream_t st);
cudaError_t launch_p2p_plan(const P2PDev* p, const unsigned* my_flags, int W, int me, unsigned epoch, int32_t* choice,
                            int L, cudaStream_t st);
// device-side layout of a plan (W > 1 without a host round trip): DevPlan per layer
// (payload offsets, R7) and the shard bounds (R13) into p->bb / p->rb
cudaError_t launch_plan_qsgd_layout(const int32_t* choice, const int32_t* params, int K, const DevLayer* layers,
                                    const int64_t* bucket0, int L, int64_t R, int B, DevPlan* plan, P2PDev* p,
                                    unsigned* flag, cudaStream_t st);

// Algorithm 1 DP (dp.cu)
struct SolveArgs {
  const double* err; const int64_t* bits; int L; int K;
  const int32_t* default_idx; const int32_t* compress; int D; uint32_t flags;
  int32_t* choice; lgreco_solve_info* info;
  uint8_t* pd; int32_t* act;  // workspace: L*(D+1) bytes, L ints
};
size_t solve_workspace_bytes(int L, int K, int D);
cudaError_t launch_weight_costs(const int64_t* bits, const int64_t* w, int L, int K, int64_t* out, cudaStream_t st);
cudaError_t launch_solve(const SolveArgs& a, void* workspace, cudaStream_t st);

}  // namespace lg
