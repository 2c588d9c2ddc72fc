/*
 * lgreco.h -- C ABI of the B200-native L-GreCo data-parallel hot path.
 *
 * L-GreCo (Alimohammadi, Markov, Frantar, Alistarh, MLSys'23, arXiv 2210.17357)
 * chooses one compression parameter per layer by (1) profiling the L2 error of
 * every candidate on every layer, (2) solving the knapsack DP of Algorithm 1 and
 * (3) compressing + exchanging the gradient with the chosen parameters.
 * Citations: PAPER.md = the paper's text; DESIGN.md lists readings R1..R21 for
 * every point the paper leaves open.
 *
 * Conventions (all entry points):
 *  - Return value: LGRECO_OK (0) or a negative status; no exception crosses the
 *    ABI.  lgreco_last_error() returns a thread-local message for the last error.
 *  - Pointers prefixed d_ are DEVICE pointers (cuda:current), h_ are HOST pointers.
 *    The caller owns every buffer it passes; the library never frees them.
 *  - `stream` is a cudaStream_t passed as void*.  All device work is enqueued on
 *    it, asynchronously, unless stated otherwise.  No entry point allocates device
 *    memory except lgreco_ctx_create.
 *  - Flat gradient layout: one contiguous fp32 vector of N elements; layer l owns
 *    [offset, offset+numel) (DDP-style flattening).
 *  - Non-finite gradient values (PAPER.md is silent) set a sticky
 *    device flag read by lgreco_ctx_check(); non-finite error tables make
 *    lgreco_solve report LGRECO_ENONFINITE in info->status.
 */
#ifndef LGRECO_H
#define LGRECO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LGRECO_OK 0
#define LGRECO_EINVAL (-1)      /* bad argument (layer table, K, params, D ...) */
#define LGRECO_ENONFINITE (-2)  /* NaN/Inf in the gradient or in the error table */
#define LGRECO_EINFEASIBLE (-3) /* reserved: the solve falls back to the defaults instead */
#define LGRECO_ECUDA (-4)       /* a CUDA runtime call failed */
#define LGRECO_ENCCL (-5)       /* an NCCL call failed */
#define LGRECO_ENOMEM (-6)      /* allocation failed (ctx_create only) */
#define LGRECO_EUNSUPPORTED (-7)

/* compressor families */
#define LGRECO_QSGD 0     /* bucketed min/max stochastic quantisation, params = bits 1..16 */
#define LGRECO_TOPK 1     /* per-layer TopK, params = density in ppm (1..1e6) */
#define LGRECO_POWERSGD 2 /* PowerSGD rank-r, params = rank >= 1 */

/* lgreco_solve flags (R1, R16) */
#define LGRECO_METRIC_SQ 1u   /* use squared L2 instead of L2 (PAPER.md:180 vs :183) */
#define LGRECO_DISC_FLOOR 2u  /* floor discretisation instead of ceil */
#define LGRECO_SOLVE_SINGLE_CTA 4u  /* run Algorithm 1 on one CTA (no 8-SM cluster); same result */
#define LGRECO_SOLVE_NARROW 8u  /* clusters of 8 CTAs instead of 16 (fewer SMs for longer): for a
                                   solve that runs beside other work, e.g. next to the fused pass of
                                   the pipelined schedule (lgreco_profile_compress); same result */

/* One layer of the flat gradient.  rows*cols == numel for matrices (the view is
 * (shape[0], numel/shape[0])); rows == 0 marks a vector.  compress == 0 sends the
 * layer lossless (raw fp32) and excludes it from the DP (R8). */
typedef struct {
    int64_t offset, numel;
    int32_t rows, cols, compress;
} lgreco_layer;

/* Candidate set C = {c^1..c^K} (Alg.1 input), ascending fidelity. */
typedef struct {
    int32_t family;        /* LGRECO_QSGD | LGRECO_TOPK | LGRECO_POWERSGD */
    int32_t K;             /* number of candidates, 1..255 */
    const int32_t* params; /* HOST array of K parameters */
    int32_t qbucket;       /* QSGD bucket size B, a multiple of 128 (<= 8192) */
    int32_t power_steps;   /* PowerSGD power steps for the profile (5) */
    uint64_t seed;         /* Philox key (R3) */
} lgreco_candidates;

/* Result summary of lgreco_solve (device-resident struct). */
typedef struct {
    double emax;          /* Emax = sum_l metric(err[l][default_l])  (Alg.1 line 2) */
    double total_err;     /* sum_l metric(err[l][choice_l]) of the returned plan */
    int64_t total_bits;   /* sum_l bits[l][choice_l] */
    int64_t default_bits; /* sum_l bits[l][default_l] */
    int32_t used_default; /* 1 if the defaults were returned (R20) */
    int32_t n_active;     /* layers with compress != 0 */
    int32_t status;       /* LGRECO_OK or LGRECO_ENONFINITE / LGRECO_EINVAL */
    int32_t pad;
} lgreco_solve_info;

typedef struct lgreco_ctx lgreco_ctx;

const char* lgreco_last_error(void);
int32_t lgreco_version(void);

/* Writes a fresh 128-byte ncclUniqueId into h_out (rank 0 calls this and
 * broadcasts the bytes over its own process group). */
int lgreco_nccl_unique_id(void* h_out);

/* Create a context for one rank of a `world`-rank data-parallel group.
 * layers: HOST array of L layers (ascending, non-overlapping); cand: candidate set.
 * nccl_unique_id: HOST 128 bytes (ignored when world == 1).  Allocates every
 * workspace the hot calls need and, for world > 1, an NCCL communicator on the
 * current device.  Owns PowerSGD warm-start state. */
int lgreco_ctx_create(lgreco_ctx** out, const lgreco_layer* layers, int32_t L,
                      const lgreco_candidates* cand, int32_t rank, int32_t world,
                      const void* nccl_unique_id, void* stream);
void lgreco_ctx_destroy(lgreco_ctx* ctx);

/* Synchronises `stream` and returns LGRECO_EINVAL if a device-plan entry point
 * (lgreco_compress_allreduce_dev) met a choice outside [0, K) for a compressed
 * layer (it used candidate 0 there), else LGRECO_ENONFINITE if any kernel saw a
 * non-finite gradient value since the last check; either clears the flags. */
int lgreco_ctx_check(lgreco_ctx* ctx, void* stream);

/* Number of kernels this ctx has launched (evidence counter). */
int64_t lgreco_ctx_launches(lgreco_ctx* ctx);

/* Measurement hook (bench.py roofline): while enabled (enable != 0), every
 * lgreco_profile call of a QSGD ctx records a CUDA event pair on its stream
 * immediately around the K1 launch (k_qprofile, the dominant kernel).  Costs one
 * event pair per call; off by default.  Returns LGRECO_EINVAL for a null ctx. */
int lgreco_ctx_timing(lgreco_ctx* ctx, int32_t enable);

/* Synchronises the recorded event pairs, writes their summed elapsed time (ms) to
 * *total_ms and their number to *count, then releases them.  LGRECO_ECUDA if an
 * event failed (the sum then covers the others). */
int lgreco_ctx_kernel_ms(lgreco_ctx* ctx, double* total_ms, int64_t* count);

/* (a1) Paper-mode accumulation ("we accumulate per-layer gradients in
 * auxiliary buffers", :318): d_G[i] = fl32(d_G[i] + d_g[i]) for i < n, one IEEE fp32
 * round-to-nearest add per element, enqueued on `stream` (kernel K0).  Between replans the
 * caller accumulates every step's local gradient into G and profiles G with d_ef = NULL.
 * d_G (in/out) and d_g are DEVICE pointers, 4-byte aligned (128-bit path when both share
 * their alignment mod 16); n = 0 is a no-op.  LGRECO_EINVAL on a negative n, null or
 * misaligned pointers; LGRECO_ECUDA if the launch fails. */
int lgreco_accumulate(float* d_G, const float* d_g, int64_t n, void* stream);

/* (a2-a4) Profile: for every layer l and candidate j, d_err[l*K+j] = the L2 norm of
 * x_l - decompress(compress(x_l, c^j)) and d_bits[l*K+j] = its transmitted size in
 * bits ("simulate the compression/decompression ... without
 * applying error feedback").  x = d_g + d_ef (d_ef nullable: x = d_g, the paper's
 * accumulated-gradient mode).  The EF buffer is read, never written.  `step`
 * selects the Philox counter (QSGD: the same uniforms the compress call of this
 * step draws, R6).  Lossless layers: err 0, bits 32*numel.
 * d_err: L*K doubles, d_bits: L*K int64, row-major by layer.  QSGD accepts any 4-byte
 * aligned d_g / d_ef; TopK and PowerSGD need 16-byte aligned base pointers (EINVAL). */
int lgreco_profile(lgreco_ctx* ctx, const float* d_g, const float* d_ef, uint64_t step,
                   double* d_err, int64_t* d_bits, void* stream);

/* (a4, NEXT-2) PowerSGD profile by singular values: for every layer l
 * and candidate rank r, d_err[l*K+j] = sqrt(sum_{i > r} sigma_i^2) of the m x k view of
 * x = d_g + d_ef (the optimal rank-r error, Eckart-Young), d_bits as lgreco_profile
 * (32 r (m + k), or 32 numel for lossless candidates / layers).  Squared singular
 * values = eigenvalues of the fp64 Gram matrix of the smaller side (the library's own
 * solver: Householder tridiagonalisation + Sturm bisection, one CTA per matrix, every
 * matrix of the table at once); the paper's choice when the rank range is large.
 * PowerSGD ctx only (LGRECO_EUNSUPPORTED otherwise, or when a matrix has min(m, k) > 4096);
 * synchronises the stream only when its workspace grows.  d_g / d_ef 4-byte aligned;
 * d_err L*K doubles, d_bits L*K int64. */
/* (NEXT-2) The PowerSGD profile method lgreco_profile uses ("the best
 * of both worlds": power steps when the rank range is small, singular values when it is
 * large).  LGRECO_PSGD_POWER (the default: R11), LGRECO_PSGD_SVD (= lgreco_psgd_profile_svd),
 * LGRECO_PSGD_AUTO: the cheaper of the two by a cost model resolved once per ctx on the
 * host -- power sum_l steps * m k r_max(l) x 1.9e-13 s (one r_max run covers every rank:
 * the pinned prefix property, so O(m k r_max) and not the paper's O(m k r_max^2)), + 3e-5 s
 * of launch latency per power step, against SVD sum_l (m k n x 1e-13 + n^3 x
 * 2.2e-12) + n_max x 2e-6 s, n = min(m, k) (the fp64 Gram + the eigensolver's traffic and
 * step latency), constants measured on B200 (R22).  lgreco_psgd_method returns
 * the resolved method (POWER or SVD).  EINVAL on a bad method / non-PowerSGD ctx. */
enum { LGRECO_PSGD_POWER = 0, LGRECO_PSGD_SVD = 1, LGRECO_PSGD_AUTO = 2 };
int lgreco_psgd_set_method(lgreco_ctx* ctx, int32_t method);
int lgreco_psgd_method(lgreco_ctx* ctx);
int lgreco_psgd_profile_svd(lgreco_ctx* ctx, const float* d_g, const float* d_ef, double* d_err,
                            int64_t* d_bits, void* stream);

/* Device workspace bytes lgreco_solve needs for (L, K, D). */
size_t lgreco_solve_workspace_bytes(int32_t L, int32_t K, int32_t D);

/* (a5-a6) Algorithm 1: Emax from the defaults, discretise
 * errors into D bins of Emax/D (ceil, R16), minimise sum bits s.t. sum disc <= D
 * by DP over layers, argmin + backtrack; falls back to the defaults when the plan
 * is not strictly within bits and raw error (R20).  All pointers are DEVICE:
 * d_err/d_bits L*K (from lgreco_profile or any table), d_default_idx L,
 * d_compress L (nullable: all active), d_choice L (out; -1 for inactive layers),
 * d_info (out), d_workspace of lgreco_solve_workspace_bytes(L,K,D) bytes.
 * Host mode: when d_err, d_bits, d_default_idx, d_compress (if given), d_choice and d_info
 * are all HOST pointers, they are staged through device scratch around the same kernels
 * (d_workspace ignored, may be NULL) and the call returns after the plan and the info are
 * back on the host (stream-synchronous); mixing host and device pointers is EINVAL.
 * Cluster (or single-CTA) DP on `stream`, launched after ALL prior work of the stream has
 * completed (no programmatic overlap on its start); it lets its successor be scheduled
 * once it runs (a compress reading d_choice still waits for it); no host synchronisation. */
int lgreco_solve(const double* d_err, const int64_t* d_bits, int32_t L, int32_t K,
                 const int32_t* d_default_idx, const int32_t* d_compress, int32_t D,
                 uint32_t flags, int32_t* d_choice, lgreco_solve_info* d_info,
                 void* d_workspace, size_t workspace_bytes, void* stream);

/* Weighted objective ("minimize sum size(l, c^l) *
 * T(l)" and PAPER.md:680-682 bucket priorities "multiplying the size of each layer by the
 * index of the bucket"): d_out[l*K + c] = d_bits[l*K + c] * d_weight[l] (int64, exact) for
 * lgreco_solve to minimise.  A negative weight or a product that overflows int64 writes
 * -1 (lgreco_solve then reports LGRECO_EINVAL).  Real-valued coefficients T(l) are
 * quantised by the caller (paper_2210_17357_b200/objectives.py).  All pointers DEVICE:
 * d_bits, d_out L*K, d_weight L; d_out may alias d_bits. */
int lgreco_weight_costs(const int64_t* d_bits, const int64_t* d_weight, int32_t L, int32_t K,
                        int64_t* d_out, void* stream);

/* Per-layer gradient norms (the Accordion-style default schedule,
 * PAPER.md:596 "used these parameters as the default set of parameters in L-GreCo"):
 * d_norm[l] = sqrt(sum_i x_i^2) over layer l of x = d_g (+ d_ef, nullable), fp64,
 * fixed-order (deterministic).  d_norm: L doubles (DEVICE). */
int lgreco_layer_norms(lgreco_ctx* ctx, const float* d_g, const float* d_ef, double* d_norm, void* stream);

/* (a7) Plan agreement: broadcast d_choice (L int32) from rank 0.
 * No-op when world == 1; NCCL broadcast, or over peer memory for a ctx set up with
 * lgreco_p2p_open / _set_peers (rank 0 stores its plan into every peer's flag area and
 * releases an epoch word the others acquire). */
int lgreco_plan_broadcast(lgreco_ctx* ctx, int32_t* d_choice, void* stream);

/* (a8-a10) Compress with the plan h_choice (HOST, L candidate indices; ignored for
 * lossless layers), update error feedback and exchange: d_out (N fp32) receives the
 * mean over ranks of the decompressed gradients, identical on every rank.
 * x = d_g + d_ef; d_ef <- x - decompress_stage1(x) (d_ef nullable: no EF).
 * QSGD: pack -> all-to-all of byte-balanced bucket shards -> ordered dequantise-
 * sum-requantise on the owner -> all-gather -> decode (R13).  TopK: select ->
 * all-gather (idx,val) -> ordered sparse sum (R10).  PowerSGD: P=MQ, all-reduce,
 * orthogonalise, Q=M^T P, all-reduce, out = P Q^T (R12).  d_g, d_ef and d_out must be
 * 16-byte aligned (cudaMalloc / torch allocations are); LGRECO_EINVAL otherwise. */
int lgreco_compress_allreduce(lgreco_ctx* ctx, const int32_t* h_choice, const float* d_g,
                              float* d_ef, float* d_out, uint64_t step, void* stream);

/* Same as lgreco_compress_allreduce with the plan in DEVICE memory (d_choice, e.g. the
 * lgreco_solve output).  For world == 1 QSGD / TopK the plan is consumed on the device
 * (no host synchronisation: profile -> solve -> compress is one asynchronous stream
 * sequence and can be captured in a CUDA graph); otherwise the plan is copied to the
 * host (stream synchronisation) because the exchange sizes depend on it. */
int lgreco_compress_allreduce_dev(lgreco_ctx* ctx, const int32_t* d_choice, const float* d_g, float* d_ef,
                                  float* d_out, uint64_t step, void* stream);

/* (a2 + a8, fused) The per-step pass of the paper's schedule (the
 * plan in force -- chosen by a preceding solve -- compresses the step, while the profile
 * of the same step feeds the next solve).  Defined as, and bit-identical to,
 *   lgreco_profile(ctx, d_g, d_ef, step, d_err, d_bits, stream);
 *   lgreco_compress_allreduce_dev(ctx, d_choice, d_g, d_ef, d_out, step, stream);
 * i.e. d_err / d_bits profile x = d_g + d_ef (the EF as it was on entry) and d_choice
 * (DEVICE, L) compresses the same x (d_ef <- x - decompress(x), d_out <- the mean).  For a
 * QSGD ctx with B = 128 this is ONE pass over d_g and d_ef (kernel K1 with the compress of
 * K5 fused: the planned candidate's code comes from the same registers and Philox
 * uniforms, then K1b) -- at world == 1 writing the decoded output, at world > 1 over peer
 * memory (lgreco_p2p_open / _set_peers) storing the stage-1 records straight into their
 * owners' windows, followed by the peer-memory exchange of lgreco_compress_allreduce_dev;
 * otherwise (NCCL exchange, B > 128, d_ef = NULL, other families) the two calls.  d_choice must not alias the
 * output of a solve that reads d_err.  flags: LGRECO_PC_CONCURRENT -- the caller asserts
 * that the kernel enqueued immediately before this call on `stream` (typically the
 * lgreco_solve of the previous step, writing a plan other than d_choice) produces nothing
 * this call reads -- in particular d_err / d_bits must not be the tables that solve reads
 * (alternate two pairs) and d_choice not the plan it writes; the fused kernel may then
 * run beside it on the SMs it leaves free.  (lgreco_solve is a plain launch: it waits for
 * all prior work of the stream, the previous solve included.)  d_g, d_ef, d_out 16-byte
 * aligned (EINVAL otherwise); d_err L*K doubles, d_bits L*K int64. */
#define LGRECO_PC_CONCURRENT 1u
int lgreco_profile_compress(lgreco_ctx* ctx, const int32_t* d_choice, const float* d_g, float* d_ef, float* d_out,
                            uint64_t step, double* d_err, int64_t* d_bits, uint32_t flags, void* stream);

/* ---- NEXT-4: mixed-family plans ("combining different compression
 * techniques inside the same model") ------------------------------------------------
 * A hybrid plan picks, per layer, a (family, parameter) column of a table that holds F
 * families' candidate lists side by side; one ctx per family (same layer table) compresses
 * the layers whose column is its own.  LGRECO_CHOICE_SKIP in a ctx's choice vector marks
 * a compressed layer that another family's ctx owns: that ctx leaves the layer's EF and
 * output untouched (world == 1 device paths of QSGD and TopK; PowerSGD's host path at
 * any world size); on a layer sent lossless (compress == 0) it marks a ctx that must not
 * handle it either (lgreco_hybrid_split leaves those to family 0 alone: a second raw pass
 * would read the EF the first one already zeroed).
 * lgreco_hybrid_table: err_out[l][c0_f + j] = err_f[l][j] (likewise bits) for the F
 *   family tables (DEVICE pointers, L x K_f row-major; h_K: HOST K_f), c0_f the prefix
 *   sum of K.  lgreco_hybrid_split: d_choice (L, a column of that table or -1) -> F
 *   per-family vectors d_choice_f[f] (f's own index, LGRECO_CHOICE_SKIP for a column of
 *   another family; -1 (lossless) kept for family 0, LGRECO_CHOICE_SKIP for the others).  Both enqueued on `stream`; EINVAL on bad sizes. */
#define LGRECO_CHOICE_SKIP (-2)
int lgreco_hybrid_table(const double* const* h_err_f, const int64_t* const* h_bits_f, const int32_t* h_K, int32_t F,
                        int32_t L, double* d_err_out, int64_t* d_bits_out, void* stream);
int lgreco_hybrid_split(const int32_t* d_choice, const int32_t* h_K, int32_t F, int32_t L, int32_t* const* h_choice_f,
                        void* stream);

/* ---- peer-memory exchange (QSGD, 1 < world <= 8, no NCCL on the data path) ----------
 * A QSGD ctx created with world > 1 and nccl_unique_id == NULL exchanges through the
 * peers' device memory (NVLink P2P stores; R13 unchanged: same shards, same sums, same
 * bytes): K5 stores every stage-1 record straight into its owner's receive window, a
 * system-scope release of a per-(stage, sender) epoch word tells the owner, the owner
 * reduces (K8) and stores its stage-2 shard into every peer's stage-2 payload, K9
 * decodes after the second epoch.  Setup: lgreco_p2p_export (3 CUDA IPC handles, 192
 * bytes) on every rank, all-gather the blobs over the process group, lgreco_p2p_open
 * (W x 192 bytes, rank order); or, for ranks simulated in one process,
 * lgreco_p2p_local + lgreco_p2p_set_peers.  lgreco_compress_allreduce then runs the
 * three stages (lgreco_p2p_stage 1, 2, 3) -- or, from lgreco_compress_allreduce_dev,
 * the whole step with the plan laid out on the device (no host synchronisation); every
 * rank must call it the same number of times (the epoch) with the same plan (use
 * lgreco_plan_broadcast).  Errors: LGRECO_EINVAL for other families / ctxs without the
 * buffers, LGRECO_ECUDA when an IPC handle cannot be opened. */
int lgreco_p2p_local(lgreco_ctx* ctx, void** h_ptrs3 /* out: recv window, stage-2 payload, flags */);
int lgreco_p2p_export(lgreco_ctx* ctx, void* h_blob /* out: 3 cudaIpcMemHandle_t */);
int lgreco_p2p_open(lgreco_ctx* ctx, const void* h_blobs /* world x 3 handles, rank order */);
int lgreco_p2p_set_peers(lgreco_ctx* ctx, void* const* h_recv, void* const* h_stage2, void* const* h_flags);
int lgreco_p2p_stage(lgreco_ctx* ctx, const int32_t* h_choice, const float* d_g, float* d_ef, float* d_out,
                     uint64_t step, int32_t stage /* 1, 2, 3 */, void* stream);

/* ---- stage entry points (the steps lgreco_compress_allreduce composes; used by
 * ---- the parity tests to simulate W ranks on one GPU) ------------------------ */

/* Payload bytes S of the packed stage-1 gradient under plan h_choice. */
int64_t lgreco_payload_bytes(lgreco_ctx* ctx, const int32_t* h_choice);

/* Record (bucket) bounds and byte bounds of the W byte-balanced shards (R13):
 * h_rec_bounds, h_byte_bounds: W+1 int64 each. */
int lgreco_shard_bounds(lgreco_ctx* ctx, const int32_t* h_choice, int32_t W,
                        int64_t* h_rec_bounds, int64_t* h_byte_bounds);

/* Host-only (no device, no ctx): payload bytes S of plan h_choice and, for QSGD,
 * the W byte-balanced shard bounds (R13) -- every rank computes the same bounds.
 * TopK/PowerSGD: S = bytes of the pair arrays / raw layers; bounds (0..0, S). */
int lgreco_plan_layout(const lgreco_layer* layers, int32_t L, const lgreco_candidates* cand,
                       const int32_t* h_choice, int32_t W, int64_t* h_S, int64_t* h_rec_bounds,
                       int64_t* h_byte_bounds);

/* QSGD stage 1 (K5): pack x = d_g + d_ef for rank field `rank` into d_payload
 * (S bytes, record layout R7), update d_ef (nullable), write decoded values to
 * d_dec (nullable). */
int lgreco_qsgd_pack(lgreco_ctx* ctx, const int32_t* h_choice, const float* d_g, float* d_ef,
                     uint8_t* d_payload, float* d_dec, uint32_t rank, uint64_t step, void* stream);

/* QSGD owner reduce (K8): records [rec_begin, rec_end) (one shard).  d_recv holds W
 * copies of that shard's stage-1 bytes, rank-major (W * shard_bytes); writes the
 * stage-2 records to d_stage2 + (byte offset of rec_begin). */
int lgreco_qsgd_reduce(lgreco_ctx* ctx, const int32_t* h_choice, int32_t W, int64_t rec_begin,
                       int64_t rec_end, const uint8_t* d_recv, uint8_t* d_stage2, uint64_t step,
                       void* stream);

/* QSGD decode (K9): d_payload (S bytes) -> d_out (N fp32). */
int lgreco_qsgd_unpack(lgreco_ctx* ctx, const int32_t* h_choice, const uint8_t* d_payload,
                       float* d_out, void* stream);

/* TopK stage 1 (K2 select with the chosen densities + K6 compaction): pairs
 * (u32 idx, f32 val) ascending per layer into d_payload (S bytes, nullable), e' into
 * d_ef (nullable), the decoded values (kept at idx, 0 elsewhere) into d_out (nullable). */
int lgreco_topk_pack(lgreco_ctx* ctx, const int32_t* h_choice, const float* d_g, float* d_ef,
                     uint8_t* d_payload, float* d_out, void* stream);

/* TopK exchange combine (K10): d_gathered = W payloads of S bytes, rank-major (the
 * all-gather result); d_out <- ordered mean over ranks (R10). */
int lgreco_topk_combine(lgreco_ctx* ctx, const int32_t* h_choice, int32_t W, const uint8_t* d_gathered,
                        float* d_out, void* stream);

/* PowerSGD stages (K7, R12).  Factor buffers use per-layer slots sized for the
 * largest candidate rank: P slots hold m x r (column-major) per compressed matrix
 * layer, Q slots k x r; lgreco_psgd_sizes returns the slot-area sizes (elements). */
int lgreco_psgd_sizes(lgreco_ctx* ctx, int64_t* h_p_elems, int64_t* h_q_elems);
/* The ctx's current PowerSGD factors (R12), for inspection / parity tests: d_Phat (P elems)
 * <- Phat = orthonormalise(Psum / W) of the last lgreco_psgd_q (or compress) call, d_Q
 * (Q elems) <- the warm-start Q = Qsum / W of the last lgreco_psgd_out (or compress) call.
 * Slot layout: compressed matrix layers in layer order, each owning rows*rmax (P) and
 * cols*rmax (Q) elements, rmax = the largest candidate rank that is not lossless for the
 * layer (0: none); the current rank-r factor is stored column-major (m x r, k x r) at the
 * slot start.  Either pointer nullable.  Enqueued on `stream`. */
int lgreco_psgd_factors(lgreco_ctx* ctx, float* d_Phat, float* d_Q, void* stream);
/* P_w = M_w Q_ws (Q_ws re-initialised from Philox stream 2 at `step` where the rank
 * changed) into d_P. */
int lgreco_psgd_p(lgreco_ctx* ctx, const int32_t* h_choice, const float* d_g, const float* d_ef, float* d_P,
                  uint64_t step, void* stream);
/* Phat = orthonormalise(d_Psum / W) (kept in ctx); Q_w = M_w^T Phat into d_Q. */
int lgreco_psgd_q(lgreco_ctx* ctx, const int32_t* h_choice, const float* d_g, const float* d_ef,
                  const float* d_Psum, int32_t W, float* d_Q, void* stream);
/* Q_ws = d_Qsum / W; d_out = Phat Q_ws^T (matrix layers); d_ef <- x - d_out. */
int lgreco_psgd_out(lgreco_ctx* ctx, const int32_t* h_choice, const float* d_g, float* d_ef,
                    const float* d_Qsum, int32_t W, float* d_out, void* stream);
/* Raw layers (vectors, lossless-equivalent ranks): payload = x (S = lgreco_payload_bytes),
 * e' = 0, d_out = x (nullable each); combine: d_out = ordered mean of W raw payloads. */
int lgreco_psgd_raw_pack(lgreco_ctx* ctx, const int32_t* h_choice, const float* d_g, float* d_ef,
                         uint8_t* d_payload, float* d_out, void* stream);
int lgreco_psgd_raw_combine(lgreco_ctx* ctx, const int32_t* h_choice, int32_t W, const uint8_t* d_gathered,
                            float* d_out, void* stream);

/* Debug: P = M Q through the tcgen05 kind::tf32 (3xTF32) path for one matrix:
 * M = d_g + d_e (m x k row-major, d_e nullable), d_Q k x r column-major (r <= 64),
 * d_P m x r column-major.  Synchronises `stream`. */
int lgreco_debug_tc_mq(const float* d_g, const float* d_e, int64_t m, int32_t k, const float* d_Q, int32_t r,
                       float* d_P, void* stream);

/* Debug: Q = M^T P through the tcgen05 path (A operand MN-major): d_P m x r and d_Q
 * k x r column-major.  Synchronises `stream`. */
int lgreco_debug_tc_mtp(const float* d_g, const float* d_e, int64_t m, int32_t k, const float* d_P, int32_t r,
                        float* d_Q, void* stream);

/* Debug: Philox4x32-10 of n counters (d_ctr: n*4 u32, key) -> d_out n*4 u32. */
int lgreco_debug_philox(const uint32_t* d_ctr, uint32_t key0, uint32_t key1, int64_t n,
                        uint32_t* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LGRECO_H */
