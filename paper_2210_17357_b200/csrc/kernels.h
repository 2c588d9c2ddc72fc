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

struct CandS { float s[16]; };  // s_j = 2^{b_j} - 1, passed by value (constant bank)

struct QProfileArgs {
  const float* g; const float* e;
  const DevLayer* layers; int L;
  const ProfChunk* chunks; int nchunks; const int32_t* layer_chunk0;
  int B; CandS cs; const int32_t* params; int K;
  uint32_t k0, k1, rankfield, step;
  double* partial; double* err; int64_t* bits;
};

struct QPackArgs {
  const float* g; float* ef; uint8_t* payload; float* dec;
  const DevLayer* layers; const DevPlan* plan; const ProfChunk* chunks; int nchunks; int B;
  uint32_t k0, k1, rankfield, step; unsigned* flag;
};

struct QUnpackArgs {
  const uint8_t* payload; float* out;
  const DevLayer* layers; const DevPlan* plan; const ProfChunk* chunks; int nchunks; int B;
};

struct QReduceArgs {
  const uint8_t* recv; int64_t shard_bytes; int64_t byte0; uint8_t* stage2;
  const DevLayer* layers; const DevPlan* plan; const int64_t* bucket0; int L;
  int64_t r0, r1; int B; int W; uint32_t k0, k1, step;
};

cudaError_t launch_qprofile(const QProfileArgs& a, cudaStream_t st);
cudaError_t launch_qpack(const QPackArgs& a, cudaStream_t st);
cudaError_t launch_qunpack(const QUnpackArgs& a, cudaStream_t st);
cudaError_t launch_qreduce(const QReduceArgs& a, cudaStream_t st);
cudaError_t launch_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, int64_t n, uint32_t* out,
                          cudaStream_t st);

// Algorithm 1 DP (dp.cu)
struct SolveArgs {
  const double* err; const int64_t* bits; int L; int K;
  const int32_t* default_idx; const int32_t* compress; int D; uint32_t flags;
  int32_t* choice; lgreco_solve_info* info;
  uint8_t* pd; int32_t* act;  // workspace: L*(D+1) bytes, L ints
};
size_t solve_workspace_bytes(int L, int K, int D);
cudaError_t launch_solve(const SolveArgs& a, void* workspace, cudaStream_t st);

}  // namespace lg
