// Diagnostic microbenchmark (not part of the product): cost of one cluster barrier
// (barrier.cluster arrive.release + wait.acquire, and the relaxed arrive) vs
// __syncthreads, for clusters of 2/4/8 CTAs of 640 threads.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/ubench_cluster scripts/ubench_cluster.cu
#include <cstdio>
#define N_IT 2000
template <int MODE>
__global__ void kern(long long* out) {
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t0 = clock64();
  for (int i = 0; i < N_IT; ++i) {
    if (MODE == 0) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (MODE == 1) __syncthreads();
    if (MODE == 2) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    if (MODE == 3) {
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
template <int MODE>
void run(const char* name, int nc, int nt) {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = nc; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(nc); cfg.blockDim = dim3(nt); cfg.attrs = attr; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern<MODE>, d);
  cudaLaunchKernelEx(&cfg, kern<MODE>, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-34s nc=%d nt=%4d cycles/iter = %.1f (%s)\n", name, nc, nt, (double)h[0] / N_IT, cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  for (int nc : {2, 4, 8})
    for (int nt : {128, 640}) {
      run<0>("cluster arrive.release/wait.acquire", nc, nt);
      run<1>("__syncthreads", nc, nt);
      run<2>("cluster arrive.relaxed/wait", nc, nt);
      run<3>("fence.acq_rel.cluster + relaxed", nc, nt);
    }
  return 0;
}
