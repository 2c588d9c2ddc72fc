// Diagnostic microbenchmark (not part of the product): per-SM issue throughput of
// the fp32 instruction forms the QSGD profile kernel is built from, scalar vs the
// packed f32x2 forms of sm_100a.  One CTA per SM, 8..32 warps, long dependent-free
// chains; prints warp-instructions per cycle per SM.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/ubench_pipes scripts/ubench_pipes.cu
#include <cstdio>
#include <cstdint>

#define N_ITER 4096
typedef unsigned long long u64;

template <int OP>
__global__ void kern(float* out, long long* cyc, float seed) {
  float a[8];
  u64 p[8];
  for (int i = 0; i < 8; ++i) {
    a[i] = seed + threadIdx.x * 0.001f + i;
    float lo = a[i], hi = a[i] + 1.f;
    asm volatile("mov.b64 %0, {%1,%2};" : "=l"(p[i]) : "f"(lo), "f"(hi));
  }
  const float b = 1.0001f + threadIdx.x * 1e-9f, c = 0.5f + threadIdx.x * 1e-9f;
  u64 bp, cp;
  asm volatile("mov.b64 %0, {%1,%2};" : "=l"(bp) : "f"(b), "f"(b));
  asm volatile("mov.b64 %0, {%1,%2};" : "=l"(cp) : "f"(c), "f"(c));
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
      if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(bp), "l"(cp));
      if (OP == 2) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
      if (OP == 3) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(bp));
      if (OP == 4) asm volatile("min.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
      if (OP == 5) asm volatile("add.rm.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(bp));
      if (OP == 6) {  // mixed: fma pipe + alu pipe
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
        asm volatile("min.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
      }
      if (OP == 7) {  // setp + selp
        float r;
        asm volatile("{.reg .pred q; setp.lt.f32 q, %1, %2; selp.f32 %0, %1, %2, q;}" : "=f"(r) : "f"(a[i]), "f"(b));
        a[i] = r;
      }
      if (OP == 8) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i) {
    float lo, hi;
    asm volatile("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[i]));
    s += a[i] + lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps, int ipl) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  kern<OP><<<148, warps * 32>>>(out, cyc, 1.f);
  kern<OP><<<148, warps * 32>>>(out, cyc, 1.f);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double instr = (double)warps * N_ITER * 8 * ipl;
  printf("%-22s warps=%2d  warp-instr/clk/SM = %.3f\n", name, warps, instr / (double)h[0]);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {8, 16, 32}) {
    run<0>("FFMA", w, 1);
    run<1>("FFMA2 (f32x2)", w, 1);
    run<2>("FADD", w, 1);
    run<3>("FADD2 (f32x2)", w, 1);
    run<5>("FADD2.RM (f32x2)", w, 1);
    run<8>("FMUL", w, 1);
    run<4>("FMNMX", w, 1);
    run<6>("FFMA+FMNMX", w, 2);
    run<7>("FSETP+FSEL", w, 2);
  }
  return 0;
}
