// Diagnostic microbenchmark (not part of the product): SM issue throughput of the K1
// candidate-element sequence and of its single instruction forms (reg vs immediate
// operands) on sm_100a.  One CTA per SM, W warps, 8 independent chains per thread.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/ubench_k1 scripts/ubench_k1.cu
#include <cstdio>

#define N_ITER 2048

template <int OP>
__global__ void kern(float* out, long long* cyc, float seed) {
  float a[8], acc[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed + threadIdx.x * 0.001f + i; acc[i] = 0.f; }
  const float b = 1.0001f + threadIdx.x * 1e-9f, c = 0.5f + threadIdx.x * 1e-9f, u = 0.25f + threadIdx.x * 1e-9f;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
      if (OP == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F800347, 0f3F000000;" : "+f"(a[i]));
      if (OP == 2) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
      if (OP == 3) asm volatile("add.rp.f32 %0, %0, 0f4B000001;" : "+f"(a[i]));
      if (OP == 4) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
      if (OP == 5) asm volatile("fma.rp.f32 %0, %1, 0fB3800000, %0;" : "+f"(a[i]) : "f"(u));
      if (OP == 6) {  // the K1 candidate-element sequence (8 instructions)
        float v, w, q, d, dec;
        asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(v) : "f"(a[i]), "f"(b));
        asm volatile("fma.rp.f32 %0, %1, 0fB3800000, %2;" : "=f"(w) : "f"(u), "f"(v));
        asm volatile("add.rp.f32 %0, %1, 0f4B000001;" : "=f"(q) : "f"(w));
        asm volatile("add.rn.f32 %0, %1, 0fCB000001;" : "=f"(q) : "f"(q));
        asm volatile("min.f32 %0, %1, 0f437F0000;" : "=f"(q) : "f"(q));
        asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(dec) : "f"(q), "f"(c), "f"(b));
        asm volatile("sub.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a[i]), "f"(dec));
        asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+f"(acc[i]) : "f"(d));
        asm volatile("add.rn.f32 %0, %0, 0f33800000;" : "+f"(a[i]));
      }
      if (OP == 7) asm volatile("min.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
      if (OP == 8) asm volatile("add.rn.f32 %0, %0, 0f3F800000;" : "+f"(a[i]));
      if (OP == 9) asm volatile("cvt.rpi.f32.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 10) {  // IMAD.WIDE.U32
        unsigned long long p;
        const unsigned x = __float_as_uint(a[i]);
        asm volatile("mul.wide.u32 %0, %1, 3528531795;" : "=l"(p) : "r"(x));
        a[i] = __uint_as_float((unsigned)p ^ (unsigned)(p >> 32));
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += a[i] + acc[i];
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
  printf("%-28s warps=%2d  warp-instr/clk/SM = %.3f\n", name, warps, instr / (double)h[0]);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {8, 24}) {
    run<0>("FFMA reg", w, 1);
    run<1>("FFMA imm", w, 1);
    run<2>("FADD reg", w, 1);
    run<3>("FADD.RP imm", w, 1);
    run<8>("FADD imm", w, 1);
    run<4>("FMUL reg", w, 1);
    run<5>("FFMA.RP reg,imm,reg", w, 1);
    run<7>("FMNMX", w, 1);
    run<9>("FRND.CEIL", w, 1);
    run<10>("IMAD.WIDE+LOP", w, 2);
    run<6>("K1 cand-elem seq (9 ops)", w, 9);
  }
  return 0;
}
