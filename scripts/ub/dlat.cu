// latency microbench: dependent chains of 64 DADD / FADD / DFMA (unrolled), clock64 per chain
#include <cstdio>
__global__ void k(double* out, const double* in, long long* t) {
  double a = in[0], b = in[1];
  float f = (float)in[3], fb = (float)in[1];
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) f = __fadd_rn(f, fb);
  long long t2 = clock64();
  double c = in[2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c = __ddiv_rn(c, b);
  long long t3 = clock64();
  out[0] = a + c + f; t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2;
}
int main() {
  double *o, *in; long long* t; cudaMallocManaged(&o, 64); cudaMallocManaged(&in, 64); cudaMallocManaged(&t, 64);
  in[0] = 1.0; in[1] = 1e-7; in[2] = 3.0; in[3] = 1.0;
  for (int r = 0; r < 3; ++r) { k<<<1, 1>>>(o, in, t); cudaDeviceSynchronize(); }
  printf("dadd %.1f fadd %.1f ddiv %.1f cycles/op\n", t[0] / 64.0, t[1] / 64.0, t[2] / 8.0);
}
