// Latency of primitives used by the reductions: dependent DFMA, LDS.64, warp_sum(double), DADD.
#include <cstdio>
#include "common.cuh"
__global__ void lb(double* out, long long* cyc, double a) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i * 1e-3;
  __syncthreads();
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < 100; ++i) x = fma(x, a, 1e-9);
  long long t1 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < 100; ++i) { double v = s[idx]; idx = (int)(v * 1e-9) + ((idx + 33) & 1023); }
  long long t2 = clock64();
  double y = x;
  for (int i = 0; i < 20; ++i) y = warp_sum(y) * 1e-3;
  long long t3 = clock64();
  double z = x;
  for (int i = 0; i < 100; ++i) z = z + a;
  long long t4 = clock64();
  float f = x;
  for (int i = 0; i < 20; ++i) { f += __shfl_xor_sync(0xffffffffu, f, 1); }
  long long t5 = clock64();
  double q = x;
  for (int i = 0; i < 20; ++i) q = sqrt(q + 1.0);
  long long t6 = clock64();
  double d = x + 2.0;
  for (int i = 0; i < 20; ++i) d = 1.0 / d + 1.0;
  long long t7 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 100; cyc[1] = (t2 - t1) / 100; cyc[2] = (t3 - t2) / 20; cyc[3] = (t4 - t3) / 100;
    cyc[4] = (t5 - t4) / 20; cyc[5] = (t6 - t5) / 20; cyc[6] = (t7 - t6) / 20;
  }
  out[threadIdx.x] = x + idx + y + z + f + q + d;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8192); cudaMalloc(&c, 64);
  for (int th : {32, 256, 1024}) {
    for (int r = 0; r < 2; ++r) lb<<<1, th>>>(o, c, 1.0000001);
    long long h[7]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("threads %4d: dfma %lld  lds64 %lld  warp_sum(f64) %lld  dadd %lld  shfl(f32)+fadd %lld  sqrt %lld  rcp+add %lld cycles\n",
           th, h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
  }
  return 0;
}
