// Micro-benchmark of the shared-memory Householder primitive (hh_factor) on an m x R panel:
// per-phase cycle counts of warp 0 to find the critical path.  nvcc -arch=sm_100a -O3 -I../../paper_2112_10855_b200/csrc
#include <cstdio>
#include <cstdlib>
#include "qr_kernels.cuh"
using namespace cpqr;

__global__ void bench(const double* A, int m, int R, long long* cyc, double* out) {
  extern __shared__ double sm[];
  __shared__ double tau[64], beta[64], w[64], np[64];
  for (int e = threadIdx.x; e < m * R; e += blockDim.x) sm[e] = A[e];
  __syncthreads();
  long long t0 = clock64();
  DenseCols M{sm, m, m};
  hh_factor(M, R, tau, beta, w, np);
  long long t1 = clock64();
  hh_formq(M, R, tau, w);
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  for (int e = threadIdx.x; e < m * R; e += blockDim.x) out[e] = sm[e];
}

int main() {
  int ms[] = {128, 256, 1024};
  int Rs[] = {8, 16, 32};
  double *A, *out; long long* cyc;
  cudaMalloc(&A, 1024 * 32 * 8); cudaMalloc(&out, 1024 * 32 * 8); cudaMalloc(&cyc, 16);
  double* h = (double*)malloc(1024 * 32 * 8);
  for (int i = 0; i < 1024 * 32; ++i) h[i] = (double)rand() / RAND_MAX - 0.5;
  cudaMemcpy(A, h, 1024 * 32 * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int threads : {128, 256, 512, 1024})
    for (int mi = 0; mi < 3; ++mi)
      for (int ri = 0; ri < 3; ++ri) {
        int m = ms[mi], R = Rs[ri];
        if ((size_t)m * R * 8 > 200 * 1024) continue;
        for (int rep = 0; rep < 2; ++rep) bench<<<1, threads, m * R * 8>>>(A, m, R, cyc, out);
        long long hc[2];
        cudaMemcpy(hc, cyc, 16, cudaMemcpyDeviceToHost);
        printf("threads %4d m %5d R %2d  factor %8lld cyc (%6lld/col)  formq %8lld cyc (%6lld/col)\n", threads, m, R,
               hc[0], hc[0] / R, hc[1], hc[1] / R);
      }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
