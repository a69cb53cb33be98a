// Phase timing of one dorg2r-style column step (dots -> barrier -> update -> barrier) in shared memory.
#include <cstdio>
#include "qr_kernels.cuh"
using namespace cpqr;
__global__ void pb(double* A, int m, int R, long long* out) {
  extern __shared__ double sm[];
  __shared__ double w[64];
  __shared__ long long ts[64][6];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int e = tid; e < m * R; e += nt) sm[e] = A[e];
  __syncthreads();
  for (int j = R - 1; j >= 0; --j) {
    long long t0 = clock64();
    double* cj = sm + (size_t)m * j;
    for (int k = j + 1 + wid; k < R; k += nw) {
      const double* ck = sm + (size_t)m * k;
      double d0 = 0, d1 = 0, d2 = 0, d3 = 0;
      int i = j + 1 + lane;
      for (; i + 96 < m; i += 128) { d0 = fma(cj[i], ck[i], d0); d1 = fma(cj[i+32], ck[i+32], d1); d2 = fma(cj[i+64], ck[i+64], d2); d3 = fma(cj[i+96], ck[i+96], d3); }
      for (; i < m; i += 32) d0 = fma(cj[i], ck[i], d0);
      const double d = warp_sum((d0 + d1) + (d2 + d3));
      if (lane == 0) w[k] = 0.5 * (ck[j] + d);
    }
    long long t1 = clock64();
    __syncthreads();
    long long t2 = clock64();
    for (int i = tid; i < m; i += nt) {
      if (i >= j && j < R - 1) {
        const double vi = (i == j) ? 1.0 : cj[i];
#pragma unroll 8
        for (int k = j + 1; k < R; ++k) sm[i + (size_t)m * k] -= w[k] * vi;
      }
      cj[i] = (i < j) ? 0.0 : ((i == j) ? 0.5 : -0.5 * cj[i]);
    }
    long long t3 = clock64();
    __syncthreads();
    long long t4 = clock64();
    if (lane == 0 && j == R / 2) { ts[wid][0] = t0; ts[wid][1] = t1; ts[wid][2] = t2; ts[wid][3] = t3; ts[wid][4] = t4; }
  }
  __syncthreads();
  if (tid < nw) for (int q = 0; q < 5; ++q) out[tid * 5 + q] = ts[tid][q];
}
int main() {
  double* A; long long* o; cudaMalloc(&A, 256 * 32 * 8); cudaMemset(A, 0, 256 * 32 * 8); cudaMalloc(&o, 64 * 5 * 8);
  cudaFuncSetAttribute(pb, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int th : {256, 512}) {
    for (int r = 0; r < 2; ++r) pb<<<1, th, 256 * 32 * 8>>>(A, 256, 32, o);
    long long h[64 * 5]; cudaMemcpy(h, o, sizeof h, cudaMemcpyDeviceToHost);
    long long base = h[0];
    printf("threads %d (column j=16)\n", th);
    for (int w = 0; w < th / 32; ++w) printf(" warp %2d: start %6lld dots_end %6lld bar1 %6lld upd_end %6lld bar2 %6lld\n", w, h[w*5]-base, h[w*5+1]-base, h[w*5+2]-base, h[w*5+3]-base, h[w*5+4]-base);
  }
  return 0;
}
