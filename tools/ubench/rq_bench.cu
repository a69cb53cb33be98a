// Cycles per column of the register-resident Householder (rowqr_factor / rowqr_formq) and of
// vec_reduce alone.
#include <cstdio>
#include <cstdlib>
#include "rowqr.cuh"
using namespace cpqr;
template <int RB>
__global__ void rb(const double* A, int m, int R, long long* cyc, double* out) {
  __shared__ double tau[RB], beta[RB], rowbuf[2 * RB], red[8 * RB], fin[2 * RB];
  const int row = threadIdx.x < m ? threadIdx.x : -1;
  double a[RB];
#pragma unroll
  for (int k = 0; k < RB; ++k) a[k] = (row >= 0 && k < R) ? A[row + m * k] : 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 32; ++rep) {
    double v[RB];
#pragma unroll
    for (int k = 0; k < RB; ++k) v[k] = a[k] * (rep + 1);
    vec_reduce<RB>(v, red, fin + (rep & 1) * RB);
  }
  long long t1 = clock64();
  rowqr_factor<RB>(a, row, R, tau, beta, rowbuf, red, fin);
  __syncthreads();
  long long t2 = clock64();
  rowqr_formq<RB>(a, row, R, tau, rowbuf, red, fin);
  __syncthreads();
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 32; cyc[1] = (t2 - t1) / R; cyc[2] = (t3 - t2) / R; }
#pragma unroll
  for (int k = 0; k < RB; ++k) if (row >= 0) out[row + m * k] = a[k] + fin[k];
}
int main() {
  double *A, *o; long long* c; cudaMalloc(&A, 256 * 32 * 8); cudaMalloc(&o, 256 * 32 * 8); cudaMalloc(&c, 64);
  double* h = (double*)malloc(256 * 32 * 8);
  for (int i = 0; i < 256 * 32; ++i) h[i] = (double)rand() / RAND_MAX - 0.5;
  cudaMemcpy(A, h, 256 * 32 * 8, cudaMemcpyHostToDevice);
  for (int m : {64, 128, 256}) {
    long long hc[3];
    for (int r = 0; r < 2; ++r) rb<32><<<1, m>>>(A, m, 32, c, o);
    cudaMemcpy(hc, c, 24, cudaMemcpyDeviceToHost);
    printf("RB 32 m %3d: vec_reduce %lld  factor %lld/col  formq %lld/col\n", m, hc[0], hc[1], hc[2]);
    for (int r = 0; r < 2; ++r) rb<16><<<1, m>>>(A, m, 16, c, o);
    cudaMemcpy(hc, c, 24, cudaMemcpyDeviceToHost);
    printf("RB 16 m %3d: vec_reduce %lld  factor %lld/col  formq %lld/col\n", m, hc[0], hc[1], hc[2]);
    for (int r = 0; r < 2; ++r) rb<8><<<1, m>>>(A, m, 8, c, o);
    cudaMemcpy(hc, c, 24, cudaMemcpyDeviceToHost);
    printf("RB  8 m %3d: vec_reduce %lld  factor %lld/col  formq %lld/col\n", m, hc[0], hc[1], hc[2]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
