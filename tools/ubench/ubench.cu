// Step-0 micro-benchmarks (SURVEY.md §7 "µB"): the roofline denominators that
// MEASURED_PEAKS.json does not carry for an fp64 path.
//   1. DFMA peak      — FP64 FMA pipe, independent chains per thread
//   2. DMMA peak      — mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA.8x8x4)
//   3. HBM read BW    — read-only streaming of a 4 GiB fp64 buffer (double2 loads)
//   4. HBM copy BW    — read+write, for comparison with MEASURED_PEAKS.json
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double c[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = fma(c[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) { acc[j][0] = 0; acc[j][1] = 0; }
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += acc[j][0] + acc[j][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void read_kernel(const double2* __restrict__ x, size_t n2, double* out) {
  double s0 = 0, s1 = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 v0 = __ldcs(x + i), v1 = __ldcs(x + i + stride), v2 = __ldcs(x + i + 2 * stride), v3 = __ldcs(x + i + 3 * stride);
    s0 += v0.x + v1.x + v2.x + v3.x; s1 += v0.y + v1.y + v2.y + v3.y;
  }
  for (; i < n2; i += stride) { double2 v = x[i]; s0 += v.x; s1 += v.y; }
  if (s0 + s1 == 1234.5) out[0] = s0;
}

__global__ void copy_kernel(const double2* __restrict__ x, double2* __restrict__ y, size_t n2) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) y[i] = x[i];
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"clock_khz\": %d}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, clk);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // --- DFMA
  for (int tpb : {256, 512}) {
    int blocks = sms * (2048 / tpb);
    int iters = 20000;
    dfma_kernel<<<blocks, tpb>>>(out, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_kernel<<<blocks, tpb>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double fl = 2.0 * 8 * iters * (double)blocks * tpb;
    printf("{\"test\": \"dfma\", \"tpb\": %d, \"tflops\": %.2f, \"ms\": %.3f}\n", tpb, fl / best / 1e9, best);
  }
  // --- DMMA
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (2048 / tpb);
    int iters = 5000;
    dmma_kernel<<<blocks, tpb>>>(out, 10);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dmma_kernel<<<blocks, tpb>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double fl = 2.0 * 256 * 4 * (double)iters * blocks * (tpb / 32);
    printf("{\"test\": \"dmma_m8n8k4\", \"tpb\": %d, \"tflops\": %.2f, \"ms\": %.3f}\n", tpb, fl / best / 1e9, best);
  }
  // also DMMA at 1 block of 4 warps per SM (latency view)
  {
    int iters = 5000; float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0); dmma_kernel<<<sms, 128>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double fl = 2.0 * 256 * 4 * (double)iters * sms * 4;
    printf("{\"test\": \"dmma_m8n8k4_4warps_per_sm\", \"tflops\": %.2f}\n", fl / best / 1e9);
  }
  // --- HBM
  size_t bytes = (size_t)4 << 30;
  double2 *x, *y; CK(cudaMalloc(&x, bytes)); CK(cudaMalloc(&y, bytes));
  CK(cudaMemset(x, 0, bytes)); CK(cudaMemset(y, 0, bytes));
  size_t n2 = bytes / 16;
  for (int mult : {1, 2, 4, 8}) {
    int blocks = sms * mult; float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0); read_kernel<<<blocks, 512>>>(x, n2, out); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    printf("{\"test\": \"hbm_read\", \"blocks\": %d, \"gbs\": %.1f}\n", blocks, bytes / best / 1e6);
  }
  {
    float best = 1e30f; size_t half = n2 / 2;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0); copy_kernel<<<sms * 4, 512>>>(x, y, n2); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    (void)half;
    printf("{\"test\": \"hbm_copy\", \"gbs\": %.1f}\n", 2.0 * bytes / best / 1e6);
  }
  // sustained DFMA / DMMA for ~3 s each (clock under FP64 load)
  {
    int blocks = sms * 4; cudaEventRecord(e0);
    for (int r = 0; r < 30; ++r) dfma_kernel<<<blocks, 512>>>(out, 20000, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 30 * 2.0 * 8 * 20000 * (double)blocks * 512;
    printf("{\"test\": \"dfma_sustained\", \"tflops\": %.2f, \"ms\": %.1f}\n", fl / ms / 1e9, ms);
    cudaEventRecord(e0);
    for (int r = 0; r < 30; ++r) dmma_kernel<<<blocks, 512>>>(out, 5000);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    fl = 30 * 2.0 * 256 * 4 * 5000.0 * blocks * 16;
    printf("{\"test\": \"dmma_sustained\", \"tflops\": %.2f, \"ms\": %.1f}\n", fl / ms / 1e9, ms);
  }
  return 0;
}
