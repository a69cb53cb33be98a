// Do FP64 DMMA (mma.sync m8n8k4 f64) and DFMA share one pipe on sm_100a?  Warps of one CTA split:
// warps < nd run DMMA chains, the rest DFMA chains; time each alone and both together.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mix_bench mix_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mix_kernel(double* out, int iters, int nd, int dfma_scale) {
  const int w = threadIdx.x >> 5;
  double s = 0;
  if (w < nd) {
    double acc[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc[j][0] = 0; acc[j][1] = 0; }
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) s += acc[j][0] + acc[j][1];
  } else {
    double c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = threadIdx.x * 1e-3 + j;
    const double a = 0.999999, b = 1e-7;
    for (int i = 0; i < iters * dfma_scale; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = fma(c[j], a, b);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j];
  }
  if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 4096 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000, tpb = 512;  // 16 warps
  struct Case { int nd; int ndfma; const char* name; } cases[] = {
    {8, 0, "dmma 8 warps alone"}, {0, 8, "dfma 8 warps alone"}, {8, 8, "dmma 8 + dfma 8"},
    {16, 0, "dmma 16 warps"}, {0, 16, "dfma 16 warps"}, {4, 12, "dmma 4 + dfma 12"}, {12, 4, "dmma 12 + dfma 4"}};
  for (auto& c : cases) {
    const int nthreads = (c.nd + c.ndfma) * 32;
    const int scale = 1;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      mix_kernel<<<sms * 2, nthreads>>>(out, iters, c.nd, scale);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fd = 2.0 * sms * c.nd * (double)iters * 4 * 512;          // DMMA flops (512 per m8n8k4)
    const double ff = 2.0 * sms * c.ndfma * 32.0 * iters * scale * 8 * 2;   // DFMA flops
    printf("{\"case\": \"%s\", \"ms\": %.3f, \"dmma_tf\": %.2f, \"dfma_tf\": %.2f, \"total_tf\": %.2f}\n", c.name, ms,
           fd / ms / 1e9, ff / ms / 1e9, (fd + ff) / ms / 1e9);
  }
  (void)tpb;
  return 0;
}
