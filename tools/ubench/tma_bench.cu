// Read ceiling of the stream kernels' TMA pattern (no math): a persistent grid streams X(a, i) of a
// strided TTM (C3 mode 4: A = 128^3, I = 128) through an S-stage mbarrier ring of 32 KB stages.
//   mode 0: 16 boxes {16 a, 16 i} per stage, SWIZZLE_128B (the production k_strided_tma pattern)
//   mode 1: 16 cp.async.bulk (non-tensor) copies of one 2 KB row each per stage
//   mode 2: one box {256 a, 16 i} per stage, no swizzle
//   mode 3: the fused slice kernel's pattern on X(i1, f), I1 = I: one box {16 i1, 128 f} per stage
//           (128 B pieces of 128 fibres 8 I1 bytes apart; 8 stages revisit each fibre)
//   mode 4: the same bytes as 1 KB runs: X viewed {16, I1/16, F}, box {16, 8, 16} (16 fibres x 128 i1)
// NP producer warps split the copies of a stage; 8 consumer warps wait, touch, release.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2112_10855_b200/csrc -o tma_bench tma_bench.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "tma_kernels.cuh"
using namespace cpqr;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(12 * 32, 1)
k_read(const __grid_constant__ CUtensorMap tm, const double* X, int64_t A, int I, int S, int NP, double* out) {
  extern __shared__ uint8_t smraw[];
  constexpr uint32_t STAGE = 16 * kBoxBytes;
  uint64_t *full, *empty;
  uint8_t* st0 = tma_carve(smraw, S, full, empty);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kCW); }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t nA = A / 256, units = nA;
  const int KS = I / kBK;
  if (warp >= kCW) {
    const int pw = warp - kCW;
    if (pw >= NP || lane != 0) return;
    const uint64_t pol = policy_evict_first();
    uint32_t it = 0;
    const int per = (MODE == 2 ? 1 : 16) / (MODE == 2 ? 1 : NP);
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int a0 = (int)(u * 256);
      for (int ks = 0; ks < KS; ++ks, ++it) {
        const int s = it % S;
        mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
        if (pw == 0) mbar_expect_tx(&full[s], STAGE);
        uint8_t* dst = st0 + (size_t)s * STAGE;
        if (MODE == 0) {
          for (int q = pw * per; q < (pw + 1) * per; ++q)
            tma_load_3d_ef(dst + q * kBoxBytes, &tm, a0 + 16 * q, ks * kBK, 0, &full[s], pol);
        } else if (MODE == 1) {
          for (int q = pw * per; q < (pw + 1) * per; ++q)
            bulk_load(dst + q * 2048, X + (int64_t)(ks * kBK + q) * A + a0, 2048, &full[s], pol);
        } else if (MODE == 2) {
          if (pw == 0) tma_load_2d_ef(dst, &tm, a0, ks * kBK, &full[s], pol);
        } else if (MODE == 3) {  // unit = 128 fibres, KS = I / 16 stages of {16 i1, 128 f}; 2 boxes (32 KB)
          if (pw == 0)
            for (int q = 0; q < 2; ++q) tma_load_2d_ef(dst + q * 16384, &tm, ks * kBK, (int)(u * 256 + 128 * q), &full[s], pol);
        } else {  // MODE 4: unit = 256 fibres in 16-fibre boxes of all i1 (I = 128 -> 16 KB per box)
          if (pw == 0)
            for (int q = 0; q < 2; ++q) {
              const int f0 = (int)(u * 256) + (ks * 2 + q) * 16;
              asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_u32(dst + q * 16384)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(0), "r"(f0), "r"(smem_u32(&full[s])), "l"(pol) : "memory");
            }
        }
      }
    }
    return;
  }
  double acc = 0;
  uint32_t it = 0;
  const uint32_t sbase = smem_u32(st0);
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x)
    for (int ks = 0; ks < KS; ++ks, ++it) {
      const int s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      acc += lds64(sbase + s * STAGE + warp * 4096 + lane * 8);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  if (acc == 1234.5) out[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t A = argc > 1 ? atoll(argv[1]) : 128ll * 128 * 128;
  const int I = argc > 2 ? atoi(argv[2]) : 128;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* X; cudaMalloc(&X, sizeof(double) * A * I);
  cudaMemset(X, 0, sizeof(double) * A * I);
  double* out; cudaMalloc(&out, 64);
  void* f = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  CUtensorMap m3, m2;
  {
    cuuint64_t d[3] = {(cuuint64_t)A, (cuuint64_t)I, 1}, st[2] = {(cuuint64_t)A * 8, (cuuint64_t)A * I * 8};
    cuuint32_t box[3] = {16, 16, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, X, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("enc3 %d\n", r);
  }
  bool ok2;
  {
    cuuint64_t d[2] = {(cuuint64_t)A, (cuuint64_t)I}, st[1] = {(cuuint64_t)A * 8};
    cuuint32_t box[2] = {256, 16}, es[2] = {1, 1};
    CUresult r = enc(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, X, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    ok2 = r == 0;
    if (r) printf("enc2 %d\n", r);
  }
  CUtensorMap ms3, ms4;
  {
    cuuint64_t d[2] = {(cuuint64_t)I, (cuuint64_t)A}, st[1] = {(cuuint64_t)I * 8};
    cuuint32_t box[2] = {16, 128}, es[2] = {1, 1};
    CUresult r = enc(&ms3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, X, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("enc s3 %d\n", r);
  }
  {
    cuuint64_t d[3] = {16, (cuuint64_t)I / 16, (cuuint64_t)A}, st[2] = {128, (cuuint64_t)I * 8};
    cuuint32_t box[3] = {16, 8, 16}, es[3] = {1, 1, 1};
    CUresult r = enc(&ms4, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, X, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("enc s4 %d\n", r);
  }
  cudaFuncSetAttribute(k_read<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k_read<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k_read<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k_read<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k_read<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct C { int mode, NP, S, grid_mult; } cs[] = {
    {0, 1, 6, 0}, {0, 2, 6, 0}, {0, 4, 6, 0}, {0, 2, 4, 0}, {0, 2, 3, 0}, {0, 2, 6, 1}, {0, 4, 3, 2},
    {1, 1, 6, 0}, {1, 2, 6, 0}, {1, 4, 6, 0}, {1, 2, 3, 2},
    {2, 1, 6, 0}, {2, 1, 3, 2}, {2, 1, 4, 0},
    {3, 1, 4, 0}, {3, 1, 6, 0}, {4, 1, 4, 0}, {4, 1, 6, 0}};
  for (auto& c : cs) {
    if (c.mode == 2 && !ok2) continue;
    const int grid = c.grid_mult == 0 ? sms - 1 : c.grid_mult == 1 ? sms : 2 * sms;
    const size_t smem = 1024 + 2048 + (size_t)c.S * 16 * kBoxBytes;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (c.mode == 0) k_read<0><<<grid, 12 * 32, smem>>>(m3, X, A, I, c.S, c.NP, out);
      if (c.mode == 1) k_read<1><<<grid, 12 * 32, smem>>>(m3, X, A, I, c.S, c.NP, out);
      if (c.mode == 2) k_read<2><<<grid, 12 * 32, smem>>>(m2, X, A, I, c.S, c.NP, out);
      if (c.mode == 3) k_read<3><<<grid, 12 * 32, smem>>>(ms3, X, A, I, c.S, c.NP, out);
      if (c.mode == 4) k_read<4><<<grid, 12 * 32, smem>>>(ms4, X, A, I, c.S, c.NP, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("{\"mode\": %d, \"NP\": %d, \"S\": %d, \"grid\": %d, \"us\": %.1f, \"gbs\": %.0f, \"err\": \"%s\"}\n", c.mode,
           c.NP, c.S, grid, best * 1e3, 8.0 * A * I / best / 1e6, cudaGetErrorString(err));
  }
  return 0;
}
