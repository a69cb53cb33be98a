// Shared device helpers for libcpqr (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define CPQR_WARP 32

// Tensor order limit of the library (N <= kMaxModes): the 10-way sine of sums.
constexpr int kMaxModes = 10;

// FP64 tensor-core MMA, D(8x8) += A(8x4) * B(4x8) (SASS DMMA.8x8x4).  tcgen05 has no f64 kind
// on sm_100a (SURVEY.md §7 hard part 1), so the warp-level mma.sync is the FP64 tensor path.
// Fragment ownership, lane = 4*g + t (g = lane>>2, t = lane&3):
//   a = A[g][t],  b = B[t][g],  d0 = D[g][2t], d1 = D[g][2t+1].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Programmatic dependent launch (PDL).  A kernel launched with the programmatic-serialization
// attribute may start while its predecessor on the stream drains; pdl_wait() (griddepcontrol.wait)
// blocks until the predecessor grid has completed and its memory is visible, so every kernel of the
// per-mode chain calls it after its prologue (shared-memory / barrier set-up, tensor-map prefetch)
// and before its first global access.  Without the attribute it returns at once.  (The launches use
// the attribute only with CPQR_PDL=1: measured slower, see cpqr.cu.)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block reduction (deterministic).  `red` must hold blockDim.x/32 doubles.
// All threads must call; returns the total on every thread.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];
  return s;
}

// Asynchronous 8-byte global -> shared copy (LDGSTS): a rolled loop of these does not wait on
// each load, so the run-once tail kernels issue all their inputs at once and wait a single time.
__device__ __forceinline__ void cp_async8(double* dst_smem, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst_smem)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Streaming (evict-first) 16-byte load for the tensor pass.
__device__ __forceinline__ double2 ldg_stream2(const double* p) {
  return __ldcs(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double ldg_stream1(const double* p) { return __ldcs(p); }
