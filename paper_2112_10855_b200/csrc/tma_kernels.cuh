// TMA-pipelined Multi-TTM stream-X kernels (sm_100a): the Blackwell mainloop for the dominant
// step of CP-ALS-QR (Alg. 2 line 8; cost Eq. (TTMcost)).
//
// Producer warp(s) after the consumer warps issue cp.async.bulk.tensor loads of each stage -- an X
// tile plus the matching rows of the (transposed, zero-padded) Q panel -- into an S-stage ring of
// shared-memory buffers, signalling `full[s]` via mbarrier complete_tx.  The consumer warps run FP64
// tensor-core MMAs (DMMA m8n8k4) straight from the swizzled tiles and release each stage on
// `empty[s]`.  X is read from HBM exactly once; Q rows come from L2 alongside each X tile, so no
// panel has to fit in shared memory whole (C5's Q_k is 256 KB).  Out-of-range rows/fibres are
// zero-filled by TMA, which handles every ragged edge.
//
// Swizzle: every box has 128-byte rows (16 doubles) and SWIZZLE_128B: the 16-byte chunk c of
// row r lives at chunk c ^ (r & 7).  MMA k-steps use the permuted k sets {2t} / {2t+1} (see
// ttm_kernels.cuh), which makes every fragment load below bank-conflict free.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace cpqr {

constexpr int kCW = 8;                 // consumer warps
constexpr int kTmaThreads = (kCW + 1) * 32;
constexpr int kBK = 16;                // K (contraction index) per stage
constexpr int kBoxBytes = 16 * 128;    // {16 doubles x 16 rows} box = 2 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef CPQR_RELEASE_MODE
#define CPQR_RELEASE_MODE 1
#endif
// OR of the raw bits of a warp's accumulator array: a value that depends on every DMMA of the stage
template <int M, int N>
__device__ __forceinline__ unsigned long long acc_dep(const double (&acc)[M][N][2]) {
  unsigned long long d = 0;
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int n = 0; n < N; ++n) d |= __double_as_longlong(acc[m][n][0]) | __double_as_longlong(acc[m][n][1]);
  return d;
}
// Consumer release of a ring stage (write-after-read hazard with the producer's next TMA into it).
// The stage was read with generic-proxy ld.shared; the refill is an async-proxy write.  Each thread
// orders its reads before the release with fence.proxy.async, then the warp's lane 0 arrives with
// release semantics.  dep: a value computed from the stage's data (the warp's accumulators), so the
// arrive also waits on the loads' results (mode 2).
__device__ __forceinline__ void consumer_release(uint64_t* bar, int lane, unsigned long long dep) {
#if CPQR_RELEASE_MODE >= 1
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
#endif
  __syncwarp();
#if CPQR_RELEASE_MODE == 2
  if (lane == 0 && dep != 0x7ff4dead0000beefull)
#else
  (void)dep;
  if (lane == 0)
#endif
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
#ifdef CPQR_DEBUG_HANG
// debugging build (CPQR_DEBUG_HANG=1 python -m paper_2112_10855_b200.build): a wait that spins too
// long reports block / thread / barrier / parity and traps instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (long long spin = 0;; ++spin) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (spin == (1ll << 24)) {
      printf("HANG block %d thread %d bar smem 0x%x parity %u\n", blockIdx.x, threadIdx.x, smem_u32(bar), parity);
      __trap();
    }
  }
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
#endif
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// L2 evict-first policy for the single-use tensor stream: X passes through L2 without evicting
// the small reused working set (Q panels, W, factors) and, above all, the code of the per-mode
// tail kernels, whose cold instruction fetches from DRAM otherwise dominate their run time.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_ef(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_ef(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                               uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
template <int NTH>
__device__ __forceinline__ void consumers_sync_n() {  // named barrier over NTH consumer threads
  asm volatile("bar.sync 1, %0;\n" ::"n"(NTH) : "memory");
}
__device__ __forceinline__ void consumers_sync() {  // named barrier over the consumer warps only
  asm volatile("bar.sync 1, %0;\n" ::"n"(kCW * 32) : "memory");
}
// byte offset of (row, 16-byte chunk) inside a 128B-swizzled box whose base is 1024-B aligned
__device__ __forceinline__ uint32_t swz(int row, int chunk) { return row * 128 + (((chunk ^ row) & 7) << 4); }

__device__ __forceinline__ double2 lds128(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// Position in an S-stage ring: slot s and the parity of its current phase, advanced without the
// integer division (`it % S`, `it / S` with a runtime S) that cost ~20 instructions per stage.
struct RingPos {
  int s = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next(int S) {
    if (++s == S) { s = 0; ph ^= 1u; }
  }
};

struct TmaSmem {
  uint32_t base;  // 1024-aligned shared address of stage 0
  uint64_t* full;
  uint64_t* empty;
};

// Carve the dynamic shared memory: [barriers (2 KB)] [stage 0] ... [stage S-1] [extra]
__device__ __forceinline__ uint8_t* tma_carve(uint8_t* raw, int S, uint64_t*& full, uint64_t*& empty) {
  uintptr_t p = reinterpret_cast<uintptr_t>(raw);
  p = (p + 1023) & ~uintptr_t(1023);
  full = reinterpret_cast<uint64_t*>(p);
  empty = full + S;
  return reinterpret_cast<uint8_t*>(p + 2048);
}

// ======================================================================= strided (mode k > 1)
// T(a, r, b) = sum_i X(a, i, b) Q(i, r).  Unit = 32 CW consecutive a (CW consumer warps x 32 rows)
// of one b; X map 3D {A, I, B}, box {16, 16, 1} (2 CW boxes per stage, split over NP producer
// warps); Q map 2D {RQ, I} over the transposed padded panel Qt[i*RQ + r], box {16, 16} (NT/2
// boxes).  Consumer warp w owns rows 32w..32w+31: M-tiles mt = 2p + s hold rows 16(2w+p) + 2g + s
// (one 16-byte load feeds two tiles).  CW = 4 runs two CTAs per SM (see launch_tma).
//
// Work decomposition.  P == nullptr: unit u goes to CTA u mod G (persistent round robin).  With
// few units per CTA that leaves a ragged last wave (C5 at 8 slabs: 500 units on 147 CTAs = 3.4
// waves, 15 % idle), so P != nullptr selects a stream-K split: the W = units x KS k-steps are cut
// into G equal contiguous ranges, one per CTA.  A unit covered by one CTA is stored to T; a unit
// cut by a range boundary leaves each CTA's partial sum in a slot P[(2 c + h) * 32 CW * R] (h = 0:
// the CTA's first unit, 1: its last).  The last of the unit's CTAs to arrive (arrival counter
// cnt[c0], c0 = the unit's first CTA; self re-arming) adds the slots in CTA order c0..c1 and stores
// T: fixed order, so bitwise reproducible, and no fix-up launch (k_strided_fixup, kept for
// CPQR_SK_FIXUP=1, computes the same sums in the same order).
struct SkRange {  // the k-step range [it0, it1) of CTA c under the stream-K split
  int64_t it0, it1;
  __device__ __forceinline__ SkRange(int64_t W, int c, int G) : it0(W * c / G), it1(W * (c + 1) / G) {}
};
// the CTA whose stream-K range [W c / G, W (c+1) / G) holds k-step it: the largest c with
// floor(W c / G) <= it, i.e. c = ceil((it + 1) G / W) - 1
__device__ __forceinline__ int sk_cta_of(int64_t it, int64_t W, int G) {
  return (int)(((it + 1) * G + W - 1) / W) - 1;
}

//
// Short slices (wa < CW).  A unit is 32 wa rows of wb = CW / wa consecutive slices b: warp w owns
// rows 32 (w mod wa) .. +31 of slice b0 + w / wa.  With A < 32 CW rows per slice (intermediates
// whose leading modes are already contracted, A = R; the paper's 75^5 shape, A = 76) a unit of one
// slice would leave most of its M-tiles empty; the host picks the wa in {1, 2, 4, 8} that fills
// them best (launch_tma).  wa = CW is the layout above; the stream-K split needs it.
template <int NT, int NP = 1, int CW = kCW>
__global__ void __launch_bounds__((CW + NP) * 32, CW == 4 ? 2 : 1)
k_strided_tma(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmQ, int64_t A,
              int I, int64_t B, int R, double* __restrict__ T, int S, double* __restrict__ P,
              unsigned* __restrict__ cnt, int wa) {
  extern __shared__ uint8_t smraw[];
  constexpr int NQB = (NT + 1) / 2;
  constexpr uint32_t XBYTES = 2 * CW * kBoxBytes, QBYTES = NQB * kBoxBytes, STAGE = XBYTES + QBYTES;
  uint64_t *full, *empty;
  uint8_t* st0 = tma_carve(smraw, S, full, empty);
  // the fused fix-up's "last to arrive" flag: in the carved barrier block (no static shared memory)
  volatile int& sk_last = *reinterpret_cast<volatile int*>(reinterpret_cast<uint8_t*>(full) + 1024);
  const uint32_t sbase = smem_u32(st0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CW); }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) prefetch_tmap(&tmX);
  pdl_wait();                // the predecessor (previous mode's tail: Q panels) has completed
  const int wb = CW / wa;
  const int64_t nA = (A + 32 * wa - 1) / (32 * wa);
  const int64_t units = nA * ((B + wb - 1) / wb);
  const int KS = (I + kBK - 1) / kBK;
  const SkRange rg(units * KS, blockIdx.x, gridDim.x);
  // the unit segments [ks0, ks1) of this CTA, in order: round robin (P == nullptr) or stream-K
  auto segments = [&](auto&& body) {
    if (P == nullptr) {
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) body(u, 0, KS);
    } else {
      for (int64_t it = rg.it0; it < rg.it1;) {
        const int64_t u = it / KS;
        const int ks0 = (int)(it - u * KS);
        const int64_t rem = rg.it1 - it;
        const int ks1 = (rem < (int64_t)(KS - ks0)) ? ks0 + (int)rem : KS;
        body(u, ks0, ks1);
        it += ks1 - ks0;
      }
    }
  };
  if (warp >= CW) {  // ---------------------------------------------------------- producer(s)
    // NP producer warps split the 16 X boxes of a stage (the per-box TMA issue cost bounds the
    // HBM-bound passes); producer 0 also loads Q and does the arrive.expect_tx for the whole stage
    // (bytes of the other producers may land first: the tx count just dips below zero meanwhile)
    const int pw = warp - CW;
    if (lane == 0) {
      prefetch_tmap(&tmX);
      if (pw == 0) prefetch_tmap(&tmQ);
      const uint64_t pol = policy_evict_first();
      RingPos rp;
      segments([&](int64_t u, int ks0, int ks1) {
        const int64_t bq = u / nA;
        const int a0 = (int)((u - bq * nA) * 32 * wa);
        const int64_t b0 = bq * wb;
        // box q belongs to warp q / 2: rows a0 + 32 (w mod wa) + 16 (q & 1) of slice b0 + w / wa; a
        // warp beyond the unit's wb slices (CW not a multiple of wa) gets slice B: zero fill, no read
        int qa[2 * CW / NP], qb[2 * CW / NP];
#pragma unroll
        for (int j = 0; j < 2 * CW / NP; ++j) {
          const int q = pw * (2 * CW / NP) + j, w = q >> 1;
          qa[j] = a0 + 32 * (w % wa) + 16 * (q & 1);
          const int64_t bb = b0 + w / wa;
          qb[j] = (w / wa < wb && bb < B) ? (int)bb : (int)B;
        }
        for (int ks = ks0; ks < ks1; ++ks, rp.next(S)) {
          const int s = rp.s;
          mbar_wait(&empty[s], rp.ph ^ 1);
          if (pw == 0) mbar_expect_tx(&full[s], STAGE);
          uint8_t* dst = st0 + (size_t)s * STAGE;
#pragma unroll
          for (int j = 0; j < 2 * CW / NP; ++j)
            tma_load_3d_ef(dst + (pw * (2 * CW / NP) + j) * kBoxBytes, &tmX, qa[j], ks * kBK, qb[j], &full[s], pol);
          if (pw == 0)
#pragma unroll
            for (int q = 0; q < NQB; ++q) tma_load_2d(dst + XBYTES + q * kBoxBytes, &tmQ, 16 * q, ks * kBK, &full[s]);
        }
      });
    }
    return;
  }
  // --------------------------------------------------------------------------------- consumers
  const int g = lane >> 2, t = lane & 3;
  const int64_t first_u = rg.it0 / KS;
  RingPos rp;
  const int wai = warp % wa, wbi = warp / wa;
  segments([&](int64_t u, int ks0, int ks1) {
    const int64_t bq = u / nA;
    const int64_t a0 = (u - bq * nA) * 32 * wa;
    const int64_t b = bq * wb + wbi;  // this warp's slice (beyond B or the unit's wb slices: idle)
    double acc[4][NT][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    for (int ks = ks0; ks < ks1; ++ks, rp.next(S)) {
      const int s = rp.s;
      mbar_wait(&full[s], rp.ph);
      const uint32_t xs = sbase + s * STAGE, qs = xs + XBYTES;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int sk = 0; sk < 2; ++sk) {
          const int k = 8 * h + 2 * t + sk;  // row (k index) inside the stage
          double2 xa[2];
#pragma unroll
          for (int p = 0; p < 2; ++p) xa[p] = lds128(xs + (2 * warp + p) * kBoxBytes + swz(k, g));
          double qb[NT];
#pragma unroll
          for (int n = 0; n < NT; ++n)
            qb[n] = lds64(qs + (n >> 1) * kBoxBytes + swz(k, 4 * (n & 1) + (g >> 1)) + 8 * (g & 1));
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            dmma(acc[0][n][0], acc[0][n][1], xa[0].x, qb[n]);
            dmma(acc[1][n][0], acc[1][n][1], xa[0].y, qb[n]);
            dmma(acc[2][n][0], acc[2][n][1], xa[1].x, qb[n]);
            dmma(acc[3][n][0], acc[3][n][1], xa[1].y, qb[n]);
          }
        }
      consumer_release(&empty[s], lane, acc_dep(acc));
    }
    if (ks0 == 0 && ks1 == KS) {  // the whole unit: straight to T
      // M-tiles 2p and 2p + 1 hold the adjacent rows 2g and 2g + 1 of the same columns: one 16-byte
      // store per column (A is even -- the TMA map requires it -- so the pair is aligned and inside
      // A together), and the 8 lanes g of a column write 128 contiguous bytes
      double* __restrict__ Tb = T + A * (int64_t)R * b;
      const bool live = wbi < wb && b < B;
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int64_t row = a0 + 32 * wai + 16 * p + 2 * g;
        if (row >= A || !live) continue;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int r0 = 8 * n + 2 * t;
          if (r0 < R)
            *reinterpret_cast<double2*>(Tb + row + A * r0) = make_double2(acc[2 * p][n][0], acc[2 * p + 1][n][0]);
          if (r0 + 1 < R)
            *reinterpret_cast<double2*>(Tb + row + A * (r0 + 1)) = make_double2(acc[2 * p][n][1], acc[2 * p + 1][n][1]);
        }
      }
    } else {  // a stream-K partial: this CTA's slot (first or last unit of its range)
      double* __restrict__ Pb = P + ((int64_t)2 * blockIdx.x + (u == first_u ? 0 : 1)) * (32 * CW) * R;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int row = 32 * warp + 16 * (m >> 1) + 2 * g + (m & 1);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int r0 = 8 * n + 2 * t;
          if (r0 < R) Pb[row + 32 * CW * r0] = acc[m][n][0];
          if (r0 + 1 < R) Pb[row + 32 * CW * (r0 + 1)] = acc[m][n][1];
        }
      }
      if (cnt == nullptr) return;  // CPQR_SK_FIXUP=1: k_strided_fixup sums the slots
      // fused fix-up: the unit's CTAs c0..c1 each leave one slot; the last to arrive sums them
      const int64_t W = units * KS;
      const int c0 = sk_cta_of(u * KS, W, gridDim.x), c1 = sk_cta_of((u + 1) * KS - 1, W, gridDim.x);
      __threadfence();
      consumers_sync_n<CW * 32>();
      if (threadIdx.x == 0) sk_last = (atomicAdd(&cnt[c0], 1u) == (unsigned)(c1 - c0)) ? 1 : 0;
      consumers_sync_n<CW * 32>();
      if (sk_last) {
        __threadfence();
        const int h0 = ((W * c0 / gridDim.x) / KS == u) ? 0 : 1;  // u is c0's first unit, or its last
        constexpr int UR = 32 * CW;
        for (int e = threadIdx.x; e < UR * R; e += CW * 32) {
          const int row = e % UR, r = e / UR;
          double v = __ldcg(P + ((int64_t)2 * c0 + h0) * UR * R + e);
          for (int cc = c0 + 1; cc <= c1; ++cc) v += __ldcg(P + ((int64_t)2 * cc) * UR * R + e);
          if (a0 + row < A) T[a0 + row + A * ((int64_t)r + (int64_t)R * b)] = v;
        }
        if (threadIdx.x == 0) cnt[c0] = 0u;  // re-armed for the next launch (graph replay)
      }
    }
  });
}

// ============================================ strided, the last two modes in one pass (R <= 8)
// T(a, r, q) = sum_b Q2(b, q) sum_i X(a, i, b) Q(i, r): the two slowest modes of an (A, I, B) view
// contracted in ONE pass over X, so the (R / I)-sized intermediate T1(a, r, b) of the first
// contraction never goes to HBM (C4 48^5 R = 8, modes 1-2: 340 MB written and read back per mode).
// A unit is 128 rows of a (8 consumer warps x one 16-row box) over ALL b: per slice b the warp
// contracts i on DMMA (acc1, rows 2g / 2g + 1 of its box), then folds the slice into the unit's
// output acc2(a, r, q) += acc1(a, r) Q2(b, q) with R plain FMAs per element (R / I of the DMMA work;
// Q2's row b comes from the transposed panel through L1, uniform across the warp).  acc2 is 2 x 2 x R
// doubles per thread, which bounds R at 8 (one N-tile).  X is read once, T written once.
template <int NP = 2>
__global__ void __launch_bounds__((8 + NP) * 32, 1)
k_strided2_tma(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmQ, int64_t A, int I,
               int B, int R, const double* __restrict__ Q2t, int rq, double* __restrict__ T, int S) {
  extern __shared__ uint8_t smraw[];
  constexpr int CW = 8;
  constexpr uint32_t XBYTES = CW * kBoxBytes, STAGE = XBYTES + kBoxBytes;
  uint64_t *full, *empty;
  uint8_t* st0 = tma_carve(smraw, S, full, empty);
  const uint32_t sbase = smem_u32(st0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CW); }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) prefetch_tmap(&tmX);
  pdl_wait();
  const int64_t units = (A + 16 * CW - 1) / (16 * CW);
  const int KS = (I + kBK - 1) / kBK;
  if (warp >= CW) {  // ---------------------------------------------------------- producer(s)
    const int pw = warp - CW;
    if (lane == 0) {
      prefetch_tmap(&tmX);
      if (pw == 0) prefetch_tmap(&tmQ);
      const uint64_t pol = policy_evict_first();
      RingPos rp;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int a0 = (int)(u * 16 * CW);
        for (int b = 0; b < B; ++b)
          for (int ks = 0; ks < KS; ++ks, rp.next(S)) {
            const int s = rp.s;
            mbar_wait(&empty[s], rp.ph ^ 1);
            if (pw == 0) mbar_expect_tx(&full[s], STAGE);
            uint8_t* dst = st0 + (size_t)s * STAGE;
#pragma unroll
            for (int q = pw * (CW / NP); q < (pw + 1) * (CW / NP); ++q)
              tma_load_3d_ef(dst + q * kBoxBytes, &tmX, a0 + 16 * q, ks * kBK, b, &full[s], pol);
            if (pw == 0) tma_load_2d(dst + XBYTES, &tmQ, 0, ks * kBK, &full[s]);
          }
      }
    }
    return;
  }
  // --------------------------------------------------------------------------------- consumers
  const int g = lane >> 2, t = lane & 3;
  RingPos rp;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t a0 = u * 16 * CW;
    double acc2[2][2][8];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc2[m][j][q] = 0.0;
    for (int b = 0; b < B; ++b) {
      double acc[2][1][2];
      acc[0][0][0] = acc[0][0][1] = acc[1][0][0] = acc[1][0][1] = 0.0;
      for (int ks = 0; ks < KS; ++ks, rp.next(S)) {
        const int s = rp.s;
        mbar_wait(&full[s], rp.ph);
        const uint32_t xs = sbase + s * STAGE, qs = xs + XBYTES;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int sk = 0; sk < 2; ++sk) {
            const int k = 8 * h + 2 * t + sk;  // row (k index) inside the stage
            const double2 xa = lds128(xs + warp * kBoxBytes + swz(k, g));
            const double qb = lds64(qs + swz(k, g >> 1) + 8 * (g & 1));
            dmma(acc[0][0][0], acc[0][0][1], xa.x, qb);
            dmma(acc[1][0][0], acc[1][0][1], xa.y, qb);
          }
        consumer_release(&empty[s], lane, acc_dep(acc));
      }
      // fold slice b: acc2(a, r, q) += acc1(a, r) Q2(b, q)
      const double2* q2 = reinterpret_cast<const double2*>(Q2t + (int64_t)b * rq);
      double qv[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 v = __ldg(q2 + q);
        qv[2 * q] = v.x;
        qv[2 * q + 1] = v.y;
      }
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int q = 0; q < 8; ++q) acc2[m][j][q] = fma(acc[m][0][j], qv[q], acc2[m][j][q]);
    }
    // rows 2g and 2g + 1 of the warp's box are adjacent: one 16-byte store per (r, q) column
    const int64_t row = a0 + 16 * warp + 2 * g;
    if (row < A) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = 2 * t + j;
        if (r >= R) continue;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < R)
            *reinterpret_cast<double2*>(T + row + A * ((int64_t)r + (int64_t)R * q)) =
                make_double2(acc2[0][j][q], acc2[1][j][q]);
      }
    }
  }
}

// Stream-K fix-up of k_strided_tma: one CTA of 1024 threads per range boundary c = 1..G-1.  A
// boundary that cuts a unit and is the first boundary inside it sums the segments of CTAs
// c0 = c-1 .. c1 in that order into T.  Each thread issues the loads of its (up to) 8 entries
// before any add: one CTA per boundary with every load in flight (a CTA per 256 entries was bound
// by CTA launch rate at ~20 us, a looped CTA by load latency at ~35 us).
__global__ void __launch_bounds__(1024) k_strided_fixup(const double* __restrict__ P, int64_t A, int R, int64_t B,
                                                        int KS, int UR, int G, double* __restrict__ T) {
  pdl_wait();
  const int c = 1 + blockIdx.x;
  const int64_t nA = (A + UR - 1) / UR;
  const int64_t W = nA * B * KS;
  const int64_t it = W * c / G;
  const int64_t u = it / KS;
  if (it == u * KS) return;                           // boundary on a unit edge: nothing cut
  const int64_t itp = W * (c - 1) / G;
  if (itp > u * KS) return;                           // not the first boundary inside u
  int c1 = c;                                         // last CTA with a segment in u
  while (c1 + 1 < G && W * (c1 + 1) / G < (u + 1) * KS) ++c1;
  const int c0 = c - 1;
  const int h0 = (itp / KS == u) ? 0 : 1;              // u is c0's first unit, or its last
  const int64_t b = u / nA, a0 = (u - b * nA) * UR;
  const int n = UR * R;
  constexpr int kPer = 8;
  double v[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int e = threadIdx.x + q * blockDim.x;
    v[q] = (e < n) ? P[((int64_t)2 * c0 + h0) * n + e] : 0.0;
  }
  for (int cc = c; cc <= c1; ++cc) {
    double w[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int e = threadIdx.x + q * blockDim.x;
      w[q] = (e < n) ? P[((int64_t)2 * cc) * n + e] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) v[q] += w[q];
  }
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int e = threadIdx.x + q * blockDim.x;
    const int row = e % UR, r = e / UR;
    if (e < n && a0 + row < A) T[a0 + row + A * ((int64_t)r + (int64_t)R * b)] = v[q];
  }
}

// ======================================================== fibre kernels (mode 1 / fused slice)
// X map 3D {I1, F2, L} (F2 = fibres per slice), box {16, 128, 1}: a stage is 16 i x 128 fibres,
// rows = fibres.  Q1 (A operand) map 2D over Qt1 {RQ, I1}, box {16, 16}.  Consumer warp w owns
// fibres 16w..16w+15 of the block; N-tile n (0/1), lane g -> fibre 16w + 8n + fmap(g) with
// fmap(g) = (g>>1) + 4(g&1) (makes the 16-byte X loads conflict free under the swizzle).
__device__ __forceinline__ int fmap(int g) { return (g >> 1) + 4 * (g & 1); }
// leading dimension of the fused slice kernel's per-warp Y in shared memory: the smallest ldy >= R
// with ldy = 2 (mod 8) (k_slice_tma)
__host__ __device__ inline int slice_ldy(int R) { return R + ((10 - R % 8) % 8); }

// One stage of the first contraction: acc[m][n] += Q1^T(r1, i) X(i, fibre) over the 16 i, for the
// warp's NF N-tiles of 8 fibres (fibre rows FW*warp + 8n + fmap(g) of the stage box).
template <int MT, int NF = 2>
__device__ __forceinline__ void fiber_stage(uint32_t xs, uint32_t qs, int warp, int g, int t,
                                            double (&acc)[MT][NF][2]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double2 xb[NF];
#pragma unroll
    for (int n = 0; n < NF; ++n) xb[n] = lds128(xs + swz(8 * NF * warp + 8 * n + fmap(g), 4 * h + t));
#pragma unroll
    for (int sk = 0; sk < 2; ++sk) {
      const int k = 8 * h + 2 * t + sk;
      double qa[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m)
        qa[m] = lds64(qs + (m >> 1) * kBoxBytes + swz(k, 4 * (m & 1) + (g >> 1)) + 8 * (g & 1));
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NF; ++n) dmma(acc[m][n][0], acc[m][n][1], qa[m], sk ? xb[n].y : xb[n].x);
    }
  }
}

// T(r, f) = sum_i Q(i, r) X(i, f), f < F (= F2 * L fibres, 2D map with L = 1).  Unit = 128 fibres.
template <int MT, int CW = kCW>
__global__ void __launch_bounds__((CW + 1) * 32, CW == 4 ? 2 : 1)
k_fiber_tma(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmQ, int I,
            int64_t F, int R, double* __restrict__ T, int S) {
  extern __shared__ uint8_t smraw[];
  constexpr int NQB = (MT + 1) / 2;
  constexpr int NF = 16 / CW;  // fibre tiles of 8 per warp: CW warps x 8 NF = 128 fibres per unit
  constexpr uint32_t XBYTES = 128 * 128, QBYTES = NQB * kBoxBytes, STAGE = XBYTES + QBYTES;
  uint64_t *full, *empty;
  uint8_t* st0 = tma_carve(smraw, S, full, empty);
  const uint32_t sbase = smem_u32(st0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CW); }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  const int64_t units = (F + 127) / 128;
  const int KS = (I + kBK - 1) / kBK;
  if (warp == CW) {
    if (lane == 0) {
      prefetch_tmap(&tmX);
      prefetch_tmap(&tmQ);
      const uint64_t pol = policy_evict_first();
      RingPos rp;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x)
        for (int ks = 0; ks < KS; ++ks, rp.next(S)) {
          const int s = rp.s;
          mbar_wait(&empty[s], rp.ph ^ 1);
          mbar_expect_tx(&full[s], STAGE);
          uint8_t* dst = st0 + (size_t)s * STAGE;
          tma_load_2d_ef(dst, &tmX, ks * kBK, (int)(u * 128), &full[s], pol);
#pragma unroll
          for (int q = 0; q < NQB; ++q) tma_load_2d(dst + XBYTES + q * kBoxBytes, &tmQ, 16 * q, ks * kBK, &full[s]);
        }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  RingPos rp;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    double acc[MT][NF][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < NF; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    for (int ks = 0; ks < KS; ++ks, rp.next(S)) {
      const int s = rp.s;
      mbar_wait(&full[s], rp.ph);
      const uint32_t xs = sbase + s * STAGE;
      fiber_stage<MT, NF>(xs, xs + XBYTES, warp, g, t, acc);
      consumer_release(&empty[s], lane, acc_dep(acc));
    }
    const int64_t f0 = u * 128 + 8 * NF * warp;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int r = 8 * m + g;
      if (r >= R) continue;
#pragma unroll
      for (int n = 0; n < NF; ++n)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int64_t f = f0 + 8 * n + fmap(2 * t + j);
          if (f < F) T[r + (int64_t)R * f] = acc[m][n][j];
        }
    }
  }
}

// Fused two-mode slice kernel (modes 1 and 2 of X(I1, I2, L) in one pass, n >= 3):
//   Y(r1, r2, l) = sum_{i2} [sum_{i1} Q1(i1, r1) X(i1, i2, l)] Q2(i2, r2).
// Units u = l * nfb + fb (fibre blocks of 128 within slice l), contiguous balanced ranges per CTA
// (u0 = c U / G).  After a unit's K loop each warp chains its first-contraction fragments into the
// second contraction (acc[m][n][j] is the A fragment of k-step (n, j), whose k index t maps to
// fibre fmap(2t+j)), accumulating Y in registers over the run of units of the same slice.  At a
// slice change the 8 warps' Y are summed in a fixed order through shared memory and written to
// Yout[l] when the run covers the whole slice, else to the partial slot P[l][c - cta_of(l nfb)]
// (fixed-order fix-up by k_slice_fixup).  Deterministic, no atomics.
template <int MT, int NF, int CW = kCW>
__global__ void __launch_bounds__((CW + 1) * 32, CW == 4 ? 2 : 1)
k_slice_tma(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmQ, int I1, int I2,
            int64_t L, const double* __restrict__ Q2, int64_t ldq2, int R, double* __restrict__ Yout,
            double* __restrict__ P, int nslots, int S) {
  extern __shared__ uint8_t smraw[];
  constexpr int NQB = (MT + 1) / 2;
  constexpr int BN = CW * 8 * NF;  // fibres per unit (box height)
  constexpr uint32_t XBYTES = BN * 128, QBYTES = NQB * kBoxBytes, STAGE = XBYTES + QBYTES;
  uint64_t *full, *empty;
  uint8_t* st0 = tma_carve(smraw, S, full, empty);
  double* red = reinterpret_cast<double*>(st0 + (size_t)S * STAGE);  // CW x (ldy x R): per-warp Y
  const uint32_t sbase = smem_u32(st0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int RR = R * R;
  // leading dimension of the per-warp Y (r1 + ldy r2): ldy = 2 mod 8, so that the four lanes t of a
  // half-warp (r2 = 8 m2 + 2 t + j, stride 2 ldy doubles) fall into different 4-double bank groups
  // (ldy = R = 16 put them in the same banks: 18 % of C3's shared-memory wavefronts were conflicts)
  const int ldy = slice_ldy(R), WY = ldy * R;
  for (int e = threadIdx.x; e < CW * WY; e += blockDim.x) red[e] = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CW); }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  const int nfb = (I2 + BN - 1) / BN;
  const int64_t U = L * nfb;
  const int64_t G = gridDim.x;
  const int64_t u0 = (int64_t)blockIdx.x * U / G, u1 = ((int64_t)blockIdx.x + 1) * U / G;
  const int KS = (I1 + kBK - 1) / kBK;
  if (warp == CW) {
    if (lane == 0) {
      prefetch_tmap(&tmX);
      prefetch_tmap(&tmQ);
      const uint64_t pol = policy_evict_first();
      RingPos rp;
      for (int64_t u = u0; u < u1; ++u) {
        const int l = (int)(u / nfb), fb = (int)(u - (int64_t)l * nfb);
        for (int ks = 0; ks < KS; ++ks, rp.next(S)) {
          const int s = rp.s;
          mbar_wait(&empty[s], rp.ph ^ 1);
          mbar_expect_tx(&full[s], STAGE);
          uint8_t* dst = st0 + (size_t)s * STAGE;
          tma_load_3d_ef(dst, &tmX, ks * kBK, fb * BN, l, &full[s], pol);
#pragma unroll
          for (int q = 0; q < NQB; ++q) tma_load_2d(dst + XBYTES + q * kBoxBytes, &tmQ, 16 * q, ks * kBK, &full[s]);
        }
      }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  double* yw = red + warp * WY;  // this warp's running Y (r1 + ldy r2)
  // NF == 2 (few stages per unit): Y stays in registers between flushes; NF == 4: in smem (yw),
  // which frees the registers the 4 N-tiles of the first contraction need
  constexpr bool YREG = NF <= 2;
  double yreg[YREG ? MT : 1][YREG ? MT : 1][2];
#pragma unroll
  for (int m = 0; m < (YREG ? MT : 1); ++m)
#pragma unroll
    for (int m2 = 0; m2 < (YREG ? MT : 1); ++m2) yreg[m][m2][0] = yreg[m][m2][1] = 0.0;
  RingPos rp;
  int64_t run_start = u0;
  for (int64_t u = u0; u < u1; ++u) {
    const int64_t l = u / nfb;
    const int fb = (int)(u - l * nfb);
    double acc[MT][NF][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < NF; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    for (int ks = 0; ks < KS; ++ks, rp.next(S)) {
      const int s = rp.s;
      mbar_wait(&full[s], rp.ph);
      const uint32_t xs = sbase + s * STAGE;
      fiber_stage<MT, NF>(xs, xs + XBYTES, warp, g, t, acc);
      consumer_release(&empty[s], lane, acc_dep(acc));
    }
    if constexpr (YREG) {
#pragma unroll
      for (int n = 0; n < NF; ++n)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i2 = fb * BN + 8 * NF * warp + 8 * n + fmap(2 * t + j);
          double qb[MT];
#pragma unroll
          for (int m2 = 0; m2 < MT; ++m2) {
            const int r2 = 8 * m2 + g;
            qb[m2] = (i2 < I2 && r2 < R) ? __ldg(Q2 + i2 + ldq2 * r2) : 0.0;
          }
#pragma unroll
          for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int m2 = 0; m2 < MT; ++m2) dmma(yreg[m][m2][0], yreg[m][m2][1], acc[m][n][j], qb[m2]);
        }
    } else {
      // second contraction over this warp's 8 NF fibres (i2), accumulated into the warp's Y in smem;
      // one 8-row block of Y (r1 in [8m, 8m+8)) live at a time keeps the register peak low
  #pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int r1 = 8 * m + g;
        double yacc[MT][2];
  #pragma unroll
        for (int m2 = 0; m2 < MT; ++m2)
  #pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int r2 = 8 * m2 + 2 * t + j;
            yacc[m2][j] = (r1 < R && r2 < R) ? yw[r1 + ldy * r2] : 0.0;
          }
  #pragma unroll
        for (int n = 0; n < NF; ++n)
  #pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int i2 = fb * BN + 8 * NF * warp + 8 * n + fmap(2 * t + j);
  #pragma unroll
            for (int m2 = 0; m2 < MT; ++m2) {
              const int r2 = 8 * m2 + g;
              const double qb = (i2 < I2 && r2 < R) ? __ldg(Q2 + i2 + ldq2 * r2) : 0.0;
              dmma(yacc[m2][0], yacc[m2][1], acc[m][n][j], qb);
            }
          }
  #pragma unroll
        for (int m2 = 0; m2 < MT; ++m2)
  #pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int r2 = 8 * m2 + 2 * t + j;
            if (r1 < R && r2 < R) yw[r1 + ldy * r2] = yacc[m2][j];
          }
      }
    }
    const bool flush = (u + 1 == u1) || ((u + 1) / nfb != l);
    if (flush) {  // fixed-order reduction of the CW warps' partial Y
      if constexpr (YREG) {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int m2 = 0; m2 < MT; ++m2)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int r1 = 8 * m + g, r2 = 8 * m2 + 2 * t + j;
              if (r1 < R && r2 < R) yw[r1 + ldy * r2] = yreg[m][m2][j];
              yreg[m][m2][j] = 0.0;
            }
      }
      consumers_sync_n<CW * 32>();
      const bool whole = (run_start == l * nfb) && (u == l * nfb + nfb - 1);
      double* dst;
      if (whole) {
        dst = Yout + l * RR;
      } else {
        const int64_t first_cta = ((l * nfb + 1) * G - 1) / U;  // owner of unit l*nfb
        dst = P + (l * nslots + (blockIdx.x - first_cta)) * RR;
      }
      for (int e = threadIdx.x; e < RR; e += CW * 32) {
        const int r2 = e / R, o = (e - r2 * R) + ldy * r2;
        double v = 0.0;
        for (int w = 0; w < CW; ++w) v += red[w * WY + o];
        dst[e] = v;
      }
      consumers_sync_n<CW * 32>();
      for (int e = threadIdx.x; e < CW * WY; e += CW * 32) red[e] = 0.0;
      consumers_sync_n<CW * 32>();
      run_start = u + 1;
    }
  }
}

// Small-slice variant (I2 <= 64, I2 % 8 == 0): a stage is the 3D box {16 i1, I2 fibres, 8 slices};
// consumer warp w owns slice 8u + w entirely (nf2 = I2/8 N-tiles), chains the second contraction
// itself and writes Y(:, :, l) directly -- no cross-warp reduction, no partial slots.
template <int MT>
__global__ void __launch_bounds__(kTmaThreads, 1)
k_slice_small_tma(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmQ, int I1,
                  int I2, int64_t L, const double* __restrict__ Q2, int64_t ldq2, int R,
                  double* __restrict__ Yout, int S) {
  extern __shared__ uint8_t smraw[];
  constexpr int NQB = (MT + 1) / 2;
  const uint32_t XBYTES = (uint32_t)I2 * 8 * 128, STAGE = XBYTES + NQB * kBoxBytes;
  uint64_t *full, *empty;
  uint8_t* st0 = tma_carve(smraw, S, full, empty);
  const uint32_t sbase = smem_u32(st0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kCW); }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  const int nf2 = I2 / 8;
  const int64_t units = (L + 7) / 8;
  const int KS = (I1 + kBK - 1) / kBK;
  if (warp == kCW) {
    if (lane == 0) {
      prefetch_tmap(&tmX);
      prefetch_tmap(&tmQ);
      const uint64_t pol = policy_evict_first();
      RingPos rp;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x)
        for (int ks = 0; ks < KS; ++ks, rp.next(S)) {
          const int s = rp.s;
          mbar_wait(&empty[s], rp.ph ^ 1);
          mbar_expect_tx(&full[s], STAGE);
          uint8_t* dst = st0 + (size_t)s * STAGE;
          tma_load_3d_ef(dst, &tmX, ks * kBK, 0, (int)(u * 8), &full[s], pol);
#pragma unroll
          for (int q = 0; q < NQB; ++q) tma_load_2d(dst + XBYTES + q * kBoxBytes, &tmQ, 16 * q, ks * kBK, &full[s]);
        }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  RingPos rp;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    double acc[MT][8][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < 8; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    const int rowbase = warp * I2;
    for (int ks = 0; ks < KS; ++ks, rp.next(S)) {
      const int s = rp.s;
      mbar_wait(&full[s], rp.ph);
      const uint32_t xs = sbase + s * STAGE, qs = xs + XBYTES;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double2 xb[8];
#pragma unroll
        for (int n = 0; n < 8; ++n)
          if (n < nf2) xb[n] = lds128(xs + swz(rowbase + 8 * n + fmap(g), 4 * h + t));
#pragma unroll
        for (int sk = 0; sk < 2; ++sk) {
          const int k = 8 * h + 2 * t + sk;
          double qa[MT];
#pragma unroll
          for (int m = 0; m < MT; ++m)
            qa[m] = lds64(qs + (m >> 1) * kBoxBytes + swz(k, 4 * (m & 1) + (g >> 1)) + 8 * (g & 1));
#pragma unroll
          for (int n = 0; n < 8; ++n)
            if (n < nf2)
#pragma unroll
              for (int m = 0; m < MT; ++m) dmma(acc[m][n][0], acc[m][n][1], qa[m], sk ? xb[n].y : xb[n].x);
        }
      }
      consumer_release(&empty[s], lane, acc_dep(acc));
    }
    const int64_t l = u * 8 + warp;
    double yacc[MT][MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < MT; ++n) yacc[m][n][0] = yacc[m][n][1] = 0.0;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      if (n >= nf2) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int i2 = 8 * n + fmap(2 * t + j);
        double qb[MT];
#pragma unroll
        for (int m2 = 0; m2 < MT; ++m2) {
          const int r2 = 8 * m2 + g;
          qb[m2] = (r2 < R) ? __ldg(Q2 + i2 + ldq2 * r2) : 0.0;
        }
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int m2 = 0; m2 < MT; ++m2) dmma(yacc[m][m2][0], yacc[m][m2][1], acc[m][n][j], qb[m2]);
      }
    }
    if (l < L) {
      double* o = Yout + l * R * R;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int r1 = 8 * m + g;
        if (r1 >= R) continue;
#pragma unroll
        for (int m2 = 0; m2 < MT; ++m2)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int r2 = 8 * m2 + 2 * t + j;
            if (r2 < R) o[r1 + R * r2] = yacc[m][m2][j];
          }
      }
    }
  }
}

// Sum the partial slots of the slices split across CTA ranges (fixed order).
__global__ void k_slice_fixup(const double* __restrict__ P, int nslots, int64_t L, int nfb, int64_t G, int RR,
                              double* __restrict__ Y) {
  pdl_wait();
  const int64_t U = L * nfb;
  for (int64_t l = blockIdx.x; l < L; l += gridDim.x) {
    const int64_t c0 = ((l * nfb + 1) * G - 1) / U;
    const int64_t c1 = ((l * nfb + nfb) * G - 1) / U;
    if (c0 == c1) continue;
    for (int e = threadIdx.x; e < RR; e += blockDim.x) {
      double v = 0.0;
      for (int64_t c = 0; c <= c1 - c0; ++c) v += P[(l * nslots + c) * RR + e];
      Y[l * RR + e] = v;
    }
  }
}

// Qt[i * RQ + r] = Q[i + ldq * r] (r < R), 0 for R <= r < RQ: the TMA-friendly panel copy.
__global__ void k_transpose_pad(const double* __restrict__ Q, int64_t ldq, int I, int R, int RQ,
                                double* __restrict__ Qt) {
  const int64_t n = (int64_t)I * RQ;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / RQ), r = (int)(e - (int64_t)i * RQ);
    Qt[e] = (r < R) ? Q[i + ldq * r] : 0.0;
  }
}

}  // namespace cpqr
