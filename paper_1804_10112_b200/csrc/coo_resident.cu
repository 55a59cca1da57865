// coo_resident.cu — K1s: COO SpMV on unconverted coordinates for matrices
// whose per-SM share of (rows, cols, vals) fits in shared memory.
//
// Reference semantics as in spmv.cu (engine.py:636-713 run_fused over the COO
// chain, _ScatterWriter engine.py:281-320): y[i] = ((+0.0 + a1*x1) + a2*x2) ...
// in storage order, one rounding per product and per sum; rows without
// nonzeros are zero.  One thread carries each row's sum, so y is bit-identical.
//
// B200 design.  A small matrix (D1: 2M nonzeros, 32 MB of coordinates and
// values) is a ~5 us stream; tiled kernels spend more than that ramping up and
// draining (K1: 1024-nonzero tiles, K2r behind a row-pointer pass: 18-20 us).
// Here the nonzeros are cut into one contiguous range per SM and each CTA
// (1024 threads, one per SM) asks for its WHOLE range at kernel start: a few
// large bulk copies (TMA) per array into ~216 KB of shared memory, one
// mbarrier per 2048-element chunk, so HBM sees 148 x 216 KB in flight from the
// first microsecond.  As chunks land, every thread gathers x for two of the
// chunk's elements and overwrites the staged value with the product (the
// gathers of chunk c stay in flight while chunk c + 1 is awaited).  After one
// block barrier each thread walks a slice of ~14 consecutive elements and sums
// the rows that START in its slice in storage order, reading on through the
// following slices to the row's end; leading elements of a row started earlier
// are skipped.  A 32-element halo past the CTA's range is staged too, so a row
// cut by the range end is finished from shared memory by its owner (longer
// rows continue from global memory).  No row pointer, no workspace, no second
// kernel: the coordinates are read once.
//
// MEASURED AND NOT CHOSEN (A/B build only; SL_COO_KERNEL=res): D1 26.5 us
// against 18.4 us for the row-pointer pass + K2r.  Per-CTA timestamps
// (tools/cr_timing.py, SL_CR_TIMING): all seven chunks are in shared memory
// 2.5 us after the kernel starts when nothing else runs, but the products are
// done only at 17.5 us — the 13.5K random x gathers per SM run at 0.46 per
// clock, half the rate calibrated with the whole L1 available, because the
// 229 KB stage leaves ~27 KB of L1 for the gathers' outstanding misses (and
// gathers issued while chunks are still landing delay those chunks to 15 us);
// the slice walk adds 4.5 us.  profiles/r2_ab_coo_resident.txt.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "tma.cuh"

namespace sl {

constexpr int kCrThreads = 1024;
constexpr int kCrChunk = 2048;                    // elements per arrival barrier
constexpr int kCrMaxChunks = 7;
constexpr int kCrCap = kCrChunk * kCrMaxChunks;   // staged elements (range + halo): 14,336
constexpr int kCrHalo = 32;
constexpr int kCrHeader = 128;                    // mbarriers
#ifndef SL_CR_BATCH
#define SL_CR_BATCH 7
#endif
constexpr int kCrBatch = SL_CR_BATCH;             // gathers a thread issues together

SL_DEV double ldx(const double* p) {
#if defined(SL_CR_NOALLOC)
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#else
  return ldg(p);
#endif
}

#ifdef SL_CR_TIMING
// A/B build only: per-CTA phase timestamps (globaltimer ns): 0 start, 1..7 chunk
// arrivals (thread 0), 8 products done, 9 thread 0's slice done
__device__ unsigned long long g_cr_t[160 * 12];
SL_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CR_T(i) do { if (tid == 0) g_cr_t[blockIdx.x * 12 + (i)] = gtime(); } while (0)
#else
#define CR_T(i) do { } while (0)
#endif

__global__ void __launch_bounds__(kCrThreads, 1)
spmv_coo_resident_kernel(int64_t nrows, int64_t nnz, int32_t per_cta, int32_t cap,
                         const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                         const double* __restrict__ vals, const double* __restrict__ x,
                         double* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double* s_val = reinterpret_cast<double*>(smem_raw + kCrHeader);
  int32_t* s_row = reinterpret_cast<int32_t*>(s_val + cap);
  int32_t* s_col = s_row + cap;
  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * per_cta;
  const int n = (int)min64(per_cta, nnz - e0);               // owned elements (row starts)
  const int n_st = (int)min64(per_cta + kCrHalo, nnz - e0);  // staged elements
  const int nch = (n_st + kCrChunk - 1) / kCrChunk;
  int32_t prev0 = -1;                                        // row of the element before the range
  CR_T(0);
  if (tid == 0) {
    for (int c = 0; c < nch; ++c) mbar_init(&bar[c], 1);
    fence_mbar_init();
    for (int c = 0; c < nch; ++c) {
      const int c0 = c * kCrChunk;
      const int cn = min(kCrChunk, n_st - c0);
      // whole 16-byte granules (the last chunk of the last range may read up
      // to 12 bytes past nnz inside the array's last granule, never used)
      const uint32_t bi = (uint32_t)((cn + 3) & ~3) * 4u, bd = (uint32_t)((cn + 1) & ~1) * 8u;
      mbar_arrive_expect_tx(&bar[c], 2u * bi + bd);
      bulk_g2s(s_row + c0, rows + e0 + c0, bi, &bar[c]);
      bulk_g2s(s_col + c0, cols + e0 + c0, bi, &bar[c]);
      bulk_g2s(s_val + c0, vals + e0 + c0, bd, &bar[c]);
    }
    if (e0 > 0) prev0 = ldg(rows + e0 - 1);
  }
  __syncthreads();                                           // barriers initialised
#ifdef SL_CR_TIMING
  if (tid == 0)
    for (int c = 0; c < nch; ++c) {
      mbar_wait(&bar[c], 0);
      CR_T(1 + c);
    }
#endif

  // ---- products in place as the copies land: thread t owns elements t, t + 1024, ...;
  // the gathers of a batch of kCrBatch elements are issued together and stay in
  // flight while the next batch's chunks are awaited and its gathers issued
#ifdef SL_CR_WAITALL
  for (int c = 0; c < nch; ++c) mbar_wait(&bar[c], 0);
#endif
  double xv[kCrBatch];
#pragma unroll
  for (int u = 0; u < kCrBatch; ++u) xv[u] = 0.0;
  const int nb = (n_st + kCrBatch * kCrThreads - 1) / (kCrBatch * kCrThreads);
  for (int b = 0; b <= nb; ++b) {
    double xn[kCrBatch];
#pragma unroll
    for (int u = 0; u < kCrBatch; ++u) xn[u] = 0.0;
    if (b < nb) {
#pragma unroll
      for (int u = 0; u < kCrBatch; ++u) {
        const int q = (b * kCrBatch + u) * kCrThreads + tid;
        if (q < n_st) {
#ifndef SL_CR_WAITALL
          mbar_wait(&bar[q / kCrChunk], 0);
#endif
          xn[u] = ldx(x + s_col[q]);
        }
      }
    }
    if (b > 0) {
#pragma unroll
      for (int u = 0; u < kCrBatch; ++u) {
        const int q = ((b - 1) * kCrBatch + u) * kCrThreads + tid;
        if (q < n_st) s_val[q] = dmul(s_val[q], xv[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kCrBatch; ++u) xv[u] = xn[u];
  }
  __syncthreads();
  CR_T(8);

  // ---- slices: each thread sums the rows starting in its slice, in storage
  // order.  One flat loop over the elements from the slice start, everything
  // predicated, so a warp's 32 walks stay converged (nested per-row loops
  // left ~3 of 32 threads active: ncu, 10M of the kernel's 12M instructions).
  const int S = ((n + kCrThreads - 1) / kCrThreads) | 1;     // odd stride: conflict-free walks
  const int s0 = tid * S;
  if (s0 >= n) return;
  const int s1 = min(n, s0 + S);
  int32_t rprev = s0 == 0 ? prev0 : s_row[s0 - 1];
  bool own = false;                   // accumulating a row that started in this slice
  int32_t rc = 0;
  double acc = 0.0;
  for (int u = s0; u < n_st; ++u) {
    if (!own && u >= s1) break;       // nothing of this slice left to finish
    const int32_t r = s_row[u];
    const double p = s_val[u];
    if (r != rprev) {                 // a row starts at u
      if (own) y[rc] = acc;
      own = u < s1;
      if (!own) break;                // the next slice's row
      for (int32_t z = rprev + 1; z < r; ++z) y[z] = 0.0;     // empty rows before r
      rc = r;
      rprev = r;
      acc = 0.0;
    }
    if (own) acc = dadd(acc, p);
  }
  CR_T(9);
  if (!own) return;
  // still inside its row at the end of the stage: the rest from global memory
  int64_t g = e0 + n_st;
  while (g < nnz && ldg(rows + g) == rc) {
    acc = dadd(acc, dmul(ldg(vals + g), ldg(x + ldg(cols + g))));
    ++g;
  }
  y[rc] = acc;
  if (g == nnz)                                               // the matrix's last row
    for (int64_t z = (int64_t)rc + 1; z < nrows; ++z) y[z] = 0.0;
}

}  // namespace sl

using namespace sl;

#ifdef SL_CR_TIMING
extern "C" int sl_debug_coo_resident_times(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_cr_t, sizeof(unsigned long long) * 160 * 12);
}
#endif

// Launches K1s when the matrix fits (nnz <= SMs x (kCrCap - kCrHalo)) and the
// arrays are 16-byte aligned; returns false (nothing launched) otherwise.
bool sl_host::launch_coo_resident(int64_t nrows, int64_t nnz, const int32_t* rows,
                                  const int32_t* cols, const double* vals, const double* x,
                                  double* y, cudaStream_t s) {
  if (nnz <= 0 || !aligned16(rows) || !aligned16(cols) || !aligned16(vals)) return false;
  const int sms = sm_count();
  int64_t per = (nnz + sms - 1) / sms;
  if (per < kCrChunk) per = kCrChunk;          // small inputs: fewer, fuller ranges
  per = (per + 3) & ~int64_t(3);               // 16-byte aligned range starts
  if (per > kCrCap - kCrHalo) return false;
  const int cap = (int)((per + kCrHalo + 3) & ~int64_t(3));
  const size_t smem = kCrHeader + (size_t)cap * 16;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_set[dev]) {
    cudaFuncSetAttribute(spmv_coo_resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kCrHeader + kCrCap * 16);
    attr_set[dev] = true;
  }
  const int grid = (int)((nnz + per - 1) / per);
  spmv_coo_resident_kernel<<<grid, kCrThreads, smem, s>>>(nrows, nnz, (int32_t)per, cap, rows,
                                                         cols, vals, x, y);
  return true;
}
