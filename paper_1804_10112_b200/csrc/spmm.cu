// spmm.cu — Y(i,k) = A(i,j) * X(j,k): A CSR, X and Y dense row-major
// (the paper's SpDM kernel on the same level structs).
//
// Reference: the loop nest (i, j, k) with Y located densely and the scatter
// writer (engine.py:591-634, 281-320): every Y(i,k) receives A(i,j)*X(j,k)
// for the row's j in storage order, accumulated from +0.0.  The kernel keeps
// that order per output element (one lane owns Y(i,k) for the whole row) and
// uses __dmul_rn/__dadd_rn (no contraction), so Y is bit-identical.
//
// Layout: a group of G lanes (G = the power of two >= K, at most 32) owns a
// row; lane l of the group owns columns k = l, l + G, ...  The row's column
// indices and values are read G at a time by the group (coalesced) and
// broadcast with shuffles; each nonzero then costs one K-wide row gather of X
// (256 B for K = 32, one sector per 4 columns) — X rows are the reuse target
// of L1/L2 on banded matrices.
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <algorithm>

#include "common.cuh"

namespace sl {

template <int G, int kB = 4>
__global__ void __launch_bounds__(256)
spmm_csr_kernel(int64_t nrows, int64_t K, const int32_t* __restrict__ pos,
                const int32_t* __restrict__ crd, const double* __restrict__ vals,
                const double* __restrict__ X, double* __restrict__ Y,
                int32_t long_min = INT32_MAX) {
  constexpr int kRowsPerWarp = 32 / G;
  const int lane = threadIdx.x & 31;
  const int g = lane / G, gl = lane % G;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w * kRowsPerWarp < nrows; w += nwarps) {
    const int64_t row = w * kRowsPerWarp + g;
    const int32_t b = row < nrows ? ldg(pos + row) : 0;
    int32_t e = row < nrows ? ldg(pos + row + 1) : 0;
    // rows longer than long_min belong to spmm_long_rows_kernel
    const bool live = row < nrows && e - b <= long_min;
    if (!live) e = b;
    for (int64_t k0 = 0; k0 < K; k0 += G) {
      const int64_t k = k0 + gl;
      const bool kin = live && k < K;
      double acc = 0.0;
      // the group walks its row; lanes of the group load the row's entries
      // G at a time and broadcast them inside the group
      for (int32_t c0 = b; c0 < e; c0 += G) {
        const int32_t q = c0 + gl;
        const int32_t cq = q < e ? ldg(crd + q) : 0;
        const double vq = q < e ? ldg(vals + q) : 0.0;
        const int n = min(G, e - c0);
        const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (g * G));
        int u = 0;
        for (; u + kB <= n; u += kB) {
          int32_t c[kB];
          double a[kB], xv[kB];
#pragma unroll
          for (int t = 0; t < kB; ++t) {
            c[t] = __shfl_sync(gmask, cq, u + t, G);
            a[t] = __shfl_sync(gmask, vq, u + t, G);
          }
#pragma unroll
          for (int t = 0; t < kB; ++t) xv[t] = kin ? ldg(X + (int64_t)c[t] * K + k) : 0.0;
#pragma unroll
          for (int t = 0; t < kB; ++t) acc = dadd(acc, dmul(a[t], xv[t]));
        }
        for (; u < n; ++u) {
          const int32_t c = __shfl_sync(gmask, cq, u, G);
          const double a = __shfl_sync(gmask, vq, u, G);
          const double xv = kin ? ldg(X + (int64_t)c * K + k) : 0.0;
          acc = dadd(acc, dmul(a, xv));
        }
      }
      if (kin) Y[row * K + k] = acc;
    }
  }
}

// Two columns per lane (K even, X and Y 16-byte aligned): a group of G lanes
// covers 2G columns with one 16-byte load per lane and nonzero, so a K = 16
// row gather is 8 lanes and a warp walks four rows at once — half the
// shuffles, loads and loop instructions per nonzero of the kernel above, which
// ncu shows issue-bound (the 64^3 stencil, K = 16: 34M warp instructions).
// The next G entries of the row are loaded while the current ones are used.
// Same order per output element: acc = dadd(acc, dmul(a, x)) over the row in
// storage order, so Y is bit-identical.
SL_DEV double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

#ifndef SL_SPMM_KB
#define SL_SPMM_KB 4
#endif
template <int G, int kB = SL_SPMM_KB, int kE = 2>
__global__ void __launch_bounds__(256)
spmm_csr_vec2_kernel(int64_t nrows, int64_t K, const int32_t* __restrict__ pos,
                     const int32_t* __restrict__ crd, const double* __restrict__ vals,
                     const double* __restrict__ X, double* __restrict__ Y,
                     int32_t long_min = INT32_MAX) {
  constexpr int kRowsPerWarp = 32 / G;
  constexpr int kChunk = kE * G;          // row entries per load step (kE per lane)
  const int lane = threadIdx.x & 31;
  const int g = lane / G, gl = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (g * G));
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w * kRowsPerWarp < nrows; w += nwarps) {
    const int64_t row = w * kRowsPerWarp + g;
    const int32_t b = row < nrows ? ldg(pos + row) : 0;
    int32_t e = row < nrows ? ldg(pos + row + 1) : 0;
    const bool live = row < nrows && e - b <= long_min;   // longer rows: spmm_long_rows_kernel
    if (!live) e = b;
    for (int64_t k0 = 0; k0 < K; k0 += 2 * G) {
      const int64_t k = k0 + 2 * gl;
      const bool kin = live && k < K;
      double acc0 = 0.0, acc1 = 0.0;
      int32_t cq[kE];
      double vq[kE];
#pragma unroll
      for (int h = 0; h < kE; ++h) {
        const int32_t q = b + h * G + gl;
        cq[h] = q < e ? ldg(crd + q) : 0;
        vq[h] = q < e ? ldg(vals + q) : 0.0;
      }
      for (int32_t c0 = b; c0 < e; c0 += kChunk) {
        int32_t cn[kE];
        double vn[kE];
#pragma unroll
        for (int h = 0; h < kE; ++h) {
          cn[h] = cq[h];
          vn[h] = vq[h];
          const int32_t q = c0 + kChunk + h * G + gl;      // the next chunk, in flight
          cq[h] = q < e ? ldg(crd + q) : 0;
          vq[h] = q < e ? ldg(vals + q) : 0.0;
        }
#pragma unroll
        for (int h = 0; h < kE; ++h) {
          const int n = min(G, e - c0 - h * G);             // entries of this register (<= 0: none)
          int u = 0;
          for (; u + kB <= n; u += kB) {
            int32_t c[kB];
            double a[kB];
            double2 xv[kB];
#pragma unroll
            for (int t = 0; t < kB; ++t) {
              c[t] = __shfl_sync(gmask, cn[h], u + t, G);
              a[t] = __shfl_sync(gmask, vn[h], u + t, G);
            }
#pragma unroll
            for (int t = 0; t < kB; ++t)
              xv[t] = kin ? ldg2(X + (int64_t)c[t] * K + k) : make_double2(0.0, 0.0);
#pragma unroll
            for (int t = 0; t < kB; ++t) {
              acc0 = dadd(acc0, dmul(a[t], xv[t].x));
              acc1 = dadd(acc1, dmul(a[t], xv[t].y));
            }
          }
          for (; u < n; ++u) {
            const int32_t c = __shfl_sync(gmask, cn[h], u, G);
            const double a = __shfl_sync(gmask, vn[h], u, G);
            const double2 xv = kin ? ldg2(X + (int64_t)c * K + k) : make_double2(0.0, 0.0);
            acc0 = dadd(acc0, dmul(a, xv.x));
            acc1 = dadd(acc1, dmul(a, xv.y));
          }
        }
      }
      if (kin) *reinterpret_cast<double2*>(Y + row * K + k) = make_double2(acc0, acc1);
    }
  }
}

// Rows longer than long_min, listed by spmm_mark_long_kernel: one CTA per
// row.  A lone group walking a power-law row keeps only kB gathers in flight
// per lane, so a 10^5-nonzero row costs ~10^5/kB dependent gather latencies.
// Here all eight warps gather a chunk of the row's X rows — a warp covers
// 32/G nonzeros x G columns per step, kPer steps — and form the products A(i,j)*X(j,k) in shared
// memory; then warp 0 (lane l < G owning column k0 + l) adds them in storage
// order.  dadd(acc, dmul(a, x)) in the same order as the group kernel:
// bit-identical.  The add chain (one dependent dadd per nonzero per column)
// is the floor the ordered sum imposes.
template <int G, int kPer>
__global__ void __launch_bounds__(256)
spmm_long_rows_kernel(int64_t K, const int32_t* __restrict__ pos, const int32_t* __restrict__ crd,
                      const double* __restrict__ vals, const double* __restrict__ X,
                      double* __restrict__ Y, const int32_t* __restrict__ list,
                      const int32_t* __restrict__ count) {
  constexpr int kRows = 32 / G, kChunk = 8 * kRows * kPer;
  extern __shared__ double smem_p[];
  double(*P)[G + 1] = reinterpret_cast<double(*)[G + 1]>(smem_p);  // +1: conflict-free columns
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gl = lane % G, gr = lane / G;
  const int n = *count;
  for (int li = blockIdx.x; li < n; li += gridDim.x) {
    const int64_t row = list[li];
    const int32_t b = ldg(pos + row), e = ldg(pos + row + 1);
    for (int64_t k0 = 0; k0 < K; k0 += G) {
      const int64_t k = k0 + gl;
      const int64_t kc = k < K ? k : K - 1;          // in-bounds column for idle lanes
      double acc = 0.0;
      for (int32_t c0 = b; c0 < e; c0 += kChunk) {
        const int nc = min(kChunk, e - c0);
        int32_t c[kPer];
        double a[kPer], xv[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int t = (warp + 8 * u) * kRows + gr;
          const int tt = min(t, nc - 1);
          c[u] = ldg(crd + c0 + tt);
          a[u] = ldg(vals + c0 + tt);
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) xv[u] = ldg(X + (int64_t)c[u] * K + kc);
#pragma unroll
        for (int u = 0; u < kPer; ++u) P[(warp + 8 * u) * kRows + gr][gl] = dmul(a[u], xv[u]);
        __syncthreads();
        if (warp == 0 && lane < G) {
          int t = 0;
          for (; t + 4 <= nc; t += 4) {
            const double p0 = P[t][lane], p1 = P[t + 1][lane], p2 = P[t + 2][lane],
                         p3 = P[t + 3][lane];
            acc = dadd(dadd(dadd(dadd(acc, p0), p1), p2), p3);
          }
          for (; t < nc; ++t) acc = dadd(acc, P[t][lane]);
        }
        __syncthreads();
      }
      if (warp == 0 && lane < G && k < K) Y[row * K + k] = acc;
    }
  }
}

__global__ void spmm_mark_long_kernel(int64_t nrows, const int32_t* __restrict__ pos,
                                      int32_t long_min, int32_t* __restrict__ list,
                                      int32_t* __restrict__ count) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x)
    if (ldg(pos + r + 1) - ldg(pos + r) > long_min) list[atomicAdd(count, 1)] = (int32_t)r;
}

}  // namespace sl

using namespace sl;
using sl_host::as_stream;
using sl_host::ceil_div;

namespace {

int spmm_launch(int64_t nrows, int64_t ncols, int64_t K, const int32_t* pos, const int32_t* crd,
                const double* vals, const double* X, double* Y, int32_t long_min,
                cudaStream_t s, int64_t nnz = -1) {
  // Even K >= 8, 16-byte aligned X and Y, rows averaging >= 16 nonzeros: two
  // columns per lane (64^3 stencil, K = 8 / 16 / 32: 76.2 / 115.9 / 204.7 ->
  // 55.7 / 92.2 / 152.7 us).  Short ragged rows stay with one column per lane:
  // a warp walking four rows waits for the longest (D1, K = 16: 56.9 us there,
  // 61.8 us here).  Gathers in flight per lane 1 / 2 / 4 / 8: 123.0 / 96.9 /
  // 92.2 / 104.4 us (K = 16).  A/B knob SL_SPMM_VEC2=0 / 1 (1: whatever the rows).
  static const int vec2_knob = [] {
    const char* e = getenv("SL_SPMM_VEC2");
    return e ? (e[0] == '0' ? 0 : 2) : 1;
  }();
  const bool rows_ok = vec2_knob == 2 || (nnz >= 0 && nnz >= 16 * nrows);
  if (vec2_knob && rows_ok && K >= 8 && K % 2 == 0 && sl_host::aligned16(X) &&
      sl_host::aligned16(Y)) {
    const int G2 = K > 32 ? 32 : (K > 16 ? 16 : (K > 8 ? 8 : 4));
    const int64_t rpb = 8 * (32 / G2);
    const int grid2 = (int)std::min<int64_t>(ceil_div(nrows, rpb), (int64_t)sl_host::sm_count() * 64);
    switch (G2) {
      case 32: spmm_csr_vec2_kernel<32><<<grid2, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y, long_min); break;
      case 16: spmm_csr_vec2_kernel<16><<<grid2, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y, long_min); break;
      case 8: spmm_csr_vec2_kernel<8><<<grid2, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y, long_min); break;
      default: spmm_csr_vec2_kernel<4><<<grid2, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y, long_min); break;
    }
    return sl_host::launch_status();
  }
  const int G = K >= 32 ? 32 : (K > 8 ? 16 : (K > 4 ? 8 : (K > 2 ? 4 : (K > 1 ? 2 : 1))));
  const int64_t rows_per_block = 8 * (32 / G);
  const int grid = (int)std::min<int64_t>(ceil_div(nrows, rows_per_block),
                                          (int64_t)sl_host::sm_count() * 64);
  switch (G) {
    case 32: spmm_csr_kernel<32><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y, long_min); break;
    case 16:   // gathers 2 at a time: 122.9 us vs 130.0 / 133.4 / 244.0 us with 4 / 8 / 16
               // (64^3 stencil, K = 16: throughput-, not latency-bound; tools/ab_spmm.py)
      spmm_csr_kernel<16, 2><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y, long_min);
      break;
    case 8: spmm_csr_kernel<8><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y, long_min); break;
    case 4: spmm_csr_kernel<4><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y, long_min); break;
    case 2: spmm_csr_kernel<2><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y, long_min); break;
    default: spmm_csr_kernel<1><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y, long_min); break;
  }
  return sl_host::launch_status();
}

int spmm_check(int64_t nrows, int64_t ncols, int64_t K, const int32_t* pos, const double* X,
               double* Y) {
  if (nrows < 0 || ncols < 0 || K < 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || ncols > INT32_MAX || K > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0 || K == 0) return SL_OK;
  if (!pos || !Y || (ncols > 0 && !X)) return SL_ERR_INVALID;
  return -1;
}

}  // namespace

extern "C" int sl_spmm_csr_f64(int64_t nrows, int64_t ncols, int64_t K, const int32_t* pos,
                               const int32_t* crd, const double* vals, const double* X, double* Y,
                               void* stream) {
  const int st = spmm_check(nrows, ncols, K, pos, X, Y);
  if (st >= 0) return st;
  return spmm_launch(nrows, ncols, K, pos, crd, vals, X, Y, INT32_MAX, as_stream(stream));
}

extern "C" int sl_spmm_csr_nnz_f64(int64_t nrows, int64_t ncols, int64_t K, int64_t nnz,
                                   const int32_t* pos, const int32_t* crd, const double* vals,
                                   const double* X, double* Y, void* stream) {
  const int st = spmm_check(nrows, ncols, K, pos, X, Y);
  if (st >= 0) return st;
  return spmm_launch(nrows, ncols, K, pos, crd, vals, X, Y, INT32_MAX, as_stream(stream), nnz);
}

extern "C" int64_t sl_spmm_csr_split_workspace_bytes(int64_t nrows, int64_t nnz,
                                                     int32_t long_min) {
  if (nrows <= 0 || long_min < 0) return 0;
  const int64_t nlong = std::min<int64_t>(nrows, nnz / ((int64_t)long_min + 1) + 1);
  return 16 + 4 * nlong;
}

extern "C" int sl_spmm_csr_split_f64(int64_t nrows, int64_t ncols, int64_t K, int64_t nnz,
                                     const int32_t* pos, const int32_t* crd, const double* vals,
                                     const double* X, double* Y, int32_t long_min, void* ws,
                                     int64_t ws_bytes, void* stream) {
  const int st = spmm_check(nrows, ncols, K, pos, X, Y);
  if (st >= 0) return st;
  if (long_min < 0) return SL_ERR_INVALID;
  if (!ws || ws_bytes < sl_spmm_csr_split_workspace_bytes(nrows, nnz, long_min))
    return SL_ERR_WORKSPACE;
  cudaStream_t s = as_stream(stream);
  int32_t* count = static_cast<int32_t*>(ws);
  int32_t* list = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + 16);
  if (cudaMemsetAsync(count, 0, sizeof(int32_t), s) != cudaSuccess) return SL_ERR_CUDA;
  spmm_mark_long_kernel<<<std::min<int64_t>(ceil_div(nrows, 256), 8LL * sl_host::sm_count()), 256,
                          0, s>>>(nrows, pos, long_min, list, count);
  int rc = sl_host::launch_status();
  if (rc != SL_OK) return rc;
  rc = spmm_launch(nrows, ncols, K, pos, crd, vals, X, Y, long_min, s, nnz);
  if (rc != SL_OK) return rc;
  const int64_t nlong = std::min<int64_t>(nrows, nnz / ((int64_t)long_min + 1) + 1);
  const int lgrid = (int)std::min<int64_t>(nlong, 4LL * sl_host::sm_count());
  // chunk depth: 32 loads per lane for G <= 16, 24 for G = 32 (the giant-row
  // time is per-chunk gather latency; measured in round 1 with
  // tools/spmm_skew_prof.py, log not retained)
  auto go = [&](auto kern, int g, int per) {
    const size_t smem = (size_t)8 * (32 / g) * per * (g + 1) * sizeof(double);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
      return;
    kern<<<lgrid, 256, smem, s>>>(K, pos, crd, vals, X, Y, list, count);
  };
  if (K > 16) go(spmm_long_rows_kernel<32, 24>, 32, 24);
  else if (K > 8) go(spmm_long_rows_kernel<16, 32>, 16, 32);
  else if (K > 4) go(spmm_long_rows_kernel<8, 32>, 8, 32);
  else go(spmm_long_rows_kernel<4, 32>, 4, 32);
  return sl_host::launch_status();
}
