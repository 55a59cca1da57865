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
                const double* __restrict__ X, double* __restrict__ Y) {
  constexpr int kRowsPerWarp = 32 / G;
  const int lane = threadIdx.x & 31;
  const int g = lane / G, gl = lane % G;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w * kRowsPerWarp < nrows; w += nwarps) {
    const int64_t row = w * kRowsPerWarp + g;
    const bool live = row < nrows;
    const int32_t b = live ? ldg(pos + row) : 0, e = live ? ldg(pos + row + 1) : 0;
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

}  // namespace sl

using namespace sl;
using sl_host::as_stream;
using sl_host::ceil_div;

extern "C" int sl_spmm_csr_f64(int64_t nrows, int64_t ncols, int64_t K, const int32_t* pos,
                               const int32_t* crd, const double* vals, const double* X, double* Y,
                               void* stream) {
  if (nrows < 0 || ncols < 0 || K < 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || ncols > INT32_MAX || K > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0 || K == 0) return SL_OK;
  if (!pos || !Y || (ncols > 0 && !X)) return SL_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  const int G = K >= 32 ? 32 : (K > 8 ? 16 : (K > 4 ? 8 : (K > 2 ? 4 : (K > 1 ? 2 : 1))));
  const int64_t rows_per_block = 8 * (32 / G);
  const int grid = (int)std::min<int64_t>(ceil_div(nrows, rows_per_block),
                                          (int64_t)sl_host::sm_count() * 64);
  switch (G) {
    case 32: spmm_csr_kernel<32><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y); break;
    case 16:   // gathers 2 at a time: 122.9 us vs 130.0 / 133.4 / 244.0 us with 4 / 8 / 16
               // (64^3 stencil, K = 16: throughput-, not latency-bound; tools/ab_spmm.py)
      spmm_csr_kernel<16, 2><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y);
      break;
    case 8: spmm_csr_kernel<8><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y); break;
    case 4: spmm_csr_kernel<4><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y); break;
    case 2: spmm_csr_kernel<2><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y); break;
    default: spmm_csr_kernel<1><<<grid, 256, 0, s>>>(nrows, K, pos, crd, vals, X, Y); break;
  }
  return sl_host::launch_status();
}
