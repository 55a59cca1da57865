// tensor3.cu — the paper's 3-tensor kernels beyond MTTKRP
// on the same CSF / COO-3 level structs:
//   TTV     Y(i,j)   = X(i,j,k) * v(k)     (dense or CSR output)
//   TTM     Y(i,j,r) = X(i,j,k) * U(k,r)   (dense output)
//   INNER   a()      = X(i,j,k) * Z(i,j,k) (scalar)
//
// TTV and TTM reduce over k only, inside each (i, j) fiber of a CSF tensor:
// the fiber sums are exactly a CSR SpMV (TTV) or SpMM (TTM) whose rows are
// the fibers (pos2 / crd2 / vals), run by the row-block SpMV and SpMM kernels
// (bit-identical ordered sums).  This file adds the pieces around them: the
// scatter of per-fiber rows into the dense output (absent fibers 0.0), and the
// row pointer of the CSR output (gather writer, engine.py:330-434: one entry
// per fiber, rows = slices).
//
// INNER intersects two sorted COO-3 tensors (merge_visits at every level,
// engine.py:211-225).  The reference reduces per fiber, then per slice, then
// overall; this kernel reduces per tile of X in a fixed tree order, so the
// result is deterministic and within the fp64-reduction tolerance (rtol 1e-12
// condition-scaled) of the reference.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace sl {

// slice s holding fiber f: pos1[s] <= f < pos1[s + 1]
SL_DEV int64_t slice_of(const int32_t* __restrict__ pos1, int64_t nslices, int64_t f) {
  int64_t lo = 0, hi = nslices - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (ldg(pos1 + mid) <= f) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void fill_zero_kernel3(double* __restrict__ a, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = 0.0;
}

// out[(crd0[s] * J + crd1[f]) * R + r] = rows[f * R + r]
__global__ void fiber_scatter_kernel(int64_t J, int64_t R, int64_t nslices, int64_t nfibers,
                                     const int32_t* __restrict__ crd0,
                                     const int32_t* __restrict__ pos1,
                                     const int32_t* __restrict__ crd1,
                                     const double* __restrict__ rows, double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nfibers * R; t += stride) {
    const int64_t f = t / R, r = t - f * R;
    const int64_t s = slice_of(pos1, nslices, f);
    out[((int64_t)ldg(crd0 + s) * J + ldg(crd1 + f)) * R + r] = ldg(rows + t);
  }
}

// CSR row pointer over i of the fiber structure: pos_out[i] = first fiber of
// the first slice with crd0 >= i
__global__ void fiber_rowptr_kernel(int64_t I, int64_t nslices, const int32_t* __restrict__ crd0,
                                    const int32_t* __restrict__ pos1, int32_t* __restrict__ pos_out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= I; i += stride) {
    int64_t lo = 0, hi = nslices;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ldg(crd0 + mid) < i) lo = mid + 1; else hi = mid;
    }
    pos_out[i] = ldg(pos1 + lo);
  }
}

// ---- inner product ----------------------------------------------------------
constexpr int kInThreads = 256;
constexpr int kInIpt = 8;
constexpr int kInTile = kInThreads * kInIpt;
constexpr int kInZCap = 4096;    // Z keys staged per tile (a power of two)

SL_DEV int64_t key3(const int32_t* i, const int32_t* j, const int32_t* k, int64_t p, int64_t J,
                    int64_t K) {
  return ((int64_t)ldg(i + p) * J + ldg(j + p)) * K + ldg(k + p);
}

// block b: partial[b] = sum over its X tile of x * z where Z holds the same
// coordinate (binary search over Z's keys; a repeated Z coordinate summed),
// reduced in a fixed tree order
__global__ void __launch_bounds__(kInThreads)
inner_tile_kernel(int64_t J, int64_t K, int64_t nx, const int32_t* __restrict__ xi,
                  const int32_t* __restrict__ xj, const int32_t* __restrict__ xk,
                  const double* __restrict__ xv, int64_t nz, const int32_t* __restrict__ zi,
                  const int32_t* __restrict__ zj, const int32_t* __restrict__ zk,
                  const double* __restrict__ zv, double* __restrict__ partial) {
  __shared__ double s_warp[kInThreads / 32];
  __shared__ int64_t s_zlo, s_zhi;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t e0 = (int64_t)blockIdx.x * kInTile;
  const int64_t e1 = min64(e0 + kInTile, nx);
  // the Z range that can match this tile: [lb(key(x[e0])), ub(key(x[e1 - 1])))
  // (warp 0: lower bound, warp 1: upper bound; a 32-ary search — each step the
  // warp probes 32 evenly spaced keys and keeps the one gap that can hold the
  // answer: 6 dependent rounds over Z instead of a thread's 26)
  if (warp < 2) {
    const int64_t target = key3(xi, xj, xk, warp == 0 ? e0 : e1 - 1, J, K);
    int64_t lo = 0, hi = nz;
    while (hi > lo) {
      const int64_t span = hi - lo;
      const int64_t p = lo + (span * lane) / 32;
      const int64_t km = key3(zi, zj, zk, p, J, K);
      const int c = __popc(__ballot_sync(0xffffffffu, warp == 0 ? km < target : km <= target));
      const int64_t nlo = c > 0 ? lo + (span * (c - 1)) / 32 + 1 : lo;
      hi = c < 32 ? lo + (span * c) / 32 : hi;
      lo = nlo;
    }
    if (lane == 0) {
      if (warp == 0) s_zlo = lo; else s_zhi = lo;
    }
  }
  __syncthreads();
  const int64_t zlo = s_zlo, zhi = s_zhi;
  double acc = 0.0;
  // Z's matching range usually is about as long as the tile: its keys are
  // staged in shared memory once (coalesced loads of the three coordinate
  // arrays) and every thread runs its kInIpt lower-bound searches there,
  // interleaved and branch-free (13 fixed steps of one 8-byte shared load each)
  // — D5 with itself 0.995 -> 0.732 ms, and 0.570 ms with the 32-ary boundary
  // search above; searching the global arrays cost three loads per probe.  Longer ranges fall through to the global search below.
  __shared__ int64_t s_zkey[kInZCap];
  const bool staged = zhi - zlo <= kInZCap;          // block-uniform
  if (staged) {
    const int nzr = (int)(zhi - zlo);
    for (int q = tid; q < nzr; q += kInThreads) s_zkey[q] = key3(zi, zj, zk, zlo + q, J, K);
    __syncthreads();
    int64_t kx[kInIpt];
    int pos[kInIpt];
#pragma unroll
    for (int t = 0; t < kInIpt; ++t) {
      const int64_t e = e0 + t * kInThreads + tid;
      kx[t] = e < e1 ? key3(xi, xj, xk, e, J, K) : INT64_MAX;
      pos[t] = 0;
    }
    for (int step = kInZCap; step > 0; step >>= 1) {
#pragma unroll
      for (int t = 0; t < kInIpt; ++t) {
        const int np = pos[t] + step;
        if (np <= nzr && s_zkey[np - 1] < kx[t]) pos[t] = np;
      }
    }
#pragma unroll
    for (int t = 0; t < kInIpt; ++t) {
      const int64_t e = e0 + t * kInThreads + tid;
      if (e < e1 && pos[t] < nzr && s_zkey[pos[t]] == kx[t]) {
        double gz = ldg(zv + zlo + pos[t]);          // Z's repeats: one grouped visit (below)
        for (int q = pos[t] + 1; q < nzr && s_zkey[q] == kx[t]; ++q) gz = dadd(gz, ldg(zv + zlo + q));
        acc = dadd(acc, dmul(ldg(xv + e), gz));
      }
    }
  }
#pragma unroll 1
  for (int t = 0; t < kInIpt && !staged; ++t) {
    const int64_t e = e0 + t * kInThreads + tid;
    if (e >= e1) break;
    const int64_t kx = key3(xi, xj, xk, e, J, K);
    int64_t lo = zlo, hi = zhi;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (key3(zi, zj, zk, mid, J, K) < kx) lo = mid + 1; else hi = mid;
    }
    if (lo < zhi && key3(zi, zj, zk, lo, J, K) == kx) {
      // Z's repeats of the coordinate are one grouped visit (engine.py:107-149,
      // 527): the product takes their sum (X's repeats each add their own
      // product — the same value up to reassociation, inside the reduction's
      // tolerance)
      double gz = ldg(zv + lo);
      for (int64_t q = lo + 1; q < zhi && key3(zi, zj, zk, q, J, K) == kx; ++q)
        gz = dadd(gz, ldg(zv + q));
      acc = dadd(acc, dmul(ldg(xv + e), gz));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = dadd(acc, __shfl_down_sync(0xffffffffu, acc, o));
  if (lane == 0) s_warp[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kInThreads / 32; ++w) s = dadd(s, s_warp[w]);
    partial[blockIdx.x] = s;
  }
}

// out = sum of the partials in a fixed order (one block)
__global__ void __launch_bounds__(1024)
inner_final_kernel(int64_t n, const double* __restrict__ partial, double* __restrict__ out) {
  __shared__ double s_warp[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double acc = 0.0;
  for (int64_t i = tid; i < n; i += 1024) acc = dadd(acc, partial[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = dadd(acc, __shfl_down_sync(0xffffffffu, acc, o));
  if (lane == 0) s_warp[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < 32; ++w) s = dadd(s, s_warp[w]);
    *out = s;
  }
}

}  // namespace sl

using namespace sl;
using sl_host::as_stream;
using sl_host::ceil_div;

extern "C" int sl_csf_fiber_scatter_f64(int64_t I, int64_t J, int64_t R, int64_t nslices,
                                        int64_t nfibers, const int32_t* crd0, const int32_t* pos1,
                                        const int32_t* crd1, const double* rows, double* out,
                                        void* stream) {
  if (I < 0 || J < 0 || R < 0 || nslices < 0 || nfibers < 0) return SL_ERR_INVALID;
  if (!out && I * J * R > 0) return SL_ERR_INVALID;
  if (nfibers > 0 && (!crd0 || !pos1 || !crd1 || !rows)) return SL_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  const int sms = sl_host::sm_count();
  const int64_t n = I * J * R;
  if (n > 0) fill_zero_kernel3<<<min(ceil_div(n, 256), 16 * sms), 256, 0, s>>>(out, n);
  if (nfibers > 0 && R > 0)
    fiber_scatter_kernel<<<min(ceil_div(nfibers * R, 256), 16 * sms), 256, 0, s>>>(
        J, R, nslices, nfibers, crd0, pos1, crd1, rows, out);
  return sl_host::launch_status();
}

extern "C" int sl_csf_fiber_rowptr(int64_t I, int64_t nslices, const int32_t* crd0,
                                   const int32_t* pos1, int32_t* pos_out, void* stream) {
  if (I < 0 || nslices < 0 || !pos_out || !pos1 || (nslices > 0 && !crd0)) return SL_ERR_INVALID;
  fiber_rowptr_kernel<<<min(ceil_div(I + 1, 256), 16 * sl_host::sm_count()), 256, 0,
                        as_stream(stream)>>>(I, nslices, crd0, pos1, pos_out);
  return sl_host::launch_status();
}

extern "C" size_t sl_inner_coo3_workspace_bytes(int64_t nx) {
  return (size_t)(ceil_div(nx, kInTile) + 1) * sizeof(double) + 256;
}

extern "C" int sl_inner_coo3_f64(int64_t I, int64_t J, int64_t K, int64_t nx, const int32_t* xi,
                                 const int32_t* xj, const int32_t* xk, const double* xv,
                                 int64_t nz, const int32_t* zi, const int32_t* zj,
                                 const int32_t* zk, const double* zv, double* out, void* ws,
                                 size_t ws_bytes, void* stream) {
  if (I < 0 || J < 0 || K < 0 || nx < 0 || nz < 0 || !out) return SL_ERR_INVALID;
  if (nx > 0 && (!xi || !xj || !xk || !xv)) return SL_ERR_INVALID;
  if (nz > 0 && (!zi || !zj || !zk || !zv)) return SL_ERR_INVALID;
  if (!ws || ws_bytes < sl_inner_coo3_workspace_bytes(nx)) return SL_ERR_WORKSPACE;
  cudaStream_t s = as_stream(stream);
  double* partial = static_cast<double*>(ws);
  const int64_t tiles = ceil_div(nx, kInTile);
  if (tiles > 0 && nz > 0) {
    inner_tile_kernel<<<(int)tiles, kInThreads, 0, s>>>(J, K, nx, xi, xj, xk, xv, nz, zi, zj, zk,
                                                        zv, partial);
    inner_final_kernel<<<1, 1024, 0, s>>>(tiles, partial, out);
  } else {
    fill_zero_kernel3<<<1, 32, 0, s>>>(out, 1);
  }
  return sl_host::launch_status();
}
