// spmv.cu — y(i) = A(i,j) * x(j) for COO, CSR, ELL, DIA and CSR x hash-vector.
//
// Reference semantics ("Exact arithmetic"): every format
// computes y[i] = ((+0.0 + a_i,j1*x_j1) + a_i,j2*x_j2) + ... in storage order,
// one rounding per product and per sum (engine.py:303 zero-fill, :320 scatter
// +=, :606-633 CSR accumulation, :528-529 a*x).  All kernels here keep that
// order: products are formed in parallel (they are order-free), and each row's
// sum is carried by ONE thread in storage order, so y is bit-identical to the
// reference.  Rows are short in every BASELINE config (<= 27 for the stencils,
// Poisson(10) for D1), so the sequential add chain is off the critical path;
// the kernels are HBM-bound on the streamed index/value arrays.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "levels.cuh"

namespace sl {

// ---------------------------------------------------------------------------
// zero fill (nnz == 0 / empty rows beyond the last stored row)

__global__ void fill_zero_kernel(double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = 0.0;
}

// ---------------------------------------------------------------------------
// K1: COO SpMV on unconverted, row-sorted coordinates.
//
// A tile of kCooTile consecutive nonzeros is loaded coalesced (16-byte vector
// loads of rows/cols/vals), x is gathered, and the products land in shared
// memory.  Row starts inside the tile are compacted with a block scan; the
// thread that owns a row start sums that row in storage order and writes y
// once.  A row that runs past the tile end is finished by its owner from
// global memory (a few elements), so no carry-out/fix-up pass exists.  Rows
// with no nonzeros between two stored rows are zeroed by the owner of the
// later row's start: y needs no memset.  (engine.py:636-713 run_fused over the
// COO chain, _ScatterWriter engine.py:281-320.)

constexpr int kCooThreads = 256;
constexpr int kCooVec = 4;                       // elements per vector load
constexpr int kCooVecPerThread = 2;
constexpr int kCooIpt = kCooVec * kCooVecPerThread;  // 8 items per thread
constexpr int kCooTile = kCooThreads * kCooIpt;      // 2048 nonzeros per tile

__global__ void __launch_bounds__(kCooThreads)
spmv_coo_kernel(int64_t nrows, int64_t nnz, const int32_t* __restrict__ rows,
                const int32_t* __restrict__ cols, const double* __restrict__ vals,
                const double* __restrict__ x, double* __restrict__ y, bool vec_ok) {
  __shared__ __align__(16) int32_t s_row[kCooTile + 4];   // s_row[4 + q] = row of item q
  __shared__ __align__(16) double s_prod[kCooTile];
  __shared__ int32_t s_start[kCooTile];
  __shared__ int32_t s_warp[kCooThreads / 32];
  __shared__ int32_t s_nstart;

  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * kCooTile;
  const int n_in = (int)min64(kCooTile, nnz - e0);

  // ---- stage: rows + products (coalesced, vectorised on full tiles)
  if (vec_ok && n_in == kCooTile) {
    int4 r4[kCooVecPerThread], c4[kCooVecPerThread];
    double2 va[kCooVecPerThread], vb[kCooVecPerThread];
#pragma unroll
    for (int k = 0; k < kCooVecPerThread; ++k) {
      const int64_t g = e0 + (int64_t)(k * kCooThreads + tid) * kCooVec;
      r4[k] = ld_stream(reinterpret_cast<const int4*>(rows + g));
      c4[k] = ld_stream(reinterpret_cast<const int4*>(cols + g));
      va[k] = ld_stream(reinterpret_cast<const double2*>(vals + g));
      vb[k] = ld_stream(reinterpret_cast<const double2*>(vals + g + 2));
    }
#pragma unroll
    for (int k = 0; k < kCooVecPerThread; ++k) {
      const double x0 = ldg(x + c4[k].x), x1 = ldg(x + c4[k].y);
      const double x2 = ldg(x + c4[k].z), x3 = ldg(x + c4[k].w);
      const int q = (k * kCooThreads + tid) * kCooVec;
      *reinterpret_cast<int4*>(s_row + 4 + q) = r4[k];
      *reinterpret_cast<double2*>(s_prod + q) = make_double2(dmul(va[k].x, x0), dmul(va[k].y, x1));
      *reinterpret_cast<double2*>(s_prod + q + 2) = make_double2(dmul(vb[k].x, x2), dmul(vb[k].y, x3));
    }
  } else {
#pragma unroll 4
    for (int q = tid; q < n_in; q += kCooThreads) {
      const int64_t g = e0 + q;
      s_row[4 + q] = ld_stream(rows + g);
      s_prod[q] = dmul(ld_stream(vals + g), ldg(x + ld_stream(cols + g)));
    }
  }
  if (tid == 0) s_row[3] = e0 == 0 ? -1 : rows[e0 - 1];
  __syncthreads();

  // ---- compact row starts (q is a start iff row[q] != row[q-1])
  int flags = 0, cnt = 0;
  {
    const int q0 = tid * kCooIpt;
    int prev = s_row[3 + q0];
#pragma unroll
    for (int t = 0; t < kCooIpt; ++t) {
      const int q = q0 + t;
      if (q < n_in) {
        const int r = s_row[4 + q];
        if (r != prev) { flags |= 1 << t; ++cnt; }
        prev = r;
      }
    }
  }
  const int lane = tid & 31, warp = tid >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int v = lane < kCooThreads / 32 ? s_warp[lane] : 0;
    int sc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, sc, o);
      if (lane >= o) sc += u;
    }
    if (lane < kCooThreads / 32) s_warp[lane] = sc - v;   // exclusive warp offsets
    if (lane == kCooThreads / 32 - 1) s_nstart = sc;
  }
  __syncthreads();
  {
    int o = s_warp[warp] + incl - cnt;
#pragma unroll
    for (int t = 0; t < kCooIpt; ++t)
      if (flags & (1 << t)) s_start[o++] = tid * kCooIpt + t;
  }
  __syncthreads();

  // ---- owners: sum each row in storage order, zero the gap before it
  const int nstart = s_nstart;
  const bool last_tile = e0 + n_in == nnz;
  for (int s = tid; s < nstart; s += kCooThreads) {
    const int q = s_start[s];
    const int r = s_row[4 + q];
    const int rp = s_row[3 + q];
    const int qe = s + 1 < nstart ? s_start[s + 1] : n_in;
    double acc = 0.0;
    for (int u = q; u < qe; ++u) acc = dadd(acc, s_prod[u]);
    bool reached_end = last_tile && s + 1 == nstart;
    if (s + 1 == nstart && !last_tile) {
      // the row may continue into later tiles: finish it from global memory
      int64_t g = e0 + n_in;
      for (; g < nnz && ldg(rows + g) == r; ++g)
        acc = dadd(acc, dmul(ldg(vals + g), ldg(x + ldg(cols + g))));
      reached_end = g == nnz;
    }
    y[r] = acc;
    for (int rr = rp + 1; rr < r; ++rr) y[rr] = 0.0;
    if (reached_end)  // the matrix's last stored row: zero the empty rows after it
      for (int64_t rr = (int64_t)r + 1; rr < nrows; ++rr) y[rr] = 0.0;
  }
}

// ---------------------------------------------------------------------------
// K2a: CSR row-block SpMV.  A block owns kCsrRows consecutive rows; their
// nonzeros are a contiguous range, staged in coalesced chunks of kCsrChunk
// products through shared memory; the thread of row r adds the chunk's
// products that belong to r in storage order.  (engine.py:591-634.)

constexpr int kCsrThreads = 256;
constexpr int kCsrRows = kCsrThreads;
constexpr int kCsrChunk = 2048;

template <bool kHashX>
struct XOperand;

template <>
struct XOperand<false> {            // dense x: locate = parent*n + c (levels.py:268-269)
  const double* x;
  SL_DEV double term(double a, int32_t c) const { return dmul(a, ldg(x + c)); }
};

template <>
struct XOperand<true> {             // hashed x: probe (levels.py:270-280), miss -> no term
  HashedLevel lv;
  const double* xv;
  // A miss contributes no term.  The row accumulator starts at +0.0 and can
  // never become -0.0 under round-to-nearest, so "no term" == "+0.0 term".
  SL_DEV double term(double a, int32_t c) const {
    const PosFound pf = lv.locate(0, c);
    return pf.found ? dmul(a, ldg(xv + pf.pos)) : 0.0;
  }
};

template <bool kHashX>
__global__ void __launch_bounds__(kCsrThreads)
spmv_csr_rowblock_kernel(int64_t nrows, const int32_t* __restrict__ pos,
                         const int32_t* __restrict__ crd, const double* __restrict__ vals,
                         XOperand<kHashX> xop, double* __restrict__ y) {
  __shared__ int32_t s_pos[kCsrRows + 1];
  __shared__ __align__(16) double s_prod[kCsrChunk];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kCsrRows;
  const int nr = (int)min64(kCsrRows, nrows - r0);
  for (int t = tid; t <= nr; t += kCsrThreads) s_pos[t] = ldg(pos + r0 + t);
  __syncthreads();
  const int32_t eb = s_pos[0], ee = s_pos[nr];
  const bool mine = tid < nr;
  const int32_t rb = mine ? s_pos[tid] : 0, re = mine ? s_pos[tid + 1] : 0;
  double acc = 0.0;
  for (int32_t cs = eb; cs < ee; cs += kCsrChunk) {
    const int n_in = min(kCsrChunk, ee - cs);
#pragma unroll 8
    for (int q = tid; q < n_in; q += kCsrThreads)
      s_prod[q] = xop.term(ld_stream(vals + cs + q), ld_stream(crd + cs + q));
    __syncthreads();
    const int lo = max(rb, cs) - cs, hi = min(re, cs + n_in) - cs;
    for (int u = lo; u < hi; ++u) acc = dadd(acc, s_prod[u]);
    __syncthreads();
  }
  if (mine) y[r0 + tid] = acc;
}

// K2b: CSR vector-per-row.  One warp per row: lanes load 32 nonzeros at a time
// coalesced, then the products are shuffled to every lane in order and added
// sequentially (the same order as the reference).  Best for long rows.
template <bool kHashX>
__global__ void __launch_bounds__(256)
spmv_csr_vector_kernel(int64_t nrows, const int32_t* __restrict__ pos,
                       const int32_t* __restrict__ crd, const double* __restrict__ vals,
                       XOperand<kHashX> xop, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nrows) return;
  const int32_t b = ldg(pos + r), e = ldg(pos + r + 1);
  double acc = 0.0;
  for (int32_t c0 = b; c0 < e; c0 += 32) {
    const int32_t q = c0 + lane;
    const double t = q < e ? xop.term(ld_stream(vals + q), ld_stream(crd + q)) : 0.0;
    const int n = min(32, e - c0);
    for (int u = 0; u < n; ++u) acc = dadd(acc, __shfl_sync(0xffffffffu, t, u));
  }
  if (lane == 0) y[r] = acc;
}

// K2c: CSR merge-path.  The merge of (row ends, nonzeros) is cut into tiles of
// kMpItems items; each tile's start coordinate comes from a diagonal search
// done by a partition kernel.  A row is owned by the tile holding its end
// item; its owner re-reads the row's head from earlier tiles if the row
// started before the tile, so every row is still summed in order by one thread.
constexpr int kMpThreads = 256;
constexpr int kMpItems = 2048;

__device__ __forceinline__ void merge_path_search(int64_t diag, const int32_t* pos, int64_t nrows,
                                                  int64_t nnz, int64_t& row, int64_t& e) {
  // find the largest row count r in [max(0, diag-nnz), min(diag, nrows)] with
  // pos[r] <= diag - r  (row ends come first on ties).
  int64_t lo = diag > nnz ? diag - nnz : 0, hi = diag < nrows ? diag : nrows;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (ldg(pos + mid) <= diag - mid) lo = mid; else hi = mid - 1;
  }
  row = lo;
  e = diag - lo;
}

__global__ void csr_merge_partition_kernel(const int32_t* __restrict__ pos, int64_t nrows,
                                           int64_t nnz, int64_t ntiles, int64_t* __restrict__ part) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  int64_t diag = t * kMpItems;
  if (diag > nrows + nnz) diag = nrows + nnz;
  int64_t row, e;
  merge_path_search(diag, pos, nrows, nnz, row, e);
  part[t] = row;
}

template <bool kHashX>
__global__ void __launch_bounds__(kMpThreads)
spmv_csr_merge_kernel(int64_t nrows, const int32_t* __restrict__ pos,
                      const int32_t* __restrict__ crd, const double* __restrict__ vals,
                      XOperand<kHashX> xop, const int64_t* __restrict__ part,
                      double* __restrict__ y) {
  __shared__ __align__(16) double s_prod[kMpItems];
  const int tid = threadIdx.x;
  const int64_t rb = part[blockIdx.x], re = part[blockIdx.x + 1];
  // rows [rb, re) end inside this tile; their nonzeros span [pos[rb], pos[re]).
  if (rb >= re) return;
  const int64_t eb = ldg(pos + rb), ee = ldg(pos + re);
  for (int64_t cs = eb; cs < ee; cs += kMpItems) {
    const int n_in = (int)min64(kMpItems, ee - cs);
#pragma unroll 8
    for (int q = tid; q < n_in; q += kMpThreads)
      s_prod[q] = xop.term(ld_stream(vals + cs + q), ld_stream(crd + cs + q));
    __syncthreads();
    // rows are few per tile (<= kMpItems) — thread-per-row over the chunk
    for (int64_t r = rb + tid; r < re; r += kMpThreads) {
      const int64_t b = ldg(pos + r), e = ldg(pos + r + 1);
      const int64_t lo = max64(b, cs) - cs, hi = min64(e, cs + n_in) - cs;
      double acc = cs == eb ? 0.0 : y[r];
      for (int64_t u = lo; u < hi; ++u) acc = dadd(acc, s_prod[u]);
      y[r] = acc;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K3: ELL SpMV, slot-major.  Thread per row; slot s of consecutive rows is
// contiguous, so every load is coalesced; slots are added in slot order
// (= the row's column order, padding last: formats.py:322-335, 443-455).

template <int kRowsPerThread>
__global__ void __launch_bounds__(256)
spmv_ell_kernel(int64_t nrows, int32_t nslots, const int32_t* __restrict__ crd,
                const double* __restrict__ vals, const double* __restrict__ x,
                double* __restrict__ y) {
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRowsPerThread;
  if (i0 >= nrows) return;
  if (kRowsPerThread == 2 && i0 + 1 < nrows) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll 9
    for (int32_t s = 0; s < nslots; ++s) {
      const int64_t p = (int64_t)s * nrows + i0;
      const int2 c = ld_stream(reinterpret_cast<const int2*>(crd + p));  // 8B aligned: nrows, i0 even
      const double2 v = ld_stream(reinterpret_cast<const double2*>(vals + p));
      a0 = dadd(a0, dmul(v.x, ldg(x + c.x)));
      a1 = dadd(a1, dmul(v.y, ldg(x + c.y)));
    }
    y[i0] = a0;
    y[i0 + 1] = a1;
  } else {
    for (int64_t i = i0; i < i0 + kRowsPerThread && i < nrows; ++i) {
      double a = 0.0;
#pragma unroll 9
      for (int32_t s = 0; s < nslots; ++s) {
        const int64_t p = (int64_t)s * nrows + i;
        a = dadd(a, dmul(ld_stream(vals + p), ldg(x + ld_stream(crd + p))));
      }
      y[i] = a;
    }
  }
}

// ---------------------------------------------------------------------------
// K4: DIA SpMV, diagonal-major.  Thread per row; for each stored diagonal in
// ascending-offset order the row takes a term iff its column is inside the
// range level's bounds (levels.py:220-222): out-of-range slots are never read.
// Offsets travel as a kernel parameter (constant bank) when ndiag <= 32.

constexpr int kDiaMaxParam = 32;
struct DiaOffsets { int32_t v[kDiaMaxParam]; };

__global__ void __launch_bounds__(256)
spmv_dia_kernel(int64_t nrows, int64_t ncols, int32_t ndiag, DiaOffsets offs,
                const int32_t* __restrict__ doffs, const double* __restrict__ vals,
                const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double a = 0.0;
  if (doffs == nullptr) {
#pragma unroll
    for (int d = 0; d < kDiaMaxParam; ++d) {
      if (d < ndiag) {
        const int64_t j = i + offs.v[d];
        if (j >= 0 && j < ncols) a = dadd(a, dmul(ld_stream(vals + (int64_t)d * nrows + i), ldg(x + j)));
      }
    }
  } else {
    for (int d = 0; d < ndiag; ++d) {
      const int64_t j = i + ldg(doffs + d);
      if (j >= 0 && j < ncols) a = dadd(a, dmul(ld_stream(vals + (int64_t)d * nrows + i), ldg(x + j)));
    }
  }
  y[i] = a;
}

}  // namespace sl

// ===========================================================================
// C ABI

using namespace sl;
using sl_host::as_stream;
using sl_host::ceil_div;

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

extern "C" int sl_spmv_coo_f64(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* rows,
                               const int32_t* cols, const double* vals, const double* x,
                               double* y, void* stream) {
  if (nrows < 0 || ncols < 0 || nnz < 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || ncols > INT32_MAX || nnz > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0) return SL_OK;
  if (!y || (nnz > 0 && (!rows || !cols || !vals || !x))) return SL_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  if (nnz == 0) {
    fill_zero_kernel<<<min(ceil_div(nrows, 256), 4 * sl_host::sm_count()), 256, 0, s>>>(y, nrows);
    return sl_host::launch_status();
  }
  const bool vec_ok = aligned16(rows) && aligned16(cols) && aligned16(vals);
  spmv_coo_kernel<<<ceil_div(nnz, kCooTile), kCooThreads, 0, s>>>(nrows, nnz, rows, cols, vals,
                                                                   x, y, vec_ok);
  return sl_host::launch_status();
}

extern "C" size_t sl_spmv_csr_workspace_bytes(int64_t nrows, int64_t nnz, int32_t variant) {
  if (variant != 2) return 0;
  const int64_t ntiles = (nrows + nnz + kMpItems - 1) / kMpItems;
  return (size_t)(ntiles + 1) * sizeof(int64_t);
}

template <bool kHashX>
static int launch_csr(int64_t nrows, const int32_t* pos, const int32_t* crd, const double* vals,
                      XOperand<kHashX> xop, double* y, int32_t variant, void* ws,
                      size_t ws_bytes, cudaStream_t s) {
  if (variant == 0) {
    spmv_csr_rowblock_kernel<kHashX><<<ceil_div(nrows, kCsrRows), kCsrThreads, 0, s>>>(
        nrows, pos, crd, vals, xop, y);
  } else if (variant == 1) {
    spmv_csr_vector_kernel<kHashX><<<ceil_div(nrows * 32, 256), 256, 0, s>>>(nrows, pos, crd,
                                                                            vals, xop, y);
  } else if (variant == 2) {
    return SL_ERR_INVALID;  // handled by caller (needs nnz)
  } else {
    return SL_ERR_INVALID;
  }
  (void)ws;
  (void)ws_bytes;
  return sl_host::launch_status();
}

extern "C" int sl_spmv_csr_f64(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* pos,
                               const int32_t* crd, const double* vals, const double* x,
                               double* y, int32_t variant, void* ws, size_t ws_bytes,
                               void* stream) {
  if (nrows < 0 || ncols < 0 || nnz < 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || ncols > INT32_MAX || nnz > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0) return SL_OK;
  if (!pos || !y || !x) return SL_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  XOperand<false> xop{x};
  if (variant == 2) {
    const int64_t ntiles = (nrows + nnz + kMpItems - 1) / kMpItems;
    if (!ws || ws_bytes < sl_spmv_csr_workspace_bytes(nrows, nnz, 2)) return SL_ERR_WORKSPACE;
    int64_t* part = static_cast<int64_t*>(ws);
    csr_merge_partition_kernel<<<ceil_div(ntiles + 1, 256), 256, 0, s>>>(pos, nrows, nnz, ntiles,
                                                                       part);
    spmv_csr_merge_kernel<false><<<(int)ntiles, kMpThreads, 0, s>>>(nrows, pos, crd, vals, xop,
                                                                   part, y);
    return sl_host::launch_status();
  }
  return launch_csr<false>(nrows, pos, crd, vals, xop, y, variant, ws, ws_bytes, s);
}

extern "C" int sl_spmv_csr_hashx_f64(int64_t nrows, const int32_t* pos, const int32_t* crd,
                                     const double* vals, int64_t w, const int32_t* x_crd,
                                     const double* x_vals, double* y, void* stream) {
  if (nrows < 0 || w <= 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || w > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0) return SL_OK;
  if (!pos || !y || !x_crd || !x_vals) return SL_ERR_INVALID;
  XOperand<true> xop{HashedLevel{x_crd, w}, x_vals};
  return launch_csr<true>(nrows, pos, crd, vals, xop, y, 0, nullptr, 0, as_stream(stream));
}

extern "C" int sl_spmv_ell_f64(int64_t nrows, int64_t ncols, int32_t nslots, const int32_t* crd,
                               const double* vals, const double* x, double* y, void* stream) {
  if (nrows < 0 || ncols < 0 || nslots < 0) return SL_ERR_INVALID;
  if ((int64_t)nslots * nrows > INT32_MAX || ncols > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0) return SL_OK;
  if (!y || (nslots > 0 && (!crd || !vals || !x))) return SL_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  const bool pair = (nrows % 2 == 0) && aligned16(vals) &&
                    (reinterpret_cast<uintptr_t>(crd) & 7u) == 0;
  if (pair)
    spmv_ell_kernel<2><<<ceil_div(ceil_div(nrows, 2), 256), 256, 0, s>>>(nrows, nslots, crd, vals,
                                                                          x, y);
  else
    spmv_ell_kernel<1><<<ceil_div(nrows, 256), 256, 0, s>>>(nrows, nslots, crd, vals, x, y);
  return sl_host::launch_status();
}

extern "C" int sl_spmv_dia_f64(int64_t nrows, int64_t ncols, int32_t ndiag, const int32_t* offsets,
                               int32_t offsets_on_host, const double* vals, const double* x,
                               double* y, void* stream) {
  if (nrows < 0 || ncols < 0 || ndiag < 0) return SL_ERR_INVALID;
  if ((int64_t)ndiag * nrows > INT32_MAX || ncols > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0) return SL_OK;
  if (!y || (ndiag > 0 && (!offsets || !vals || !x))) return SL_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  DiaOffsets p{};
  const int32_t* doffs = nullptr;
  if (offsets_on_host && ndiag <= kDiaMaxParam) {
    for (int d = 0; d < ndiag; ++d) p.v[d] = offsets[d];
  } else if (offsets_on_host) {
    return SL_ERR_INVALID;  // > 32 diagonals: pass a device array
  } else {
    doffs = offsets;
  }
  spmv_dia_kernel<<<ceil_div(nrows, 256), 256, 0, s>>>(nrows, ncols, ndiag, p, doffs, vals, x, y);
  return sl_host::launch_status();
}
