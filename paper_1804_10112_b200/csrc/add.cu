// add.cu — C(i,j) = A(i,j) + B(i,j) with A CSR, B COO (or CSR), C CSR.
//
// Reference: the i-lattice {A0,B0} -> {A0} and j-lattice {A1,B1} -> {A1} ->
// {B1} co-iteration (engine.py:591-634) feeding the
// gather-append writer (engine.py:330-434).  Per row the output is the
// sorted union of A's and B's columns; a coordinate present in both gets
// a + b, otherwise the copy; B's duplicate coordinates are grouped and summed
// (+0.0 + b1 + b2 ..., engine.py:107-149, 524-527); the stored value is
// 0.0 + value (engine.py:404, 413, 625-631).  Explicit zeros are kept.
//
// B200 design (two passes over the operands, scan-based assembly):
//   0. rowptr   (COO B only) one pass over B's row coordinates yields the
//               row groups the reference's dedup-chained iterator walks
//               (Grouped over compressed(~U), engine.py:107-149) as a row
//               pointer; cols/vals are never moved — B is not converted.
//   1. count    thread per row merges the two sorted column lists and counts
//               distinct coordinates; a decoupled look-back scan across
//               blocks turns counts into the final c_pos in the same launch.
//   2. fill     thread per row merges again and writes (crd, val) at c_pos[r].
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace sl {

constexpr int kAddThreads = 256;

// ---- pass 0: row pointer of a row-sorted COO level ---------------------------
__global__ void coo_rowptr_kernel(int64_t nrows, int64_t nnz, const int32_t* __restrict__ rows,
                                  int32_t* __restrict__ rowptr) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e > nnz) return;
  // rowptr[r] = first e with rows[e] >= r, for r in [0, nrows]
  const int64_t lo = e == 0 ? 0 : (int64_t)ldg(rows + e - 1) + 1;
  const int64_t hi = e == nnz ? nrows : (int64_t)ldg(rows + e);
  for (int64_t r = lo; r <= hi; ++r) rowptr[r] = (int32_t)e;
}

// ---- merge of one row ----------------------------------------------------------
// Visits the union of A's row [alo, ahi) and B's row [blo, bhi) in ascending
// column order, B duplicates grouped.  F(col, value) is called per output.
template <bool kValues, typename F>
SL_DEV int merge_row(int32_t alo, int32_t ahi, const int32_t* __restrict__ a_crd,
                     const double* __restrict__ a_vals, int32_t blo, int32_t bhi,
                     const int32_t* __restrict__ b_cols, const double* __restrict__ b_vals,
                     F&& emit) {
  int n = 0;
  int32_t pa = alo, pb = blo;
  int32_t ca = pa < ahi ? ldg(a_crd + pa) : INT32_MAX;
  int32_t cb = pb < bhi ? ldg(b_cols + pb) : INT32_MAX;
  while (pa < ahi || pb < bhi) {
    const int32_t c = ca < cb ? ca : cb;
    double e = 0.0;
    const bool has_a = ca == c, has_b = cb == c;
    double a = 0.0;
    if (has_a) {
      if (kValues) a = ldg(a_vals + pa);
      ++pa;
      ca = pa < ahi ? ldg(a_crd + pa) : INT32_MAX;
    }
    if (has_b) {
      double b = kValues ? ldg(b_vals + pb) : 0.0;
      int32_t q = pb + 1;
      int32_t cq = q < bhi ? ldg(b_cols + q) : INT32_MAX;
      if (cq == c) {
        // duplicates: Python sum() over the group, 0 + b1 + b2 + ...
        if (kValues) b = dadd(0.0, b);
        while (cq == c) {
          if (kValues) b = dadd(b, ldg(b_vals + q));
          ++q;
          cq = q < bhi ? ldg(b_cols + q) : INT32_MAX;
        }
      }
      pb = q;
      cb = cq;
      e = has_a ? dadd(a, b) : b;
    } else {
      e = a;
    }
    emit(n, c, dadd(0.0, e));
    ++n;
  }
  return n;
}

struct NoEmit {
  SL_DEV void operator()(int, int32_t, double) const {}
};

// ---- pass 1: count + decoupled look-back scan -------------------------------------
// status[b] packs (flag << 62) | value: flag 1 = block aggregate, 2 = inclusive prefix.
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kAddThreads)
add_count_kernel(int64_t nrows, const int32_t* __restrict__ a_pos, const int32_t* __restrict__ a_crd,
                 const int32_t* __restrict__ b_pos, const int32_t* __restrict__ b_cols,
                 int32_t* __restrict__ c_pos, unsigned long long* __restrict__ status,
                 unsigned int* __restrict__ ticket) {
  __shared__ int32_t s_warp[kAddThreads / 32];
  __shared__ int64_t s_prefix;
  __shared__ unsigned int s_bid;
  if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);   // in-order block ids: look-back progress
  __syncthreads();
  const int64_t bid = s_bid;
  const int64_t r = bid * kAddThreads + threadIdx.x;
  int cnt = 0;
  if (r < nrows)
    cnt = merge_row<false>(ldg(a_pos + r), ldg(a_pos + r + 1), a_crd, nullptr, ldg(b_pos + r),
                           ldg(b_pos + r + 1), b_cols, nullptr, NoEmit{});
  // block inclusive scan of counts
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int v = lane < kAddThreads / 32 ? s_warp[lane] : 0;
    int sc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, sc, o);
      if (lane >= o) sc += u;
    }
    if (lane < kAddThreads / 32) s_warp[lane] = sc - v;
    const int total = __shfl_sync(0xffffffffu, sc, kAddThreads / 32 - 1);
    // decoupled look-back (warp 0)
    int64_t prefix = 0;
    if (bid == 0) {
      if (lane == 0) atomicExch(status, kFlagInc | (uint64_t)total);
    } else {
      if (lane == 0) atomicExch(status + bid, kFlagAgg | (uint64_t)total);
      int64_t look = bid - 1;
      while (true) {
        const int64_t idx = look - lane;
        uint64_t st = 0;
        if (idx >= 0) {
          do {
            st = *reinterpret_cast<volatile unsigned long long*>(status + idx);
          } while ((st >> 62) == 0);
        } else {
          st = kFlagInc;   // before block 0: inclusive zero
        }
        const unsigned inc_mask = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        // lanes up to (and including) the first inclusive one contribute
        const int stop = inc_mask ? __ffs(inc_mask) - 1 : 31;
        uint64_t v = lane <= stop ? (st & kValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        prefix += (int64_t)__shfl_sync(0xffffffffu, v, 0);
        if (inc_mask) break;
        look -= 32;
      }
      if (lane == 0) atomicExch(status + bid, kFlagInc | (uint64_t)(prefix + total));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  if (r < nrows) c_pos[r + 1] = (int32_t)(s_prefix + s_warp[warp] + incl);
  if (r == 0) c_pos[0] = 0;
}

// ---- pass 2: fill ------------------------------------------------------------------
struct FillEmit {
  int32_t* crd;
  double* vals;
  SL_DEV void operator()(int n, int32_t c, double v) const {
    crd[n] = c;
    vals[n] = v;
  }
};

__global__ void __launch_bounds__(kAddThreads)
add_fill_kernel(int64_t nrows, const int32_t* __restrict__ a_pos, const int32_t* __restrict__ a_crd,
                const double* __restrict__ a_vals, const int32_t* __restrict__ b_pos,
                const int32_t* __restrict__ b_cols, const double* __restrict__ b_vals,
                const int32_t* __restrict__ c_pos, int32_t* __restrict__ c_crd,
                double* __restrict__ c_vals) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int32_t o = ldg(c_pos + r);
  merge_row<true>(ldg(a_pos + r), ldg(a_pos + r + 1), a_crd, a_vals, ldg(b_pos + r),
                  ldg(b_pos + r + 1), b_cols, b_vals, FillEmit{c_crd + o, c_vals + o});
}

}  // namespace sl

using namespace sl;
using sl_host::as_stream;
using sl_host::ceil_div;

// workspace: [ticket u32, pad][status u64 x nblocks][rowptr i32 x (nrows+1)]
static size_t add_status_bytes(int64_t nrows) {
  const int64_t nblocks = (nrows + kAddThreads - 1) / kAddThreads;
  return 256 + (size_t)nblocks * 8;
}

extern "C" size_t sl_add_csr_workspace_bytes(int64_t nrows, int64_t b_nnz) {
  (void)b_nnz;
  return add_status_bytes(nrows) + (size_t)(nrows + 1) * sizeof(int32_t) + 256;
}

static const int32_t* add_rowptr(int64_t nrows, int64_t b_nnz, const int32_t* b_pos,
                                 const int32_t* b_rows, void* ws, bool build, cudaStream_t s) {
  if (b_pos) return b_pos;
  int32_t* rp = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + add_status_bytes(nrows));
  if (build) coo_rowptr_kernel<<<ceil_div(b_nnz + 1, 256), 256, 0, s>>>(nrows, b_nnz, b_rows, rp);
  return rp;
}

extern "C" int sl_add_csr_count(int64_t nrows, const int32_t* a_pos, const int32_t* a_crd,
                                int64_t b_nnz, const int32_t* b_pos, const int32_t* b_rows,
                                const int32_t* b_cols, int32_t* c_pos, void* ws, size_t ws_bytes,
                                void* stream) {
  if (nrows < 0 || b_nnz < 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || b_nnz > INT32_MAX) return SL_ERR_RANGE;
  if (!c_pos || !a_pos || (!b_pos && !b_rows && b_nnz > 0)) return SL_ERR_INVALID;
  if (!ws || ws_bytes < sl_add_csr_workspace_bytes(nrows, b_nnz)) return SL_ERR_WORKSPACE;
  cudaStream_t s = as_stream(stream);
  if (nrows == 0) {
    return cudaMemsetAsync(c_pos, 0, sizeof(int32_t), s) == cudaSuccess ? SL_OK : SL_ERR_CUDA;
  }
  const int64_t nblocks = ceil_div(nrows, kAddThreads);
  if (cudaMemsetAsync(ws, 0, add_status_bytes(nrows), s) != cudaSuccess) return SL_ERR_CUDA;
  const int32_t* bp = add_rowptr(nrows, b_nnz, b_pos, b_rows, ws, true, s);
  unsigned int* ticket = static_cast<unsigned int*>(ws);
  auto* status = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 256);
  add_count_kernel<<<(int)nblocks, kAddThreads, 0, s>>>(nrows, a_pos, a_crd, bp, b_cols, c_pos,
                                                        status, ticket);
  return sl_host::launch_status();
}

extern "C" int sl_add_csr_fill(int64_t nrows, const int32_t* a_pos, const int32_t* a_crd,
                               const double* a_vals, int64_t b_nnz, const int32_t* b_pos,
                               const int32_t* b_rows, const int32_t* b_cols, const double* b_vals,
                               const int32_t* c_pos, int32_t* c_crd, double* c_vals, void* ws,
                               size_t ws_bytes, void* stream) {
  if (nrows < 0 || b_nnz < 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || b_nnz > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0) return SL_OK;
  if (!c_pos || !a_pos || (!b_pos && !b_rows && b_nnz > 0)) return SL_ERR_INVALID;
  if ((!c_crd || !c_vals) && b_nnz > 0) return SL_ERR_INVALID;
  if (!b_pos && (!ws || ws_bytes < sl_add_csr_workspace_bytes(nrows, b_nnz)))
    return SL_ERR_WORKSPACE;
  cudaStream_t s = as_stream(stream);
  // the row pointer of a COO B was built by sl_add_csr_count in the same workspace
  const int32_t* bp = add_rowptr(nrows, b_nnz, b_pos, b_rows, ws, false, s);
  add_fill_kernel<<<ceil_div(nrows, kAddThreads), kAddThreads, 0, s>>>(
      nrows, a_pos, a_crd, a_vals, bp, b_cols, b_vals, c_pos, c_crd, c_vals);
  return sl_host::launch_status();
}
