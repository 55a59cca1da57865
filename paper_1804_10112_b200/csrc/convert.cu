// convert.cu — format conversion on the device.
//
// Reference: formats.convert (formats.py:583-587) re-stores a tensor through
// an identity assignment evaluated by the interpreter, i.e. through the
// append (compressed/singleton) and insert (dense) protocols of the output
// levels (levels.py:303-394) in the layouts of formats.assemble
// (formats.py:361-501).  The B200 versions produce exactly those layouts:
//   COO-SoA -> CSR : the row pointer of the row-sorted COO level (the append
//                    protocol's pos, one pass over the row coordinates);
//                    crd / vals are the COO column / value arrays unchanged.
//   CSR -> ELL     : slot s of row i = the row's s-th entry at s*N + i,
//                    padding (col 0, 0.0) (formats.py:322-335, 443-455).
//   COO -> DIA     : diagonal set = sorted distinct (c - r) (formats.py:313),
//                    vals[d*N + i] (formats.py:405-412), other slots 0.0.
// Matrices are canonical (unique coordinates, as assemble guarantees for the
// unique formats CSR/ELL/DIA).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace sl {

// row lengths' maximum (ELL slot count)
__global__ void csr_max_row_kernel(int64_t nrows, const int32_t* __restrict__ pos,
                                   const double* __restrict__ vals, int32_t* __restrict__ out) {
  int32_t m = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int32_t kept = 0;   // entries that survive assemble's zero filter
    for (int32_t p = ldg(pos + r); p < ldg(pos + r + 1); ++p) kept += ldg(vals + p) != 0.0;
    m = max(m, kept);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// thread per row: its entries into slots 0 .. len-1, padding in the rest
__global__ void csr_to_ell_kernel(int64_t nrows, int32_t nslots, const int32_t* __restrict__ pos,
                                  const int32_t* __restrict__ crd, const double* __restrict__ vals,
                                  int32_t* __restrict__ ecrd, double* __restrict__ evals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const int32_t b = ldg(pos + i), e = ldg(pos + i + 1);
  int32_t s = 0;
  for (int32_t q = b; q < e && s < nslots; ++q) {
    const double v = ldg(vals + q);
    if (v == 0.0) continue;                         // assemble drops exact zeros
    const int64_t p = (int64_t)s * nrows + i;
    ecrd[p] = ldg(crd + q);
    evals[p] = dadd(0.0, v);
    ++s;
  }
  for (; s < nslots; ++s) {
    const int64_t p = (int64_t)s * nrows + i;
    ecrd[p] = 0;
    evals[p] = 0.0;
  }
}

// mark the diagonals present: flag[(c - r) + nrows - 1] = 1
__global__ void dia_mark_kernel(int64_t nnz, int64_t nrows, const int32_t* __restrict__ rows,
                                const int32_t* __restrict__ cols, const double* __restrict__ vals,
                                int32_t* __restrict__ flag) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    if (ldg(vals + e) != 0.0) flag[(int64_t)ldg(cols + e) - ldg(rows + e) + nrows - 1] = 1;
}

// compact the flags into the sorted offset list; index[o] = diagonal index
// (single block: the flag array has nrows + ncols - 1 entries)
__global__ void __launch_bounds__(1024)
dia_compact_kernel(int64_t nflags, int64_t nrows, const int32_t* __restrict__ flag,
                   int32_t* __restrict__ index, int32_t* __restrict__ offsets,
                   int32_t* __restrict__ ndiag) {
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_base = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nflags; b0 += 1024) {
    const int64_t o = b0 + tid;
    const int f = o < nflags ? flag[o] : 0;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    int before = s_base;
    for (int w = 0; w < warp; ++w) before += s_warp[w];
    const int idx = before + __popc(m & ((1u << lane) - 1u));
    if (f) {
      index[o] = idx;
      offsets[idx] = (int32_t)(o - (nrows - 1));
    }
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < 32; ++w) t += s_warp[w];
      s_base += t;
    }
    __syncthreads();
  }
  if (tid == 0) *ndiag = s_base;
}

__global__ void dia_scatter_kernel(int64_t nnz, int64_t nrows, const int32_t* __restrict__ rows,
                                   const int32_t* __restrict__ cols, const double* __restrict__ vals,
                                   const int32_t* __restrict__ index, double* __restrict__ dvals) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = ldg(vals + e);
    if (v == 0.0) continue;
    const int64_t r = ldg(rows + e);
    const int64_t d = ldg(index + ((int64_t)ldg(cols + e) - r + nrows - 1));
    dvals[d * nrows + r] = dadd(0.0, v);
  }
}

// COO row coordinates of a CSR matrix: rows[p] = i for p in [pos[i], pos[i+1])
__global__ void csr_rows_kernel(int64_t nrows, const int32_t* __restrict__ pos,
                                int32_t* __restrict__ rows) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += stride)
    for (int32_t p = ldg(pos + i); p < ldg(pos + i + 1); ++p) rows[p] = (int32_t)i;
}

__global__ void fill_zero_f64_kernel(double* __restrict__ a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = 0.0;
}

}  // namespace sl

using namespace sl;
using sl_host::as_stream;
using sl_host::ceil_div;

extern "C" int sl_convert_coo_to_csr(int64_t nrows, int64_t nnz, const int32_t* rows,
                                     int32_t* pos, void* stream) {
  if (nrows < 0 || nnz < 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || nnz > INT32_MAX) return SL_ERR_RANGE;
  if (!pos || (nnz > 0 && !rows)) return SL_ERR_INVALID;
  sl_host::launch_coo_rowptr(nrows, nnz, rows, pos, as_stream(stream));
  return sl_host::launch_status();
}

extern "C" int sl_csr_max_row_length(int64_t nrows, const int32_t* pos, const double* vals,
                                     int32_t* out_dev, void* stream) {
  if (nrows < 0 || !pos || !out_dev) return SL_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(out_dev, 0, sizeof(int32_t), s) != cudaSuccess) return SL_ERR_CUDA;
  if (nrows == 0) return SL_OK;
  csr_max_row_kernel<<<min(ceil_div(nrows, 256), 4 * sl_host::sm_count()), 256, 0, s>>>(
      nrows, pos, vals, out_dev);
  return sl_host::launch_status();
}

extern "C" int sl_convert_csr_to_ell(int64_t nrows, int32_t nslots, const int32_t* pos,
                                     const int32_t* crd, const double* vals, int32_t* ecrd,
                                     double* evals, void* stream) {
  if (nrows < 0 || nslots < 0) return SL_ERR_INVALID;
  if ((int64_t)nslots * nrows > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0 || nslots == 0) return SL_OK;
  if (!pos || !ecrd || !evals) return SL_ERR_INVALID;
  csr_to_ell_kernel<<<ceil_div(nrows, 256), 256, 0, as_stream(stream)>>>(nrows, nslots, pos, crd,
                                                                        vals, ecrd, evals);
  return sl_host::launch_status();
}

extern "C" size_t sl_convert_coo_to_dia_workspace_bytes(int64_t nrows, int64_t ncols) {
  return (size_t)(nrows + ncols) * 2 * sizeof(int32_t) + 256;
}

extern "C" int sl_convert_coo_to_dia_offsets(int64_t nrows, int64_t ncols, int64_t nnz,
                                             const int32_t* rows, const int32_t* cols,
                                             const double* vals, int32_t* offsets,
                                             int32_t* ndiag_dev, void* ws, size_t ws_bytes,
                                             void* stream) {
  if (nrows <= 0 || ncols <= 0 || nnz < 0) return SL_ERR_INVALID;
  if (nrows + ncols > INT32_MAX || nnz > INT32_MAX) return SL_ERR_RANGE;
  if (!offsets || !ndiag_dev || (nnz > 0 && (!rows || !cols || !vals))) return SL_ERR_INVALID;
  if (!ws || ws_bytes < sl_convert_coo_to_dia_workspace_bytes(nrows, ncols)) return SL_ERR_WORKSPACE;
  cudaStream_t s = as_stream(stream);
  const int64_t nflags = nrows + ncols - 1;
  int32_t* flag = static_cast<int32_t*>(ws);
  int32_t* index = flag + nflags;
  if (cudaMemsetAsync(flag, 0, (size_t)nflags * sizeof(int32_t), s) != cudaSuccess)
    return SL_ERR_CUDA;
  if (nnz > 0)
    dia_mark_kernel<<<min(ceil_div(nnz, 256), 8 * sl_host::sm_count()), 256, 0, s>>>(
        nnz, nrows, rows, cols, vals, flag);
  dia_compact_kernel<<<1, 1024, 0, s>>>(nflags, nrows, flag, index, offsets, ndiag_dev);
  return sl_host::launch_status();
}

extern "C" int sl_convert_coo_to_dia_values(int64_t nrows, int64_t ncols, int64_t nnz,
                                            int32_t ndiag, const int32_t* rows,
                                            const int32_t* cols, const double* vals,
                                            double* dvals, void* ws, size_t ws_bytes,
                                            void* stream) {
  if (nrows <= 0 || ncols <= 0 || nnz < 0 || ndiag < 0) return SL_ERR_INVALID;
  if ((int64_t)ndiag * nrows > INT32_MAX) return SL_ERR_RANGE;
  if ((ndiag > 0 && !dvals) || (nnz > 0 && (!rows || !cols || !vals))) return SL_ERR_INVALID;
  if (!ws || ws_bytes < sl_convert_coo_to_dia_workspace_bytes(nrows, ncols)) return SL_ERR_WORKSPACE;
  cudaStream_t s = as_stream(stream);
  const int64_t n = (int64_t)ndiag * nrows;
  if (n > 0)
    fill_zero_f64_kernel<<<min(ceil_div(n, 256), 8 * sl_host::sm_count()), 256, 0, s>>>(dvals, n);
  const int32_t* index = static_cast<const int32_t*>(ws) + (nrows + ncols - 1);
  if (nnz > 0)
    dia_scatter_kernel<<<min(ceil_div(nnz, 256), 8 * sl_host::sm_count()), 256, 0, s>>>(
        nnz, nrows, rows, cols, vals, index, dvals);
  return sl_host::launch_status();
}

extern "C" int sl_csr_row_indices(int64_t nrows, const int32_t* pos, int32_t* rows, void* stream) {
  if (nrows < 0 || !pos) return SL_ERR_INVALID;
  if (nrows == 0) return SL_OK;
  csr_rows_kernel<<<min(ceil_div(nrows, 256), 16 * sl_host::sm_count()), 256, 0,
                    as_stream(stream)>>>(nrows, pos, rows);
  return sl_host::launch_status();
}
