// mttkrp.cu — A(i,r) = X(i,j,k) * B(j,r) * C(k,r) over COO-3 and CSF.
//
// Reference: loop order (i, j, k, r), scatter into dense A at depth 3,
// term (x * B[j,r]) * C[k,r] (engine.py:528-529 evaluates Mul(Mul(X,B),C)),
// every output row summed over its slice's nonzeros.
//
// B200 design.  Work unit: a chunk of kMtChunk consecutive nonzeros per warp
// (nnz-balanced, so Zipf-heavy slices are split across warps); lane l owns
// rank columns r = l + 32q, so each factor-row gather is one coalesced
// 256-byte load (R = 32).  Per element the term keeps the reference
// association; per output row the warp accumulates sequentially in storage
// order.  A row that lies entirely inside one chunk is stored directly; the
// partial sums of rows cut by chunk boundaries go to a carry workspace and a
// fix-up kernel adds them in a fixed order (deterministic run to run).  The
// slice sum is therefore a chunked reduction: A matches the sequential
// reference within |d| <= 1e-12 * sum|terms| (not bit-exact).  Rows of A with
// no nonzeros are zeroed by the chunk that owns the gap (no memset).
//
// CSF: the chunk's starting fiber/slice come from a bandwidth-bound pre-pass
// (each fiber/slice marks the chunk starts it contains — no searches); the
// B row is loaded once per fiber and held in registers while the fiber's k
// coordinates stream past.
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "common.cuh"

namespace sl {

constexpr int kMtWarps = 8;
constexpr int kMtThreads = kMtWarps * 32;
constexpr int kMtChunk = 2048;
constexpr int kMtBatch = 8;   // products issued ahead of the accumulation chain

struct CarryWs {
  int32_t* first_row;  // [nchunks] row of the chunk's first nonzero
  int32_t* head_row;   // [nchunks] row of the head carry (-1: none)
  int32_t* tail_row;   // [nchunks] row of the tail carry (-1: none)
  int32_t* fstart;     // [nchunks] CSF: fiber of the chunk's first nonzero
  int32_t* sstart;     // [nchunks] CSF: slice of the chunk's first nonzero
  double* head;        // [nchunks][R]
  double* tail;        // [nchunks][R]
};

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static CarryWs carve(void* ws, int64_t nchunks, int R) {
  char* p = static_cast<char*>(ws);
  CarryWs c;
  const size_t ib = align_up((size_t)nchunks * 4);
  c.first_row = reinterpret_cast<int32_t*>(p); p += ib;
  c.head_row = reinterpret_cast<int32_t*>(p); p += ib;
  c.tail_row = reinterpret_cast<int32_t*>(p); p += ib;
  c.fstart = reinterpret_cast<int32_t*>(p); p += ib;
  c.sstart = reinterpret_cast<int32_t*>(p); p += ib;
  const size_t db = align_up((size_t)nchunks * R * 8);
  c.head = reinterpret_cast<double*>(p); p += db;
  c.tail = reinterpret_cast<double*>(p);
  return c;
}

static size_t carry_bytes(int64_t nchunks, int R) {
  return 5 * align_up((size_t)nchunks * 4) + 2 * align_up((size_t)nchunks * R * 8);
}

template <int RPL>
struct RowAcc {
  double v[RPL];
  SL_DEV void zero() {
#pragma unroll
    for (int q = 0; q < RPL; ++q) v[q] = 0.0;
  }
};

template <int RPL>
SL_DEV void store_row(double* __restrict__ dst, const RowAcc<RPL>& a, int lane, int R) {
#pragma unroll
  for (int q = 0; q < RPL; ++q) {
    const int r = lane + 32 * q;
    if (r < R) dst[r] = a.v[q];
  }
}

SL_DEV void zero_rows(double* __restrict__ A, int64_t lo, int64_t hi, int lane, int R) {
  // rows [lo, hi) of A, R contiguous doubles each
  for (int64_t q = lo * R + lane; q < hi * R; q += 32) A[q] = 0.0;
}

// Flush one finished (or cut) row of the chunk.
template <int RPL>
SL_DEV void flush_row(int32_t row, const RowAcc<RPL>& acc, bool is_first, bool is_last,
                      bool head_partial, bool tail_cont, int64_t c, CarryWs cw, double* A,
                      int lane, int R) {
  if (is_first && head_partial) {
    store_row(cw.head + c * R, acc, lane, R);
    if (lane == 0) cw.head_row[c] = row;
  } else if (is_last && tail_cont) {
    store_row(cw.tail + c * R, acc, lane, R);
    if (lane == 0) cw.tail_row[c] = row;
  } else {
    store_row(A + (int64_t)row * R, acc, lane, R);
  }
}

// ---- K7: COO-3 ---------------------------------------------------------------------
template <int RPL>
__global__ void __launch_bounds__(kMtThreads)
mttkrp_coo3_kernel(int64_t I, int R, int64_t nnz, int64_t nchunks, const int32_t* __restrict__ ii,
                   const int32_t* __restrict__ jj, const int32_t* __restrict__ kk,
                   const double* __restrict__ vals, const double* __restrict__ B,
                   const double* __restrict__ C, double* __restrict__ A, CarryWs cw) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * kMtWarps + (threadIdx.x >> 5);
  if (c >= nchunks) return;
  const int64_t e0 = c * kMtChunk;
  const int64_t e1 = min64(e0 + kMtChunk, nnz);
  const int32_t row_first = ldg(ii + e0);
  const int32_t prev_row = e0 > 0 ? ldg(ii + e0 - 1) : -1;
  const bool head_partial = prev_row == row_first;
  const bool tail_cont = e1 < nnz && ldg(ii + e1) == ldg(ii + e1 - 1);
  if (lane == 0) {
    cw.first_row[c] = row_first;
    cw.head_row[c] = -1;
    cw.tail_row[c] = -1;
  }
  if (!head_partial) zero_rows(A, prev_row + 1, row_first, lane, R);

  RowAcc<RPL> acc;
  acc.zero();
  int32_t cur = row_first;
  bool first = true;
  for (int64_t base = e0; base < e1; base += 32) {
    const int n = (int)min64(32, e1 - base);
    int32_t li = 0, lj = 0, lk = 0;
    double lv = 0.0;
    if (lane < n) {
      li = ld_stream(ii + base + lane);
      lj = ld_stream(jj + base + lane);
      lk = ld_stream(kk + base + lane);
      lv = ld_stream(vals + base + lane);
    }
    for (int u0 = 0; u0 < n; u0 += kMtBatch) {
      // issue the factor gathers of kMtBatch nonzeros before the add chain
      double t[kMtBatch][RPL];
      int32_t rows[kMtBatch];
#pragma unroll
      for (int b = 0; b < kMtBatch; ++b) {
        const int u = u0 + b < n ? u0 + b : n - 1;
        rows[b] = __shfl_sync(0xffffffffu, li, u);
        const int32_t j = __shfl_sync(0xffffffffu, lj, u);
        const int32_t k = __shfl_sync(0xffffffffu, lk, u);
        const double v = __shfl_sync(0xffffffffu, lv, u);
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int r = lane + 32 * q;
          t[b][q] = r < R ? dmul(dmul(v, ldg(B + (int64_t)j * R + r)), ldg(C + (int64_t)k * R + r))
                          : 0.0;
        }
      }
#pragma unroll
      for (int b = 0; b < kMtBatch; ++b) {
        if (u0 + b >= n) break;
        if (rows[b] != cur) {
          flush_row(cur, acc, first, false, head_partial, tail_cont, c, cw, A, lane, R);
          zero_rows(A, (int64_t)cur + 1, rows[b], lane, R);
          acc.zero();
          cur = rows[b];
          first = false;
        }
#pragma unroll
        for (int q = 0; q < RPL; ++q) acc.v[q] = dadd(acc.v[q], t[b][q]);
      }
    }
  }
  flush_row(cur, acc, first, true, head_partial, tail_cont, c, cw, A, lane, R);
  if (e1 == nnz) zero_rows(A, (int64_t)cur + 1, I, lane, R);
}

// ---- K8: CSF ----------------------------------------------------------------------------
// Pre-pass: fiber f marks the chunks whose first nonzero it holds; slice s
// marks the chunks whose first nonzero lies in its nonzero range.
__global__ void csf_chunk_starts_kernel(int64_t nslices, int64_t nfibers,
                                        const int32_t* __restrict__ pos1,
                                        const int32_t* __restrict__ pos2, CarryWs cw) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nfibers) {
    const int64_t lo = ldg(pos2 + t), hi = ldg(pos2 + t + 1);
    for (int64_t c = (lo + kMtChunk - 1) / kMtChunk; c * kMtChunk < hi; ++c) cw.fstart[c] = (int32_t)t;
  }
  if (t < nslices) {
    const int64_t lo = ldg(pos2 + ldg(pos1 + t)), hi = ldg(pos2 + ldg(pos1 + t + 1));
    for (int64_t c = (lo + kMtChunk - 1) / kMtChunk; c * kMtChunk < hi; ++c) cw.sstart[c] = (int32_t)t;
  }
}

template <int RPL>
__global__ void __launch_bounds__(kMtThreads)
mttkrp_csf_kernel(int64_t I, int R, int64_t nslices, int64_t nfibers, int64_t nnz, int64_t nchunks,
                  const int32_t* __restrict__ crd0, const int32_t* __restrict__ pos1,
                  const int32_t* __restrict__ crd1, const int32_t* __restrict__ pos2,
                  const int32_t* __restrict__ crd2, const double* __restrict__ vals,
                  const double* __restrict__ B, const double* __restrict__ C,
                  double* __restrict__ A, CarryWs cw) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * kMtWarps + (threadIdx.x >> 5);
  if (c >= nchunks) return;
  const int64_t e0 = c * kMtChunk;
  const int64_t e1 = min64(e0 + kMtChunk, nnz);
  int64_t f = ldg(cw.fstart + c);
  int64_t s = ldg(cw.sstart + c);
  const int32_t row_first = ldg(crd0 + s);
  const bool head_partial = ldg(pos2 + ldg(pos1 + s)) < e0;
  const int32_t prev_row = head_partial ? row_first : (s > 0 ? ldg(crd0 + s - 1) : -1);
  if (lane == 0) {
    cw.first_row[c] = row_first;
    cw.head_row[c] = -1;
    cw.tail_row[c] = -1;
  }
  if (!head_partial) zero_rows(A, prev_row + 1, row_first, lane, R);

  // current fiber / slice state (warp-uniform)
  int64_t fend = ldg(pos2 + f + 1);               // first nonzero after fiber f
  int64_t s_fend = ldg(pos1 + s + 1);             // first fiber after slice s
  int32_t cur = row_first;
  double b[RPL];
  {
    const int64_t j = ldg(crd1 + f);
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int r = lane + 32 * q;
      b[q] = r < R ? ldg(B + j * R + r) : 0.0;
    }
  }
  RowAcc<RPL> acc;
  acc.zero();
  bool first = true;
  for (int64_t base = e0; base < e1; base += 32) {
    const int n = (int)min64(32, e1 - base);
    int32_t lk = 0;
    double lv = 0.0;
    if (lane < n) {
      lk = ld_stream(crd2 + base + lane);
      lv = ld_stream(vals + base + lane);
    }
    for (int u0 = 0; u0 < n; u0 += kMtBatch) {
      double cg[kMtBatch][RPL];
      double vb[kMtBatch];
#pragma unroll
      for (int bb = 0; bb < kMtBatch; ++bb) {
        const int u = u0 + bb < n ? u0 + bb : n - 1;
        const int32_t k = __shfl_sync(0xffffffffu, lk, u);
        vb[bb] = __shfl_sync(0xffffffffu, lv, u);
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int r = lane + 32 * q;
          cg[bb][q] = r < R ? ldg(C + (int64_t)k * R + r) : 0.0;
        }
      }
#pragma unroll
      for (int bb = 0; bb < kMtBatch; ++bb) {
        if (u0 + bb >= n) break;
        const int64_t e = base + u0 + bb;
        if (e >= fend) {
          // next non-empty fiber, possibly crossing slices
          do {
            ++f;
            while (f >= s_fend) {
              ++s;
              s_fend = ldg(pos1 + s + 1);
            }
            fend = ldg(pos2 + f + 1);
          } while (e >= fend);
          const int32_t row = ldg(crd0 + s);
          if (row != cur) {
            flush_row(cur, acc, first, false, head_partial, false, c, cw, A, lane, R);
            zero_rows(A, (int64_t)cur + 1, row, lane, R);
            acc.zero();
            cur = row;
            first = false;
          }
          const int64_t j = ldg(crd1 + f);
#pragma unroll
          for (int q = 0; q < RPL; ++q) {
            const int r = lane + 32 * q;
            b[q] = r < R ? ldg(B + j * R + r) : 0.0;
          }
        }
#pragma unroll
        for (int q = 0; q < RPL; ++q)
          acc.v[q] = dadd(acc.v[q], dmul(dmul(vb[bb], b[q]), cg[bb][q]));
      }
    }
  }
  // does the last slice continue past this chunk?
  const bool tail_cont = e1 < nnz && ldg(pos2 + s_fend) > e1;
  flush_row(cur, acc, first, true, head_partial, tail_cont, c, cw, A, lane, R);
  if (e1 == nnz) zero_rows(A, (int64_t)cur + 1, I, lane, R);
  (void)nslices;
  (void)nfibers;
}

// ---- fix-up: rows cut by chunk boundaries ---------------------------------------------
// Block per chunk c that holds a tail carry: the row continues through chunks
// c+1 .. ce (their first rows equal it and they hold head carries).  ce is
// found by a warp-wide 32-ary search over the monotone first_row array; the
// 8 warps sum strided subsets of the heads, combined in a fixed order.
template <int RPL>
__global__ void __launch_bounds__(kMtThreads)
mttkrp_fixup_kernel(int R, int64_t nchunks, CarryWs cw, double* __restrict__ A) {
  const int64_t c = blockIdx.x;
  const int32_t row = cw.tail_row[c];
  if (row < 0) return;
  __shared__ int64_t s_end;
  __shared__ double s_part[kMtWarps][32 * RPL];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    // last chunk ce >= c with first_row[ce'] == row for all c < ce' <= ce
    int64_t lo = c, hi = nchunks - 1;   // answer in [lo, hi]
    while (lo < hi) {
      const int64_t span = hi - lo;
      const int64_t step = (span + 31) / 32;
      const int64_t probe = lo + (int64_t)(lane + 1) * step;
      const bool ok = probe <= hi && ldg(cw.first_row + probe) == row;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      // ok is monotone: true for a prefix of lanes
      const int nok = __popc(m);
      const int64_t new_lo = lo + (int64_t)nok * step;
      const int64_t new_hi = min64(hi, lo + (int64_t)(nok + 1) * step - 1);
      lo = new_lo;
      hi = new_hi;
    }
    if (lane == 0) s_end = lo;
  }
  __syncthreads();
  const int64_t ce = s_end;
  RowAcc<RPL> part;
  part.zero();
  for (int64_t q = c + 1 + warp; q <= ce; q += kMtWarps) {
#pragma unroll
    for (int p = 0; p < RPL; ++p) {
      const int r = lane + 32 * p;
      if (r < R) part.v[p] = dadd(part.v[p], cw.head[q * R + r]);
    }
  }
#pragma unroll
  for (int p = 0; p < RPL; ++p) s_part[warp][lane + 32 * p] = part.v[p];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int p = 0; p < RPL; ++p) {
      const int r = lane + 32 * p;
      if (r < R) {
        double tot = cw.tail[c * R + r];
        for (int w = 0; w < kMtWarps; ++w) tot = dadd(tot, s_part[w][r]);
        A[(int64_t)row * R + r] = tot;
      }
    }
  }
}

__global__ void fill_zero_f64(double* __restrict__ a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = 0.0;
}

}  // namespace sl

using namespace sl;
using sl_host::as_stream;
using sl_host::ceil_div;

static int64_t mt_nchunks(int64_t nnz) { return (nnz + kMtChunk - 1) / kMtChunk; }

extern "C" size_t sl_mttkrp_workspace_bytes(int64_t nnz, int32_t R) {
  return carry_bytes(mt_nchunks(nnz) + 1, R);
}

template <typename Launch>
static int dispatch_rpl(int R, Launch&& launch) {
  if (R <= 32) return launch(std::integral_constant<int, 1>{});
  if (R <= 64) return launch(std::integral_constant<int, 2>{});
  if (R <= 128) return launch(std::integral_constant<int, 4>{});
  return SL_ERR_RANGE;
}

static int mt_check(int64_t I, int64_t J, int64_t K, int32_t R, int64_t nnz) {
  if (I < 0 || J < 0 || K < 0 || R <= 0 || nnz < 0) return SL_ERR_INVALID;
  if (I > INT32_MAX || J > INT32_MAX || K > INT32_MAX || nnz > INT32_MAX || R > 128)
    return SL_ERR_RANGE;
  return SL_OK;
}

extern "C" int sl_mttkrp_coo3_f64(int64_t I, int64_t J, int64_t K, int32_t R, int64_t nnz,
                                  const int32_t* i, const int32_t* j, const int32_t* k,
                                  const double* vals, const double* B, const double* C, double* A,
                                  void* ws, size_t ws_bytes, void* stream) {
  int st = mt_check(I, J, K, R, nnz);
  if (st != SL_OK) return st;
  if (I == 0) return SL_OK;
  if (!A) return SL_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  if (nnz == 0) {
    fill_zero_f64<<<min(ceil_div(I * R, 256), 1024), 256, 0, s>>>(A, I * R);
    return sl_host::launch_status();
  }
  if (!i || !j || !k || !vals || !B || !C) return SL_ERR_INVALID;
  if (!ws || ws_bytes < sl_mttkrp_workspace_bytes(nnz, R)) return SL_ERR_WORKSPACE;
  const int64_t nch = mt_nchunks(nnz);
  CarryWs cw = carve(ws, nch + 1, R);
  const int grid = ceil_div(nch, kMtWarps);
  return dispatch_rpl(R, [&](auto rpl) {
    constexpr int RPL = decltype(rpl)::value;
    mttkrp_coo3_kernel<RPL><<<grid, kMtThreads, 0, s>>>(I, R, nnz, nch, i, j, k, vals, B, C, A, cw);
    mttkrp_fixup_kernel<RPL><<<(int)nch, kMtThreads, 0, s>>>(R, nch, cw, A);
    return sl_host::launch_status();
  });
}

extern "C" int sl_mttkrp_csf_f64(int64_t I, int64_t J, int64_t K, int32_t R, int64_t nslices,
                                 int64_t nfibers, int64_t nnz, const int32_t* crd0,
                                 const int32_t* pos1, const int32_t* crd1, const int32_t* pos2,
                                 const int32_t* crd2, const double* vals, const double* B,
                                 const double* C, double* A, void* ws, size_t ws_bytes,
                                 void* stream) {
  int st = mt_check(I, J, K, R, nnz);
  if (st != SL_OK) return st;
  if (nslices < 0 || nfibers < 0) return SL_ERR_INVALID;
  if (I == 0) return SL_OK;
  if (!A) return SL_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  if (nnz == 0) {
    fill_zero_f64<<<min(ceil_div(I * R, 256), 1024), 256, 0, s>>>(A, I * R);
    return sl_host::launch_status();
  }
  if (!crd0 || !pos1 || !crd1 || !pos2 || !crd2 || !vals || !B || !C) return SL_ERR_INVALID;
  if (!ws || ws_bytes < sl_mttkrp_workspace_bytes(nnz, R)) return SL_ERR_WORKSPACE;
  const int64_t nch = mt_nchunks(nnz);
  CarryWs cw = carve(ws, nch + 1, R);
  const int64_t nt = nslices > nfibers ? nslices : nfibers;
  csf_chunk_starts_kernel<<<ceil_div(nt, 256), 256, 0, s>>>(nslices, nfibers, pos1, pos2, cw);
  const int grid = ceil_div(nch, kMtWarps);
  return dispatch_rpl(R, [&](auto rpl) {
    constexpr int RPL = decltype(rpl)::value;
    mttkrp_csf_kernel<RPL><<<grid, kMtThreads, 0, s>>>(I, R, nslices, nfibers, nnz, nch, crd0,
                                                       pos1, crd1, pos2, crd2, vals, B, C, A, cw);
    mttkrp_fixup_kernel<RPL><<<(int)nch, kMtThreads, 0, s>>>(R, nch, cw, A);
    return sl_host::launch_status();
  });
}
