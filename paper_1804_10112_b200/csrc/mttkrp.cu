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
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"

namespace sl {

constexpr int kMtWarps = 4;     // 2 / 4 / 8 / 16 warps per block at 16 warps/SM: COO-3 0.957 / 0.958 / 0.965 / 0.974 ms
constexpr int kMtThreads = kMtWarps * 32;
constexpr int kMtChunk = 1024;   // 512 / 1024 / 2048 / 4096: COO-3 0.990 / 0.966 / 0.990 / 1.103 ms, CSF 1.127 / 1.067 / 1.064 / 1.170 ms
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

// ---- K7 (vectorised): COO-3, R in {16, 32, 64} --------------------------------------
// kLpn = R/4 lanes per nonzero, each lane owning 4 consecutive rank columns
// read with one 256-bit load from B and one from C; 32/kLpn nonzeros per warp
// step.  Each lane group ("sub") keeps a partial sum of the current output row
// over the nonzeros it handled; when the row ends the subs' partials are
// combined with a fixed xor-shuffle tree (deterministic).  ~3x fewer
// instructions per nonzero than the lane-per-column kernel (ncu: that one is
// issue-bound at ~50 warp-instructions per nonzero).
SL_DEV double4 ld4(const double* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
      : "l"(p));
  return v;
}

SL_DEV double4 shfl_xor4(double4 a, int m) {
  return make_double4(__shfl_xor_sync(0xffffffffu, a.x, m), __shfl_xor_sync(0xffffffffu, a.y, m),
                      __shfl_xor_sync(0xffffffffu, a.z, m), __shfl_xor_sync(0xffffffffu, a.w, m));
}

SL_DEV double4 add4(double4 a, double4 b) {
  return make_double4(dadd(a.x, b.x), dadd(a.y, b.y), dadd(a.z, b.z), dadd(a.w, b.w));
}

template <int kLpn>
SL_DEV double4 combine_subs(double4 a) {
  // fixed tree over the 32/kLpn subs: xor kLpn, 2kLpn, ...
#pragma unroll
  for (int m = kLpn; m < 32; m <<= 1) a = add4(a, shfl_xor4(a, m));
  return a;
}

SL_DEV void store4(double* dst, double4 v) {
  *reinterpret_cast<double4*>(dst) = v;
}

// destination of a finished row: head carry, tail carry or A itself
SL_DEV double* row_dst(int32_t row, bool is_first, bool is_last, bool head_partial, bool tail_cont,
                       int64_t c, CarryWs cw, double* A, int R, int lane) {
  if (is_first && head_partial) {
    if (lane == 0) cw.head_row[c] = row;
    return cw.head + c * R;
  }
  if (is_last && tail_cont) {
    if (lane == 0) cw.tail_row[c] = row;
    return cw.tail + c * R;
  }
  return A + (int64_t)row * R;
}

// Per-batch sources of (i, j, k, x) for the 32 nonzeros [base, base + 32),
// lane l holding nonzero base + l.  The next batch's loads are issued before
// the current batch is consumed (double-buffered in registers).
struct CooSrc {
  const int32_t* ii;
  const int32_t* jj;
  const int32_t* kk;
  const double* vals;
  int64_t e1;
  int32_t ni, nj, nk;
  double nv;
  SL_DEV void prefetch(int64_t base, int lane) {
    if (base + lane < e1) {
      ni = ld_stream(ii + base + lane);
      nj = ld_stream(jj + base + lane);
      nk = ld_stream(kk + base + lane);
      nv = ld_stream(vals + base + lane);
    }
  }
  SL_DEV void start(int64_t e0, int lane) { prefetch(e0, lane); }
  SL_DEV void next(int64_t base, int lane, int32_t& li, int32_t& lj, int32_t& lk, double& lv) {
    li = ni; lj = nj; lk = nk; lv = nv;
    prefetch(base + 32, lane);
  }
};

// CSF: the batch's fibers and slices come from 32-wide windows of pos2/crd1
// and pos1/crd0; each lane finds its nonzero's fiber (slice) by counting the
// window's fiber (slice) ends at or before it (warp OR + popcount).

struct CsfSrc {
  const int32_t* crd0;
  const int32_t* pos1;
  const int32_t* crd1;
  const int32_t* pos2;
  const int32_t* crd2;
  const double* vals;
  int64_t nslices, nfibers, e1;
  int64_t f, s;        // fiber / slice of the batch's first nonzero (warp-uniform)
  int32_t nk;
  double nv;
  // the batch's fiber-end / fiber-j / slice-end / slice-i windows, loaded one
  // batch ahead: the next batch's first fiber and slice follow from the
  // current windows alone, so these loads are never on the critical path
  // (loading them at the start of each batch put an L2 round trip per 32
  // nonzeros in series: CSF 1.25 ms vs COO-3 1.00 ms)
  int32_t wfe, wjw, wse, wiw;
  SL_DEV void prefetch(int64_t base, int lane) {
    if (base + lane < e1) {
      nk = ld_stream(crd2 + base + lane);
      nv = ld_stream(vals + base + lane);
    }
  }
  SL_DEV void load_windows(int lane) {
    wfe = f + 1 + lane <= nfibers ? ldg(pos2 + f + 1 + lane) : INT32_MAX;
    wjw = f + lane < nfibers ? ldg(crd1 + f + lane) : 0;
    wse = s + 1 + lane <= nslices ? ldg(pos1 + s + 1 + lane) : INT32_MAX;
    wiw = s + lane < nslices ? ldg(crd0 + s + lane) : 0;
  }
  SL_DEV void start(int64_t e0, int lane) {
    prefetch(e0, lane);
    load_windows(lane);
  }
  SL_DEV void next(int64_t base, int lane, int32_t& li, int32_t& lj, int32_t& lk, double& lv) {
    const int32_t fe = wfe, jw = wjw, se = wse, iw = wiw;
    // fiber of element base + lane: the number of window fibers ending at or
    // before it.  Fiber ends inside the batch are distinct positions 1..31,
    // so one warp OR of (1 << position) and a popcount of the bits up to the
    // lane give every lane's count (a 5-step shuffle search per lane before:
    // CSF ran 20% more instructions than COO-3)
    const unsigned le_mask = 0xffffffffu >> (31 - lane);
    const int32_t pf = fe - (int32_t)base;
    const unsigned fbits = __reduce_or_sync(0xffffffffu, pf >= 0 && pf < 32 ? 1u << pf : 0u);
    const int df = __popc(fbits & le_mask);
    lj = __shfl_sync(0xffffffffu, jw, df);
    const int32_t fib = (int32_t)(f + df);
    // slices average 2000 nonzeros: a batch usually lies in one slice (the
    // first slice ends after the batch's last fiber) and skips the count
    const int32_t se0 = __shfl_sync(0xffffffffu, se, 0);
    const int32_t fib_last = __shfl_sync(0xffffffffu, fib, 31);
    if (se0 > fib_last) {
      li = __shfl_sync(0xffffffffu, iw, 0);
    } else {
      const int32_t ps = se - (int32_t)f;      // slice ends as fiber offsets 1..31
      const unsigned sbits = __reduce_or_sync(0xffffffffu, ps >= 0 && ps < 32 ? 1u << ps : 0u);
      const int ds = __popc(sbits & (0xffffffffu >> (31 - df)));
      li = __shfl_sync(0xffffffffu, iw, ds);
    }
    lk = nk;
    lv = nv;
    // advance to the next batch's first nonzero and start its loads
    f += __popc(__ballot_sync(0xffffffffu, fe <= (int32_t)(base + 32)));
    s += __popc(__ballot_sync(0xffffffffu, se <= (int32_t)f));
    prefetch(base + 32, lane);
    load_windows(lane);
  }
};

template <int kR, class Src>
SL_DEV void mttkrp_vec_body(int64_t I, int64_t e0, int64_t e1, int32_t row_first, int32_t prev_row,
                            bool head_partial, bool tail_cont, int64_t c,
                            const double* __restrict__ B, const double* __restrict__ C,
                            double* __restrict__ A, CarryWs cw, Src& src, bool reuse_b) {
  constexpr int kLpn = kR / 4, kNps = 32 / kLpn;   // lanes per nonzero, nonzeros per step
  constexpr int kSteps = 4;                        // steps whose loads are issued together
  const int lane = threadIdx.x & 31, sub = lane / kLpn, q = lane % kLpn;
  if (lane == 0) {
    cw.first_row[c] = row_first;
    cw.head_row[c] = -1;
    cw.tail_row[c] = -1;
  }
  if (!head_partial) zero_rows(A, prev_row + 1, row_first, lane, kR);
  double4 acc = make_double4(0.0, 0.0, 0.0, 0.0);
  int32_t cur = row_first;
  bool first = true;
  auto flush = [&](bool is_last) {
    const double4 tot = combine_subs<kLpn>(acc);
    double* dst = row_dst(cur, first, is_last, head_partial, tail_cont, c, cw, A, kR, lane);
    if (sub == 0) store4(dst + 4 * q, tot);
  };
  src.start(e0, lane);
  // sub s handles the kSteps CONSECUTIVE nonzeros [u0 + s*kSteps, ...) of a
  // round, so it can keep the B row of a fiber in registers across nonzeros
  // that share j (ncu: the kernel is L1-throughput bound; B reloads were half
  // of the L1 traffic)
  int32_t jprev = -1;
  double4 b = make_double4(0.0, 0.0, 0.0, 0.0);
  for (int64_t base = e0; base < e1; base += 32) {
    const int n = (int)min64(32, e1 - base);
    int32_t li, lj, lk;
    double lv;
    src.next(base, lane, li, lj, lk, lv);
    for (int u0 = 0; u0 < n; u0 += kSteps * kNps) {
      double4 t[kSteps];
#pragma unroll
      for (int st = 0; st < kSteps; ++st) {
        const int u = u0 + sub * kSteps + st;
        const int us = u < n ? u : n - 1;
        const int32_t j = __shfl_sync(0xffffffffu, lj, us);
        const int32_t k = __shfl_sync(0xffffffffu, lk, us);
        const double v = __shfl_sync(0xffffffffu, lv, us);
        if (j != jprev || !reuse_b) {
          b = ld4(B + (int64_t)j * kR + 4 * q);
          jprev = j;
        }
        const double4 cc = ld4(C + (int64_t)k * kR + 4 * q);
        t[st] = make_double4(dmul(dmul(v, b.x), cc.x), dmul(dmul(v, b.y), cc.y),
                             dmul(dmul(v, b.z), cc.z), dmul(dmul(v, b.w), cc.w));
      }
      // fast path: rows are sorted, so if the round's last nonzero is still in
      // the current row, all of them are; every sub adds its terms in order
      const int ulast = min(u0 + kSteps * kNps, n) - 1;
      if (__shfl_sync(0xffffffffu, li, ulast) == cur) {
#pragma unroll
        for (int st = 0; st < kSteps; ++st)
          if (u0 + sub * kSteps + st < n) acc = add4(acc, t[st]);
        continue;
      }
#pragma unroll
      for (int s2 = 0; s2 < kNps; ++s2) {
#pragma unroll
        for (int st = 0; st < kSteps; ++st) {
          const int u = u0 + s2 * kSteps + st;    // warp-uniform element index, storage order
          if (u < n) {
            const int32_t r = __shfl_sync(0xffffffffu, li, u);
            if (r != cur) {
              flush(false);
              zero_rows(A, (int64_t)cur + 1, r, lane, kR);
              acc = make_double4(0.0, 0.0, 0.0, 0.0);
              cur = r;
              first = false;
            }
            if (sub == s2) acc = add4(acc, t[st]);
          }
        }
      }
    }
  }
  flush(true);
  (void)I;
}

template <int kR>
__global__ void __launch_bounds__(kMtThreads, 16 / kMtWarps)
mttkrp_coo3_vec_kernel(int64_t I, int64_t nnz, int64_t nchunks, const int32_t* __restrict__ ii,
                       const int32_t* __restrict__ jj, const int32_t* __restrict__ kk,
                       const double* __restrict__ vals, const double* __restrict__ B,
                       const double* __restrict__ C, double* __restrict__ A, CarryWs cw,
                       bool reuse_b) {
  const int64_t c = (int64_t)blockIdx.x * kMtWarps + (threadIdx.x >> 5);
  if (c >= nchunks) return;
  const int64_t e0 = c * kMtChunk;
  const int64_t e1 = min64(e0 + kMtChunk, nnz);
  const int32_t row_first = ldg(ii + e0);
  const int32_t prev_row = e0 > 0 ? ldg(ii + e0 - 1) : -1;
  const bool tail_cont = e1 < nnz && ldg(ii + e1) == ldg(ii + e1 - 1);
  CooSrc src{ii, jj, kk, vals, e1, 0, 0, 0, 0.0};
  mttkrp_vec_body<kR>(I, e0, e1, row_first, prev_row, prev_row == row_first, tail_cont, c, B, C, A,
                      cw, src, reuse_b);
  if (e1 == nnz) zero_rows(A, (int64_t)ldg(ii + nnz - 1) + 1, I, threadIdx.x & 31, kR);
}

template <int kR>
__global__ void __launch_bounds__(kMtThreads, 16 / kMtWarps)
mttkrp_csf_vec_kernel(int64_t I, int64_t nslices, int64_t nfibers, int64_t nnz, int64_t nchunks,
                      const int32_t* __restrict__ crd0, const int32_t* __restrict__ pos1,
                      const int32_t* __restrict__ crd1, const int32_t* __restrict__ pos2,
                      const int32_t* __restrict__ crd2, const double* __restrict__ vals,
                      const double* __restrict__ B, const double* __restrict__ C,
                      double* __restrict__ A, CarryWs cw, bool reuse_b) {
  const int64_t c = (int64_t)blockIdx.x * kMtWarps + (threadIdx.x >> 5);
  if (c >= nchunks) return;
  const int64_t e0 = c * kMtChunk;
  const int64_t e1 = min64(e0 + kMtChunk, nnz);
  const int64_t f = ldg(cw.fstart + c), s = ldg(cw.sstart + c);
  const int32_t row_first = ldg(crd0 + s);
  const bool head_partial = ldg(pos2 + ldg(pos1 + s)) < e0;
  const int32_t prev_row = head_partial ? row_first : (s > 0 ? ldg(crd0 + s - 1) : -1);
  bool tail_cont = false;
  if (e1 < nnz) {
    const int64_t sn = ldg(cw.sstart + c + 1);        // slice of nonzero e1
    tail_cont = ldg(pos2 + ldg(pos1 + sn)) < e1;     // it started before e1
  }
  CsfSrc src{crd0, pos1, crd1, pos2, crd2, vals, nslices, nfibers, e1, f, s, 0, 0.0};
  mttkrp_vec_body<kR>(I, e0, e1, row_first, prev_row, head_partial, tail_cont, c, B, C, A, cw, src,
                      reuse_b);
  if (e1 == nnz) zero_rows(A, (int64_t)ldg(crd0 + nslices - 1) + 1, I, threadIdx.x & 31, kR);
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
// A row cut by chunk boundaries has a tail carry in the chunk where it starts
// (s) and head carries in chunks s+1 .. ce.  Two levels, fixed order
// (deterministic):
//   1. group prefix: chunks are grouped by 32; within a group, each head is
//      replaced by the running sum of the heads of its row from the group's
//      start (or the row's first head in the group) up to it;
//   2. owner: the warp of chunk s finds ce by galloping over the monotone
//      first_row array and adds tail[s] + the group prefixes at the last
//      chunk of the row in each group it spans (<= 1 + (ce - s) / 32 terms).
// The heaviest D5 slice spans ~1950 chunks: one warp summing them serially
// measured 328 us; this takes a few us.
constexpr int kFixGroup = 32;

template <int RPL>
__global__ void __launch_bounds__(kMtThreads)
mttkrp_group_prefix_kernel(int R, int64_t nchunks, CarryWs cw) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * kMtWarps + (threadIdx.x >> 5);
  const int64_t c0 = g * kFixGroup;
  if (c0 >= nchunks) return;
  const int64_t c1 = min64(c0 + kFixGroup, nchunks);
  double run[RPL];
  int32_t prow = -1;
  for (int64_t c = c0; c < c1; ++c) {
    const int32_t row = cw.head_row[c];
    if (row < 0) { prow = -1; continue; }
#pragma unroll
    for (int p = 0; p < RPL; ++p) {
      const int r = lane + 32 * p;
      if (r < R) {
        const double h = cw.head[c * R + r];
        run[p] = row == prow ? dadd(run[p], h) : h;
        cw.head[c * R + r] = run[p];
      }
    }
    prow = row;
  }
}

template <int RPL>
__global__ void __launch_bounds__(kMtThreads)
mttkrp_fixup_kernel(int R, int64_t nchunks, CarryWs cw, double* __restrict__ A) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * kMtWarps;
  for (int64_t c = (int64_t)blockIdx.x * kMtWarps + (threadIdx.x >> 5); c < nchunks; c += nwarps) {
    const int32_t row = cw.tail_row[c];
    if (row < 0) continue;
    // gallop: find ce = last chunk index with first_row == row (>= c + 1)
    int64_t lo = c + 1, step = 1;                 // first_row[lo] == row
    while (true) {
      const int64_t probe = lo + step;
      if (probe >= nchunks || ldg(cw.first_row + probe) != row) break;
      lo = probe;
      step <<= 1;
    }
    int64_t hi = min64(lo + step, nchunks) - 1;   // answer in [lo, hi]
    while (lo < hi) {
      const int64_t span = hi - lo;
      const int64_t st = (span + 31) / 32;
      const int64_t p = lo + (int64_t)(lane + 1) * st;
      const bool ok = p <= hi && ldg(cw.first_row + p) == row;
      const int nok = __popc(__ballot_sync(0xffffffffu, ok));
      const int64_t nlo = lo + (int64_t)nok * st;
      hi = min64(hi, lo + (int64_t)(nok + 1) * st - 1);
      lo = nlo;
    }
    const int64_t ce = lo;
#pragma unroll
    for (int p = 0; p < RPL; ++p) {
      const int r = lane + 32 * p;
      if (r >= R) continue;
      double tot = cw.tail[c * R + r];
      // last chunk of the row in each group from group(c + 1) to group(ce)
      for (int64_t gs = (c + 1) / kFixGroup; gs <= ce / kFixGroup; ++gs) {
        const int64_t last = min64(ce, gs * kFixGroup + kFixGroup - 1);
        tot = dadd(tot, cw.head[last * R + r]);
      }
      A[(int64_t)row * R + r] = tot;
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

static int group_grid(int64_t nch) {
  const int64_t ngroups = (nch + kFixGroup - 1) / kFixGroup;
  return (int)((ngroups + kMtWarps - 1) / kMtWarps);
}

static int fixup_grid(int64_t nch) {
  const int64_t want = (nch + kMtWarps - 1) / kMtWarps;
  const int64_t cap = 8LL * sl_host::sm_count();
  return (int)(want < cap ? want : cap);
}

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

// vectorised kernels: R in {16, 32, 64}, 32-byte aligned factor rows
static bool vec_path(const double* B, const double* C, const double* A, int R) {
  const bool aligned = (reinterpret_cast<uintptr_t>(B) & 31u) == 0 &&
                       (reinterpret_cast<uintptr_t>(C) & 31u) == 0 &&
                       (reinterpret_cast<uintptr_t>(A) & 31u) == 0;
  return aligned && (R == 16 || R == 32 || R == 64) && !getenv("SL_MTTKRP_SCALAR");
}

// group prefix + owner fix-up of the rows cut by chunk boundaries
static int launch_fixup(int R, int64_t nch, CarryWs cw, double* A, cudaStream_t s) {
  return dispatch_rpl(R, [&](auto rpl) {
    constexpr int RPL = decltype(rpl)::value;
    mttkrp_group_prefix_kernel<RPL><<<group_grid(nch), kMtThreads, 0, s>>>(R, nch, cw);
    mttkrp_fixup_kernel<RPL><<<fixup_grid(nch), kMtThreads, 0, s>>>(R, nch, cw, A);
    return sl_host::launch_status();
  });
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
  const bool reuse_b = !getenv("SL_MTTKRP_NOREUSE");
  if (vec_path(B, C, A, R)) {
    if (R == 16)
      mttkrp_coo3_vec_kernel<16><<<grid, kMtThreads, 0, s>>>(I, nnz, nch, i, j, k, vals, B, C, A,
                                                             cw, reuse_b);
    else if (R == 32)
      mttkrp_coo3_vec_kernel<32><<<grid, kMtThreads, 0, s>>>(I, nnz, nch, i, j, k, vals, B, C, A,
                                                             cw, reuse_b);
    else
      mttkrp_coo3_vec_kernel<64><<<grid, kMtThreads, 0, s>>>(I, nnz, nch, i, j, k, vals, B, C, A,
                                                             cw, reuse_b);
    return launch_fixup(R, nch, cw, A, s);
  }
  const int st2 = dispatch_rpl(R, [&](auto rpl) {
    constexpr int RPL = decltype(rpl)::value;
    mttkrp_coo3_kernel<RPL><<<grid, kMtThreads, 0, s>>>(I, R, nnz, nch, i, j, k, vals, B, C, A, cw);
    return SL_OK;
  });
  return st2 != SL_OK ? st2 : launch_fixup(R, nch, cw, A, s);
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
  const bool reuse_b = !getenv("SL_MTTKRP_NOREUSE");
  if (vec_path(B, C, A, R)) {
    if (R == 16)
      mttkrp_csf_vec_kernel<16><<<grid, kMtThreads, 0, s>>>(I, nslices, nfibers, nnz, nch, crd0,
                                                            pos1, crd1, pos2, crd2, vals, B, C, A,
                                                            cw, reuse_b);
    else if (R == 32)
      mttkrp_csf_vec_kernel<32><<<grid, kMtThreads, 0, s>>>(I, nslices, nfibers, nnz, nch, crd0,
                                                            pos1, crd1, pos2, crd2, vals, B, C, A,
                                                            cw, reuse_b);
    else
      mttkrp_csf_vec_kernel<64><<<grid, kMtThreads, 0, s>>>(I, nslices, nfibers, nnz, nch, crd0,
                                                            pos1, crd1, pos2, crd2, vals, B, C, A,
                                                            cw, reuse_b);
    return launch_fixup(R, nch, cw, A, s);
  }
  const int st2 = dispatch_rpl(R, [&](auto rpl) {
    constexpr int RPL = decltype(rpl)::value;
    mttkrp_csf_kernel<RPL><<<grid, kMtThreads, 0, s>>>(I, R, nslices, nfibers, nnz, nch, crd0,
                                                       pos1, crd1, pos2, crd2, vals, B, C, A, cw);
    return SL_OK;
  });
  return st2 != SL_OK ? st2 : launch_fixup(R, nch, cw, A, s);
}
