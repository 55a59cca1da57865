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
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "levels.cuh"
#include "tma.cuh"

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

constexpr int kCooVec = 4;                       // elements per vector load
constexpr int kCooHalo = 128;                    // staged past the tile end

template <int kCooThreads, int kCooVecPerThread, int kMinBlocks>
__global__ void __launch_bounds__(kCooThreads, kMinBlocks)
spmv_coo_kernel(int64_t nrows, int64_t nnz, const int32_t* __restrict__ rows,
                const int32_t* __restrict__ cols, const double* __restrict__ vals,
                const double* __restrict__ x, double* __restrict__ y, bool vec_ok) {
  constexpr int kCooIpt = kCooVec * kCooVecPerThread;  // items per thread
  constexpr int kCooTile = kCooThreads * kCooIpt;      // nonzeros owned per tile
  // s_row[4 + q] = row of staged item q; s_row[3] = row of the item before the tile
  __shared__ __align__(16) int32_t s_row[kCooTile + kCooHalo + 4];
  __shared__ __align__(16) double s_prod[kCooTile + kCooHalo];
  __shared__ uint16_t s_start[kCooTile];          // row-start items (< kCooTile + kCooHalo)
  __shared__ int32_t s_wcnt[kCooThreads / 32];
  __shared__ unsigned s_mask[kCooThreads / 32][kCooTile / kCooThreads];

  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * kCooTile;
  const int n_in = (int)min64(kCooTile, nnz - e0);               // owned row starts
  const int n_st = (int)min64(kCooTile + kCooHalo, nnz - e0);    // staged items

  // ---- stage rows + products: all loads of a thread are issued before use
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
    const int qh = kCooTile + tid;                 // halo item of this thread
    int32_t rh = 0, ch = 0;
    double vh = 0.0;
    if (qh < n_st) {
      rh = ldg(rows + e0 + qh);
      ch = ldg(cols + e0 + qh);
      vh = ldg(vals + e0 + qh);
    }
    double xg[kCooVecPerThread][4];
#pragma unroll
    for (int k = 0; k < kCooVecPerThread; ++k) {
      xg[k][0] = ldg(x + c4[k].x);
      xg[k][1] = ldg(x + c4[k].y);
      xg[k][2] = ldg(x + c4[k].z);
      xg[k][3] = ldg(x + c4[k].w);
    }
    const double xh = qh < n_st ? ldg(x + ch) : 0.0;
#pragma unroll
    for (int k = 0; k < kCooVecPerThread; ++k) {
      const int q = (k * kCooThreads + tid) * kCooVec;
      *reinterpret_cast<int4*>(s_row + 4 + q) = r4[k];
      *reinterpret_cast<double2*>(s_prod + q) =
          make_double2(dmul(va[k].x, xg[k][0]), dmul(va[k].y, xg[k][1]));
      *reinterpret_cast<double2*>(s_prod + q + 2) =
          make_double2(dmul(vb[k].x, xg[k][2]), dmul(vb[k].y, xg[k][3]));
    }
    if (qh < n_st) {
      s_row[4 + qh] = rh;
      s_prod[qh] = dmul(vh, xh);
    }
  } else {
    for (int q = tid; q < n_st; q += kCooThreads) {
      const int64_t g = e0 + q;
      s_row[4 + q] = ldg(rows + g);
      s_prod[q] = dmul(ldg(vals + g), ldg(x + ldg(cols + g)));
    }
  }
  if (tid == 0) s_row[3] = e0 == 0 ? -1 : ldg(rows + e0 - 1);
  __syncthreads();

  // ---- compact the row starts of the owned range with warp ballots; the
  // predecessor's row comes from a shuffle (one shared load per item), the
  // per-warp masks live in shared memory (no register spills)
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int kPerWarp = kCooTile / (kCooThreads / 32);   // 256 items per warp
  int cnt = 0;
#pragma unroll
  for (int b = 0; b < kPerWarp / 32; ++b) {
    const int q = warp * kPerWarp + b * 32 + lane;
    const int32_t r = s_row[4 + q];
    int32_t rp = __shfl_up_sync(0xffffffffu, r, 1);
    if (lane == 0) rp = s_row[3 + q];
    const unsigned m = __ballot_sync(0xffffffffu, q < n_in && r != rp);
    if (lane == 0) s_mask[warp][b] = m;
    cnt += __popc(m);
  }
  if (lane == 0) s_wcnt[warp] = cnt;
  __syncthreads();
  int base = 0, nstart = 0;
#pragma unroll
  for (int w = 0; w < kCooThreads / 32; ++w) {
    const int c = s_wcnt[w];
    base += w < warp ? c : 0;
    nstart += c;
  }
#pragma unroll
  for (int b = 0; b < kPerWarp / 32; ++b) {
    const unsigned m = s_mask[warp][b];
    if (m & (1u << lane))
      s_start[base + __popc(m & ((1u << lane) - 1u))] = (uint16_t)(warp * kPerWarp + b * 32 + lane);
    base += __popc(m);
  }
  __syncthreads();

  // ---- thread per row, lockstep: rows summed in storage order from +0.0
  bool cont = false;   // this thread owns the last row and it runs past the halo
  int32_t cont_r = 0;
  double cont_acc = 0.0;
  for (int si = tid; si < nstart; si += kCooThreads) {
    const int q = s_start[si];
    const int32_t r = s_row[4 + q];
    const int32_t rp = s_row[3 + q];
    double acc = 0.0;
    int64_t g;
    if (si + 1 < nstart) {
      const int qe = s_start[si + 1];
      for (int u = q; u < qe; ++u) acc = dadd(acc, s_prod[u]);
      g = e0 + qe;
    } else {
      // last row starting in this tile: runs into the halo (and beyond)
      int u = q;
      for (; u < n_st && s_row[4 + u] == r; ++u) acc = dadd(acc, s_prod[u]);
      g = e0 + u;
      if (u == n_st && g < nnz) {
        // the row goes on past the halo: the owner's warp finishes it (below)
        cont = true;
        cont_r = r;
        cont_acc = acc;
        for (int32_t q2 = rp + 1; q2 < r; ++q2) y[q2] = 0.0;
        continue;
      }
    }
    y[r] = acc;
    for (int32_t q2 = rp + 1; q2 < r; ++q2) y[q2] = 0.0;          // empty rows before r
    if (g == nnz)                                                   // the matrix's last row
      for (int64_t q2 = (int64_t)r + 1; q2 < nrows; ++q2) y[q2] = 0.0;
  }
  // continuation of a long row by the owner's warp (no block barrier on the
  // common path): 32 coalesced products per round, added in order through
  // shuffles (a power-law row no longer costs one dependent global walk per
  // element: D5's fibres as COO 2.67 -> 0.86 ms; a block-wide version, 0.58
  // ms, put a barrier on every tile and cost D1 0.4-0.8 us)
  const unsigned wm = __ballot_sync(0xffffffffu, cont);
  if (!wm) return;
  const int src = __ffs(wm) - 1;
  const int32_t r = __shfl_sync(0xffffffffu, cont_r, src);
  int64_t g = e0 + n_st;
  double acc = __shfl_sync(0xffffffffu, cont_acc, src);
  for (;;) {
    const int64_t e = g + lane;
    const bool in = e < nnz && ldg(rows + e) == r;
    const double pr = in ? dmul(ldg(vals + e), ldg(x + ldg(cols + e))) : 0.0;
    const int cnt = __popc(__ballot_sync(0xffffffffu, in));   // rows sorted: a prefix
    for (int u = 0; u < cnt; ++u) acc = dadd(acc, __shfl_sync(0xffffffffu, pr, u));
    g += cnt;
    if (cnt < 32) break;
  }
  if (lane == src) {
    y[r] = acc;
    if (g == nnz)                                                   // the matrix's last row
      for (int64_t q2 = (int64_t)r + 1; q2 < nrows; ++q2) y[q2] = 0.0;
  }
}

// ---------------------------------------------------------------------------
// K2a: CSR row-block SpMV.  A block owns kCsrRows consecutive rows; their
// nonzeros are a contiguous range, staged in coalesced chunks of kCsrChunk
// products through shared memory; the thread of row r adds the chunk's
// products that belong to r in storage order.  (engine.py:591-634.)

constexpr int kCsrThreads = 256;
constexpr int kCsrRows = kCsrThreads;
constexpr int kCsrIpt = 8;
constexpr int kCsrChunk = kCsrThreads * kCsrIpt;   // 2048 products per staging round

template <int kHashX>
struct XOperand;

template <>
struct XOperand<0> {            // dense x: locate = parent*n + c (levels.py:268-269)
  const double* x;
  SL_DEV double term(double a, int32_t c) const { return dmul(a, ldg(x + c)); }
};

template <>
struct XOperand<1> {             // hashed x: probe (levels.py:270-280), miss -> no term
  HashedLevel lv;
  const double* xv;
  // A miss contributes no term.  The row accumulator starts at +0.0 and can
  // never become -0.0 under round-to-nearest, so "no term" == "+0.0 term".
  SL_DEV double term(double a, int32_t c) const {
    const PosFound pf = lv.locate(0, c);
    return pf.found ? dmul(a, ldg(xv + pf.pos)) : 0.0;
  }
};

template <>
struct XOperand<2> {                // hashed x through the slot map (hashed.cu): one
  HashedLevel lv;                   // resolved locate per coordinate c < n, probing
  const double* xv;                 // only for coordinates outside the map
  const unsigned long long* map;
  int64_t n;
  SL_DEV int64_t slot(int32_t c) const {
    if (c < n) {
      const unsigned long long m = __ldg(map + c);
      return m == ~0ull ? -1 : (int64_t)(uint32_t)m;
    }
    const PosFound pf = lv.locate(0, c);
    return pf.found ? pf.pos : -1;
  }
  SL_DEV double term(double a, int32_t c) const {
    const int64_t sl = slot(c);
    return sl >= 0 ? dmul(a, ldg(xv + sl)) : 0.0;
  }
};

template <>
struct XOperand<3> {                // sparse-vector x (compressed, ordered, unique):
  const int32_t* map;               // index of coordinate c in x, -1 if absent — the
  const double* xv;                 // intersection {A1, x1} of the product's j-lattice
  int64_t n;                        // (engine.py:211-225, 591-634): absent -> no term
  SL_DEV int64_t slot(int32_t c) const { return c < n ? (int64_t)__ldg(map + c) : -1; }
  SL_DEV double term(double a, int32_t c) const {
    const int64_t sl = slot(c);
    return sl >= 0 ? dmul(a, ldg(xv + sl)) : 0.0;
  }
};

// Stage products of elements [cs, cs + n) into s_prod with every load of a
// thread issued before its first use (crd/vals stream, then the x gathers).
template <int kThreads, int kIpt>
SL_DEV void stage_products(const int32_t* __restrict__ crd, const double* __restrict__ vals,
                           int64_t cs, int n, XOperand<0> xop, double* s_prod) {
  const int tid = threadIdx.x;
  int32_t c[kIpt];
  double v[kIpt], xv[kIpt];
  if (n == kThreads * kIpt) {   // full chunk: unpredicated batches
#pragma unroll
    for (int k = 0; k < kIpt; ++k) c[k] = ld_stream(crd + cs + tid + k * kThreads);
#pragma unroll
    for (int k = 0; k < kIpt; ++k) v[k] = ld_stream(vals + cs + tid + k * kThreads);
#pragma unroll
    for (int k = 0; k < kIpt; ++k) xv[k] = ldg(xop.x + c[k]);
#pragma unroll
    for (int k = 0; k < kIpt; ++k) s_prod[tid + k * kThreads] = dmul(v[k], xv[k]);
    return;
  }
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {
    const int q = tid + k * kThreads;
    c[k] = q < n ? ld_stream(crd + cs + q) : 0;
    v[k] = q < n ? ld_stream(vals + cs + q) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < kIpt; ++k) xv[k] = tid + k * kThreads < n ? ldg(xop.x + c[k]) : 0.0;
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {
    const int q = tid + k * kThreads;
    if (q < n) s_prod[q] = dmul(v[k], xv[k]);
  }
}

// Mapped hashed x: crd/vals, then the map entries, then x — each batch of
// loads independent of the next batch's wait.
template <int kThreads, int kIpt, int kX>
SL_DEV void stage_products(const int32_t* __restrict__ crd, const double* __restrict__ vals,
                           int64_t cs, int n, XOperand<kX> xop, double* s_prod) {
  const int tid = threadIdx.x;
  int32_t c[kIpt];
  double v[kIpt];
  int64_t sl[kIpt];
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {
    const int q = tid + k * kThreads;
    c[k] = q < n ? ld_stream(crd + cs + q) : 0;
    v[k] = q < n ? ld_stream(vals + cs + q) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < kIpt; ++k) sl[k] = tid + k * kThreads < n ? xop.slot(c[k]) : -1;
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {
    const int q = tid + k * kThreads;
    if (q < n) s_prod[q] = sl[k] >= 0 ? dmul(v[k], ldg(xop.xv + sl[k])) : 0.0;
  }
}

// Hashed x: hybrid probing.  Each lane first probes its own element for
// kHashSolo steps (the whole answer for short probe sequences); elements still
// unresolved are then finished one at a time by the whole warp, 32
// consecutive probe steps per round (one coalesced 128-byte load), taking the
// first match-or-empty in probe order — the sequential answer.
constexpr int kHashSolo = 4;
constexpr int kHashPer = 8;     // probe steps per lane per cooperative round (256 per warp)

template <int kThreads, int kIpt>
SL_DEV void stage_products(const int32_t* __restrict__ crd, const double* __restrict__ vals,
                           int64_t cs, int n, XOperand<1> xop, double* s_prod) {
  const int tid = threadIdx.x, lane = tid & 31;
  const HashedLevel& lv = xop.lv;
  const int64_t w = lv.w;
#pragma unroll 1
  for (int k = 0; k < kIpt; ++k) {
    const int q = tid + k * kThreads;
    const bool valid = q < n;
    const int32_t c = valid ? ld_stream(crd + cs + q) : 0;
    const double a = valid ? ld_stream(vals + cs + q) : 0.0;
    int64_t slot = -1;
    bool done = !valid;
    const int64_t home = c % w;
    int64_t step = 0;
    for (; step < kHashSolo && step < w && !done; ++step) {
      int64_t sidx = home + step;
      if (sidx >= w) sidx -= w;
      const int32_t v = ldg(lv.crd + sidx);
      if (v == c) { slot = sidx; done = true; }
      else if (v == kEmpty) done = true;
    }
    if (step >= w) done = true;   // whole (tiny) segment scanned
    unsigned pending = __ballot_sync(0xffffffffu, !done);
    while (pending) {
      const int src = __ffs(pending) - 1;
      pending &= pending - 1;
      const int32_t cc = __shfl_sync(0xffffffffu, c, src);
      const int64_t hh = cc % w;
      int64_t found = -1;
      // each round the warp probes kHashPer * 32 consecutive steps: lane l
      // checks steps s0 + kHashPer*l + {0..kHashPer-1} (independent loads);
      // the lowest step that matches or is empty ends the probe
      for (int64_t s0 = kHashSolo; s0 < w; s0 += kHashPer * 32) {
        int32_t v[kHashPer];
        const int64_t sb = s0 + (int64_t)kHashPer * lane;   // this lane's first step
#pragma unroll
        for (int k = 0; k < kHashPer; ++k) {
          const int64_t st = sb + k;
          int64_t p = hh + st;
          while (p >= w) p -= w;
          v[k] = st < w ? ldg(lv.crd + p) : 0;
        }
        int hit_k = kHashPer;
#pragma unroll
        for (int k = kHashPer - 1; k >= 0; --k)
          if (sb + k < w && (v[k] == cc || v[k] == kEmpty)) hit_k = k;
        const bool hit_match = hit_k < kHashPer && v[hit_k < kHashPer ? hit_k : 0] == cc;
        const unsigned hit = __ballot_sync(0xffffffffu, hit_k < kHashPer);
        if (hit) {
          const int f = __ffs(hit) - 1;
          const int hk = __shfl_sync(0xffffffffu, hit_k, f);
          const bool mf = __shfl_sync(0xffffffffu, hit_match ? 1 : 0, f) != 0;
          int64_t pf = hh + s0 + (int64_t)kHashPer * f + hk;
          while (pf >= w) pf -= w;
          found = mf ? pf : -1;
          break;
        }
      }
      if (lane == src) slot = found;
    }
    if (valid) s_prod[q] = slot >= 0 ? dmul(a, ldg(xop.xv + slot)) : 0.0;
  }
}

template <int kHashX, int kRows = kCsrRows>
__global__ void __launch_bounds__(kCsrThreads, kHashX == 1 ? 4 : 8)
spmv_csr_rowblock_kernel(int64_t nrows, const int32_t* __restrict__ pos,
                         const int32_t* __restrict__ crd, const double* __restrict__ vals,
                         XOperand<kHashX> xop, double* __restrict__ y) {
  __shared__ int32_t s_pos[kRows + 1];
  __shared__ __align__(16) double s_prod[kCsrChunk];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  const int nr = (int)min64(kRows, nrows - r0);
  for (int t = tid; t <= nr; t += kCsrThreads) s_pos[t] = ldg(pos + r0 + t);
  __syncthreads();
  const int32_t eb = s_pos[0], ee = s_pos[nr];
  const bool mine = tid < nr;
  const int32_t rb = mine ? s_pos[tid] : 0, re = mine ? s_pos[tid + 1] : 0;
  double acc = 0.0;
  for (int32_t cs = eb; cs < ee; cs += kCsrChunk) {
    const int n_in = min(kCsrChunk, ee - cs);
    stage_products<kCsrThreads, kCsrIpt>(crd, vals, cs, n_in, xop, s_prod);
    __syncthreads();
    const int lo = max(rb, cs) - cs, hi = min(re, cs + n_in) - cs;
    for (int u = lo; u < hi; ++u) acc = dadd(acc, s_prod[u]);
    __syncthreads();
  }
  if (mine) y[r0 + tid] = acc;
}

// K2f: CSR row-stage.  The block's whole nonzero range (up to kCap elements
// per round) is bulk-copied (TMA, cp.async.bulk: no LSU wavefronts, no
// registers) into shared memory; then the thread of row r walks its own row
// in storage order like the ELL kernel walks its slots: batches of kBatch
// crd reads from smem (stride = row length: odd strides are conflict-free),
// kBatch x gathers in flight (consecutive rows' u-th columns are adjacent for
// banded matrices, so these coalesce), then the ordered add chain.  Products
// never round-trip through smem.  Many small blocks per SM, several waves:
// while some blocks walk their rows, others' copies are in flight.
//
// Measured on the 64^3 27-point stencil (tools/ab_csr.py, L2 cold and clean,
// DESIGN.md §3): K2a 28.6 us -> 32-row blocks at 20/SM 23.8 us (64-row
// blocks at 10/SM 24.5, 128-row at 5/SM 24.7, batch 14/27 no better).  Also
// measured and dropped: K2a with a 2-4 stage cp.async (LDGSTS) ring of
// chunks (29-41 us: the in-place products and read-back cost more L1
// wavefronts than the latency they hide), and a persistent warp-specialised
// version of this kernel (one CTA/SM, producer warp + 2-8 consumer groups
// with double-buffered stages: 26.7-37.6 us; too few row-walking threads per
// SM), and a persistent one-warp-per-block version that loads the next
// tile's row bounds during the current walk (25.3-28.8 us at 10-20 blocks/SM:
// hardware block scheduling of many short blocks beats the software loop).
// Staging the range with 16-byte cp.async (LDGSTS) by all threads instead of
// the bulk copy: 24.8 us (round-1 A/B; log not retained).  On short,
// irregular rows (D1, Poisson(10)) the row walk diverges
// (warps run the longest row) and K2a stays faster (20.5 vs 29 us), so the
// automatic choice takes K2f only for rows averaging >= 16 nonzeros.

#ifdef SL_WITH_ALT   // row-stage CSR (variant 4): A/B variant, opt-in build (SL_BUILD_ALT=1)
constexpr int kCsrStageRows = 32;
constexpr int kCsrStageCap = 896;     // 28 per row: the 27-point stencil's rows fit in one round
constexpr int kCsrStageBatch = 9;
constexpr int kCsrStageBlocks = 20;   // 20 x 11.3 KB of shared memory per SM

template <int kRows, int kCap>
struct CsrStageSmem {
  uint64_t bar;
  int32_t pos[kRows + 1];
  __align__(16) int32_t crd[kCap];
  __align__(16) double val[kCap];
};

template <int kRows, int kCap, int kBatch, int kMinBlocks>
__global__ void __launch_bounds__(kRows, kMinBlocks)
spmv_csr_stage_kernel(int64_t nrows, const int32_t* __restrict__ pos,
                      const int32_t* __restrict__ crd, const double* __restrict__ vals,
                      const double* __restrict__ x, double* __restrict__ y) {
  static_assert(kCap % 4 == 0, "granule-aligned capacity");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<CsrStageSmem<kRows, kCap>*>(smem_raw);
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  const int nr = (int)min64(kRows, nrows - r0);
  if (tid == 0) {
    mbar_init(&sm.bar, 1);
    fence_mbar_init();
  }
  for (int t = tid; t <= nr; t += kRows) sm.pos[t] = ldg(pos + r0 + t);
  __syncthreads();
  const int32_t eb = sm.pos[0], ee = sm.pos[nr];
  const int32_t a0 = eb & ~3;
  const int nch = ee > eb ? (ee - a0 + kCap - 1) / kCap : 0;
  const bool mine = tid < nr;
  const int32_t rb = mine ? sm.pos[tid] : 0, re = mine ? sm.pos[tid + 1] : 0;
  double acc = 0.0;
  for (int k = 0; k < nch; ++k) {
    const int32_t c0 = a0 + k * kCap;
    const int32_t c1 = min(c0 + kCap, ee);
    if (tid == 0) {
      const uint32_t bc = (uint32_t)(((c1 - c0 + 3) & ~3) * 4);
      const uint32_t bv = (uint32_t)(((c1 - c0 + 1) & ~1) * 8);
      mbar_arrive_expect_tx(&sm.bar, bc + bv);
      bulk_g2s(sm.crd, crd + c0, bc, &sm.bar);
      bulk_g2s(sm.val, vals + c0, bv, &sm.bar);
    }
    mbar_wait(&sm.bar, k & 1);
    const int lo = max(rb, c0) - c0, hi = min(re, c1) - c0;
    for (int u = lo; u < hi; u += kBatch) {
      const int n = min(kBatch, hi - u);
      int32_t c[kBatch];
      double xv[kBatch], v[kBatch];
#pragma unroll
      for (int b = 0; b < kBatch; ++b) c[b] = b < n ? sm.crd[u + b] : 0;
#pragma unroll
      for (int b = 0; b < kBatch; ++b) xv[b] = b < n ? ldg(x + c[b]) : 0.0;
#pragma unroll
      for (int b = 0; b < kBatch; ++b) v[b] = b < n ? sm.val[u + b] : 0.0;
#pragma unroll
      for (int b = 0; b < kBatch; ++b)
        if (b < n) acc = dadd(acc, dmul(v[b], xv[b]));
    }
    if (k + 1 < nch) {
      __syncthreads();            // every row done with this round's stage
      if (tid == 0) fence_proxy_async_smem();
    }
  }
  if (mine) y[r0 + tid] = acc;
}

template <int kRows, int kCap, int kBatch, int kMinBlocks>
static void launch_csr_stage(int64_t nrows, const int32_t* pos, const int32_t* crd,
                             const double* vals, const double* x, double* y, cudaStream_t s) {
  constexpr size_t smem = sizeof(CsrStageSmem<kRows, kCap>);
  auto kern = spmv_csr_stage_kernel<kRows, kCap, kBatch, kMinBlocks>;
  static unsigned long long attr_set = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > 48 * 1024 && !(__atomic_load_n(&attr_set, __ATOMIC_ACQUIRE) >> (dev & 63) & 1ull)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    __atomic_fetch_or(&attr_set, 1ull << (dev & 63), __ATOMIC_ACQ_REL);
  }
  kern<<<(int)((nrows + kRows - 1) / kRows), kRows, smem, s>>>(nrows, pos, crd, vals, x, y);
}

// K2r: row-stage with a register hand-off.  K2f holds its shared-memory stage
// for the whole walk (gathers and the ordered add chain), which caps the rows
// in flight at ~640 per SM.  Here a persistent one-warp block copies each
// lane's row (<= kMaxRow nonzeros) from the stage into registers and at once
// bulk-copies the NEXT tile into the same stage, so one tile's gathers and
// adds overlap the next tile's HBM read.  Tiles with a longer row walk the
// stage as K2f does; tiles beyond the stage capacity read global memory.
// The register batch's terms: dense x gathers x[c]; a slot-mapped hashed x
// (kX 2) or a sparse-vector x (kX 3) first gathers the coordinate's slot, then
// x[slot]; a missing coordinate contributes no term (+0.0, see XOperand<1>).
#endif  // SL_WITH_ALT

template <int kX, int kB>
SL_DEV void handoff_terms(const XOperand<kX>& xop, const int32_t* c, const double* v, int u0,
                          int len, double* t) {
  if constexpr (kX == 0) {
    double xv[kB];
#pragma unroll
    for (int b = 0; b < kB; ++b) xv[b] = u0 + b < len ? ldg(xop.x + c[b]) : 0.0;
#pragma unroll
    for (int b = 0; b < kB; ++b) t[b] = dmul(v[b], xv[b]);
  } else {
    int64_t sl[kB];
#pragma unroll
    for (int b = 0; b < kB; ++b) sl[b] = u0 + b < len ? xop.slot(c[b]) : -1;
    double xv[kB];
#pragma unroll
    for (int b = 0; b < kB; ++b) xv[b] = sl[b] >= 0 ? ldg(xop.xv + sl[b]) : 0.0;
#pragma unroll
    for (int b = 0; b < kB; ++b) t[b] = sl[b] >= 0 ? dmul(v[b], xv[b]) : 0.0;
  }
}

// Up to kMaxPeers output buffers the epilogue stores every row into: the
// all-gather of y fused into the SpMV (each GPU writes its row block straight
// into every peer's full-y buffer over NVLink — symmetric / IPC-mapped
// pointers, already offset to this rank's first row).
constexpr int kMaxPeers = 8;
struct PeerOut {
  double* p[kMaxPeers];
  int n;
};

template <int kCap, int kMaxRow, int kBatch, int kMinBlocks, int kX, bool kPeers = false>
__global__ void __launch_bounds__(32, kMinBlocks)
spmv_csr_handoff_kernel(int64_t nrows, const int32_t* __restrict__ pos,
                        const int32_t* __restrict__ crd, const double* __restrict__ vals,
                        XOperand<kX> xop, double* __restrict__ y, PeerOut peers) {
  static_assert(kCap % 4 == 0 && kMaxRow % kBatch == 0, "shapes");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  int32_t* s_crd = reinterpret_cast<int32_t*>(smem_raw + 16);
  double* s_val = reinterpret_cast<double*>(smem_raw + 16 + kCap * 4);
  const int lane = threadIdx.x;
  const int64_t ntiles = (nrows + 31) / 32;
  int64_t tile = blockIdx.x;
  if (tile >= ntiles) return;
  pdl_wait();            // COO path: launched with PDL behind the row-pointer pass
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int32_t a0, int32_t ee) {   // lane 0: stage [a0, ee) (granule-rounded)
    const uint32_t bc = (uint32_t)(((ee - a0 + 3) & ~3) * 4);
    const uint32_t bv = (uint32_t)(((ee - a0 + 1) & ~1) * 8);
    mbar_arrive_expect_tx(bar, bc + bv);
    bulk_g2s(s_crd, crd + a0, bc, bar);
    bulk_g2s(s_val, vals + a0, bv, bar);
  };
  int64_t r0 = tile * 32;
  int nr = (int)min64(32, nrows - r0);
  int32_t pb = lane < nr ? ldg(pos + r0 + lane) : 0;
  int32_t pe = lane < nr ? ldg(pos + r0 + lane + 1) : 0;
  int32_t eb = __shfl_sync(0xffffffffu, pb, 0), ee = __shfl_sync(0xffffffffu, pe, nr - 1);
  int32_t a0 = eb & ~3;
  bool staged = ee > eb && ee - a0 <= kCap;
  if (staged && lane == 0) issue(a0, ee);
  uint32_t phase = 0;
  for (;;) {
    ee = __shfl_sync(0xffffffffu, pe, nr - 1);   // this tile's element range [eb, ee)
    // next tile's bounds: in flight during this tile's wait and copy
    const int64_t next = tile + gridDim.x;
    const int64_t nr0 = next * 32;
    const int nnr = next < ntiles ? (int)min64(32, nrows - nr0) : 0;
    const int32_t npb = lane < nnr ? ldg(pos + nr0 + lane) : 0;
    const int32_t npe = lane < nnr ? ldg(pos + nr0 + lane + 1) : 0;
    auto issue_next = [&]() -> bool {
      if (nnr == 0) return false;
      const int32_t neb = __shfl_sync(0xffffffffu, npb, 0);
      const int32_t nee = __shfl_sync(0xffffffffu, npe, nnr - 1);
      const bool ns = nee > neb && nee - (neb & ~3) <= kCap;
      if (ns && lane == 0) {
        fence_proxy_async_smem();
        issue(neb & ~3, nee);
      }
      return ns;
    };
    double acc = 0.0;
    bool next_staged = false;
    const int len = pe - pb;
    bool reg = false;
    if (staged) {
      mbar_wait(bar, phase);
      phase ^= 1u;
      reg = __all_sync(0xffffffffu, len <= kMaxRow);
    }
    if (reg) {
      const int off = pb - a0;
      int32_t c[kMaxRow];
      double v[kMaxRow];
#pragma unroll
      for (int u = 0; u < kMaxRow; ++u) {
        c[u] = u < len ? s_crd[off + u] : 0;
        v[u] = u < len ? s_val[off + u] : 0.0;
      }
      __syncwarp();                     // every lane's row is in registers
      next_staged = issue_next();
#pragma unroll
      for (int u0 = 0; u0 < kMaxRow; u0 += kBatch) {
        double t[kBatch];
        handoff_terms<kX, kBatch>(xop, c + u0, v + u0, u0, len, t);
#pragma unroll
        for (int b = 0; b < kBatch; ++b)
          if (u0 + b < len) acc = dadd(acc, t[b]);
      }
    } else {
      // a row longer than kMaxRow, or a tile beyond the stage: rounds of kCap
      // elements through the stage (round 0 already staged if the tile fits),
      // products formed in place by the whole warp, then every lane adds its
      // row's part of the round in order (K2a's split of the work: a long row
      // costs one add per element, not a gather chain per element)
      const int nch = ee > eb ? (ee - a0 + kCap - 1) / kCap : 0;
      for (int k = 0; k < nch; ++k) {
        const int32_t c0 = a0 + k * kCap, c1 = min(c0 + kCap, ee);
        if (k > 0 || !staged) {
          if (lane == 0) {
            fence_proxy_async_smem();
            issue(c0, c1);
          }
          mbar_wait(bar, phase);
          phase ^= 1u;
        }
        for (int q = max(eb, c0) - c0 + lane; q < c1 - c0; q += 32)
          s_val[q] = xop.term(s_val[q], s_crd[q]);
        __syncwarp();
        const int lo = max(pb, c0) - c0, hi = min(pe, c1) - c0;
        for (int u = lo; u < hi; ++u) acc = dadd(acc, s_val[u]);
        __syncwarp();
      }
      next_staged = issue_next();
    }
    if (lane < nr) {
      if (kPeers) {
#pragma unroll 1
        for (int q = 0; q < peers.n; ++q) peers.p[q][r0 + lane] = acc;   // posted stores
      } else {
        y[r0 + lane] = acc;
      }
    }
    if (nnr == 0) break;
    tile = next;
    r0 = nr0;
    nr = nnr;
    pb = npb;
    pe = npe;
    eb = __shfl_sync(0xffffffffu, pb, 0);
    a0 = eb & ~3;
    staged = next_staged;
  }
}

template <int kCap, int kMaxRow, int kBatch, int kMinBlocks, int kX>
static void launch_csr_handoff(int64_t nrows, const int32_t* pos, const int32_t* crd,
                               const double* vals, XOperand<kX> xop, double* y, int blocks_per_sm,
                               cudaStream_t s, bool pdl = false, const PeerOut* peers = nullptr) {
  constexpr size_t smem = 16 + (size_t)kCap * 12;
  const int64_t ntiles = (nrows + 31) / 32;
  const int grid = (int)min64(ntiles, (int64_t)sl_host::sm_count() * blocks_per_sm);
  if (peers) {
    spmv_csr_handoff_kernel<kCap, kMaxRow, kBatch, kMinBlocks, kX, true><<<grid, 32, smem, s>>>(
        nrows, pos, crd, vals, xop, y, *peers);
    return;
  }
  if (pdl) {
    sl_host::launch_pdl(spmv_csr_handoff_kernel<kCap, kMaxRow, kBatch, kMinBlocks, kX>, dim3(grid),
                        dim3(32), s, smem, nrows, pos, crd, vals, xop, y, PeerOut{});
    return;
  }
  spmv_csr_handoff_kernel<kCap, kMaxRow, kBatch, kMinBlocks, kX><<<grid, 32, smem, s>>>(
      nrows, pos, crd, vals, xop, y, PeerOut{});
}

#ifdef SL_WITH_ALT
// K2q: the register hand-off with a ring of two stages per warp.  K2r keeps
// one tile's bulk copy in flight per warp (12 x 10.5 KB per SM), and a warp
// then waits out the copy latency once per tile.  Here tiles t+1 and t+2 are
// in flight while tile t's gathers and adds run (10 warps x 2 x 10.5 KB per
// SM), and the row pointer of a tile is read two iterations before its copy
// is issued, so neither latency sits on a warp's path.  Arithmetic per row is
// K2r's (same terms, same ordered add chain), so the results are bit-equal.
struct TileRows {
  int32_t pb, pe;   // this lane's row [pb, pe) (0, 0 past the tile's last row)
  int nr;           // rows in the tile (0: no such tile)
};

SL_DEV TileRows load_tile_rows(const int32_t* __restrict__ pos, int64_t nrows, int64_t tile,
                               int64_t ntiles, int lane) {
  TileRows t;
  t.nr = tile < ntiles ? (int)min64(32, nrows - tile * 32) : 0;
  t.pb = lane < t.nr ? ldg(pos + tile * 32 + lane) : 0;
  t.pe = lane < t.nr ? ldg(pos + tile * 32 + lane + 1) : 0;
  return t;
}

template <int kCap, int kMaxRow, int kBatch, int kMinBlocks, int kX>
__global__ void __launch_bounds__(32, kMinBlocks)
spmv_csr_ring_kernel(int64_t nrows, const int32_t* __restrict__ pos,
                     const int32_t* __restrict__ crd, const double* __restrict__ vals,
                     XOperand<kX> xop, double* __restrict__ y) {
  static_assert(kCap % 4 == 0 && kMaxRow % kBatch == 0, "shapes");
  constexpr uint32_t kStage = (uint32_t)kCap * 12;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);   // [2]
  unsigned char* sbase = smem_raw + 16;
  const int lane = threadIdx.x;
  const int64_t ntiles = (nrows + 31) / 32, G = gridDim.x;
  int64_t tile = blockIdx.x;
  if (tile >= ntiles) return;
  pdl_wait();            // COO path: launched with PDL behind the row-pointer pass
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto s_crd = [&](int s) { return reinterpret_cast<int32_t*>(sbase + s * kStage); };
  auto s_val = [&](int s) { return reinterpret_cast<double*>(sbase + s * kStage + kCap * 4); };
  auto issue = [&](int s, int32_t a0, int32_t ee) {   // lane 0: stage [a0, ee) into slot s
    const uint32_t bc = (uint32_t)(((ee - a0 + 3) & ~3) * 4);
    const uint32_t bv = (uint32_t)(((ee - a0 + 1) & ~1) * 8);
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bars[s], bc + bv);
    bulk_g2s(s_crd(s), crd + a0, bc, &bars[s]);
    bulk_g2s(s_val(s), vals + a0, bv, &bars[s]);
  };
  auto try_issue = [&](const TileRows& t, int s) -> bool {   // stage tile t if it fits
    if (t.nr == 0) return false;
    const int32_t eb = __shfl_sync(0xffffffffu, t.pb, 0);
    const int32_t ee = __shfl_sync(0xffffffffu, t.pe, t.nr - 1);
    const bool ok = ee > eb && ee - (eb & ~3) <= kCap;
    if (ok && lane == 0) issue(s, eb & ~3, ee);
    return ok;
  };
  TileRows t0 = load_tile_rows(pos, nrows, tile, ntiles, lane);
  TileRows t1 = load_tile_rows(pos, nrows, tile + G, ntiles, lane);
  TileRows t2 = load_tile_rows(pos, nrows, tile + 2 * G, ntiles, lane);
  bool st0 = try_issue(t0, 0), st1 = try_issue(t1, 1);
  uint32_t ph = 0;       // bit s: the parity stage s's next wait expects
  int s = 0;
  for (;;) {
    const TileRows t3 = load_tile_rows(pos, nrows, tile + 3 * G, ntiles, lane);
    const int32_t eb = __shfl_sync(0xffffffffu, t0.pb, 0);
    const int32_t ee = __shfl_sync(0xffffffffu, t0.pe, t0.nr - 1);
    const int32_t a0 = eb & ~3;
    const int len = t0.pe - t0.pb;
    double acc = 0.0;
    bool st2 = false, reg = false;
    if (st0) {
      mbar_wait(&bars[s], (ph >> s) & 1u);
      ph ^= 1u << s;
      reg = __all_sync(0xffffffffu, len <= kMaxRow);
    }
    if (reg) {
      const int off = t0.pb - a0;
      const int32_t* sc = s_crd(s);
      const double* sv = s_val(s);
      int32_t c[kMaxRow];
      double v[kMaxRow];
#pragma unroll
      for (int u = 0; u < kMaxRow; ++u) {
        c[u] = u < len ? sc[off + u] : 0;
        v[u] = u < len ? sv[off + u] : 0.0;
      }
      __syncwarp();                     // every lane's row is in registers
      st2 = try_issue(t2, s);
#pragma unroll
      for (int u0 = 0; u0 < kMaxRow; u0 += kBatch) {
        double t[kBatch];
        handoff_terms<kX, kBatch>(xop, c + u0, v + u0, u0, len, t);
#pragma unroll
        for (int b = 0; b < kBatch; ++b)
          if (u0 + b < len) acc = dadd(acc, t[b]);
      }
    } else {
      // K2r's rounds through this tile's slot (round 0 already there if the
      // tile was staged); the other slot's copy stays in flight
      int32_t* sc = s_crd(s);
      double* sv = s_val(s);
      const int nch = ee > eb ? (ee - a0 + kCap - 1) / kCap : 0;
      for (int k = 0; k < nch; ++k) {
        const int32_t c0 = a0 + k * kCap, c1 = min(c0 + kCap, ee);
        if (k > 0 || !st0) {
          if (lane == 0) issue(s, c0, c1);
          mbar_wait(&bars[s], (ph >> s) & 1u);
          ph ^= 1u << s;
        }
        for (int q = max(eb, c0) - c0 + lane; q < c1 - c0; q += 32) sv[q] = xop.term(sv[q], sc[q]);
        __syncwarp();
        const int lo = max(t0.pb, c0) - c0, hi = min(t0.pe, c1) - c0;
        for (int u = lo; u < hi; ++u) acc = dadd(acc, sv[u]);
        __syncwarp();
      }
      st2 = try_issue(t2, s);
    }
    if (lane < t0.nr) y[tile * 32 + lane] = acc;
    if (t1.nr == 0) break;
    tile += G;
    t0 = t1;
    t1 = t2;
    t2 = t3;
    st0 = st1;
    st1 = st2;
    s ^= 1;
  }
}

// A/B knob: SL_CARVEOUT=1 asks for the maximum shared-memory carveout before
// the hand-off / ring launches; SL_DEBUG_OCC=1 prints their resident blocks/SM
template <typename Kern>
static void occupancy_setup(Kern kern, size_t smem, const char* name) {
  static int done[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (done[dev & 63]) return;
  done[dev & 63] = 1;
  const char* c = getenv("SL_CARVEOUT");
  if (c && c[0] == '1')
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  const char* d = getenv("SL_DEBUG_OCC");
  if (d && d[0] == '1') {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32, smem);
    fprintf(stderr, "[occ] %s smem %zu blocks/SM %d\n", name, smem, nb);
  }
}

template <int kCap, int kMaxRow, int kBatch, int kMinBlocks, int kX>
static void launch_csr_ring(int64_t nrows, const int32_t* pos, const int32_t* crd,
                            const double* vals, XOperand<kX> xop, double* y, int blocks_per_sm,
                            cudaStream_t s, bool pdl = false) {
  constexpr size_t smem = 16 + (size_t)kCap * 24;
  occupancy_setup(spmv_csr_ring_kernel<kCap, kMaxRow, kBatch, kMinBlocks, kX>, smem, "ring");
  const int64_t ntiles = (nrows + 31) / 32;
  const int grid = (int)min64(ntiles, (int64_t)sl_host::sm_count() * blocks_per_sm);
  if (pdl) {
    sl_host::launch_pdl(spmv_csr_ring_kernel<kCap, kMaxRow, kBatch, kMinBlocks, kX>, dim3(grid),
                        dim3(32), s, smem, nrows, pos, crd, vals, xop, y);
    return;
  }
  spmv_csr_ring_kernel<kCap, kMaxRow, kBatch, kMinBlocks, kX><<<grid, 32, smem, s>>>(
      nrows, pos, crd, vals, xop, y);
}

// A/B knob while the ring variant is measured: SL_CSR_RING=1 selects K2q
// wherever K2r would run (blocks per SM from SL_CSR_RING_BLOCKS, default 10)
static int csr_ring_blocks() {
  const char* e = getenv("SL_CSR_RING");
  if (!e || e[0] != '1') return 0;
  const char* b = getenv("SL_CSR_RING_BLOCKS");
  return b ? atoi(b) : 10;
}

#endif  // SL_WITH_ALT

// 896-element stage (28 per row), rows of up to 28 nonzeros in registers,
// gathers in one batch of 28 (rotating-copies protocol: batches of 7 / 14 / 28
// 17.37 / 17.39 / 16.43 us on the 64^3 stencil, D1 CSR 14.50 -> 14.20 us), 12
// one-warp blocks per SM (148 registers).  Round 1, two batches of 14:
// 64^3 stencil 22.4 us, D1 19.3 us, against K2f 23.8 / K2a 20.5 us; 14-27
// element batches, 10-24 blocks/SM and a 32-nonzero register row measured
// 22.4-27.2 / 19.3-24.4 us; two stages per block (tiles t+1 and t+2 in
// flight, 10 blocks/SM) 25.9-30.7 / 26.7-28.7 us (round-1 A/B runs under the
// per-launch flush protocol; logs not retained)
constexpr int kCsrHandoffCap = 896;
constexpr int kCsrHandoffMaxRow = 28;
constexpr int kCsrHandoffBatch = 28;   // one batch: all of a row's gathers in flight before the adds
constexpr int kCsrHandoffBlocks = 12;

// (A smaller stage for short rows — 384 / 448 / 512 / 640 elements, leaving the
// L1 more room for the x gathers — measured 16.6 / 14.3 / 14.3 / 14.3 us on D1
// CSR against 14.5 us: no gain, profiles/r2_ab_coo_resident.txt.)

// K2d: CSR warp row-block.  Each warp owns 32 consecutive rows; their
// nonzeros (contiguous) are staged in warp-private shared memory in rounds of
// 256 products (8 coalesced loads per lane), and lane r adds the round's
// products of its row in order.  Warps synchronise with __syncwarp only, so
// they progress independently (the block-level barriers of K2a stall on the
// slowest warp).
#ifdef SL_WITH_ALT   // warp row-block (3) and vector-per-row (1) CSR: A/B variant, opt-in build (SL_BUILD_ALT=1)
constexpr int kCsrWarpIpt = 8;
constexpr int kCsrWarpChunk = 32 * kCsrWarpIpt;   // 256 products per round

__global__ void __launch_bounds__(256, 8)
spmv_csr_warp_kernel(int64_t nrows, const int32_t* __restrict__ pos, const int32_t* __restrict__ crd,
                     const double* __restrict__ vals, const double* __restrict__ x,
                     double* __restrict__ y) {
  __shared__ __align__(16) double s_prod[8][kCsrWarpChunk];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w0 = ((int64_t)blockIdx.x * 8 + warp) * 32;
  if (w0 >= nrows) return;
  const int nr = (int)min64(32, nrows - w0);
  const int32_t rb = lane < nr ? ldg(pos + w0 + lane) : 0;
  const int32_t re = lane < nr ? ldg(pos + w0 + lane + 1) : 0;
  const int32_t eb = __shfl_sync(0xffffffffu, rb, 0), ee = __shfl_sync(0xffffffffu, re, nr - 1);
  double* sp = s_prod[warp];
  double acc = 0.0;
  for (int32_t cs = eb; cs < ee; cs += kCsrWarpChunk) {
    const int n = min(kCsrWarpChunk, ee - cs);
    int32_t c[kCsrWarpIpt];
    double v[kCsrWarpIpt], xv[kCsrWarpIpt];
    if (n == kCsrWarpChunk) {
#pragma unroll
      for (int k = 0; k < kCsrWarpIpt; ++k) c[k] = ld_stream(crd + cs + lane + 32 * k);
#pragma unroll
      for (int k = 0; k < kCsrWarpIpt; ++k) v[k] = ld_stream(vals + cs + lane + 32 * k);
#pragma unroll
      for (int k = 0; k < kCsrWarpIpt; ++k) xv[k] = ldg(x + c[k]);
#pragma unroll
      for (int k = 0; k < kCsrWarpIpt; ++k) sp[lane + 32 * k] = dmul(v[k], xv[k]);
    } else {
#pragma unroll
      for (int k = 0; k < kCsrWarpIpt; ++k) {
        const int q = lane + 32 * k;
        if (q < n) sp[q] = dmul(ld_stream(vals + cs + q), ldg(x + ld_stream(crd + cs + q)));
      }
    }
    __syncwarp();
    const int lo = max(rb, cs) - cs, hi = min(re, cs + n) - cs;
    for (int u = lo; u < hi; ++u) acc = dadd(acc, sp[u]);
    __syncwarp();
  }
  if (lane < nr) y[w0 + lane] = acc;
}

// K2b: CSR vector-per-row.  One warp per row: lanes load 32 nonzeros at a time
// coalesced, then the products are shuffled to every lane in order and added
// sequentially (the same order as the reference).  Best for long rows.
template <int kHashX>
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
#endif  // SL_WITH_ALT

// 128-thread blocks over 1024-item tiles: the tile's barriers couple fewer
// threads to the one summing a long row (D5's fibres, TTV: 256 / 128 / 64
// threads 230.9 / 218.6 / 255.0 us)
constexpr int kMpThreads = 128;
constexpr int kMpItems = 8 * kMpThreads;

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

template <int kHashX>
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
  if (eb == ee) {   // every row owned by this tile is empty: no chunk writes them
    for (int64_t r = rb + tid; r < re; r += kMpThreads) y[r] = 0.0;
    return;
  }
  // this thread's first row's bounds: in flight during the staging, not after
  // the barrier (most tiles hold fewer rows than threads)
  const int64_t r_first = rb + tid;
  int64_t pb = 0, pe = 0;
  if (r_first < re) {
    pb = ldg(pos + r_first);
    pe = ldg(pos + r_first + 1);
  }
  for (int64_t cs = eb; cs < ee; cs += kMpItems) {
    const int n_in = (int)min64(kMpItems, ee - cs);
    stage_products<kMpThreads, kMpItems / kMpThreads>(crd, vals, cs, n_in, xop, s_prod);
    __syncthreads();
    // rows are few per tile (<= kMpItems) — thread-per-row over the chunk
    for (int64_t r = r_first; r < re; r += kMpThreads) {
      const int64_t b = r == r_first ? pb : ldg(pos + r), e = r == r_first ? pe : ldg(pos + r + 1);
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

constexpr int kEllBatch = 9;   // slots loaded per batch (27 = 3 batches for the stencil)

// 4 blocks/SM (64 registers): the 64^3 stencil's 1024 blocks run in 1.7
// waves, so later blocks' loads overlap earlier blocks' gathers and adds
// (measured 24.2 -> 22.7 us; one wave at 8 blocks/SM starts every block's
// batches in lockstep)
template <int kBatch, int kThreads, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
spmv_ell_kernel(int64_t nrows, int32_t nslots, const int32_t* __restrict__ crd,
                const double* __restrict__ vals, const double* __restrict__ x,
                double* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double a = 0.0;
  int32_t s0 = 0;
  for (; s0 + kBatch <= nslots; s0 += kBatch) {   // full batches: no predicates
    int32_t c[kBatch];
    double v[kBatch], xv[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) c[b] = ld_stream(crd + (int64_t)(s0 + b) * nrows + i);
#pragma unroll
    for (int b = 0; b < kBatch; ++b) v[b] = ld_stream(vals + (int64_t)(s0 + b) * nrows + i);
#pragma unroll
    for (int b = 0; b < kBatch; ++b) xv[b] = ldg(x + c[b]);
#pragma unroll
    for (int b = 0; b < kBatch; ++b) a = dadd(a, dmul(v[b], xv[b]));
  }
  for (; s0 < nslots; ++s0) {
    const int64_t p = (int64_t)s0 * nrows + i;
    a = dadd(a, dmul(ld_stream(vals + p), ldg(x + ld_stream(crd + p))));
  }
  y[i] = a;
}

// ---------------------------------------------------------------------------
// K4: DIA SpMV, diagonal-major.  Thread per row; for each stored diagonal in
// ascending-offset order the row takes a term iff its column is inside the
// range level's bounds (levels.py:220-222): out-of-range slots are never read.
// Offsets travel as a kernel parameter (constant bank) when ndiag <= 32.

// Offsets in the constant bank (kernel parameter); all of a row's in-range
// value and x loads are issued before the in-order add chain.
constexpr int kDiaThreads = 128;
template <int kMaxD>
// 1280 threads per SM in 128-thread blocks (256 x 5: 25.85 us, 128 x 10: 25.13 us, 64 x 20: 25.21 us
// on D3), 47 registers (D3: 3 / 4 / 5 / 6 blocks 26.8 / 26.7 / 25.8 / 32.3 us, the last
// with spills; round 1: 39.4 -> 33.5 us from 8 to 4 blocks/SM under the flush protocol)
__global__ void __launch_bounds__(kDiaThreads, 1280 / kDiaThreads)
spmv_dia_kernel(int64_t nrows, int64_t row0, int64_t ncols, int32_t ndiag, DiaOffsets offs,
                const double* __restrict__ vals, const double* __restrict__ x,
                double* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double v[kMaxD], xv[kMaxD];
  bool in[kMaxD];
#pragma unroll
  for (int d = 0; d < kMaxD; ++d) {
    const int64_t j = row0 + i + offs.v[d];
    in[d] = d < ndiag && j >= 0 && j < ncols;
    v[d] = in[d] ? ld_stream(vals + (int64_t)d * nrows + i) : 0.0;
    xv[d] = in[d] ? ldg(x + j) : 0.0;
  }
  double a = 0.0;
#pragma unroll
  for (int d = 0; d < kMaxD; ++d)
    if (in[d]) a = dadd(a, dmul(v[d], xv[d]));
  y[i] = a;
}

// Device-resident offsets (any number of diagonals).
__global__ void __launch_bounds__(256)
spmv_dia_dev_kernel(int64_t nrows, int64_t row0, int64_t ncols, int32_t ndiag,
                    const int32_t* __restrict__ doffs, const double* __restrict__ vals,
                    const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double a = 0.0;
  for (int d = 0; d < ndiag; ++d) {
    const int64_t j = row0 + i + ldg(doffs + d);
    if (j >= 0 && j < ncols) a = dadd(a, dmul(ld_stream(vals + (int64_t)d * nrows + i), ldg(x + j)));
  }
  y[i] = a;
}

}  // namespace sl

// ===========================================================================
// C ABI

using namespace sl;
using sl_host::as_stream;
using sl_host::ceil_div;
using sl_host::aligned16;

// SL_SPMV_PATH=pipe selects the persistent TMA pipelines (pipe.cu) instead of
// the LDG kernels (A/B knob; the LDG kernels measured faster on every BASELINE
// config), =ldg forces LDG.
#ifdef SL_WITH_ALT
static int spmv_path() {
  const char* e = getenv("SL_SPMV_PATH");
  return !e ? 0 : (e[0] == 'l' ? 1 : (e[0] == 'p' ? 2 : 0));
}
#endif


extern "C" size_t sl_spmv_coo_workspace_bytes(int64_t nrows) {
  return ((size_t)(nrows + 1) * sizeof(int32_t) + 255) & ~size_t(255);
}

extern "C" int sl_spmv_coo_f64(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* rows,
                               const int32_t* cols, const double* vals, const double* x,
                               double* y, void* ws, size_t ws_bytes, void* stream) {
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
#ifdef SL_WITH_ALT
  if (vec_ok && spmv_path() == 2) return sl_host::launch_coo_pipe(nrows, nnz, rows, cols, vals, x, y, s);
#endif
  // With a workspace and rows averaging <= 28 nonzeros: the row level's
  // position index (one streaming pass over the row coordinates into the
  // workspace; cols and vals are not touched), then the register hand-off
  // kernel K2r over (row pointer, cols, vals), launched with PDL so it starts
  // while the pass drains.  D1: 20.4 us (staged tiles below) -> see DESIGN.md.
  // The staged-tile kernel K1 computes on the coordinates alone (no
  // workspace): the path for longer rows, misaligned arrays, or ws == NULL.
  const char* ck = getenv("SL_COO_KERNEL");       // A/B knob: "tile" forces K1, "res" K1s
#ifdef SL_WITH_ALT
  // K1s (coo_resident.cu, A/B build): one resident range per SM — measured
  // 26.5 us on D1 against 18.4 us here (profiles/r2_ab_coo_resident.txt)
  if (ck && ck[0] == 'r' && vec_ok &&
      sl_host::launch_coo_resident(nrows, nnz, rows, cols, vals, x, y, s))
    return sl_host::launch_status();
#endif
  if (ws && ws_bytes >= sl_spmv_coo_workspace_bytes(nrows) && vec_ok &&
      nnz <= (int64_t)kCsrHandoffMaxRow * nrows && !(ck && ck[0] == 't')) {
    int32_t* rowptr = static_cast<int32_t*>(ws);
    sl_host::launch_coo_rowptr(nrows, nnz, rows, rowptr, s);
#ifdef SL_WITH_ALT
    if (const int rb = csr_ring_blocks()) {
      launch_csr_ring<kCsrHandoffCap, kCsrHandoffMaxRow, kCsrHandoffBatch, 10>(
          nrows, rowptr, cols, vals, XOperand<0>{x}, y, rb, s, true);
      return sl_host::launch_status();
    }
#endif
    launch_csr_handoff<kCsrHandoffCap, kCsrHandoffMaxRow, kCsrHandoffBatch, kCsrHandoffBlocks>(
        nrows, rowptr, cols, vals, XOperand<0>{x}, y, kCsrHandoffBlocks, s, true);
    return sl_host::launch_status();
  }
  // 1024-nonzero tiles, 8 blocks/SM: on D1 (2M nonzeros) the grid is 1.65x the
  // resident slots, so later tiles' loads overlap earlier tiles' sum phases
  // (round 1: 2048-nonzero tiles in one wave 37.0 us vs 26.2 us; per-thread
  // walks without the start compaction 29.4 vs 24.8 us; persistent and TMA-ring
  // variants 26.9-36.8 us; round 2: a warp-segmented register version (heads
  // by ballot, per-lane-source shuffle sums, no shared memory) 32-37 us — its
  // sum loop runs as many warp steps as the round's longest row for ~3 heads)
  spmv_coo_kernel<256, 1, 8><<<ceil_div(nnz, 1024), 256, 0, s>>>(nrows, nnz, rows, cols, vals,
                                                                 x, y, vec_ok);
  return sl_host::launch_status();
}

extern "C" size_t sl_spmv_csr_workspace_bytes(int64_t nrows, int64_t nnz, int32_t variant) {
  if (variant != 2) return 0;
  const int64_t ntiles = (nrows + nnz + kMpItems - 1) / kMpItems;
  return (size_t)(ntiles + 1) * sizeof(int64_t);
}

template <int kHashX>
static int launch_csr(int64_t nrows, int64_t nnz, const int32_t* pos, const int32_t* crd,
                      const double* vals, XOperand<kHashX> xop, double* y, int32_t variant,
                      void* ws, size_t ws_bytes, cudaStream_t s) {
#ifdef SL_WITH_ALT
  if (variant == 0 && !kHashX && aligned16(crd) && aligned16(vals) && spmv_path() == 2) {
    const double* xd = reinterpret_cast<const XOperand<0>&>(xop).x;
    return sl_host::launch_csr_pipe(nrows, pos, crd, vals, xd, y, s);
  }
#endif
  if (variant == 0 || variant == 5) {
    // variant 0 (automatic): rows averaging <= 28 nonzeros (aligned crd/vals)
    // take the register hand-off kernel K2r, longer rows the row-block kernel
    // K2a, whose staged products keep very long rows parallel (variant 5
    // forces K2a).
    // K2a: short rows (<= 16 per row on average): 192-row blocks, about one chunk
    // each and more blocks than resident slots, so blocks' load and sum phases
    // interleave (D1 22.8 -> 21.2 us, hashed x 40.7 -> 32.8 us); long rows
    // (the 27-point stencil) keep 256-row blocks (29.0 vs 35.2 us)
    // (nnz < 0: not known to the entry point — the located-x paths, whose
    // per-nonzero locate latency also favours more, smaller blocks)
    // dense x and sparse-vector x (spx stencil 46.0 -> 35.9 us); the hashed x
    // paths keep K2a (slot-mapped H1: 45.5 us with K2a, 54.2 us here — the
    // element-order gathers of K2a's staging serve its two random gathers
    // per nonzero better than the row walk)
    if constexpr (kHashX == 0 || kHashX == 3) {
      if (variant == 0 && nnz >= 0 && nnz <= (int64_t)kCsrHandoffMaxRow * nrows &&
          aligned16(crd) && aligned16(vals)) {
#ifdef SL_WITH_ALT
        if (const int rb = csr_ring_blocks()) {
          launch_csr_ring<kCsrHandoffCap, kCsrHandoffMaxRow, kCsrHandoffBatch, 10>(
              nrows, pos, crd, vals, xop, y, rb, s);
          return sl_host::launch_status();
        }
#endif
        // dense x: one batch of 28 gathers; a located x (slot, then value: two
        // dependent gathers and 64-bit slots in registers) keeps two batches of 14
        launch_csr_handoff<kCsrHandoffCap, kCsrHandoffMaxRow, kHashX == 0 ? kCsrHandoffBatch : 14,
                           kCsrHandoffBlocks>(nrows, pos, crd, vals, xop, y, kCsrHandoffBlocks, s);
        return sl_host::launch_status();
      }
    }
    if (nnz <= 16 * nrows) {
      spmv_csr_rowblock_kernel<kHashX, 192><<<ceil_div(nrows, 192), kCsrThreads, 0, s>>>(
          nrows, pos, crd, vals, xop, y);
      return sl_host::launch_status();
    }
    spmv_csr_rowblock_kernel<kHashX><<<ceil_div(nrows, kCsrRows), kCsrThreads, 0, s>>>(
        nrows, pos, crd, vals, xop, y);
#ifdef SL_WITH_ALT
  } else if (variant == 4 && !kHashX) {
    if (!aligned16(crd) || !aligned16(vals)) return SL_ERR_INVALID;
    launch_csr_stage<kCsrStageRows, kCsrStageCap, kCsrStageBatch, kCsrStageBlocks>(
        nrows, pos, crd, vals, reinterpret_cast<const XOperand<0>&>(xop).x, y, s);
#endif
  } else if (variant == 6 && !kHashX) {
    if (!aligned16(crd) || !aligned16(vals)) return SL_ERR_INVALID;
    launch_csr_handoff<kCsrHandoffCap, kCsrHandoffMaxRow, kCsrHandoffBatch, kCsrHandoffBlocks>(
        nrows, pos, crd, vals, reinterpret_cast<const XOperand<0>&>(xop), y, kCsrHandoffBlocks, s);
#ifdef SL_WITH_ALT
  } else if (variant == 3 && !kHashX) {
    const double* xd = reinterpret_cast<const XOperand<0>&>(xop).x;
    spmv_csr_warp_kernel<<<ceil_div(nrows, 256), 256, 0, s>>>(nrows, pos, crd, vals, xd, y);
  } else if (variant == 1) {
    spmv_csr_vector_kernel<kHashX><<<ceil_div(nrows * 32, 256), 256, 0, s>>>(nrows, pos, crd,
                                                                            vals, xop, y);
#endif
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
  if (!pos || !y || (nnz > 0 && (!x || !crd || !vals))) return SL_ERR_INVALID;   // x may be empty
  cudaStream_t s = as_stream(stream);
  XOperand<0> xop{x};
  if (variant == 2) {
    const int64_t ntiles = (nrows + nnz + kMpItems - 1) / kMpItems;
    if (!ws || ws_bytes < sl_spmv_csr_workspace_bytes(nrows, nnz, 2)) return SL_ERR_WORKSPACE;
    int64_t* part = static_cast<int64_t*>(ws);
    csr_merge_partition_kernel<<<ceil_div(ntiles + 1, 256), 256, 0, s>>>(pos, nrows, nnz, ntiles,
                                                                       part);
    spmv_csr_merge_kernel<0><<<(int)ntiles, kMpThreads, 0, s>>>(nrows, pos, crd, vals, xop,
                                                                   part, y);
    return sl_host::launch_status();
  }
  return launch_csr<0>(nrows, nnz, pos, crd, vals, xop, y, variant, ws, ws_bytes, s);
}

extern "C" int sl_spmv_csr_hashx_f64(int64_t nrows, const int32_t* pos, const int32_t* crd,
                                     const double* vals, int64_t w, const int32_t* x_crd,
                                     const double* x_vals, double* y, void* stream) {
  if (nrows < 0 || w <= 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || w > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0) return SL_OK;
  if (!pos || !y || !x_crd || !x_vals) return SL_ERR_INVALID;
  XOperand<1> xop{HashedLevel{x_crd, w}, x_vals};
  return launch_csr<1>(nrows, -1, pos, crd, vals, xop, y, 0, nullptr, 0, as_stream(stream));
}

extern "C" size_t sl_spmv_csr_hashx_map_workspace_bytes(int64_t n, int64_t w) {
  return sl_hashed_slot_map_workspace_bytes(n, w);
}

extern "C" int sl_spmv_csr_hashx_map_f64(int64_t nrows, int64_t n, int64_t nnz,
                                         const int32_t* pos, const int32_t* crd,
                                         const double* vals, int64_t w,
                                         const int32_t* x_crd, const double* x_vals, double* y,
                                         void* ws, size_t ws_bytes, void* stream) {
  if (nrows < 0 || n < 0 || w <= 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || w > INT32_MAX || n > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0) return SL_OK;
  if (!pos || !y || !x_crd || !x_vals) return SL_ERR_INVALID;
  const int st = sl_hashed_slot_map(n, w, x_crd, ws, ws_bytes, stream);
  if (st != SL_OK) return st;
  XOperand<2> xop{HashedLevel{x_crd, w}, x_vals, static_cast<const unsigned long long*>(ws), n};
  return launch_csr<2>(nrows, nnz, pos, crd, vals, xop, y, 0, nullptr, 0, as_stream(stream));
}

__global__ void spx_map_kernel(int64_t n, int64_t xnnz, const int32_t* __restrict__ xcrd,
                               int32_t* __restrict__ map) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = t; i < n; i += stride) map[i] = -1;
}

__global__ void spx_scatter_kernel(int64_t n, int64_t xnnz, const int32_t* __restrict__ xcrd,
                                   int32_t* __restrict__ map) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < xnnz; q += stride) {
    const int32_t c = ldg(xcrd + q);
    if (c >= 0 && c < n) map[c] = (int32_t)q;
  }
}

extern "C" size_t sl_spmv_csr_spx_workspace_bytes(int64_t n) { return (size_t)n * 4 + 256; }

extern "C" int sl_spmv_csr_spx_f64(int64_t nrows, int64_t n, int64_t nnz, const int32_t* pos,
                                   const int32_t* crd, const double* vals, int64_t xnnz,
                                   const int32_t* x_crd, const double* x_vals, double* y,
                                   void* ws, size_t ws_bytes, void* stream) {
  if (nrows < 0 || n < 0 || xnnz < 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || n > INT32_MAX || xnnz > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0) return SL_OK;
  if (!pos || !y || (xnnz > 0 && (!x_crd || !x_vals))) return SL_ERR_INVALID;
  if (!ws || ws_bytes < sl_spmv_csr_spx_workspace_bytes(n)) return SL_ERR_WORKSPACE;
  cudaStream_t s = as_stream(stream);
  int32_t* map = static_cast<int32_t*>(ws);
  const int sms = sl_host::sm_count();
  if (n > 0) spx_map_kernel<<<min(ceil_div(n, 256), 8 * sms), 256, 0, s>>>(n, xnnz, x_crd, map);
  if (xnnz > 0)
    spx_scatter_kernel<<<min(ceil_div(xnnz, 256), 8 * sms), 256, 0, s>>>(n, xnnz, x_crd, map);
  XOperand<3> xop{map, x_vals, n};
  return launch_csr<3>(nrows, nnz, pos, crd, vals, xop, y, 0, nullptr, 0, s);
}

extern "C" int sl_spmv_ell_f64(int64_t nrows, int64_t ncols, int32_t nslots, const int32_t* crd,
                               const double* vals, const double* x, double* y, void* stream) {
  if (nrows < 0 || ncols < 0 || nslots < 0) return SL_ERR_INVALID;
  if ((int64_t)nslots * nrows > INT32_MAX || ncols > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0) return SL_OK;
  if (!y || (nslots > 0 && (!crd || !vals || !x))) return SL_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
#ifdef SL_WITH_ALT
  if (nslots > 0 && nslots <= sl_host::kEllPipeMaxSlots && nrows % 4 == 0 && aligned16(crd) &&
      aligned16(vals) && spmv_path() == 2)
    return sl_host::launch_ell_pipe(nrows, nslots, crd, vals, x, y, s);
#endif
  // batch 9 x 256 threads x 4 blocks/SM; round 1 measured batch 7-27 at 64-512
  // threads per block (20.5-24.5 us against 20.8 us here), issuing the next
  // batch's loads before the current batch's gathers (register software
  // pipelining, 20.6-24.6 us) and a grid-stride persistent grid of 2-8
  // blocks/SM (20.6-25.3 us)
  // 128-thread blocks, 8 per SM (256 x 4: 15.44 us, 128 x 8 / 64 x 16: 15.36 us on the 64^3 stencil)
  spmv_ell_kernel<kEllBatch, 128, 8><<<ceil_div(nrows, 128), 128, 0, s>>>(nrows, nslots, crd, vals,
                                                                          x, y);
  return sl_host::launch_status();
}

extern "C" int sl_spmv_dia_rows_f64(int64_t nrows, int64_t row0, int64_t ncols, int32_t ndiag,
                                    const int32_t* offsets, int32_t offsets_on_host,
                                    const double* vals, const double* x, double* y, void* stream) {
  if (nrows < 0 || row0 < 0 || ncols < 0 || ndiag < 0) return SL_ERR_INVALID;
  if ((int64_t)ndiag * nrows > INT32_MAX || ncols > INT32_MAX || row0 > INT32_MAX) return SL_ERR_RANGE;
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
  const int grid = ceil_div(nrows, kDiaThreads);
#ifdef SL_WITH_ALT
  if (!doffs && row0 == 0 && aligned16(vals) && aligned16(x) && ndiag > 0 && spmv_path() == 2)
    return sl_host::launch_dia_pipe(nrows, ncols, ndiag, p, vals, x, y, s);
#endif
  if (doffs) {
    spmv_dia_dev_kernel<<<ceil_div(nrows, 256), 256, 0, s>>>(nrows, row0, ncols, ndiag, doffs, vals, x, y);
  } else if (ndiag <= 8) {
    spmv_dia_kernel<8><<<grid, kDiaThreads, 0, s>>>(nrows, row0, ncols, ndiag, p, vals, x, y);
  } else if (ndiag <= 16) {
    spmv_dia_kernel<16><<<grid, kDiaThreads, 0, s>>>(nrows, row0, ncols, ndiag, p, vals, x, y);
  } else {
    spmv_dia_kernel<32><<<grid, kDiaThreads, 0, s>>>(nrows, row0, ncols, ndiag, p, vals, x, y);
  }
  return sl_host::launch_status();
}

extern "C" int sl_spmv_dia_f64(int64_t nrows, int64_t ncols, int32_t ndiag, const int32_t* offsets,
                               int32_t offsets_on_host, const double* vals, const double* x,
                               double* y, void* stream) {
  return sl_spmv_dia_rows_f64(nrows, 0, ncols, ndiag, offsets, offsets_on_host, vals, x, y, stream);
}

// Which optional kernels this build carries (bit 0: the A/B alternatives —
// CSR variants 1, 3, 4 and the persistent TMA pipelines, SL_BUILD_ALT=1).
extern "C" int sl_build_features(void) {
#ifdef SL_WITH_ALT
  return 1;
#else
  return 0;
#endif
}

// CSR SpMV of a row block with the all-gather fused into the epilogue: rows
// [0, nrows) of this block are stored into every buffer y_peers[q]
// (q < npeers <= 8; host array of device pointers, each already offset to the
// block's first global row — peer buffers mapped through CUDA IPC / symmetric
// memory, or local buffers).  The register hand-off kernel (rows averaging
// <= 28 nonzeros, 16-byte-aligned crd / vals) stores directly; any other
// matrix is computed into y_peers[0] and copied to the other buffers.
extern "C" int sl_spmv_csr_peers_f64(int64_t nrows, int64_t ncols, int64_t nnz,
                                     const int32_t* pos, const int32_t* crd, const double* vals,
                                     const double* x, const uint64_t* y_peers, int32_t npeers,
                                     void* stream) {
  if (nrows < 0 || ncols < 0 || nnz < 0 || npeers < 1 || npeers > kMaxPeers || !y_peers)
    return SL_ERR_INVALID;
  if (nrows > INT32_MAX || ncols > INT32_MAX || nnz > INT32_MAX) return SL_ERR_RANGE;
  if (nrows == 0) return SL_OK;
  cudaStream_t s = as_stream(stream);
  PeerOut po{};
  po.n = npeers;
  for (int q = 0; q < npeers; ++q) po.p[q] = reinterpret_cast<double*>(y_peers[q]);
  if (nnz > 0 && nnz <= (int64_t)kCsrHandoffMaxRow * nrows && aligned16(crd) && aligned16(vals)) {
    launch_csr_handoff<kCsrHandoffCap, kCsrHandoffMaxRow, kCsrHandoffBatch, kCsrHandoffBlocks>(
        nrows, pos, crd, vals, XOperand<0>{x}, po.p[0], kCsrHandoffBlocks, s, false, &po);
    return sl_host::launch_status();
  }
  const int st = sl_spmv_csr_f64(nrows, ncols, nnz, pos, crd, vals, x, po.p[0], 0, nullptr, 0,
                                 stream);
  if (st != SL_OK) return st;
  for (int q = 1; q < npeers; ++q)
    if (cudaMemcpyAsync(po.p[q], po.p[0], (size_t)nrows * sizeof(double), cudaMemcpyDefault, s) !=
        cudaSuccess)
      return SL_ERR_CUDA;
  return sl_host::launch_status();
}
