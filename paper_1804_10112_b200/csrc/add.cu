// add.cu — C(i,j) = A(i,j) + B(i,j) with A CSR, B COO (or CSR), C CSR.
//
// Reference: the i-lattice {A0,B0} -> {A0} and j-lattice {A1,B1} -> {A1} ->
// {B1} co-iteration (engine.py:591-634) feeding the
// gather-append writer (engine.py:330-434).  Per row the output is the
// sorted union of A's and B's columns; a coordinate present in both gets
// a + b, otherwise the copy; B's duplicate coordinates are grouped and summed
// (Python's sum() over the group, engine.py:107-149, 524-527: `PySum`,
// common.cuh); the stored value is
// 0.0 + value (engine.py:404, 413, 625-631).  Explicit zeros are kept.
//
// B200 design (two passes over the operands, scan-based assembly):
//   0. rowptr   (COO B only) one pass over B's row coordinates yields the
//               row groups the reference's dedup-chained iterator walks
//               (Grouped over compressed(~U), engine.py:107-149) as a row
//               pointer; cols/vals are never moved — B is not converted.
//   1. count    128-row tiles; the tile's column slices are bulk-copied to
//               shared memory (TMA), thread per row merges the two sorted
//               lists and counts distinct coordinates; tile-local inclusive
//               scan -> c_pos, tile total -> workspace.
//   2. scan     one block scans the tile totals (no cross-block look-back
//               chain: with thousands of small tiles a decoupled look-back
//               advanced only ~32 tiles per L2 round trip — measured 150 us).
//   3. fill     tiles staged again (values too), merged, outputs written at
//               their final positions; the fused entry also finalises c_pos
//               here, the two-pass entry finalises it at the end of count.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "tma.cuh"

namespace sl {


// ---- pass 0: row pointer of a row-sorted COO level ---------------------------
// kRowptrIpt elements per thread (16-byte loads when aligned): 8 behind A + B's
// 5M coordinates (4 / 8 / 16: 82.7 / 81.7 / 85.0 us for the chain), 4 for the
// SpMV / SpDM row pointer (D1's 2M coordinates: 17.3 / 18.2 / 18.9 us for the
// COO SpMV) — the smaller pass wants more, shorter threads
#ifndef SL_ROWPTR_IPT_SPMV
#define SL_ROWPTR_IPT_SPMV 4
#endif
template <int kRowptrIpt>
__global__ void __launch_bounds__(256)
coo_rowptr_kernel(int64_t nrows, int64_t nnz, const int32_t* __restrict__ rows,
                  int32_t* __restrict__ rowptr, int64_t* __restrict__ zero, int64_t nzero) {
  pdl_trigger();                           // the count pass may begin launching
  // the count pass's super-tile totals start at zero (saves a memset node)
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nzero;
       q += (int64_t)gridDim.x * blockDim.x)
    zero[q] = 0;
  // rowptr[r] = first e with rows[e] >= r, r in [0, nrows]: element e writes the
  // entries r in (rows[e-1], rows[e]] (e = nnz closes the trailing rows)
  const int64_t e0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRowptrIpt;
  if (e0 > nnz) return;
  int32_t r[kRowptrIpt];
  const bool vec = e0 + kRowptrIpt <= nnz && ((reinterpret_cast<uintptr_t>(rows + e0) & 15u) == 0);
  if (vec) {
    int4 q[kRowptrIpt / 4];
#pragma unroll
    for (int t = 0; t < kRowptrIpt / 4; ++t)
      q[t] = ld_stream(reinterpret_cast<const int4*>(rows + e0 + 4 * t));
#pragma unroll
    for (int t = 0; t < kRowptrIpt / 4; ++t) {
      r[4 * t] = q[t].x; r[4 * t + 1] = q[t].y; r[4 * t + 2] = q[t].z; r[4 * t + 3] = q[t].w;
    }
  } else {
#pragma unroll
    for (int t = 0; t < kRowptrIpt; ++t) r[t] = e0 + t < nnz ? ldg(rows + e0 + t) : (int32_t)nrows;
  }
  // positions past the end read as row nrows, so element nnz closes the
  // trailing rows (rowptr[nrows] = nnz) and later ones write nothing
  int32_t prev = e0 == 0 ? -1 : ldg(rows + e0 - 1);
  // a row change almost always advances by one row: one predicated store per
  // element; the gap loop (empty rows) runs out of line.  (A per-change
  // counted loop cost ~42 instructions per element: ncu, 6.7M warp
  // instructions for D4's 5M coordinates.)
  unsigned gaps = 0;
#pragma unroll
  for (int t = 0; t < kRowptrIpt; ++t) {
    const int32_t cur = r[t];
    const int32_t pv = t == 0 ? prev : r[t - 1];
    if (cur != pv) rowptr[cur] = (int32_t)(e0 + t);
    gaps |= (cur - pv > 1 ? 1u : 0u) << t;
  }
  if (gaps) {
#pragma unroll
    for (int t = 0; t < kRowptrIpt; ++t) {
      if (gaps >> t & 1u) {
        const int32_t lo = t == 0 ? prev : r[t - 1];
        for (int32_t q = lo + 1; q < r[t]; ++q) rowptr[q] = (int32_t)(e0 + t);
      }
    }
  }
}

// ---- merge of one row ----------------------------------------------------------
// Visits the union of A's row [alo, ahi) and B's row [blo, bhi) in ascending
// column order, B duplicates grouped.  emit(n, col, value) is called per output.
// Element accessors read the tile's shared-memory stage (or global memory past
// the stage's capacity).
template <bool kValues, typename Acc, typename F>
SL_DEV int merge_row(int32_t alo, int32_t ahi, int32_t blo, int32_t bhi, const Acc& acc,
                     F&& emit) {
  int n = 0;
  int32_t pa = alo, pb = blo;
  int32_t ca = pa < ahi ? acc.acol(pa) : INT32_MAX;
  int32_t cb = pb < bhi ? acc.bcol(pb) : INT32_MAX;
  while (pa < ahi || pb < bhi) {
    const int32_t c = ca < cb ? ca : cb;
    double e = 0.0;
    const bool has_a = ca == c, has_b = cb == c;
    double a = 0.0;
    if (has_a) {
      if (kValues) a = acc.aval(pa);
      ++pa;
      ca = pa < ahi ? acc.acol(pa) : INT32_MAX;
    }
    if (has_b) {
      double b = kValues ? acc.bval(pb) : 0.0;
      int32_t q = pb + 1;
      int32_t cq = q < bhi ? acc.bcol(q) : INT32_MAX;
      if (cq == c) {
        // duplicates: Python's sum() over the group (PySum)
        PySum g;
        if (kValues) g.start(b);
        while (cq == c) {
          if (kValues) g.add(acc.bval(q));
          ++q;
          cq = q < bhi ? acc.bcol(q) : INT32_MAX;
        }
        if (kValues) b = g.value();
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

// Count-only merge over the tile's unified column stage (A's slice at
// [ia, iah), B's at [ib, ibh) of one shared array, 32-bit indices): the number
// of distinct columns in A's row (unique) union B's row (sorted, possibly
// repeated).  One element of either operand is consumed per iteration (A
// first on ties) and a new output starts whenever the column differs from the
// previous one, so matches and duplicate-B groups need no separate paths.
// (ncu, D4: the pairwise merge with a duplicate look-ahead ran 30M warp
// instructions at 90% issue; this form, with one shared load per element and
// no 64-bit pointer selects, is what the count pass executes.)
SL_DEV int count_row_idx(int ia, int iah, int ib, int ibh, const int32_t* s_col) {
  // explicit 32-bit shared addresses: with generic indexing the compiler
  // rematerialised the shared-window base (S2R CgaCtaId + 3 ops) per load
  const uint32_t base = smem_u32(s_col);
  int n = 0;
  int32_t last = -1;
  int32_t ca = lds32(base + 4u * ia);      // the stage holds one slack element past B's end
  int32_t cb = lds32(base + 4u * ib);
  ca = ia < iah ? ca : INT32_MAX;
  cb = ib < ibh ? cb : INT32_MAX;
  for (int it = (iah - ia) + (ibh - ib); it > 0; --it) {
    const bool ta = ca <= cb;
    const int32_t c = ta ? ca : cb;
    n += c != last;
    last = c;
    ia += ta;
    ib += !ta;
    const int idx = ta ? ia : ib;
    const int32_t v = lds32(base + 4u * idx);
    const int32_t nx = idx < (ta ? iah : ibh) ? v : INT32_MAX;
    ca = ta ? nx : ca;
    cb = ta ? cb : nx;
  }
  return n;
}

// Fill merge over staged columns only: per output its column and its sources,
// packed as bits 0-10 = A's stage index + 1 (0: no A entry), bits 11-21 = the
// first stage index (relative to B's region) + 1 of B's run (0: none), bits
// 22-31 = the run's length.  A's row holds unique columns (a non-unique CSR
// is grouped before it gets here), and A comes first on ties, so an A entry is
// always the first of its output.  The values are read from global memory by
// emit_outputs, coalesced across the tile's consecutive outputs.
SL_DEV void fill_row_src(int ia, int iah, int ib, int ibh, int kcs, const int32_t* s_col,
                         uint2* out) {
  const uint32_t base = smem_u32(s_col);
  // one 8-byte record (column, sources) per output, rewritten by every
  // element of the output (a single st.shared.v2 and one running address per
  // step; two arrays cost a second store and a second address)
  uint32_t po = smem_u32(out) - 8u;                            // output n at po + 8 (n + 1)
  int32_t last = -1;
  uint32_t src = 0;
  int32_t ca = lds32(base + 4u * ia);
  int32_t cb = lds32(base + 4u * ib);
  ca = ia < iah ? ca : INT32_MAX;
  cb = ib < ibh ? cb : INT32_MAX;
  for (int it = (iah - ia) + (ibh - ib); it > 0; --it) {
    const bool ta = ca <= cb;
    const int32_t c = ta ? ca : cb;
    const bool fresh = c != last;
    po += fresh ? 8u : 0u;
    last = c;
    src = fresh ? 0u : src;
    const uint32_t bsrc = ((src >> 11) & 0x7ffu) ? src : (src | ((uint32_t)(ib - kcs + 1) << 11));
    src = ta ? (src | (uint32_t)(ia + 1)) : bsrc + (1u << 22);
    sts64(po, (uint32_t)c, src);
    ia += ta;
    ib += !ta;
    const int idx = ta ? ia : ib;
    const int32_t v = lds32(base + 4u * idx);
    const int32_t nx = idx < (ta ? iah : ibh) ? v : INT32_MAX;
    ca = ta ? nx : ca;
    cb = ta ? cb : nx;
  }
}

// Writes outputs [0, n) of a staged run: column from the stage, value
// 0 + (a + bgroup | a | bgroup) from the global A / B values (a0 / b0: the
// global index of stage index 0 of each), four outputs per thread in flight.
#ifndef SL_EMIT_UNROLL
#define SL_EMIT_UNROLL 2
#endif
constexpr int kEmitUnroll = SL_EMIT_UNROLL;

template <int kThreads>
SL_DEV void emit_outputs(int n, const uint2* s_out, int64_t a0,
                         int64_t b0, const double* __restrict__ a_vals,
                         const double* __restrict__ b_vals, int32_t* gc, double* gv) {
  const double* ap = a_vals + a0 - 1;      // source fields hold stage index + 1
  const double* bp = b_vals + b0 - 1;
  for (int q0 = threadIdx.x; q0 < n; q0 += kEmitUnroll * kThreads) {
    uint32_t src[kEmitUnroll];
    int32_t col[kEmitUnroll];
    double av[kEmitUnroll], bv[kEmitUnroll];
#pragma unroll
    for (int u = 0; u < kEmitUnroll; ++u) {
      const int q = q0 + u * kThreads;
      const uint2 o = q < n ? s_out[q] : make_uint2(0u, 0u);
      col[u] = (int32_t)o.x;
      src[u] = o.y;
    }
#pragma unroll
    for (int u = 0; u < kEmitUnroll; ++u) {
      const uint32_t sa = src[u] & 0x7ffu, sb = (src[u] >> 11) & 0x7ffu;
      av[u] = sa ? ldg(ap + sa) : 0.0;
      bv[u] = sb ? ldg(bp + sb) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kEmitUnroll; ++u) {
      const int q = q0 + u * kThreads;
      if (q < n) {
        const uint32_t sb = (src[u] >> 11) & 0x7ffu, nbv = src[u] >> 22;
        double g = bv[u];
        if (nbv > 1) {                       // a repeated B coordinate: Python's sum()
          PySum p;
          p.start(g);
          for (uint32_t k = 1; k < nbv; ++k) p.add(ldg(bp + sb + k));
          g = p.value();
        }
        // a + g with the absent side read as +0.0: the stored value 0.0 + e is
        // then bit-identical to 0.0 + a / 0.0 + g of the reference's copy
        // cases (x + 0.0 is x except for -0.0, which 0.0 + x turns into +0.0
        // either way) — no selects on the 64-bit values (ncu: 6 of the
        // emitter's ~46 instructions per output)
        const double e = dadd(av[u], g);
        gc[q] = col[u];
        gv[q] = dadd(0.0, e);
      }
    }
  }
}

// first index in [lo, hi) of a sorted global int32 range whose value is >= c
SL_DEV int32_t lower_bound_g(const int32_t* __restrict__ a, int32_t lo, int32_t hi, int32_t c) {
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (ldg(a + mid) < c) lo = mid + 1; else hi = mid;
  }
  return lo;
}

struct NoEmit {
  SL_DEV void operator()(int, int32_t, double) const {}
};

struct FillEmit {
  int32_t* crd;
  double* vals;
  SL_DEV void operator()(int n, int32_t c, double v) const {
    crd[n] = c;
    vals[n] = v;
  }
};

// ---- tile kernel: kAddRows rows per block, operands staged in shared memory ----
// kMode 0: count   -> c_pos[r + 1] = tile-local inclusive count, tile_tot[tile],
//                     super_tot[tile / kSuper] += tile total
// kMode 1: fill    (c_pos final)
// kMode 2: fill + finalise c_pos from the tile-local counts and the tile prefix

constexpr int kAddRows = 128;
// staged elements per operand per tile (Poisson(5) x 128 rows: 640 +- 25;
// larger tiles take the grouped path): the count stages columns only and is
// thread-bound at 16 blocks/SM, so it keeps the roomier stage; the fill's
// 704-element stage lets 6 instead of 5 blocks share an SM (85.1 -> 81.4 us)
constexpr int kAddCapCount = 768;
constexpr int kAddCapFill = 704;
constexpr int kSuper = 64;       // tiles per super-tile of the two-level prefix

// Accessor for tiles that exceed the stage capacity (or unaligned operands):
// elements read from global memory.
struct GlobalAcc {
  const int32_t* a_crd;
  const double* a_vals;
  const int32_t* b_cols;
  const double* b_vals;
  SL_DEV int32_t acol(int32_t p) const { return ldg(a_crd + p); }
  SL_DEV double aval(int32_t p) const { return ldg(a_vals + p); }
  SL_DEV int32_t bcol(int32_t p) const { return ldg(b_cols + p); }
  SL_DEV double bval(int32_t p) const { return ldg(b_vals + p); }
};

// inclusive block scan of one int per thread (kAddRows threads)
SL_DEV int block_incl_scan(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  int before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kAddRows / 32; ++w) {
    const int c = s_warp[w];
    before += w < warp ? c : 0;
    tot += c;
  }
  *total = tot;
  return before + incl;
}

// One row beyond the stage, merged by the whole block (merge path): thread t
// takes diagonals [t E, (t + 1) E) of the row's merged sequence (A first on
// ties), found by one binary search along the diagonal, and walks them from
// global memory (L1 catches each thread's sequential reads).  An output
// starts at an item whose column differs from the item before it; its owner
// (the thread holding that item) reads ahead through B's run of the column,
// even past its segment, and the items of a run inside another thread's
// segment are skipped there.  Count mode returns the row's output count
// (every thread); fill mode writes the outputs at oc / ov, 0 + (a + g | a | g)
// with g Python's sum() of B's run.  O((|A| + |B|) / 128 + log) per thread,
// whatever the row's shape (repeated B coordinates included).
template <bool kFill>
SL_DEV int merge_long_row(int32_t a0, int32_t a1, int32_t b0, int32_t b1,
                          const int32_t* __restrict__ a_crd, const double* __restrict__ a_vals,
                          const int32_t* __restrict__ b_cols, const double* __restrict__ b_vals,
                          int32_t* oc, double* ov, int* s_warp) {
  const int tid = threadIdx.x;
  const int na = a1 - a0, nb = b1 - b0, T = na + nb;
  const int E = (T + blockDim.x - 1) / blockDim.x;
  const int d0 = min(T, tid * E), d1 = min(T, d0 + E);
  int lo = max(0, d0 - nb), hi = min(d0, na);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ldg(a_crd + a0 + mid) <= ldg(b_cols + b0 + d0 - mid - 1)) lo = mid + 1; else hi = mid;
  }
  const int ia0 = lo, ib0 = d0 - lo;
  int32_t before = -1;                      // column of the item before diagonal d0
  if (d0 > 0) {
    const int32_t la = ia0 > 0 ? ldg(a_crd + a0 + ia0 - 1) : -1;
    const int32_t lb = ib0 > 0 ? ldg(b_cols + b0 + ib0 - 1) : -1;
    before = max(la, lb);
  }
  int cnt = 0;
  {
    int pa = ia0, pb = ib0;
    int32_t last = before;
    for (int d = d0; d < d1; ++d) {
      const int32_t ca = pa < na ? ldg(a_crd + a0 + pa) : INT32_MAX;
      const int32_t cb = pb < nb ? ldg(b_cols + b0 + pb) : INT32_MAX;
      const bool ta = ca <= cb;
      const int32_t c = ta ? ca : cb;
      cnt += c != last;
      last = c;
      pa += ta;
      pb += !ta;
    }
  }
  int total;
  const int incl = block_incl_scan(cnt, s_warp, &total);
  if (!kFill) {
    __syncthreads();                        // s_warp reused by the caller
    return total;
  }
  int q = incl - cnt;
  int pa = ia0, pb = ib0;
  int32_t last = before;
  for (int d = d0; d < d1; ++d) {
    const int32_t ca = pa < na ? ldg(a_crd + a0 + pa) : INT32_MAX;
    const int32_t cb = pb < nb ? ldg(b_cols + b0 + pb) : INT32_MAX;
    const bool ta = ca <= cb;
    const int32_t c = ta ? ca : cb;
    if (c != last) {                        // this thread owns the output of column c
      const double a = ta ? ldg(a_vals + a0 + pa) : 0.0;
      int u = ta ? pb : pb;                 // B's run of c starts at pb either way
      double g = 0.0;
      int nbr = 0;
      PySum ps;
      for (; u < nb && ldg(b_cols + b0 + u) == c; ++u, ++nbr) {
        const double bv = ldg(b_vals + b0 + u);
        if (nbr == 0) g = bv; else { if (nbr == 1) ps.start(g); ps.add(bv); }
      }
      if (nbr > 1) g = ps.value();
      const double e = ta ? (nbr ? dadd(a, g) : a) : g;
      oc[q] = c;
      ov[q] = dadd(0.0, e);
      ++q;
    }
    last = c;
    pa += ta;
    pb += !ta;
  }
  __syncthreads();
  return total;
}

// exclusive prefix of all tile totals before `tile` (one warp; lane 0 result)
SL_DEV int64_t tile_prefix(int64_t tile, const int64_t* tile_tot, const int64_t* super_tot) {
  const int lane = threadIdx.x & 31;
  const int64_t sup = tile / kSuper;
  int64_t acc = 0;
  for (int64_t u = lane; u < sup; u += 32) acc += ldg(super_tot + u);
  for (int64_t u = sup * kSuper + lane; u < tile; u += 32) acc += ldg(tile_tot + u);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  return acc;
}

// count: 32 registers keep 16 blocks (64 warps) resident; fill: columns-only
// staging (~17 KB of shared memory) and <= 40 registers keep 12
template <int kMode>
__global__ void __launch_bounds__(kAddRows, kMode == 0 ? 16 : 10)
add_tile_kernel(int64_t nrows, const int32_t* __restrict__ a_pos, const int32_t* __restrict__ a_crd,
                const double* __restrict__ a_vals, const int32_t* __restrict__ b_pos,
                const int32_t* __restrict__ b_cols, const double* __restrict__ b_vals,
                int32_t* __restrict__ c_pos, int32_t* __restrict__ c_crd,
                double* __restrict__ c_vals, int64_t* __restrict__ tile_tot,
                int64_t* __restrict__ super_tot, bool staged_ok,
                const int32_t* __restrict__ guard = nullptr, uint8_t* __restrict__ perm = nullptr) {
  constexpr bool kValues = kMode != 0;
  constexpr int kAddCap = kValues ? kAddCapFill : kAddCapCount;
  if (guard != nullptr) {                  // nothing to merge (see the exact convert)
    pdl_wait();
    if (ldg(guard) == 0) return;
  }
  __shared__ int32_t s_apos[kAddRows + 1], s_bpos[kAddRows + 1];
  // unified stages: A's slice at [0, kCS), B's at [kCS, 2 kCS); a value is
  // staged at the same index as its column
  constexpr int kCS = kAddCap + 8;
  __shared__ __align__(16) int32_t s_col[2 * kCS + 4];   // + slack read past B's end
  __shared__ int32_t s_rbase[kAddRows];         // row output offsets within the tile
  __shared__ int s_warp[kAddRows / 32];
  __shared__ int64_t s_tile_out;
  __shared__ __align__(8) uint64_t bar;
  // output stage (fill modes): the tile's outputs are contiguous in C; per
  // output its column and its sources (fill_row_src) — the values are read
  // from global memory when the stage is written out, so only columns are
  // staged and the block's shared memory stays at ~17 KB
  __shared__ __align__(8) uint2 s_out[kValues ? 2 * kAddCap : 1];
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  const int64_t tile = blockIdx.x;
  const int64_t r0 = tile * kAddRows;
  const int nr = (int)min64(kAddRows, nrows - r0);
  if (kMode == 0) {
    // launched with PDL behind the row-pointer pass: its b_pos and zeroed
    // super-tile totals must be visible; then let the fill begin launching
    // (it reads b_pos before its own wait: complete once this wait returns)
    pdl_wait();
    pdl_trigger();
  }
  for (int t = tid; t <= nr; t += kAddRows) {
    s_apos[t] = ldg(a_pos + r0 + t);
    s_bpos[t] = ldg(b_pos + r0 + t);
  }
  __syncthreads();
  const int32_t ea0 = s_apos[0], eb0 = s_bpos[0];
  const int32_t ea1 = s_apos[nr], eb1 = s_bpos[nr];
  const int na = ea1 - ea0, nb = eb1 - eb0;
  const bool fits = staged_ok && na <= kAddCap && nb <= kAddCap;   // block-uniform
  BulkRange32 ra{}, rb{};
  if (fits) {
    ra = plan_granules32(a_crd, ea0, ea1);
    rb = plan_granules32(b_cols, eb0, eb1);
    // element p of A lands at s_col[p - ra.lo0] (B: kCS + p - rb.lo0)
    if (tid == 0) {
      mbar_arrive_expect_tx(&bar, ra.tx_bytes + rb.tx_bytes);
      issue_range32(a_crd, ra, s_col, &bar);
      issue_range32(b_cols, rb, s_col + kCS, &bar);
      if (kValues) {            // the values the emitter reads after the merge: to L2 now
        prefetch_l2(a_vals + ea0, na);
        prefetch_l2(b_vals + eb0, nb);
      }
    }
    __syncthreads();
    // the fill waits for the copy only after reading its row bases and tile
    // prefix (global loads that then overlap the bulk copy)
    if (!kValues) mbar_wait(&bar, 0);
  }
  // ---- tiles beyond the stage (denser or power-law rows): consecutive row
  // groups whose A and B slices fit are staged and merged one after another
  // (a group of one oversized row merges from global memory)
  __shared__ int s_g1;
  uint32_t gphase = 0;
  auto oversized = [&](int r) {            // one row alone beyond the stage
    return s_apos[r + 1] - s_apos[r] > kAddCap || s_bpos[r + 1] - s_bpos[r] > kAddCap;
  };
  auto group_end = [&](int g0) {           // block-uniform: last row bound that still fits
    if (tid == 0) {
      int lo = g0 + 1, hi = nr;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_apos[mid] - s_apos[g0] <= kAddCap && s_bpos[mid] - s_bpos[g0] <= kAddCap) lo = mid;
        else hi = mid - 1;
      }
      s_g1 = lo;
    }
    __syncthreads();
    return s_g1;
  };
  // stage the slices of rows [g0, g1); returns the stage index offsets of A and B
  auto stage_group = [&](int g0, int g1, int32_t& oa, int32_t& ob) {
    const int32_t alo = s_apos[g0], ahi = s_apos[g1], blo = s_bpos[g0], bhi = s_bpos[g1];
    const BulkRange32 ga = plan_granules32(a_crd, alo, ahi), gb = plan_granules32(b_cols, blo, bhi);
    if (tid == 0) {
      fence_proxy_async_smem();          // the previous group's reads precede these writes
      mbar_arrive_expect_tx(&bar, ga.tx_bytes + gb.tx_bytes);
      issue_range32(a_crd, ga, s_col, &bar);
      issue_range32(b_cols, gb, s_col + kCS, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, gphase);
    gphase ^= 1u;
    oa = (int32_t)ga.lo0;
    ob = (int32_t)gb.lo0;
  };
  const bool grouped = !fits && staged_ok;   // block-uniform

  const bool mine = tid < nr;
  const GlobalAcc gacc{a_crd, a_vals, b_cols, b_vals};
  // Rows of a staged tile are merged in order of their merge length (a
  // counting sort over lengths clamped to 31; ties in any order), so each
  // warp's 32 rows have similar lengths and fewer lanes idle while the
  // longest row of the warp finishes (Poisson(5)+Poisson(5) rows: a warp's
  // longest row is ~1.6x the mean).  Returns the row this thread merges.
  __shared__ int s_hist[32];
  __shared__ uint8_t s_perm[kAddRows];
  auto sorted_row = [&]() -> int {
    if (tid < 32) s_hist[tid] = 0;
    __syncthreads();
    const int len = mine ? min((s_apos[tid + 1] - s_apos[tid]) + (s_bpos[tid + 1] - s_bpos[tid]), 31)
                         : 31;
    const int rank = atomicAdd(&s_hist[len], 1);
    __syncthreads();
    if (tid < 32) {                        // exclusive scan of the 32 bucket sizes
      const int v = s_hist[tid];
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += u;
      }
      s_hist[tid] = incl - v;
    }
    __syncthreads();
    s_perm[s_hist[len] + rank] = (uint8_t)tid;
    __syncthreads();
    return s_perm[tid];
  };
  // ---- per-row counts (count mode) / row bases (fill modes)
  if (kMode == 0) {
    int cnt = 0;
    if (grouped) {
      for (int g0 = 0; g0 < nr;) {
        if (oversized(g0)) {               // merged by its own thread below, in parallel
          ++g0;
          continue;
        }
        const int g1 = group_end(g0);
        int32_t oa, ob;
        stage_group(g0, g1, oa, ob);
        const int row = g0 + tid;
        if (row < g1)
          s_rbase[row] = count_row_idx(s_apos[row] - oa, s_apos[row + 1] - oa,
                                       kCS + s_bpos[row] - ob, kCS + s_bpos[row + 1] - ob, s_col);
        __syncthreads();                   // counts written, stage free
        g0 = g1;
      }
      // rows alone beyond the stage: merged by the whole block (merge path)
      const bool any_big = __syncthreads_or(mine && oversized(tid));
      for (int r = 0; any_big && r < nr; ++r) {
        if (!oversized(r)) continue;
        const int n = merge_long_row<false>(s_apos[r], s_apos[r + 1], s_bpos[r], s_bpos[r + 1],
                                            a_crd, nullptr, b_cols, nullptr, nullptr, nullptr,
                                            s_warp);
        if (tid == 0) s_rbase[r] = n;
        __syncthreads();
      }
      cnt = mine ? s_rbase[tid] : 0;
    } else if (fits) {
      const int row = sorted_row();
      // the fill merges the same rows in the same order: it reads the
      // permutation back instead of sorting again (four barriers per tile)
      if (perm) perm[tile * kAddRows + tid] = (uint8_t)row;
      if (row < nr)
        s_rbase[row] = count_row_idx(s_apos[row] - (int32_t)ra.lo0, s_apos[row + 1] - (int32_t)ra.lo0,
                                     kCS + s_bpos[row] - (int32_t)rb.lo0,
                                     kCS + s_bpos[row + 1] - (int32_t)rb.lo0, s_col);
      __syncthreads();
      cnt = mine ? s_rbase[tid] : 0;
    } else if (mine) {
      cnt = merge_row<false>(s_apos[tid], s_apos[tid + 1], s_bpos[tid], s_bpos[tid + 1], gacc,
                             NoEmit{});
    }
    int total;
    const int incl = block_incl_scan(cnt, s_warp, &total);
    if (mine) c_pos[r0 + tid + 1] = incl;           // tile-local; finalised later
    if (tid == 0) {
      tile_tot[tile] = total;
      atomicAdd(reinterpret_cast<unsigned long long*>(super_tot + tile / kSuper),
                (unsigned long long)total);
    }
    return;
  }

  int64_t tile_out, n_out;
  // fill launched with PDL behind the count pass: the stage copies above are
  // in flight; the counts, totals and c_pos it wrote are read from here on
  pdl_wait();
  // a tile that fits the fill's stage fitted the count's: its merge order is in perm
  const int prow = fits && perm ? (int)ldg(perm + tile * kAddRows + tid) : -1;
  if (kMode == 1) {
    tile_out = ldg(c_pos + r0);
    n_out = ldg(c_pos + r0 + nr) - tile_out;
    if (mine) s_rbase[tid] = (int32_t)(ldg(c_pos + r0 + tid) - tile_out);
  } else {
    if (tid < 32) {
      const int64_t pre = tile_prefix(tile, tile_tot, super_tot);
      if (tid == 0) s_tile_out = pre;
    }
    // c_pos holds tile-local inclusive counts
    const int32_t prev_local = mine && tid > 0 ? ldg(c_pos + r0 + tid) : 0;
    const int32_t own_local = mine ? ldg(c_pos + r0 + tid + 1) : 0;
    if (mine) s_rbase[tid] = prev_local;
    __syncthreads();   // prefix known; every predecessor count read before any write
    tile_out = s_tile_out;
    n_out = ldg(tile_tot + tile);
    if (mine) c_pos[r0 + tid + 1] = (int32_t)(tile_out + own_local);
    if (r0 + tid == 0) c_pos[0] = 0;
  }
  __syncthreads();
  if (grouped) {
    for (int g0 = 0; g0 < nr;) {
      if (oversized(g0)) {                 // merged by its own thread below, in parallel
        ++g0;
        continue;
      }
      const int g1 = group_end(g0);
      const int32_t ob0 = s_rbase[g0];                       // group's first output (tile-local)
      const int32_t ob1 = g1 < nr ? s_rbase[g1] : (int32_t)n_out;
      {
        int32_t oa, ob;
        stage_group(g0, g1, oa, ob);
        const int row = g0 + tid;
        if (row < g1)
          fill_row_src(s_apos[row] - oa, s_apos[row + 1] - oa, kCS + s_bpos[row] - ob,
                       kCS + s_bpos[row + 1] - ob, kCS, s_col, s_out + (s_rbase[row] - ob0));
        __syncthreads();
        // the group's outputs, coalesced
        emit_outputs<kAddRows>(ob1 - ob0, s_out, oa, ob, a_vals, b_vals,
                               c_crd + tile_out + ob0, c_vals + tile_out + ob0);
      }
      __syncthreads();                     // stages free for the next group
      g0 = g1;
    }
    // rows alone beyond the stage: merged by the whole block (merge path)
    const bool any_big = __syncthreads_or(mine && oversized(tid));
    for (int r = 0; any_big && r < nr; ++r) {
      if (!oversized(r)) continue;
      merge_long_row<true>(s_apos[r], s_apos[r + 1], s_bpos[r], s_bpos[r + 1], a_crd, a_vals,
                           b_cols, b_vals, c_crd + tile_out + s_rbase[r],
                           c_vals + tile_out + s_rbase[r], s_warp);
    }
    return;
  }
  if (fits) {
    const int row = perm ? prow : sorted_row();
    mbar_wait(&bar, 0);
    // n_out <= na + nb <= 2 kAddCap: the tile's outputs fit the output stage
    if (row < nr)
      fill_row_src(s_apos[row] - (int32_t)ra.lo0, s_apos[row + 1] - (int32_t)ra.lo0,
                   kCS + s_bpos[row] - (int32_t)rb.lo0, kCS + s_bpos[row + 1] - (int32_t)rb.lo0,
                   kCS, s_col, s_out + s_rbase[row]);
    __syncthreads();
    emit_outputs<kAddRows>((int)n_out, s_out, ra.lo0, rb.lo0, a_vals, b_vals,
                           c_crd + tile_out, c_vals + tile_out);
  } else if (mine) {                       // unaligned operands: merged from global memory
    merge_row<true>(s_apos[tid], s_apos[tid + 1], s_bpos[tid], s_bpos[tid + 1], gacc,
                    FillEmit{c_crd + tile_out + s_rbase[tid], c_vals + tile_out + s_rbase[tid]});
  }
}

// ---- COO -> CSR identity copy (formats.convert), duplicate-free fast path ----
// The reference's copy into CSR (engine.identity_copy, engine.py:775-779) is
// the A+B gather-append with an empty A: per row, B's coordinates in order,
// repeated ones summed, every value stored as 0.0 + v.  Without repeated
// coordinates that is B's row pointer, cols unchanged and 0.0 + vals, which
// this single pass writes (16 B read, 12 B written per nonzero); it also
// flags any repeated coordinate, in which case the guarded A+B passes that
// follow redo the conversion exactly (they exit at once when the flag is 0).
constexpr int kCvIpt = 4;

__global__ void __launch_bounds__(256)
coo_csr_copy_kernel(int64_t nrows, int64_t nnz, const int32_t* __restrict__ rows,
                    const int32_t* __restrict__ cols, const double* __restrict__ vals,
                    int32_t* __restrict__ rowptr, int32_t* __restrict__ c_pos,
                    int32_t* __restrict__ c_crd, double* __restrict__ c_vals,
                    int32_t* __restrict__ dup_flag, bool vec_ok, int32_t* __restrict__ a_pos,
                    int64_t* __restrict__ super_tot, int64_t nsuper) {
  // the guarded fallback's inputs: an all-zero A row pointer, zeroed super-tile totals
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q <= nrows;
       q += (int64_t)gridDim.x * blockDim.x) {
    a_pos[q] = 0;
    if (q < nsuper) super_tot[q] = 0;
  }
  const int64_t e0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kCvIpt;
  if (e0 > nnz) return;
  int32_t r[kCvIpt], c[kCvIpt];
  double v[kCvIpt];
  const bool vec = vec_ok && e0 + kCvIpt <= nnz;
  if (vec) {
    const int4 a = ld_stream(reinterpret_cast<const int4*>(rows + e0));
    const int4 b = ld_stream(reinterpret_cast<const int4*>(cols + e0));
    const double2 v0 = ld_stream(reinterpret_cast<const double2*>(vals + e0));
    const double2 v1 = ld_stream(reinterpret_cast<const double2*>(vals + e0 + 2));
    r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
    c[0] = b.x; c[1] = b.y; c[2] = b.z; c[3] = b.w;
    v[0] = v0.x; v[1] = v0.y; v[2] = v1.x; v[3] = v1.y;
  } else {
#pragma unroll
    for (int t = 0; t < kCvIpt; ++t) {
      const bool ok = e0 + t < nnz;
      r[t] = ok ? ldg(rows + e0 + t) : (int32_t)nrows;
      c[t] = ok ? ldg(cols + e0 + t) : -1;
      v[t] = ok ? ldg(vals + e0 + t) : 0.0;
    }
  }
  const int32_t prev_r = e0 == 0 ? -1 : ldg(rows + e0 - 1);
  const int32_t prev_c = e0 == 0 ? -1 : ldg(cols + e0 - 1);
  unsigned gaps = 0;
  bool dup = false;
#pragma unroll
  for (int t = 0; t < kCvIpt; ++t) {
    const int32_t pr = t == 0 ? prev_r : r[t - 1];
    const int32_t pc = t == 0 ? prev_c : c[t - 1];
    if (r[t] != pr) {
      rowptr[r[t]] = (int32_t)(e0 + t);
      c_pos[r[t]] = (int32_t)(e0 + t);
    }
    gaps |= (r[t] - pr > 1 ? 1u : 0u) << t;
    dup |= e0 + t < nnz && r[t] == pr && c[t] == pc;
  }
  if (gaps) {
#pragma unroll
    for (int t = 0; t < kCvIpt; ++t)
      if (gaps >> t & 1u) {
        const int32_t lo = t == 0 ? prev_r : r[t - 1];
        for (int32_t q = lo + 1; q < r[t]; ++q) {
          rowptr[q] = (int32_t)(e0 + t);
          c_pos[q] = (int32_t)(e0 + t);
        }
      }
  }
  if (dup) atomicOr(dup_flag, 1);
  if (vec) {
    *reinterpret_cast<int4*>(c_crd + e0) = make_int4(c[0], c[1], c[2], c[3]);
    *reinterpret_cast<double2*>(c_vals + e0) = make_double2(dadd(0.0, v[0]), dadd(0.0, v[1]));
    *reinterpret_cast<double2*>(c_vals + e0 + 2) = make_double2(dadd(0.0, v[2]), dadd(0.0, v[3]));
  } else {
#pragma unroll
    for (int t = 0; t < kCvIpt; ++t)
      if (e0 + t < nnz) {
        c_crd[e0 + t] = c[t];
        c_vals[e0 + t] = dadd(0.0, v[t]);
      }
  }
}

// two-pass count: c_pos[r + 1] += prefix of its tile; c_pos[0] = 0
__global__ void __launch_bounds__(kAddRows)
pos_finalize_kernel(int64_t nrows, const int64_t* __restrict__ tile_tot,
                    const int64_t* __restrict__ super_tot, int32_t* __restrict__ c_pos) {
  __shared__ int64_t s_off;
  const int64_t tile = blockIdx.x;
  if (threadIdx.x < 32) {
    const int64_t pre = tile_prefix(tile, tile_tot, super_tot);
    if (threadIdx.x == 0) s_off = pre;
  }
  __syncthreads();
  const int64_t r = tile * kAddRows + threadIdx.x;
  if (r < nrows) c_pos[r + 1] = (int32_t)(c_pos[r + 1] + s_off);
  if (r == 0) c_pos[0] = 0;
}

}  // namespace sl

using namespace sl;
using sl_host::as_stream;
using sl_host::ceil_div;

// workspace: [tile totals i64 x ntiles][super-tile totals i64 x nsuper][rowptr i32 x (nrows+1)]
static int64_t add_ntiles(int64_t nrows) { return (nrows + kAddRows - 1) / kAddRows; }
static int64_t add_nsuper(int64_t nrows) { return (add_ntiles(nrows) + kSuper - 1) / kSuper; }
static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
static size_t add_tiles_bytes(int64_t nrows) { return al256((size_t)add_ntiles(nrows) * 8); }
static size_t add_super_bytes(int64_t nrows) { return al256((size_t)add_nsuper(nrows) * 8); }

static size_t add_rowptr_bytes(int64_t nrows) { return al256((size_t)(nrows + 1) * sizeof(int32_t)); }
static size_t add_perm_bytes(int64_t nrows) { return al256((size_t)add_ntiles(nrows) * kAddRows); }

extern "C" size_t sl_add_csr_workspace_bytes(int64_t nrows, int64_t b_nnz) {
  (void)b_nnz;
  return add_tiles_bytes(nrows) + add_super_bytes(nrows) + add_rowptr_bytes(nrows) +
         add_perm_bytes(nrows) + 256;
}

// the fill stages values at their columns' indices: needs 16-byte-aligned operands
static bool add_staged_ok(const int32_t* ac, const double* av, const int32_t* bc,
                          const double* bv) {
  return sl_host::aligned16(ac) && sl_host::aligned16(av) && sl_host::aligned16(bc) &&
         sl_host::aligned16(bv);
}

struct AddWs {
  int64_t* tiles;
  int64_t* supers;
  int32_t* rowptr;
  uint8_t* perm;       // [ntiles][kAddRows]: each staged tile's merge order (count -> fill)
};

static AddWs add_ws(void* ws, int64_t nrows) {
  char* p = static_cast<char*>(ws);
  char* rp = p + add_tiles_bytes(nrows) + add_super_bytes(nrows);
  return AddWs{reinterpret_cast<int64_t*>(p), reinterpret_cast<int64_t*>(p + add_tiles_bytes(nrows)),
               reinterpret_cast<int32_t*>(rp),
               reinterpret_cast<uint8_t*>(rp + add_rowptr_bytes(nrows))};
}

void sl_host::launch_coo_rowptr(int64_t nrows, int64_t nnz, const int32_t* rows,
                                int32_t* rowptr, cudaStream_t s) {
  coo_rowptr_kernel<SL_ROWPTR_IPT_SPMV>
      <<<ceil_div(ceil_div(nnz + 1, SL_ROWPTR_IPT_SPMV), 256), 256, 0, s>>>(
          nrows, nnz, rows, rowptr, (int64_t*)nullptr, (int64_t)0);
}

static const int32_t* add_rowptr(int64_t nrows, int64_t b_nnz, const int32_t* b_pos,
                                 const int32_t* b_rows, const AddWs& w, bool build, cudaStream_t s) {
  if (b_pos) return b_pos;
  if (build) sl_host::launch_coo_rowptr(nrows, b_nnz, b_rows, w.rowptr, s);
  return w.rowptr;
}

static int add_check(int64_t nrows, int64_t b_nnz, const int32_t* a_pos, const int32_t* b_pos,
                     const int32_t* b_rows, const int32_t* c_pos, void* ws, size_t ws_bytes) {
  if (nrows < 0 || b_nnz < 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || b_nnz > INT32_MAX) return SL_ERR_RANGE;
  if (!c_pos || !a_pos || (!b_pos && !b_rows && b_nnz > 0)) return SL_ERR_INVALID;
  if (!ws || ws_bytes < sl_add_csr_workspace_bytes(nrows, b_nnz)) return SL_ERR_WORKSPACE;
  return SL_OK;
}

// count pass: rowptr (COO B; it also zeroes the super-tile totals), tile
// counts (tile-local c_pos, tile and super-tile totals), the count launched
// with PDL behind the row pointer
static const int32_t* add_count_pass(int64_t nrows, const int32_t* a_pos, const int32_t* a_crd,
                                     int64_t b_nnz, const int32_t* b_pos, const int32_t* b_rows,
                                     const int32_t* b_cols, int32_t* c_pos, const AddWs& w,
                                     cudaStream_t s) {
  const int32_t* bp = b_pos;
  if (b_pos) {
    cudaMemsetAsync(w.supers, 0, (size_t)add_nsuper(nrows) * 8, s);
  } else {
    coo_rowptr_kernel<8><<<ceil_div(ceil_div(b_nnz + 1, 8), 256), 256, 0, s>>>(
        nrows, b_nnz, b_rows, w.rowptr, w.supers, add_nsuper(nrows));
    bp = w.rowptr;
  }
  sl_host::launch_pdl(add_tile_kernel<0>, dim3((unsigned)add_ntiles(nrows)), dim3(kAddRows), s,
                      (size_t)0, nrows, a_pos, a_crd, (const double*)nullptr, bp, b_cols,
                      (const double*)nullptr, c_pos, (int32_t*)nullptr, (double*)nullptr, w.tiles,
                      w.supers, true, (const int32_t*)nullptr, w.perm);
  return bp;
}

extern "C" int sl_add_csr_count(int64_t nrows, const int32_t* a_pos, const int32_t* a_crd,
                                int64_t b_nnz, const int32_t* b_pos, const int32_t* b_rows,
                                const int32_t* b_cols, int32_t* c_pos, void* ws, size_t ws_bytes,
                                void* stream) {
  const int st = add_check(nrows, b_nnz, a_pos, b_pos, b_rows, c_pos, ws, ws_bytes);
  if (st != SL_OK) return st;
  cudaStream_t s = as_stream(stream);
  if (nrows == 0)
    return cudaMemsetAsync(c_pos, 0, sizeof(int32_t), s) == cudaSuccess ? SL_OK : SL_ERR_CUDA;
  const AddWs w = add_ws(ws, nrows);
  add_count_pass(nrows, a_pos, a_crd, b_nnz, b_pos, b_rows, b_cols, c_pos, w, s);
  pos_finalize_kernel<<<(int)add_ntiles(nrows), kAddRows, 0, s>>>(nrows, w.tiles, w.supers, c_pos);
  return sl_host::launch_status();
}

extern "C" int sl_add_csr_fill(int64_t nrows, const int32_t* a_pos, const int32_t* a_crd,
                               const double* a_vals, int64_t b_nnz, const int32_t* b_pos,
                               const int32_t* b_rows, const int32_t* b_cols, const double* b_vals,
                               const int32_t* c_pos, int32_t* c_crd, double* c_vals, void* ws,
                               size_t ws_bytes, void* stream) {
  const int st = add_check(nrows, b_nnz, a_pos, b_pos, b_rows, c_pos, ws, ws_bytes);
  if (st != SL_OK) return st;
  if ((!c_crd || !c_vals) && b_nnz > 0) return SL_ERR_INVALID;
  if (nrows == 0) return SL_OK;
  cudaStream_t s = as_stream(stream);
  const AddWs w = add_ws(ws, nrows);
  // a COO B's row pointer was built by sl_add_csr_count in the same workspace
  const int32_t* bp = add_rowptr(nrows, b_nnz, b_pos, b_rows, w, false, s);
  add_tile_kernel<1><<<(int)add_ntiles(nrows), kAddRows, 0, s>>>(
      nrows, a_pos, a_crd, a_vals, bp, b_cols, b_vals, const_cast<int32_t*>(c_pos), c_crd, c_vals,
      w.tiles, w.supers, add_staged_ok(a_crd, a_vals, b_cols, b_vals), nullptr, w.perm);
  return sl_host::launch_status();
}

extern "C" int sl_add_csr_f64(int64_t nrows, const int32_t* a_pos, const int32_t* a_crd,
                              const double* a_vals, int64_t b_nnz, const int32_t* b_pos,
                              const int32_t* b_rows, const int32_t* b_cols, const double* b_vals,
                              int32_t* c_pos, int32_t* c_crd, double* c_vals, void* ws,
                              size_t ws_bytes, void* stream) {
  const int st = add_check(nrows, b_nnz, a_pos, b_pos, b_rows, c_pos, ws, ws_bytes);
  if (st != SL_OK) return st;
  cudaStream_t s = as_stream(stream);
  if (nrows == 0)
    return cudaMemsetAsync(c_pos, 0, sizeof(int32_t), s) == cudaSuccess ? SL_OK : SL_ERR_CUDA;
  const AddWs w = add_ws(ws, nrows);
  const int32_t* bp = add_count_pass(nrows, a_pos, a_crd, b_nnz, b_pos, b_rows, b_cols, c_pos, w, s);
  sl_host::launch_pdl(add_tile_kernel<2>, dim3((unsigned)add_ntiles(nrows)), dim3(kAddRows), s,
                      (size_t)0, nrows, a_pos, a_crd, a_vals, bp, b_cols, b_vals, c_pos, c_crd, c_vals,
                      w.tiles, w.supers, add_staged_ok(a_crd, a_vals, b_cols, b_vals),
                      (const int32_t*)nullptr, w.perm);
  return sl_host::launch_status();
}

// COO -> CSR exactly as the reference's convert (formats.py:583-587 ->
// engine.identity_copy): c_crd / c_vals hold nnz elements (the duplicate-free
// size, an upper bound); nnz(C) = c_pos[nrows].
extern "C" size_t sl_convert_coo_to_csr_exact_workspace_bytes(int64_t nrows, int64_t nnz) {
  return sl_add_csr_workspace_bytes(nrows, nnz) + al256((size_t)(nrows + 1) * sizeof(int32_t)) +
         256;
}

extern "C" int sl_convert_coo_to_csr_exact(int64_t nrows, int64_t nnz, const int32_t* rows,
                                           const int32_t* cols, const double* vals,
                                           int32_t* c_pos, int32_t* c_crd, double* c_vals,
                                           void* ws, size_t ws_bytes, void* stream) {
  if (nrows < 0 || nnz < 0) return SL_ERR_INVALID;
  if (nrows > INT32_MAX || nnz > INT32_MAX) return SL_ERR_RANGE;
  if (!c_pos || (nnz > 0 && (!rows || !cols || !vals || !c_crd || !c_vals))) return SL_ERR_INVALID;
  if (!ws || ws_bytes < sl_convert_coo_to_csr_exact_workspace_bytes(nrows, nnz))
    return SL_ERR_WORKSPACE;
  cudaStream_t s = as_stream(stream);
  if (nrows == 0)
    return cudaMemsetAsync(c_pos, 0, sizeof(int32_t), s) == cudaSuccess ? SL_OK : SL_ERR_CUDA;
  const AddWs w = add_ws(ws, nrows);
  char* tail = static_cast<char*>(ws) + sl_add_csr_workspace_bytes(nrows, nnz);
  int32_t* a_pos = reinterpret_cast<int32_t*>(tail);                 // empty A: all zeros
  int32_t* flag = reinterpret_cast<int32_t*>(tail + al256((size_t)(nrows + 1) * sizeof(int32_t)));
  cudaMemsetAsync(flag, 0, sizeof(int32_t), s);
  const bool vec_ok = sl_host::aligned16(rows) && sl_host::aligned16(cols) &&
                      sl_host::aligned16(vals) && sl_host::aligned16(c_crd) &&
                      sl_host::aligned16(c_vals);
  coo_csr_copy_kernel<<<ceil_div(ceil_div(nnz + 1, kCvIpt), 256), 256, 0, s>>>(
      nrows, nnz, rows, cols, vals, w.rowptr, c_pos, c_crd, c_vals, flag, vec_ok, a_pos, w.supers,
      add_nsuper(nrows));
  // repeated coordinates: the exact gather-append passes (no-ops otherwise)
  add_tile_kernel<0><<<(int)add_ntiles(nrows), kAddRows, 0, s>>>(
      nrows, a_pos, nullptr, nullptr, w.rowptr, cols, nullptr, c_pos, nullptr, nullptr, w.tiles,
      w.supers, true, flag);
  add_tile_kernel<2><<<(int)add_ntiles(nrows), kAddRows, 0, s>>>(
      nrows, a_pos, nullptr, nullptr, w.rowptr, cols, vals, c_pos, c_crd, c_vals, w.tiles, w.supers,
      add_staged_ok(nullptr, nullptr, cols, vals), flag);
  return sl_host::launch_status();
}
