// pipe.cu — persistent, warp-specialized TMA pipelines for the SpMV formats.
//
// One CTA per SM.  Warp 0 is the producer: its lane 0 walks the CTA's tiles
// (tile = blockIdx.x + j * gridDim.x) and, for each, bulk-copies the tile's
// index/value slices into stage j % kGroups of a shared-memory ring
// (cp.async.bulk, completion counted on the stage's `full` mbarrier).
// Consumer group g (kGroupThreads threads) owns stage g: it waits on full[g],
// computes the tile, writes y, and releases the stage on empty[g], which the
// producer waits on before refilling.  With kGroups tiles in flight per SM the
// copy engine always has the next tiles' bytes moving while the current one
// is computed: the structure the LDG kernels lacked (ncu: long-scoreboard
// bound, 1.1-wave tails).
//
// Arithmetic is the reference's: per row, products a*x added
// in storage order from +0.0, one rounding each — bit-identical to the LDG
// kernels and to the oracle.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "tma.cuh"

namespace sl {

constexpr int kPG = 4;           // consumer groups = ring stages
constexpr int kPGT = 128;        // threads per consumer group
constexpr int kPGW = kPGT / 32;  // warps per group
constexpr int kPipeThreads = 32 + kPG * kPGT;

struct PipeBars {
  uint64_t full[kPG];
  uint64_t empty[kPG];
};

SL_DEV void pipe_init(PipeBars& b) {
  if (threadIdx.x == 0) {
    for (int g = 0; g < kPG; ++g) {
      mbar_init(&b.full[g], 1);
      mbar_init(&b.empty[g], kPGW);
    }
    fence_mbar_init();
  }
  __syncthreads();
}

// producer side: stage g may be refilled once its previous tile was consumed
SL_DEV void pipe_acquire(PipeBars& b, int j) {
  const int g = j % kPG, k = j / kPG;
  if (k > 0) mbar_wait(&b.empty[g], (k - 1) & 1);
}

SL_DEV void pipe_release(PipeBars& b, int g) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&b.empty[g]);
}

// ---------------------------------------------------------------------------
// ELL: tile = kPGT rows x all slots (nslots <= kEllPipeMaxSlots).

__global__ void __launch_bounds__(kPipeThreads, 1)
spmv_ell_pipe_kernel(int64_t nrows, int32_t nslots, const int32_t* __restrict__ crd,
                     const double* __restrict__ vals, const double* __restrict__ x,
                     double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) PipeBars bars;
  const size_t stage = (size_t)nslots * kPGT * 12;
  const int64_t ntiles = (nrows + kPGT - 1) / kPGT;
  pipe_init(bars);
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (threadIdx.x == 0) {
      for (int j = 0;; ++j) {
        const int64_t tile = blockIdx.x + (int64_t)j * gridDim.x;
        if (tile >= ntiles) break;
        pipe_acquire(bars, j);
        const int g = j % kPG;
        const int64_t r0 = tile * kPGT;
        const int nr = (int)min64(kPGT, nrows - r0);
        unsigned char* st = smem + g * stage;
        mbar_arrive_expect_tx(&bars.full[g], (uint32_t)(nslots * nr * 12));
        for (int s = 0; s < nslots; ++s) {
          const int64_t p = (int64_t)s * nrows + r0;
          bulk_g2s(st + (size_t)s * kPGT * 8, vals + p, nr * 8, &bars.full[g]);
          bulk_g2s(st + (size_t)nslots * kPGT * 8 + (size_t)s * kPGT * 4, crd + p, nr * 4,
                   &bars.full[g]);
        }
      }
    }
    return;
  }
  const int g = (warp - 1) / kPGW;
  const int t = threadIdx.x - 32 - g * kPGT;
  for (int j = g;; j += kPG) {
    const int64_t tile = blockIdx.x + (int64_t)j * gridDim.x;
    if (tile >= ntiles) break;
    mbar_wait(&bars.full[g], (j / kPG) & 1);
    const int64_t r0 = tile * kPGT;
    const int nr = (int)min64(kPGT, nrows - r0);
    if (t < nr) {
      const double* sv = reinterpret_cast<const double*>(smem + g * stage);
      const int32_t* sc = reinterpret_cast<const int32_t*>(smem + g * stage + (size_t)nslots * kPGT * 8);
      double a = 0.0;
      int u = 0;
      for (; u + 9 <= nslots; u += 9) {
        double xv[9];
#pragma unroll
        for (int b = 0; b < 9; ++b) xv[b] = ldg(x + sc[(u + b) * kPGT + t]);
#pragma unroll
        for (int b = 0; b < 9; ++b) a = dadd(a, dmul(sv[(u + b) * kPGT + t], xv[b]));
      }
      for (; u < nslots; ++u) a = dadd(a, dmul(sv[u * kPGT + t], ldg(x + sc[u * kPGT + t])));
      y[r0 + t] = a;
    }
    pipe_release(bars, g);
  }
}

// ---------------------------------------------------------------------------
// DIA: tile = kPGT rows; per diagonal the in-range value slice and x window.
constexpr int kDiaPipeMax = 32;
constexpr int kDiaPipeSlot = kPGT + 4;   // + realignment slack (f64: <= 1 element per end)

struct DiaPlan {
  int64_t lo, hi;                        // in-range rows [lo, hi) of the tile
  BulkRange<double> v, xw;
};

SL_DEV DiaPlan dia_plan(const double* vals, const double* x, int64_t nrows, int64_t ncols,
                        int64_t r0, int nr, int d, int32_t off) {
  DiaPlan p;
  p.lo = max64(r0, -(int64_t)off);
  p.hi = min64(r0 + nr, ncols - off);
  if (p.hi < p.lo) p.hi = p.lo;
  p.v = plan_range(vals, (int64_t)d * nrows + p.lo, (int64_t)d * nrows + p.hi);
  p.xw = plan_range(x, p.lo + off, p.hi + off);
  return p;
}

__global__ void __launch_bounds__(kPipeThreads, 1)
spmv_dia_pipe_kernel(int64_t nrows, int64_t ncols, int32_t ndiag, DiaOffsets offs,
                     const double* __restrict__ vals, const double* __restrict__ x,
                     double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) PipeBars bars;
  __shared__ int32_t s_off[kDiaPipeMax];
  if (threadIdx.x < kDiaPipeMax) s_off[threadIdx.x] = threadIdx.x < ndiag ? offs.v[threadIdx.x] : 0;
  const size_t stage = (size_t)ndiag * 2 * kDiaPipeSlot * 8;
  const int64_t ntiles = (nrows + kPGT - 1) / kPGT;
  pipe_init(bars);
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (threadIdx.x == 0) {
      for (int j = 0;; ++j) {
        const int64_t tile = blockIdx.x + (int64_t)j * gridDim.x;
        if (tile >= ntiles) break;
        pipe_acquire(bars, j);
        const int g = j % kPG;
        const int64_t r0 = tile * kPGT;
        const int nr = (int)min64(kPGT, nrows - r0);
        double* sv = reinterpret_cast<double*>(smem + g * stage);
        double* sx = sv + (size_t)ndiag * kDiaPipeSlot;
        uint32_t tx = 0;
        for (int d = 0; d < ndiag; ++d) {
          const DiaPlan p = dia_plan(vals, x, nrows, ncols, r0, nr, d, s_off[d]);
          tx += p.v.tx_bytes + p.xw.tx_bytes;
        }
        mbar_arrive_expect_tx(&bars.full[g], tx);
        for (int d = 0; d < ndiag; ++d) {
          const DiaPlan p = dia_plan(vals, x, nrows, ncols, r0, nr, d, s_off[d]);
          if (p.v.tx_bytes)
            bulk_g2s(sv + (size_t)d * kDiaPipeSlot + (p.v.blo - p.v.lo0), vals + p.v.blo,
                     p.v.tx_bytes, &bars.full[g]);
          if (p.xw.tx_bytes)
            bulk_g2s_keep(sx + (size_t)d * kDiaPipeSlot + (p.xw.blo - p.xw.lo0), x + p.xw.blo,
                          p.xw.tx_bytes, &bars.full[g]);
        }
      }
    }
    return;
  }
  const int g = (warp - 1) / kPGW;
  const int t = threadIdx.x - 32 - g * kPGT;
  for (int j = g;; j += kPG) {
    const int64_t tile = blockIdx.x + (int64_t)j * gridDim.x;
    if (tile >= ntiles) break;
    mbar_wait(&bars.full[g], (j / kPG) & 1);
    const int64_t r0 = tile * kPGT;
    const int nr = (int)min64(kPGT, nrows - r0);
    if (t < nr) {
      const int64_t i = r0 + t;
      const double* sv = reinterpret_cast<const double*>(smem + g * stage);
      const double* sx = sv + (size_t)ndiag * kDiaPipeSlot;
      double a = 0.0;
      for (int d = 0; d < ndiag; ++d) {
        const int32_t off = s_off[d];
        const int64_t jc = i + off;
        if (jc < 0 || jc >= ncols) continue;
        const DiaPlan p = dia_plan(vals, x, nrows, ncols, r0, nr, d, off);
        const int64_t ve = (int64_t)d * nrows + i;
        const double v = (ve >= p.v.blo && ve < p.v.bhi)
                             ? sv[(size_t)d * kDiaPipeSlot + (ve - p.v.lo0)] : ldg(vals + ve);
        const double xv = (jc >= p.xw.blo && jc < p.xw.bhi)
                              ? sx[(size_t)d * kDiaPipeSlot + (jc - p.xw.lo0)] : ldg(x + jc);
        a = dadd(a, dmul(v, xv));
      }
      y[i] = a;
    }
    pipe_release(bars, g);
  }
}

// ---------------------------------------------------------------------------
// COO: tile = kCooPipeTile nonzeros + kCooPipeHalo staged past its end.
// Products in place; each consumer thread owns the row starts among 16
// consecutive items and sums those rows in storage order (halo, then global
// for rows longer than the halo).  Empty rows are zeroed by the owner of the
// next stored row (no memset).
constexpr int kCooPipeTile = 2048;
constexpr int kCooPipeHalo = 256;
constexpr int kCooPipeSt = kCooPipeTile + kCooPipeHalo;
constexpr int kCooPipeIpt = kCooPipeTile / kPGT;    // 16 owned items per thread
constexpr size_t kCooPipeStage = (size_t)kCooPipeSt * 8 + (size_t)(kCooPipeSt + 8) * 4 +
                                 (size_t)kCooPipeSt * 4;

__global__ void __launch_bounds__(kPipeThreads, 1)
spmv_coo_pipe_kernel(int64_t nrows, int64_t nnz, const int32_t* __restrict__ rows,
                     const int32_t* __restrict__ cols, const double* __restrict__ vals,
                     const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) PipeBars bars;
  const int64_t ntiles = (nnz + kCooPipeTile - 1) / kCooPipeTile;
  pipe_init(bars);
  const int warp = threadIdx.x >> 5;
  // stage layout: vals[St] | rows[4 + St + 4] | cols[St]; rows[3] = row before the tile
  auto sval = [&](int g) { return reinterpret_cast<double*>(smem + g * kCooPipeStage); };
  auto srow = [&](int g) {
    return reinterpret_cast<int32_t*>(smem + g * kCooPipeStage + (size_t)kCooPipeSt * 8);
  };
  auto scol = [&](int g) {
    return reinterpret_cast<int32_t*>(smem + g * kCooPipeStage + (size_t)kCooPipeSt * 8 +
                                      (size_t)(kCooPipeSt + 8) * 4);
  };
  if (warp == 0) {
    if (threadIdx.x == 0) {
      for (int j = 0;; ++j) {
        const int64_t tile = blockIdx.x + (int64_t)j * gridDim.x;
        if (tile >= ntiles) break;
        pipe_acquire(bars, j);
        const int g = j % kPG;
        const int64_t e0 = tile * kCooPipeTile;
        const int n_st = (int)min64(kCooPipeSt, nnz - e0);
        const int nb = n_st & ~3;   // 16-byte multiple for the 4-byte arrays
        const int nbv = n_st & ~1;
        mbar_arrive_expect_tx(&bars.full[g], (uint32_t)(nb * 8 + nbv * 8));
        if (nbv) bulk_g2s(sval(g), vals + e0, nbv * 8, &bars.full[g]);
        if (nb) {
          bulk_g2s(srow(g) + 4, rows + e0, nb * 4, &bars.full[g]);
          bulk_g2s(scol(g), cols + e0, nb * 4, &bars.full[g]);
        }
      }
    }
    return;
  }
  const int g = (warp - 1) / kPGW;
  const int t = threadIdx.x - 32 - g * kPGT;
  for (int j = g;; j += kPG) {
    const int64_t tile = blockIdx.x + (int64_t)j * gridDim.x;
    if (tile >= ntiles) break;
    const int64_t e0 = tile * kCooPipeTile;
    const int n_in = (int)min64(kCooPipeTile, nnz - e0);
    const int n_st = (int)min64(kCooPipeSt, nnz - e0);
    const int nb = n_st & ~3, nbv = n_st & ~1;
    const int32_t before = (t == 0) ? (e0 == 0 ? -1 : ldg(rows + e0 - 1)) : 0;
    mbar_wait(&bars.full[g], (j / kPG) & 1);
    double* sv = sval(g);
    int32_t* sr = srow(g);
    const int32_t* sc = scol(g);
    if (t == 0) sr[3] = before;
    // unaligned tail items (last tile only)
    for (int q = nb + t; q < n_st; q += kPGT) {
      sr[4 + q] = ldg(rows + e0 + q);
      const_cast<int32_t*>(sc)[q] = ldg(cols + e0 + q);
    }
    for (int q = nbv + t; q < n_st; q += kPGT) sv[q] = ldg(vals + e0 + q);
    group_sync(1 + g, kPGT);
    // products in place, gathers of 18 items issued together
    {
      constexpr int kIt = kCooPipeSt / kPGT;
      double xv[kIt];
#pragma unroll
      for (int k = 0; k < kIt; ++k) {
        const int q = t + k * kPGT;
        xv[k] = q < n_st ? ldg(x + sc[q]) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < kIt; ++k) {
        const int q = t + k * kPGT;
        if (q < n_st) sv[q] = dmul(sv[q], xv[k]);
      }
    }
    group_sync(1 + g, kPGT);
    const int q0 = t * kCooPipeIpt;
    if (q0 < n_in) {
      int32_t prev = sr[3 + q0];
      for (int tt = 0; tt < kCooPipeIpt; ++tt) {
        const int q = q0 + tt;
        if (q >= n_in) break;
        const int32_t r = sr[4 + q];
        if (r != prev) {
          double acc = 0.0;
          int u = q;
          for (; u < n_st && sr[4 + u] == r; ++u) acc = dadd(acc, sv[u]);
          int64_t ge = e0 + u;
          if (u == n_st) {
            for (; ge < nnz && ldg(rows + ge) == r; ++ge)
              acc = dadd(acc, dmul(ldg(vals + ge), ldg(x + ldg(cols + ge))));
          }
          y[r] = acc;
          for (int32_t q2 = prev + 1; q2 < r; ++q2) y[q2] = 0.0;
          if (ge == nnz)
            for (int64_t q2 = (int64_t)r + 1; q2 < nrows; ++q2) y[q2] = 0.0;
        }
        prev = r;
      }
    }
    group_sync(1 + g, kPGT);   // all reads of the stage done before release
    pipe_release(bars, g);
  }
}

// ---------------------------------------------------------------------------
// CSR: tile = kPGT rows; their nonzero range [pos[r0], pos[r0 + nr]) is
// staged up to kCsrPipeCap elements (the rest, for unusually dense tiles, is
// read directly).  The producer warp prefetches the tiles' pos bounds 32 at a
// time so the copies are never behind a dependent load.
constexpr int kCsrPipeCap = kPGT * 28;   // 3584: the 27-point stencil's 3456 fit
constexpr size_t kCsrPipeStage = (size_t)(kCsrPipeCap + 4) * 8 + (size_t)(kCsrPipeCap + 8) * 4;

__global__ void __launch_bounds__(kPipeThreads, 1)
spmv_csr_pipe_kernel(int64_t nrows, const int32_t* __restrict__ pos,
                     const int32_t* __restrict__ crd, const double* __restrict__ vals,
                     const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) PipeBars bars;
  const int64_t ntiles = (nrows + kPGT - 1) / kPGT;
  pipe_init(bars);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto sval = [&](int g) { return reinterpret_cast<double*>(smem + g * kCsrPipeStage); };
  auto scrd = [&](int g) {
    return reinterpret_cast<int32_t*>(smem + g * kCsrPipeStage + (size_t)(kCsrPipeCap + 4) * 8);
  };
  if (warp == 0) {
    int64_t eb_l = 0, ee_l = 0;
    for (int j = 0;; ++j) {
      const int64_t tile = blockIdx.x + (int64_t)j * gridDim.x;
      if (tile >= ntiles) break;
      if ((j & 31) == 0) {   // lanes prefetch the bounds of the next 32 tiles
        const int64_t tl = blockIdx.x + (int64_t)(j + lane) * gridDim.x;
        if (tl < ntiles) {
          eb_l = ldg(pos + tl * kPGT);
          ee_l = ldg(pos + min64(tl * kPGT + kPGT, nrows));
        }
      }
      const int64_t eb = __shfl_sync(0xffffffffu, eb_l, j & 31);
      const int64_t ee = __shfl_sync(0xffffffffu, ee_l, j & 31);
      if (lane == 0) {
        pipe_acquire(bars, j);
        const int g = j % kPG;
        const int64_t ce = min64(ee, eb + kCsrPipeCap);
        const BulkRange<int32_t> rc = plan_range(crd, eb, ce);
        const BulkRange<double> rv = plan_range(vals, eb, ce);
        mbar_arrive_expect_tx(&bars.full[g], rc.tx_bytes + rv.tx_bytes);
        issue_range(vals, rv, sval(g), &bars.full[g]);
        issue_range(crd, rc, scrd(g), &bars.full[g]);
      }
      __syncwarp();
    }
    return;
  }
  const int g = (warp - 1) / kPGW;
  const int t = threadIdx.x - 32 - g * kPGT;
  for (int j = g;; j += kPG) {
    const int64_t tile = blockIdx.x + (int64_t)j * gridDim.x;
    if (tile >= ntiles) break;
    const int64_t r0 = tile * kPGT;
    const int nr = (int)min64(kPGT, nrows - r0);
    // row bounds and tile bounds: issued before waiting on the stage
    const int64_t pb = t < nr ? ldg(pos + r0 + t) : 0;
    const int64_t pe = t < nr ? ldg(pos + r0 + t + 1) : 0;
    const int64_t eb = ldg(pos + r0), ee = ldg(pos + r0 + nr);
    const int64_t ce = min64(ee, eb + kCsrPipeCap);
    const BulkRange<int32_t> rc = plan_range(crd, eb, ce);
    const BulkRange<double> rv = plan_range(vals, eb, ce);
    mbar_wait(&bars.full[g], (j / kPG) & 1);
    double* sv = sval(g);
    const int32_t* sc = scrd(g);
    const int n = (int)(ce - eb);
    // products in place (edge elements outside the bulk ranges come from global)
    for (int q0 = 0; q0 < n; q0 += 9 * kPGT) {
      double xv[9], vv[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const int q = q0 + t + k * kPGT;
        const int64_t e = eb + q;
        if (q < n) {
          const int32_t c = (e >= rc.blo && e < rc.bhi) ? sc[e - rc.lo0] : ldg(crd + e);
          vv[k] = (e >= rv.blo && e < rv.bhi) ? sv[e - rv.lo0] : ldg(vals + e);
          xv[k] = ldg(x + c);
        }
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const int q = q0 + t + k * kPGT;
        if (q < n) sv[eb + q - rv.lo0] = dmul(vv[k], xv[k]);
      }
    }
    group_sync(1 + g, kPGT);
    if (t < nr) {
      double acc = 0.0;
      const int64_t mid = min64(pe, ce);
      for (int64_t e = pb; e < mid; ++e) acc = dadd(acc, sv[e - rv.lo0]);
      for (int64_t e = max64(pb, ce); e < pe; ++e)        // beyond the staged cap
        acc = dadd(acc, dmul(ldg(vals + e), ldg(x + ldg(crd + e))));
      y[r0 + t] = acc;
    }
    group_sync(1 + g, kPGT);
    pipe_release(bars, g);
  }
}

}  // namespace sl

// ---------------------------------------------------------------------------
// host launchers (called from spmv.cu's C ABI)

namespace sl_host {

static int pipe_grid(int64_t ntiles) {
  const int sms = sm_count();
  return (int)(ntiles < sms ? ntiles : sms);
}

template <typename K>
static bool set_smem(K kernel, size_t bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) ==
         cudaSuccess;
}

int launch_ell_pipe(int64_t nrows, int32_t nslots, const int32_t* crd, const double* vals,
                    const double* x, double* y, cudaStream_t s) {
  using namespace sl;
  const size_t smem = (size_t)kPG * nslots * kPGT * 12;
  if (!set_smem(spmv_ell_pipe_kernel, smem)) return SL_ERR_CUDA;
  const int64_t ntiles = (nrows + kPGT - 1) / kPGT;
  spmv_ell_pipe_kernel<<<pipe_grid(ntiles), kPipeThreads, smem, s>>>(nrows, nslots, crd, vals, x, y);
  return launch_status();
}

int launch_dia_pipe(int64_t nrows, int64_t ncols, int32_t ndiag, const sl::DiaOffsets& offs,
                    const double* vals, const double* x, double* y, cudaStream_t s) {
  using namespace sl;
  const size_t smem = (size_t)kPG * ndiag * 2 * kDiaPipeSlot * 8;
  if (!set_smem(spmv_dia_pipe_kernel, smem)) return SL_ERR_CUDA;
  const int64_t ntiles = (nrows + kPGT - 1) / kPGT;
  spmv_dia_pipe_kernel<<<pipe_grid(ntiles), kPipeThreads, smem, s>>>(nrows, ncols, ndiag, offs,
                                                                    vals, x, y);
  return launch_status();
}

int launch_coo_pipe(int64_t nrows, int64_t nnz, const int32_t* rows, const int32_t* cols,
                    const double* vals, const double* x, double* y, cudaStream_t s) {
  using namespace sl;
  const size_t smem = (size_t)kPG * kCooPipeStage;
  if (!set_smem(spmv_coo_pipe_kernel, smem)) return SL_ERR_CUDA;
  const int64_t ntiles = (nnz + kCooPipeTile - 1) / kCooPipeTile;
  spmv_coo_pipe_kernel<<<pipe_grid(ntiles), kPipeThreads, smem, s>>>(nrows, nnz, rows, cols, vals,
                                                                    x, y);
  return launch_status();
}

int launch_csr_pipe(int64_t nrows, const int32_t* pos, const int32_t* crd, const double* vals,
                    const double* x, double* y, cudaStream_t s) {
  using namespace sl;
  const size_t smem = (size_t)kPG * kCsrPipeStage;
  if (!set_smem(spmv_csr_pipe_kernel, smem)) return SL_ERR_CUDA;
  const int64_t ntiles = (nrows + kPGT - 1) / kPGT;
  spmv_csr_pipe_kernel<<<pipe_grid(ntiles), kPipeThreads, smem, s>>>(nrows, pos, crd, vals, x, y);
  return launch_status();
}

}  // namespace sl_host
