/*
 * sl_abi.h — C ABI of the B200-native sparse level-format kernels.
 *
 * This is the drop-in boundary for the reference's hot path: the executor
 * loop nest `_Executor.run_node` / `run_fused` (reference
 * pkg/src/sparselevels/engine.py:580-713) specialised, per SURVEY.md §8(a16),
 * to the five expression/format patterns of BASELINE.json, plus the level
 * functions those loop nests call (levels.py:215-394).
 *
 * Conventions
 *   - Every pointer is a caller-owned DEVICE pointer (cudaMalloc / torch), except
 *     where a parameter is documented as a host pointer.
 *   - Coordinates and positions are int32 (the reference uses Python ints; the
 *     configs fit int32, and sizes above INT32_MAX return SL_ERR_RANGE).
 *     Values are IEEE binary64.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Every call is asynchronous and stream-ordered; nothing here synchronises
 *     the host except the functions documented as "synchronous".
 *   - No call allocates device memory.  Scratch comes from a caller workspace
 *     sized by the matching sl_*_workspace_bytes() function.
 *   - Return value: SL_OK (0) or an SL_ERR_* code.  The Python host package
 *     maps them 1:1 onto the reference exception classes (errors.py:4-55).
 *   - Reentrant; the only global state is a cached per-device SM count.
 *   - Arrays are read in whole 16-byte granules by the bulk (TMA) copies: up to
 *     15 bytes before an array start and after an array end that are not
 *     16-byte aligned may be read (never written, never used).  Every
 *     cudaMalloc / cuMemMap / torch allocation contains those bytes; a tightly
 *     packed suballocation must leave them readable.
 *
 * Arithmetic contract ("Exact arithmetic"):
 *   SpMV     y[i] = ((+0.0 + a_i,j1*x_j1) + a_i,j2*x_j2) + ...   in storage
 *            order, one rounding per multiply and per add (no FMA contraction):
 *            bit-identical to engine.py:303,320 (scatter) / :606-633 (CSR).
 *   A+B      sorted union per row; value a+b where both stored, else the copy;
 *            explicit zeros kept (engine.py:387-413): bit-identical.  A run
 *            of repeated B coordinates is one term, Python's sum() of the run
 *            (engine.py:527; Neumaier-compensated on CPython 3.12).
 *   MTTKRP   A[i,r] = sum of (x*B[j,r])*C[k,r] (engine.py:528-529 association);
 *            the sum over a slice is a parallel reduction, so A matches the
 *            sequential reference within |d| <= 1e-12 * sum|terms|.
 */
#ifndef SL_ABI_H
#define SL_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:4-55) ------------------------------------- */
enum {
  SL_OK = 0,
  SL_ERR_INVALID = 1,              /* bad argument (null pointer, negative size)        */
  SL_ERR_UNSUPPORTED_CAPABILITY = 2,/* UnsupportedCapabilityError  errors.py:8 / levels.py:197 */
  SL_ERR_ASSEMBLY = 3,             /* AssemblyError               errors.py:16          */
  SL_ERR_HASH_SEGMENT_FULL = 4,    /* HashSegmentFullError        errors.py:20 / levels.py:330 */
  SL_ERR_UNSUPPORTED_MERGE = 5,    /* UnsupportedMergeError       errors.py:46          */
  SL_ERR_UNSUPPORTED_OUTPUT = 6,   /* UnsupportedOutputError      errors.py:50          */
  SL_ERR_RANGE = 7,                /* size beyond the int32 index contract               */
  SL_ERR_WORKSPACE = 8,            /* workspace too small                                */
  SL_ERR_CUDA = 9                  /* CUDA launch/runtime failure                        */
};

/* ---- level kinds (levels.py:25-31) -------------------------------------- */
enum {
  SL_DENSE = 0, SL_RANGE = 1, SL_COMPRESSED = 2,
  SL_SINGLETON = 3, SL_OFFSET = 4, SL_HASHED = 5
};

/* One storage level as the reference's LevelStorage (levels.py:173-191).
 * Which fields are meaningful depends on `kind`, exactly as in the reference. */
typedef struct sl_level {
  int32_t kind;
  int32_t crd_stride;      /* interleaved (AoS) crd arrays: stride, default 1     */
  int32_t crd_base;        /* interleaved (AoS) crd arrays: lane, default 0       */
  int32_t noffset;         /* length of `offset` (range/offset levels)            */
  int64_t n;               /* dense/range: dimension size                         */
  int64_t m;               /* range: the other dimension's extent                 */
  int64_t w;               /* hashed: segment width                               */
  int64_t range_n;         /* offset: enclosing range level's n                   */
  const int32_t* pos;      /* compressed                                           */
  const int32_t* crd;      /* compressed / singleton / hashed                      */
  const int32_t* offset;   /* range / offset (shared DIA offsets)                  */
} sl_level;

/* Level-function ids for sl_level_query (levels.py:215-294). */
enum {
  SL_FN_COORD_BOUNDS = 0,  /* in: a = prefix last coord      out: o0 = lo, o1 = hi     */
  SL_FN_COORD_ACCESS = 1,  /* in: a = parent_pos, b = coord  out: o0 = pos, o1 = found */
  SL_FN_POS_BOUNDS = 2,    /* in: a = parent_pos             out: o0 = lo, o1 = hi     */
  SL_FN_POS_ACCESS = 3,    /* in: a = pos, b = prefix last   out: o0 = coord, o1 = found */
  SL_FN_LOCATE = 4,        /* in: a = parent_pos, b = coord  out: o0 = pos, o1 = found */
  SL_FN_SIZE = 5           /* in: a = parent_size            out: o0 = size            */
};

/* ---- library ----------------------------------------------------------- */
int         sl_version(void);                 /* ABI version, 0x0100 = 1.0 */
const char* sl_status_string(int status);     /* static string, never NULL */
/* Synchronous: clears and returns the sticky error of the last CUDA call. */
int         sl_last_cuda_error(void);
/* Number of SMs of the current device (cached). Synchronous. */
int         sl_device_sm_count(int32_t* out);

/* ---- level functions, batched on the device ------------------------------
 * Replaces: LevelStorage.coord_bounds/coord_access/pos_bounds/pos_access/
 * locate/size (levels.py:215-294).  `lv` is a HOST pointer to the level
 * descriptor whose array pointers are device pointers.  For each query q,
 * evaluates function `fn` on (a[q], b[q]) and writes (o0[q], o1[q]).
 * Returns SL_ERR_UNSUPPORTED_CAPABILITY (without launching) when the kind
 * lacks the capability, exactly as LevelStorage._require (levels.py:197-199).
 * b and o1 may be NULL when the function does not use them. */
int sl_level_query(const sl_level* lv, int32_t fn, int64_t nq,
                   const int64_t* a, const int64_t* b,
                   int64_t* o0, int64_t* o1, void* stream);

/* ---- hashed level: locate and insert --------------------------------------
 * Replaces: LevelStorage.locate for hashed levels (levels.py:270-280) —
 * linear probing from (coord % w) inside segment parent_pos, first match wins,
 * first -1 or a full scan of the segment means "absent" (pos -1, found 0).
 * Warp-cooperative: `group` lanes (1, 4, 8, 16 or 32) probe consecutive slots
 * of one query at once; the result is the first match-or-empty in probe order.
 * parent_pos may be NULL (all queries in segment 0: a hash vector). */
int sl_hashed_locate(int64_t nq, const int32_t* parent_pos, const int32_t* coord,
                     int64_t w, const int32_t* crd,
                     int32_t* out_pos, uint8_t* out_found, int32_t group,
                     void* stream);

/* Replaces: LevelStorage.insert_init + insert_coord (levels.py:303-333) in bulk.
 * crd must already hold -1 in empty slots (sl_hashed_insert_init does that).
 * Concurrent inserts use atomicCAS, so the final slot of a coordinate is the
 * one some sequential insertion order would give; the SET of stored
 * coordinates per segment and every locate result's `found` are identical to
 * the reference's.  Idempotent.  Overflow is reported through *err_flag
 * (device int32, set to SL_ERR_HASH_SEGMENT_FULL) — the call itself is async. */
int sl_hashed_insert_init(int64_t size, int32_t* crd, void* stream);
int sl_hashed_insert(int64_t nq, const int32_t* parent_pos, const int32_t* coord,
                     int64_t w, int32_t* crd, int32_t* err_flag, void* stream);
/* The same bulk insert with the reference's exact table layout: the result
 * equals calling insert_coord(parent_pos[q], coord[q]) for q = 0, 1, ... in
 * order (every coordinate at the first slot from its home free at its turn;
 * entries already in crd keep their slots; repeated coordinates idempotent).
 * Priority race: slots hold (q << 32 | coord) updated by atomicMin, so a slot
 * only passes to earlier queries and displaced ones probe on.  size = the
 * table length (a multiple of w); workspace from
 * sl_hashed_insert_ordered_workspace_bytes(nq, size). */
size_t sl_hashed_insert_ordered_workspace_bytes(int64_t nq, int64_t size);
int sl_hashed_insert_ordered(int64_t nq, const int32_t* parent_pos, const int32_t* coord,
                             int64_t w, int64_t size, int32_t* crd, int32_t* err_flag,
                             void* ws, size_t ws_bytes, void* stream);

/* Slot map of a hash vector: for every coordinate c < n, the answer of
 * locate(c) (first slot in probe order holding c with no empty slot before
 * it), packed (probe distance << 32 | slot) in a u64 at ws[c], ~0 = absent.
 * Exact for any table contents.  Used when queries outnumber table slots
 * (one resolution per coordinate instead of one probe sequence per query). */
size_t sl_hashed_slot_map_workspace_bytes(int64_t n, int64_t w);
int sl_hashed_slot_map(int64_t n, int64_t w, const int32_t* crd, void* ws, size_t ws_bytes,
                       void* stream);

/* ---- SpMV  y(i) = A(i,j) * x(j), dense x and y --------------------------
 * COO-SoA (formats.py:132-133): rows/cols = L0/L1 crd, row-major sorted
 * (the compressed(~U) level is ordered).  Replaces run_fused over i(+)j with
 * scatter into y (engine.py:636-713, 281-320).  No conversion to CSR: tiles of
 * nonzeros are staged, products formed in parallel, and each row is summed in
 * storage order by the thread that owns the row's first nonzero.  Empty rows
 * are written as +0.0 in the same launch (no memset). */
/* CSR SpMV of a row block with the all-gather of y fused into the epilogue
 * (each GPU stores its rows straight into every peer's full-y
 * buffer over NVLink instead of an NCCL all-gather after the kernel).
 * y_peers: HOST array of npeers (1..8) device pointers — peer buffers mapped
 * through CUDA IPC / symmetric memory, or local buffers — each already offset
 * to this block's first global row.  The register hand-off kernel stores
 * directly (rows averaging <= 28 nonzeros, 16-byte-aligned crd/vals); other
 * matrices are computed into y_peers[0] and copied to the rest.  The caller
 * synchronises the ranks (a barrier) before reading its full y. */
int sl_spmv_csr_peers_f64(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* pos,
                          const int32_t* crd, const double* vals, const double* x,
                          const uint64_t* y_peers, int32_t npeers, void* stream);

/* Optional kernels this build carries: bit 0 = the A/B alternatives (CSR
 * variants 1, 3, 4 and the persistent TMA pipelines of SL_SPMV_PATH=pipe),
 * compiled only with SL_BUILD_ALT=1; without them those variants return
 * SL_ERR_INVALID. */
int sl_build_features(void);

int sl_spmv_coo_f64(int64_t nrows, int64_t ncols, int64_t nnz,
                    const int32_t* rows, const int32_t* cols, const double* vals,
                    const double* x, double* y, void* ws, size_t ws_bytes, void* stream);
/* Workspace of sl_spmv_coo_f64: the row level's position index (nrows + 1
 * ints), built per call by one streaming pass over the row coordinates; with
 * it (and rows averaging <= 28 nonzeros, 16-byte-aligned arrays) the sums run
 * in the register hand-off kernel; ws == NULL keeps the staged-tile kernel. */
size_t sl_spmv_coo_workspace_bytes(int64_t nrows);

/* CSR (formats.py:126-127). Replaces run_node(i) -> run_node(j) with
 * locate of x (engine.py:591-634).
 * variant 0 = automatic: register hand-off (variant 6) when rows average
 *             <= 28 nonzeros and crd/vals are 16-byte aligned, else row-block (5);
 * variant 1 = vector-per-row (a warp per row; lanes load the row's nonzeros
 *             coalesced, lane 0 sums them in order from registers via shuffles);
 * variant 2 = merge-path (nnz+rows balanced tiles; row-owner sums in order);
 * variant 3 = warp row-block (each warp owns 32 rows, warp-private staging);
 * variant 4 = row-stage (the block's crd/vals bulk-copied (TMA) to shared
 *             memory; thread per row walks its row in order; crd and vals
 *             must be 16-byte aligned, else SL_ERR_INVALID);
 * variant 5 = row-block (rows tiled; nonzeros of the tile staged through
 *             shared memory in coalesced chunks; thread per row sums in order);
 * variant 6 = register hand-off (persistent one-warp blocks: a 32-row tile is
 *             bulk-copied to shared memory, each lane moves its row into
 *             registers and the next tile's copy starts while this one is
 *             gathered and summed; 16-byte-aligned crd/vals, else SL_ERR_INVALID);
 * All variants are bit-identical.  ws may be NULL for every variant but 2. */
size_t sl_spmv_csr_workspace_bytes(int64_t nrows, int64_t nnz, int32_t variant);
int sl_spmv_csr_f64(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* pos,
                    const int32_t* crd, const double* vals,
                    const double* x, double* y, int32_t variant,
                    void* ws, size_t ws_bytes, void* stream);

/* ELL (formats.py:164-169): slot-major crd/vals [nslots * nrows], position
 * s*nrows + i (levels.py:230), padding (col 0, 0.0) visited like the
 * reference (its 0.0*x[0] terms are added after the row's real entries). */
int sl_spmv_ell_f64(int64_t nrows, int64_t ncols, int32_t nslots,
                    const int32_t* crd, const double* vals,
                    const double* x, double* y, void* stream);

/* DIA (formats.py:170-175): ndiag sorted offsets (HOST or device pointer,
 * see offsets_on_host), vals [ndiag * nrows] at d*nrows + i.  Row i takes the
 * term of diagonal d iff 0 <= i + offset[d] < ncols (range level bounds,
 * levels.py:220-222), in ascending-offset order. */
int sl_spmv_dia_f64(int64_t nrows, int64_t ncols, int32_t ndiag,
                    const int32_t* offsets, int32_t offsets_on_host,
                    const double* vals, const double* x, double* y, void* stream);

/* DIA row block [row0, row0 + nrows) of a larger matrix (a multi-GPU shard):
 * vals [ndiag * nrows] hold the block's slots, y the block's rows, x the whole
 * vector; row i of the block takes diagonal d iff 0 <= row0 + i + offset[d] <
 * ncols.  sl_spmv_dia_f64 is row0 = 0. */
int sl_spmv_dia_rows_f64(int64_t nrows, int64_t row0, int64_t ncols, int32_t ndiag,
                         const int32_t* offsets, int32_t offsets_on_host,
                         const double* vals, const double* x, double* y, void* stream);

/* CSR x hash-vector: y(i) = A(i,j) * x(j) with x a hashed level of width w
 * (crd[w] with -1 empties, vals[w] by slot).  x is located per nonzero
 * (engine.py:558-572 -> levels.py:270-280); a miss contributes no term. */
int sl_spmv_csr_hashx_f64(int64_t nrows, const int32_t* pos, const int32_t* crd,
                          const double* vals, int64_t w, const int32_t* x_crd,
                          const double* x_vals, double* y, void* stream);

/* ---- C(i,j) = A(i,j) + B(i,j) -> CSR --------------------------------------
 * A is CSR; B is COO-SoA (b_pos == NULL, b_rows given) or CSR (b_pos given).
 * Replaces the co-iteration of engine.py:591-634 with the gather-append
 * writer (engine.py:330-434).  Two passes:
 *   count: c_pos[0] = 0, c_pos[i+1] = |row i of A  union  row i of B|, then an
 *          in-place exclusive scan -> c_pos is the final CSR row pointer;
 *   fill:  writes c_crd/c_vals in sorted-union order.
 * nnz_c = c_pos[nrows] (read it back, or size c_crd/c_vals at nnz_a + nnz_b). */
/* CSR x hash-vector through the slot map (x has dimension n): the same
 * results as sl_spmv_csr_hashx_f64, one locate per coordinate instead of per
 * nonzero.  ws: sl_spmv_csr_hashx_map_workspace_bytes(n, w). */
size_t sl_spmv_csr_hashx_map_workspace_bytes(int64_t n, int64_t w);
int sl_spmv_csr_hashx_map_f64(int64_t nrows, int64_t n, int64_t nnz, const int32_t* pos,
                              const int32_t* crd, const double* vals, int64_t w,
                              const int32_t* x_crd,
                              const double* x_vals, double* y, void* ws, size_t ws_bytes,
                              void* stream);

/* CSR x sparse-vector x (compressed, ordered, unique; dimension n): the
 * product's j-lattice is the intersection {A1, x1} (engine.py:211-225,
 * 591-634) — only coordinates present in both contribute, in ascending j.
 * Replaces that merge with an index map (coordinate -> position in x) built
 * in ws, then the CSR row-block kernel.  ws: sl_spmv_csr_spx_workspace_bytes(n). */
size_t sl_spmv_csr_spx_workspace_bytes(int64_t n);
int sl_spmv_csr_spx_f64(int64_t nrows, int64_t n, int64_t nnz, const int32_t* pos,
                        const int32_t* crd, const double* vals, int64_t x_nnz, const int32_t* x_crd,
                        const double* x_vals, double* y, void* ws, size_t ws_bytes,
                        void* stream);

/* ---- SpMM  Y(i,k) = A(i,j) * X(j,k): A CSR, X (ncols x K) and Y (nrows x K)
 * dense row-major (dense-2).  Replaces the (i, j, k) loop nest with dense
 * scatter (engine.py:591-634, 281-320): each Y(i,k) accumulates the row's
 * products in storage order from +0.0 — bit-identical. */
int sl_spmm_csr_f64(int64_t nrows, int64_t ncols, int64_t K, const int32_t* pos,
                    const int32_t* crd, const double* vals, const double* X, double* Y,
                    void* stream);
/* The same product with the nonzero count known to the caller (nnz =
 * pos[nrows]; -1: unknown): the average row length picks the kernel shape
 * (two columns per lane for rows averaging >= 16 nonzeros).  Bit-identical
 * to sl_spmm_csr_f64; same reference loop nest. */
int sl_spmm_csr_nnz_f64(int64_t nrows, int64_t ncols, int64_t K, int64_t nnz, const int32_t* pos,
                        const int32_t* crd, const double* vals, const double* X, double* Y,
                        void* stream);
/* The same product with rows longer than long_min split out (power-law
 * rows): a device pass lists them (workspace: a counter and the list), the
 * group kernel skips them, and one CTA per listed row gathers its X rows with
 * all warps while one warp adds the products in storage order — bit-identical
 * to sl_spmm_csr_f64.  Same reference loop nest as above. */
int64_t sl_spmm_csr_split_workspace_bytes(int64_t nrows, int64_t nnz, int32_t long_min);
int sl_spmm_csr_split_f64(int64_t nrows, int64_t ncols, int64_t K, int64_t nnz,
                          const int32_t* pos, const int32_t* crd, const double* vals,
                          const double* X, double* Y, int32_t long_min, void* ws,
                          int64_t ws_bytes, void* stream);

/* ---- 3-tensor kernels beyond MTTKRP (X CSF) ----------
 * TTV Y(i,j) = X(i,j,k) v(k) and TTM Y(i,j,r) = X(i,j,k) U(k,r) reduce over k
 * inside each (i, j) fiber: the fiber sums are sl_spmv_csr_f64 /
 * sl_spmm_csr_f64 over the fibers as rows (pos2, crd2, vals), bit-identical.
 * Then, dense output: rows (nfibers x R) scattered to out (I x J x R, zero
 * elsewhere); CSR output (gather writer, engine.py:330-434): one entry per
 * fiber, pos over i from the slice structure, crd = crd1, vals = fiber sums. */
int sl_csf_fiber_scatter_f64(int64_t I, int64_t J, int64_t R, int64_t nslices, int64_t nfibers,
                             const int32_t* crd0, const int32_t* pos1, const int32_t* crd1,
                             const double* rows, double* out, void* stream);
int sl_csf_fiber_rowptr(int64_t I, int64_t nslices, const int32_t* crd0, const int32_t* pos1,
                        int32_t* pos_out, void* stream);
/* INNERPROD a() = X(i,j,k) * Z(i,j,k), both COO-3 sorted: intersection at
 * every level (engine.py:211-225).  *out (device) = the sum, reduced in a
 * fixed tree order: deterministic, within the fp64 reduction tolerance of the
 * reference's per-fiber / per-slice order.  ws: sl_inner_coo3_workspace_bytes(nx). */
size_t sl_inner_coo3_workspace_bytes(int64_t nx);
int sl_inner_coo3_f64(int64_t I, int64_t J, int64_t K, int64_t nx, const int32_t* xi,
                      const int32_t* xj, const int32_t* xk, const double* xv, int64_t nz,
                      const int32_t* zi, const int32_t* zj, const int32_t* zk, const double* zv,
                      double* out, void* ws, size_t ws_bytes, void* stream);

size_t sl_add_csr_workspace_bytes(int64_t nrows, int64_t b_nnz);
int sl_add_csr_count(int64_t nrows,
                     const int32_t* a_pos, const int32_t* a_crd,
                     int64_t b_nnz, const int32_t* b_pos, const int32_t* b_rows,
                     const int32_t* b_cols,
                     int32_t* c_pos, void* ws, size_t ws_bytes, void* stream);
int sl_add_csr_fill(int64_t nrows,
                    const int32_t* a_pos, const int32_t* a_crd, const double* a_vals,
                    int64_t b_nnz, const int32_t* b_pos, const int32_t* b_rows,
                    const int32_t* b_cols, const double* b_vals,
                    const int32_t* c_pos, int32_t* c_crd, double* c_vals,
                    void* ws, size_t ws_bytes, void* stream);

/* Fused single pass: count, decoupled look-back scan and fill in one launch
 * over the operands (each read once).  c_crd / c_vals must hold nnz_a + nnz_b
 * entries (the union's upper bound); c_pos is final on completion. */
int sl_add_csr_f64(int64_t nrows,
                   const int32_t* a_pos, const int32_t* a_crd, const double* a_vals,
                   int64_t b_nnz, const int32_t* b_pos, const int32_t* b_rows,
                   const int32_t* b_cols, const double* b_vals,
                   int32_t* c_pos, int32_t* c_crd, double* c_vals,
                   void* ws, size_t ws_bytes, void* stream);

/* ---- MTTKRP  A(i,r) = X(i,j,k) * B(j,r) * C(k,r) ----------------------------
 * B [J x R], C [K x R], A [I x R] row-major dense (dense-2 layout).
 * COO-3 (formats.py:138-140): i, j, k = L0/L1/L2 crd, lexicographically sorted.
 * CSF (formats.py:136-137): pos0/crd0 slices, pos1/crd1 fibers, pos2/crd2.
 * Rows of A with no nonzeros are written +0.0 in-kernel.  Deterministic:
 * partial sums of slices split across work chunks are combined by a fix-up
 * kernel in a fixed order. */
size_t sl_mttkrp_workspace_bytes(int64_t nnz, int32_t R);
int sl_mttkrp_coo3_f64(int64_t I, int64_t J, int64_t K, int32_t R, int64_t nnz,
                       const int32_t* i, const int32_t* j, const int32_t* k,
                       const double* vals, const double* B, const double* C,
                       double* A, void* ws, size_t ws_bytes, void* stream);
int sl_mttkrp_csf_f64(int64_t I, int64_t J, int64_t K, int32_t R,
                      int64_t nslices, int64_t nfibers, int64_t nnz,
                      const int32_t* crd0, const int32_t* pos1, const int32_t* crd1,
                      const int32_t* pos2, const int32_t* crd2,
                      const double* vals, const double* B, const double* C,
                      double* A, void* ws, size_t ws_bytes, void* stream);

/* ---- format conversion (formats.convert, formats.py:583-587) -------------
 * COO -> CSR exactly as the reference's identity copy: call the A+B entry
 * points with an empty A (a_pos all zero) and the COO as B; the structural
 * row pointer alone (row-sorted COO, unique coordinates) is: */
int sl_convert_coo_to_csr(int64_t nrows, int64_t nnz, const int32_t* rows, int32_t* pos,
                          void* stream);
/* COO -> CSR exactly (repeated coordinates summed as (0 + v1) + v2 ..., every
 * value stored as 0.0 + v; engine.identity_copy, engine.py:775-779) in one
 * streaming pass when the COO has no repeated coordinate (row pointer, cols
 * copied, 0.0 + vals), else through the A+B gather-append passes, chosen on
 * the device (no host round trip).  c_crd / c_vals hold nnz elements;
 * nnz(C) = c_pos[nrows]. */
size_t sl_convert_coo_to_csr_exact_workspace_bytes(int64_t nrows, int64_t nnz);
int sl_convert_coo_to_csr_exact(int64_t nrows, int64_t nnz, const int32_t* rows,
                                const int32_t* cols, const double* vals, int32_t* c_pos,
                                int32_t* c_crd, double* c_vals, void* ws, size_t ws_bytes,
                                void* stream);
/* CSR -> ELL: nslots = max per-row count of nonzero values (read *out_dev
 * after the stream); entries with value 0.0 are dropped and values stored as
 * 0.0 + v, as the reference's reorder writer + assemble do. */
int sl_csr_max_row_length(int64_t nrows, const int32_t* pos, const double* vals,
                          int32_t* out_dev, void* stream);
int sl_convert_csr_to_ell(int64_t nrows, int32_t nslots, const int32_t* pos,
                          const int32_t* crd, const double* vals,
                          int32_t* ell_crd, double* ell_vals, void* stream);
/* COO (unique coordinates) -> DIA: offsets of the nonzero entries' diagonals,
 * sorted (offsets needs nrows + ncols - 1 entries; *ndiag_dev is the count),
 * then the values [ndiag * nrows] (0.0 where no entry). */
size_t sl_convert_coo_to_dia_workspace_bytes(int64_t nrows, int64_t ncols);
int sl_convert_coo_to_dia_offsets(int64_t nrows, int64_t ncols, int64_t nnz,
                                  const int32_t* rows, const int32_t* cols, const double* vals,
                                  int32_t* offsets, int32_t* ndiag_dev,
                                  void* ws, size_t ws_bytes, void* stream);
int sl_convert_coo_to_dia_values(int64_t nrows, int64_t ncols, int64_t nnz, int32_t ndiag,
                                 const int32_t* rows, const int32_t* cols, const double* vals,
                                 double* dia_vals, void* ws, size_t ws_bytes, void* stream);

/* CSR -> COO-SoA row coordinates (rows[p] = i for p in [pos[i], pos[i+1])):
 * with the A+B entry points (empty B) this is the identity copy into COO and
 * the COO output of a gather-append (engine.py:330-434). */
int sl_csr_row_indices(int64_t nrows, const int32_t* pos, int32_t* rows, void* stream);

/* ---- utilities used by the benchmark ------------------------------------- */
/* Writes `bytes` of junk into `buf` to evict L2 between timed iterations. */
int sl_l2_flush(void* buf, size_t bytes, void* stream);
/* Read-only sweep of `bytes` (>= the L2 size): evicts L2 and leaves it clean,
 * so the next kernel starts cold without paying for earlier write-backs. */
int sl_l2_read(const void* buf, size_t bytes, void* sink, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SL_ABI_H */
