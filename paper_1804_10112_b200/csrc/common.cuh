// common.cuh — shared device helpers for the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sl_abi.h"

#define SL_DEV __device__ __forceinline__

namespace sl {

// The reference rounds every product and every sum separately
// (engine.py:528-531 evaluates Python floats).  The _rn intrinsics are never
// contracted into FMA, which keeps results bit-identical.
SL_DEV double dmul(double a, double b) { return __dmul_rn(a, b); }
SL_DEV double dadd(double a, double b) { return __dadd_rn(a, b); }
SL_DEV double dsub(double a, double b) { return __dsub_rn(a, b); }

// A duplicate group's value is Python's builtin sum() over it
// (engine.py:527: `sum(vals[p] for p in ps)`).  The reference runs on CPython
// 3.12, whose sum() of floats is Neumaier-compensated (bltinmodule.c,
// builtin_sum_impl): f = 0 + v1 (int 0 + float), then per item
// t = f + x, c += |f| >= |x| ? (f - t) + x : (x - t) + f, f = t; the result is
// f + c when c is nonzero and finite, else f.  Two items give the plain sum;
// three or more can differ from it in the last bit.
struct PySum {
  double f, c;
  SL_DEV void start(double v1) { f = dadd(0.0, v1); c = 0.0; }
  SL_DEV void add(double x) {
    const double t = dadd(f, x);
    c = dadd(c, fabs(f) >= fabs(x) ? dadd(dsub(f, t), x) : dadd(dsub(x, t), f));
    f = t;
  }
  SL_DEV double value() const { return (c != 0.0 && isfinite(c)) ? dadd(f, c) : f; }
};

// Programmatic dependent launch: wait for the preceding grid (its writes
// visible), and let the next grid in the stream begin launching.
SL_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SL_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Read-only loads through the non-coherent path.
template <typename T>
SL_DEV T ldg(const T* p) { return __ldg(p); }

// Streaming loads: data touched exactly once.  Not allocated in L1 and tagged
// evict-first in L2 (an L2 cache policy from createpolicy) so the reused
// operands (x, factor matrices) stay resident.
SL_DEV uint64_t policy_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
SL_DEV uint64_t policy_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
SL_DEV int32_t ld_stream(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
      : "=r"(v) : "l"(p), "l"(policy_evict_first()));
  return v;
}
SL_DEV double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
      : "=d"(v) : "l"(p), "l"(policy_evict_first()));
  return v;
}
SL_DEV int4 ld_stream(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(policy_evict_first()));
  return v;
}
SL_DEV int2 ld_stream(const int2* p) {
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.b32 {%0,%1}, [%2], %3;"
      : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(policy_evict_first()));
  return v;
}
SL_DEV double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
      : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(policy_evict_first()));
  return v;
}
// Reused operands (x, B, C): keep in L2.
SL_DEV double ld_keep(const double* p) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(policy_evict_last()));
  return v;
}
// Output stores that are never re-read by this kernel.
SL_DEV void st_stream(double* p, double v) {
  asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" :: "l"(p), "d"(v) : "memory");
}

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

template <typename T>
SL_DEV T warp_bcast(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }

}  // namespace sl

namespace sl {
constexpr int kDiaMaxParam = 32;
struct DiaOffsets { int32_t v[kDiaMaxParam]; };   // DIA offsets passed by value (constant bank)
}  // namespace sl

// Host-side helpers shared by the .cu files.
namespace sl_host {
constexpr int kEllPipeMaxSlots = 32;   // ELL pipeline: slots per staged tile
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
int launch_ell_pipe(int64_t nrows, int32_t nslots, const int32_t* crd, const double* vals,
                    const double* x, double* y, cudaStream_t s);
int launch_dia_pipe(int64_t nrows, int64_t ncols, int32_t ndiag, const sl::DiaOffsets& offs,
                    const double* vals, const double* x, double* y, cudaStream_t s);
int launch_coo_pipe(int64_t nrows, int64_t nnz, const int32_t* rows, const int32_t* cols,
                    const double* vals, const double* x, double* y, cudaStream_t s);
int launch_csr_pipe(int64_t nrows, const int32_t* pos, const int32_t* crd, const double* vals,
                    const double* x, double* y, cudaStream_t s);
void launch_coo_rowptr(int64_t nrows, int64_t nnz, const int32_t* rows, int32_t* rowptr,
                       cudaStream_t s);       // add.cu: row pointer of a row-sorted COO
bool launch_coo_resident(int64_t nrows, int64_t nnz, const int32_t* rows, const int32_t* cols,
                         const double* vals, const double* x, double* y,
                         cudaStream_t s);    // coo_resident.cu: false when the matrix does not fit
int sm_count();                              // cached per current device
inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
int launch_status();                         // SL_OK or SL_ERR_CUDA after a launch
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Launch with programmatic dependent launch (PDL): the kernel may start while
// the previous kernel in the stream drains; it must execute
// sl::pdl_wait() before reading anything that kernel writes.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s,
                       size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
}  // namespace sl_host
