// calib_l2.cu — L2 -> SM throughput on this B200 for the access shapes the
// MTTKRP kernels use (tools only; built by tools/calib_l2.py with nvcc).
//   rows:  each warp reads random 256-byte rows (R = 32 doubles) of an
//          L2-resident table (the C / B factor-row gathers) and accumulates
//   seq:   each warp streams an L2-resident buffer with .cg loads
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void gather_rows_kernel(const double* __restrict__ table, const int32_t* __restrict__ idx,
                                   int64_t n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t i = w0 * 4; i < n; i += nw * 4) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t k = i + u < n ? __ldg(idx + i + u) : 0;
      v[u] = __ldcg(table + k * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u];
  }
  if (acc == 12345.678) out[0] = acc;   // keep the loads
}

__global__ void stream_cg_kernel(const double2* __restrict__ buf, int64_t n2, int reps,
                                 double* __restrict__ out) {
  double acc = 0.0;
  for (int r = 0; r < reps; ++r)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
         i += (int64_t)gridDim.x * blockDim.x) {
      const double2 v = __ldcg(buf + i);
      acc += v.x + v.y;
    }
  if (acc == 12345.678) out[0] = acc;
}

// random 8-byte gathers y += x[idx[i]] (SpMV's x operand), 8 per thread in flight
__global__ void gather8_kernel(const double* __restrict__ x, const int32_t* __restrict__ idx,
                               int64_t n, double* __restrict__ out) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 8 * stride) {
    int32_t k[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) k[u] = i0 + u * stride < n ? __ldg(idx + i0 + u * stride) : 0;
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(x + k[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void empty_kernel() {}

extern "C" int calib_empty(int blocks, void* stream) {
  empty_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>();
  return (int)cudaGetLastError();
}

extern "C" int calib_gather8(const double* x, const int32_t* idx, int64_t n, double* out,
                             int blocks, void* stream) {
  gather8_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(x, idx, n, out);
  return (int)cudaGetLastError();
}

extern "C" int calib_gather_rows(const double* table, const int32_t* idx, int64_t n, double* out,
                                 int blocks, void* stream) {
  gather_rows_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(table, idx, n, out);
  return (int)cudaGetLastError();
}

extern "C" int calib_stream_cg(const double* buf, int64_t n_doubles, int reps, double* out,
                               int blocks, void* stream) {
  stream_cg_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const double2*>(buf), n_doubles / 2, reps, out);
  return (int)cudaGetLastError();
}
