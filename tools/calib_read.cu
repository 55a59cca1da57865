// calib_read.cu — what a cold streaming READ of N bytes costs on this B200,
// timed exactly as bench.py times a kernel: 2x-L2 write sweep, 2x-L2 read
// sweep, then CUDA events around the one launch.  The floor an HBM-bound
// read-mostly kernel (CSR / ELL / DIA SpMV) can reach at its working-set size.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/_calib_read tools/calib_read.cu
//   tools/_calib_read            # one line per (size, variant)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void flush_write(uint4* b, size_t n, uint32_t s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = make_uint4((uint32_t)i ^ s, s, 1, 2);
}
__global__ void flush_read(const uint4* b, size_t n, uint32_t* sink) {
  uint32_t a = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcg(b + i); a ^= v.x ^ v.w;
  }
  if (a == 0x12345u) *sink = a;
}

// grid-stride, U independent 16-B loads per thread per iteration
template <int U>
__global__ void rd_stride(const uint4* __restrict__ b, size_t n, uint32_t* sink) {
  uint32_t a = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(b + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) a ^= v[u].x ^ v[u].w;
  }
  for (; i < n; i += stride) { uint4 v = __ldg(b + i); a ^= v.x ^ v.w; }
  if (a == 0x12345u) *sink = a;
}

// one block per chunk (non-persistent), each thread U consecutive-strided loads
template <int U>
__global__ void rd_chunk(const uint4* __restrict__ b, size_t n, uint32_t* sink) {
  uint32_t a = 0;
  const size_t base = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x;
  uint4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { size_t i = base + (size_t)u * blockDim.x; v[u] = i < n ? __ldg(b + i) : make_uint4(0,0,0,0); }
#pragma unroll
  for (int u = 0; u < U; ++u) a ^= v[u].x ^ v[u].w;
  if (a == 0x12345u) *sink = a;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int l2; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  const size_t fl = 2 * (size_t)l2;
  uint4 *fw, *fr, *buf; uint32_t* sink;
  CK(cudaMalloc(&fw, fl)); CK(cudaMalloc(&fr, fl)); CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(fr, 1, fl));
  const size_t maxb = 300u << 20;
  CK(cudaMalloc(&buf, maxb)); CK(cudaMemset(buf, 3, maxb));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const size_t sizes[] = {35200000, 87550884, 150730764, 262406292};
  struct V { const char* name; int kind; };
  for (size_t bytes : sizes) {
    const size_t n = bytes / 16;
    for (int var = 0; var < 9; ++var) {
      std::vector<float> ts;
      const char* nm = "";
      for (int rep = 0; rep < 23; ++rep) {
        flush_write<<<4 * sms, 512>>>(fw, fl / 16, rep);
        flush_read<<<4 * sms, 512>>>(fr, fl / 16, sink);
        cudaEventRecord(e0);
        switch (var) {
          case 0: nm = "stride U1 4x148x512"; rd_stride<1><<<4 * sms, 512>>>(buf, n, sink); break;
          case 1: nm = "stride U4 2x148x512"; rd_stride<4><<<2 * sms, 512>>>(buf, n, sink); break;
          case 2: nm = "stride U4 4x148x256"; rd_stride<4><<<4 * sms, 256>>>(buf, n, sink); break;
          case 3: nm = "stride U8 2x148x256"; rd_stride<8><<<2 * sms, 256>>>(buf, n, sink); break;
          case 4: nm = "stride U8 1x148x1024"; rd_stride<8><<<sms, 1024>>>(buf, n, sink); break;
          case 5: nm = "stride U4 8x148x256"; rd_stride<4><<<8 * sms, 256>>>(buf, n, sink); break;
          case 6: nm = "chunk U4 x256"; rd_chunk<4><<<(unsigned)((n + 1023) / 1024), 256>>>(buf, n, sink); break;
          case 7: nm = "chunk U8 x256"; rd_chunk<8><<<(unsigned)((n + 2047) / 2048), 256>>>(buf, n, sink); break;
          case 8: nm = "chunk U2 x512"; rd_chunk<2><<<(unsigned)((n + 1023) / 1024), 512>>>(buf, n, sink); break;
        }
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep >= 3) ts.push_back(ms * 1000.f);
      }
      double s = 0; for (float t : ts) s += t;
      const double mean = s / ts.size();
      std::sort(ts.begin(), ts.end());
      printf("%6.1f MB  %-22s mean %7.2f us  min %7.2f  -> %6.0f GB/s (%.1f%% of 6554)\n",
             bytes / 1e6, nm, mean, ts[0], bytes / mean / 1e3, 100.0 * bytes / mean / 1e3 / 6554.6);
    }
  }
  // empty-kernel event overhead
  std::vector<float> ts;
  for (int rep = 0; rep < 23; ++rep) {
    flush_write<<<4 * sms, 512>>>(fw, fl / 16, rep);
    flush_read<<<4 * sms, 512>>>(fr, fl / 16, sink);
    cudaEventRecord(e0);
    rd_chunk<1><<<1, 32>>>(buf, 0, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep >= 3) ts.push_back(ms * 1000.f);
  }
  double s = 0; for (float t : ts) s += t;
  printf("empty kernel after the flush: mean %.2f us\n", s / ts.size());
  return 0;
}
