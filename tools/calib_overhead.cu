// calib_overhead.cu — event-bracket overhead of one launch under the bench's
// timing protocol, and variants (no flush; flush then idle; graph).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/_calib_overhead tools/calib_overhead.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <unistd.h>
#include <cuda_runtime.h>

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
__global__ void empty_k(uint32_t* sink, int v) { if (v == 12345) *sink = v; }
__global__ void small_k(uint32_t* sink, int v) { if (threadIdx.x == 999 + v) *sink = v; }

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  const size_t fl = 2 * (size_t)l2;
  uint4 *fw, *fr; uint32_t* sink;
  cudaMalloc(&fw, fl); cudaMalloc(&fr, fl); cudaMalloc(&sink, 4); cudaMemset(fr, 1, fl);
  cudaEvent_t e0, e1, e2; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  auto run = [&](const char* name, int mode) {
    double s = 0, s2 = 0; int n = 0;
    for (int rep = 0; rep < 43; ++rep) {
      if (mode == 1 || mode == 2 || mode == 4 || mode == 5) {
        flush_write<<<4 * sms, 512, 0, st>>>(fw, fl / 16, rep);
        flush_read<<<4 * sms, 512, 0, st>>>(fr, fl / 16, sink);
      }
      if (mode == 2) { cudaStreamSynchronize(st); usleep(200); }
      if (mode == 5) cudaEventRecord(e2, st);
      cudaEventRecord(e0, st);
      if (mode == 4) small_k<<<148 * 4, 256, 0, st>>>(sink, rep);
      else empty_k<<<1, 32, 0, st>>>(sink, rep);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep >= 3) { s += ms * 1000; ++n; }
      if (mode == 5) { cudaEventElapsedTime(&ms, e2, e0); if (rep >= 3) s2 += ms * 1000; }
    }
    printf("%-46s %7.2f us", name, s / n);
    if (mode == 5) printf("   (e2->e0 back to back: %.2f us)", s2 / n);
    printf("\n");
  };
  run("empty kernel, no flush", 0);
  run("empty kernel after write+read flush", 1);
  run("empty kernel after flush, sync + 200us idle", 2);
  run("592x256 no-op kernel after flush", 4);
  run("empty after flush, two events back to back", 5);
  // graph: flush, e0, empty, e1
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  flush_write<<<4 * sms, 512, 0, st>>>(fw, fl / 16, 7);
  flush_read<<<4 * sms, 512, 0, st>>>(fr, fl / 16, sink);
  cudaEventRecord(e0, st);
  empty_k<<<1, 32, 0, st>>>(sink, 1);
  cudaEventRecord(e1, st);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  double s = 0;
  for (int rep = 0; rep < 43; ++rep) {
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep >= 3) s += ms * 1000;
  }
  printf("%-46s %7.2f us\n", "graph [flush, e0, empty, e1]", s / 40);
  return 0;
}
