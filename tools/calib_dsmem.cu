// calib_dsmem.cu — random 256-byte row gathers from a table distributed over
// a thread-block cluster's shared memory (DSMEM), against the same gathers
// from an L2-resident global table, and both at once: the ceiling an MTTKRP
// holding C (10,000 x 32 fp64 = 2.56 MB) in a 16-CTA cluster would face.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/_calib_dsmem tools/calib_dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int kRowDoubles = 32;            // 256-byte rows, like an R = 32 factor row
constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// mode 0: all rows from DSMEM; 1: all from global (L2); 2: alternate
template <int kMode>
__global__ void __launch_bounds__(kThreads, 1)
gather_kernel(const double* __restrict__ gtab, int rows_per_cta, int total_rows, int iters,
              double* __restrict__ sink) {
  extern __shared__ double stab[];
  cg::cluster_group cl = cg::this_cluster();
  const int nblk = cl.num_blocks();
  const int me = cl.block_rank();
  // fill this CTA's slice from the global copy (rows [me * rpc, (me + 1) * rpc))
  for (int q = threadIdx.x; q < rows_per_cta * kRowDoubles; q += kThreads)
    stab[q] = gtab[(size_t)me * rows_per_cta * kRowDoubles + q];
  cl.sync();
  const int lane = threadIdx.x & 31, sub = lane >> 3, q = lane & 7;   // 8 lanes x 32 B per row
  const uint32_t warp_g = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t h = hash32(warp_g * 7919u + it * 4u + sub);
    const int row = (int)(h % (uint32_t)total_rows);
    const bool use_dsmem = kMode == 0 || (kMode == 2 && (it & 1));
    if (use_dsmem) {
      const int owner = row / rows_per_cta, off = row % rows_per_cta;
      const double* remote = cl.map_shared_rank(stab, owner % nblk);
      const double4 v = *reinterpret_cast<const double4*>(remote + (size_t)off * kRowDoubles + 4 * q);
      acc0 += v.x; acc1 += v.y; acc2 += v.z; acc3 += v.w;
    } else {
      const double* p = gtab + (size_t)row * kRowDoubles + 4 * q;
      double4 v;
      asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
      acc0 += v.x; acc1 += v.y; acc2 += v.z; acc3 += v.w;
    }
  }
  cl.sync();
  if (acc0 + acc1 + acc2 + acc3 == 1234.5) sink[0] = acc0;
}

template <int kMode>
float run(const double* gtab, double* sink, int cluster, int rows_per_cta, int iters, int sms,
          size_t smem) {
  auto k = gather_kernel<kMode>;
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nclusters = sms / cluster;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclusters * cluster);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  const int total = rows_per_cta * cluster;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k, gtab, rows_per_cta, total, iters / 8, sink);   // warm
  cudaEventRecord(e0);
  cudaError_t err = cudaLaunchKernelEx(&cfg, k, gtab, rows_per_cta, total, iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    printf("launch failed (cluster %d): %s\n", cluster, cudaGetErrorString(err));
    return -1;
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  // rows gathered: per warp 4 rows per iteration
  const double rows = (double)nclusters * cluster * (kThreads / 32) * 4.0 * iters;
  const double gbs = rows * 256.0 / (ms * 1e-3) / 1e9;
  printf("mode %-7s cluster %2d (%3d CTAs): %8.3f ms  %8.1f GB/s of 256-B rows (%.0f B/clk/SM at 1.9 GHz)\n",
         kMode == 0 ? "dsmem" : kMode == 1 ? "global" : "both", cluster, nclusters * cluster, ms, gbs,
         gbs * 1e9 / (nclusters * cluster) / 1.9e9);
  return ms;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int rows_total = 10000;
  double *gtab, *sink;
  cudaMalloc(&gtab, (size_t)rows_total * 256 + 16 * 256 * 1024);
  cudaMalloc(&sink, 8);
  cudaMemset(gtab, 0, (size_t)rows_total * 256);
  const int iters = 4096;
  for (int cluster : {16, 8}) {
    // cluster 16 holds the whole 10,000-row table; cluster 8 the largest that fits
    const int rpc = (rows_total + cluster - 1) / cluster > 880 ? 880 : (rows_total + cluster - 1) / cluster;
    const size_t smem = (size_t)rpc * 256;
    run<0>(gtab, sink, cluster, rpc, iters, sms, smem);
    run<1>(gtab, sink, cluster, rpc, iters, sms, smem);
    run<2>(gtab, sink, cluster, rpc, iters, sms, smem);
  }
  return 0;
}
