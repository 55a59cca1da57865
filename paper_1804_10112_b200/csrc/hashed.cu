// hashed.cu — hashed-level locate (warp-cooperative probing) and bulk insert.
//
// Reference: LevelStorage.locate for hashed levels (levels.py:270-280) and
// insert_init/insert_coord (levels.py:303-333).  Probe order is
// base + (coord + step) % W for step = 0..W-1; the first slot that holds the
// coordinate is the answer, the first empty slot (-1) or a full scan means
// "absent".  A tile of G lanes probes G consecutive steps per round and takes
// the lowest step that is a match-or-empty: exactly the sequential answer.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "levels.cuh"

namespace sl {

template <int G>
__global__ void __launch_bounds__(256)
hashed_locate_kernel(int64_t nq, const int32_t* __restrict__ parent_pos,
                     const int32_t* __restrict__ coord, HashedLevel lv,
                     int32_t* __restrict__ out_pos, uint8_t* __restrict__ out_found) {
  const int lane = threadIdx.x & 31;
  const int tile_lane = lane & (G - 1);
  const unsigned mask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  const int64_t tiles_per_grid = (int64_t)gridDim.x * (blockDim.x / G);
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; q < nq; q += tiles_per_grid) {
    const int64_t pp = parent_pos ? ldg(parent_pos + q) : 0;
    const int32_t c = ldg(coord + q);
    PosFound pf;
    if constexpr (G == 1) pf = lv.locate(pp, c);
    else pf = lv.template locate_coop<G>(pp, c, tile_lane, mask);
    if (tile_lane == 0) {
      out_pos[q] = (int32_t)pf.pos;
      out_found[q] = pf.found ? 1 : 0;
    }
  }
}

__global__ void hashed_fill_kernel(int32_t* __restrict__ crd, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    crd[i] = kEmpty;
}

// Concurrent linear-probing insert: atomicCAS(-1 -> c) on the first empty slot
// in probe order; a slot already holding c ends the probe (idempotence).
__global__ void hashed_insert_kernel(int64_t nq, const int32_t* __restrict__ parent_pos,
                                     const int32_t* __restrict__ coord, int64_t w,
                                     int32_t* __restrict__ crd, int32_t* __restrict__ err) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const int64_t base = (parent_pos ? (int64_t)parent_pos[q] : 0) * w;
  const int32_t c = coord[q];
  const int64_t home = c % w;
  for (int64_t step = 0; step < w; ++step) {
    int64_t s = home + step;
    if (s >= w) s -= w;
    int32_t* slot = crd + base + s;
    int32_t v = *reinterpret_cast<volatile int32_t*>(slot);
    if (v == c) return;
    if (v == kEmpty) {
      v = atomicCAS(slot, kEmpty, c);
      if (v == kEmpty || v == c) return;
    }
  }
  atomicExch(err, SL_ERR_HASH_SEGMENT_FULL);
}

}  // namespace sl

using namespace sl;

extern "C" int sl_hashed_locate(int64_t nq, const int32_t* parent_pos, const int32_t* coord,
                                int64_t w, const int32_t* crd, int32_t* out_pos,
                                uint8_t* out_found, int32_t group, void* stream) {
  if (nq < 0 || w <= 0) return SL_ERR_INVALID;
  if (w > INT32_MAX || nq > INT32_MAX) return SL_ERR_RANGE;
  if (nq == 0) return SL_OK;
  if (!coord || !crd || !out_pos || !out_found) return SL_ERR_INVALID;
  cudaStream_t s = sl_host::as_stream(stream);
  HashedLevel lv{crd, w};
  const int64_t threads = nq * (int64_t)group;
  const int grid = (int)std::min<int64_t>((threads + 255) / 256, 32LL * sl_host::sm_count());
  switch (group) {
    case 1: hashed_locate_kernel<1><<<grid, 256, 0, s>>>(nq, parent_pos, coord, lv, out_pos, out_found); break;
    case 4: hashed_locate_kernel<4><<<grid, 256, 0, s>>>(nq, parent_pos, coord, lv, out_pos, out_found); break;
    case 8: hashed_locate_kernel<8><<<grid, 256, 0, s>>>(nq, parent_pos, coord, lv, out_pos, out_found); break;
    case 16: hashed_locate_kernel<16><<<grid, 256, 0, s>>>(nq, parent_pos, coord, lv, out_pos, out_found); break;
    case 32: hashed_locate_kernel<32><<<grid, 256, 0, s>>>(nq, parent_pos, coord, lv, out_pos, out_found); break;
    default: return SL_ERR_INVALID;
  }
  return sl_host::launch_status();
}

extern "C" int sl_hashed_insert_init(int64_t size, int32_t* crd, void* stream) {
  if (size < 0) return SL_ERR_INVALID;
  if (size == 0) return SL_OK;
  if (!crd) return SL_ERR_INVALID;
  hashed_fill_kernel<<<std::min(sl_host::ceil_div(size, 256), 8 * sl_host::sm_count()), 256, 0,
                       sl_host::as_stream(stream)>>>(crd, size);
  return sl_host::launch_status();
}

extern "C" int sl_hashed_insert(int64_t nq, const int32_t* parent_pos, const int32_t* coord,
                                int64_t w, int32_t* crd, int32_t* err_flag, void* stream) {
  if (nq < 0 || w <= 0) return SL_ERR_INVALID;
  if (w > INT32_MAX || nq > INT32_MAX) return SL_ERR_RANGE;
  if (nq == 0) return SL_OK;
  if (!coord || !crd || !err_flag) return SL_ERR_INVALID;
  hashed_insert_kernel<<<sl_host::ceil_div(nq, 256), 256, 0, sl_host::as_stream(stream)>>>(
      nq, parent_pos, coord, w, crd, err_flag);
  return sl_host::launch_status();
}
