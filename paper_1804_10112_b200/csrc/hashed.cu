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

#include <algorithm>

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

// ---- ordered bulk insert: the table the sequential insert_coord calls build --
// insert_coord in query order q = 0, 1, ... (levels.py:312-333) places each new
// coordinate at the first slot from its home that is empty at that moment;
// the result depends on the order whenever probe sequences collide.  The
// bulk insert reproduces it exactly with priorities: a slot holds
// (order << 32 | coord) and keys race by atomicMin, so a slot can only ever be
// taken over by a higher-priority (earlier) key; the loser (or the displaced
// key) continues probing from the next slot.  Every key visits the slots from
// its home to its final slot, each of which ends up held by an earlier key,
// so its final slot is the first one from its home not taken by earlier keys
// — the sequential answer, by induction over the order.  Entries already in
// the table keep their slots (priority 0), and repeated coordinates are
// reduced to their first occurrence beforehand (a later copy could otherwise
// pass the slot the first copy only takes afterwards).
constexpr unsigned long long kPackEmpty = ~0ull;

SL_DEV unsigned long long dedup_key(int64_t pp, int32_t c) {
  return ((unsigned long long)pp << 32) | (uint32_t)c;
}
SL_DEV uint64_t dedup_home(unsigned long long key, int lg) {
  return (uint64_t)((key * 0x9E3779B97F4A7C15ull) >> (64 - lg));
}

__global__ void ordered_seed_kernel(int64_t size, const int32_t* __restrict__ crd,
                                    unsigned long long* __restrict__ P, int64_t m,
                                    unsigned long long* __restrict__ dkey,
                                    uint32_t* __restrict__ dord) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < size; i += stride) {
    const int32_t v = crd[i];
    P[i] = v == kEmpty ? kPackEmpty : (unsigned long long)(uint32_t)v;   // order 0
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    dkey[i] = kPackEmpty;
    dord[i] = 0xffffffffu;
  }
}

// first occurrence of every (segment, coordinate): min query index per key
__global__ void ordered_dedup_kernel(int64_t nq, const int32_t* __restrict__ parent_pos,
                                     const int32_t* __restrict__ coord, int lg,
                                     unsigned long long* __restrict__ dkey,
                                     uint32_t* __restrict__ dord) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const unsigned long long key = dedup_key(parent_pos ? parent_pos[q] : 0, coord[q]);
  const uint64_t mask = (1ull << lg) - 1;
  for (uint64_t h = dedup_home(key, lg);; h = (h + 1) & mask) {
    const unsigned long long old = atomicCAS(dkey + h, kPackEmpty, key);
    if (old == kPackEmpty || old == key) {
      atomicMin(dord + h, (uint32_t)q);
      return;
    }
  }
}

__global__ void ordered_insert_kernel(int64_t nq, const int32_t* __restrict__ parent_pos,
                                      const int32_t* __restrict__ coord, int64_t w, int lg,
                                      const unsigned long long* __restrict__ dkey,
                                      const uint32_t* __restrict__ dord,
                                      unsigned long long* __restrict__ P,
                                      int32_t* __restrict__ err) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const int64_t pp = parent_pos ? parent_pos[q] : 0;
  const int32_t c0 = coord[q];
  {  // only the first occurrence of a repeated coordinate inserts
    const unsigned long long key = dedup_key(pp, c0);
    const uint64_t mask = (1ull << lg) - 1;
    uint64_t h = dedup_home(key, lg);
    while (dkey[h] != key) h = (h + 1) & mask;
    if (dord[h] != (uint32_t)q) return;
  }
  unsigned long long* seg = P + pp * w;
  unsigned long long mine = ((unsigned long long)(q + 1) << 32) | (uint32_t)c0;
  int64_t s = (int64_t)(c0 % w);
  int64_t d = 0;                                  // probe distance of the key being placed
  for (;;) {
    const unsigned long long old = atomicMin(seg + s, mine);
    if (old == kPackEmpty) return;                // placed
    if ((uint32_t)old == (uint32_t)mine) return;  // already present (an earlier entry)
    if (old > mine) {                             // displaced a later key: it moves on
      mine = old;
      const int64_t home = (int64_t)((int32_t)(uint32_t)old % w);
      d = s >= home ? s - home : s + w - home;
    }
    s = s + 1 == w ? 0 : s + 1;
    if (++d >= w) {                               // probed the whole segment
      atomicExch(err, SL_ERR_HASH_SEGMENT_FULL);
      return;
    }
  }
}

__global__ void ordered_unpack_kernel(int64_t size, const unsigned long long* __restrict__ P,
                                      int32_t* __restrict__ crd) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < size; i += stride)
    crd[i] = P[i] == kPackEmpty ? kEmpty : (int32_t)(uint32_t)P[i];
}

static int ordered_lg(int64_t nq) {
  int lg = 6;
  while ((1ll << lg) < 2 * nq) ++lg;
  return lg;
}

}  // namespace sl

extern "C" size_t sl_hashed_insert_ordered_workspace_bytes(int64_t nq, int64_t size) {
  const int64_t m = 1ll << sl::ordered_lg(nq);
  return (size_t)size * 8 + (size_t)m * 12 + 256;
}

extern "C" int sl_hashed_insert_ordered(int64_t nq, const int32_t* parent_pos,
                                        const int32_t* coord, int64_t w, int64_t size,
                                        int32_t* crd, int32_t* err_flag, void* ws,
                                        size_t ws_bytes, void* stream) {
  using namespace sl;
  if (nq < 0 || w <= 0 || size < 0 || size % w != 0) return SL_ERR_INVALID;
  if (w > INT32_MAX || nq >= INT32_MAX) return SL_ERR_RANGE;
  if (nq == 0) return SL_OK;
  if (!coord || !crd || !err_flag) return SL_ERR_INVALID;
  if (!ws || ws_bytes < sl_hashed_insert_ordered_workspace_bytes(nq, size)) return SL_ERR_WORKSPACE;
  cudaStream_t s = sl_host::as_stream(stream);
  const int lg = ordered_lg(nq);
  const int64_t m = 1ll << lg;
  char* p = static_cast<char*>(ws);
  auto* P = reinterpret_cast<unsigned long long*>(p);
  auto* dkey = reinterpret_cast<unsigned long long*>(p + (size_t)size * 8);
  auto* dord = reinterpret_cast<uint32_t*>(p + (size_t)size * 8 + (size_t)m * 8);
  const int grid = (int)std::min<int64_t>(sl_host::ceil_div(std::max(size, m), 256),
                                          8 * sl_host::sm_count());
  ordered_seed_kernel<<<grid, 256, 0, s>>>(size, crd, P, m, dkey, dord);
  ordered_dedup_kernel<<<sl_host::ceil_div(nq, 256), 256, 0, s>>>(nq, parent_pos, coord, lg, dkey,
                                                                  dord);
  ordered_insert_kernel<<<sl_host::ceil_div(nq, 256), 256, 0, s>>>(nq, parent_pos, coord, w, lg,
                                                                   dkey, dord, P, err_flag);
  ordered_unpack_kernel<<<grid, 256, 0, s>>>(size, P, crd);
  return sl_host::launch_status();
}

namespace sl {

// ---- slot map: the answer of locate(c) for every coordinate c < n ------------
// For a query stream much longer than the table (CSR x hash-vector: one
// locate per nonzero, ~10 per stored coordinate), resolving each coordinate
// once is cheaper than probing per query.  locate(c) returns the first slot s
// in probe order home(c), home(c)+1, ... holding c, provided no empty slot
// comes before it; with d = (s - home(c)) mod W and L(s) = the number of
// occupied slots immediately preceding s (cyclically), s is reachable iff
// d <= L(s), and the answer is the reachable slot of c with the smallest d.
// That is exact for any table contents (not only tables built by insert).
// Map entries pack (d << 32 | s); ~0 = absent.
constexpr int kMapChunk = 1024;

// per chunk: last empty slot at or before each slot (within the chunk, -1 if
// none) and the chunk's last empty slot
__global__ void __launch_bounds__(kMapChunk)
hash_runs_kernel(int64_t w, const int32_t* __restrict__ crd, int32_t* __restrict__ last_empty,
                 int32_t* __restrict__ chunk_last, unsigned long long* __restrict__ map,
                 int64_t n) {
  __shared__ int32_t s_warp[kMapChunk / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the map starts absent (~0) — done here rather than in a launch of its own
  for (int64_t i = (int64_t)blockIdx.x * kMapChunk + tid; i < n; i += (int64_t)gridDim.x * kMapChunk)
    map[i] = ~0ull;
  const int64_t s = (int64_t)blockIdx.x * kMapChunk + tid;
  int32_t v = (s < w && ldg(crd + s) == kEmpty) ? (int32_t)s : -1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = max(v, u);
  }
  if (lane == 31) s_warp[warp] = v;
  __syncthreads();
  int32_t before = -1;
  for (int i = 0; i < warp; ++i) before = max(before, s_warp[i]);
  v = max(v, before);
  if (s < w) last_empty[s] = v;
  if (tid == kMapChunk - 1) chunk_last[blockIdx.x] = v;
}

// exclusive prefix max of the chunk maxima (one block); chunk_pre[nchunks] = overall last empty
__global__ void __launch_bounds__(1024)
hash_chunk_scan_kernel(int64_t nchunks, const int32_t* __restrict__ chunk_last,
                       int32_t* __restrict__ chunk_pre) {
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = -1;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nchunks; b0 += 1024) {
    const int64_t b = b0 + tid;
    int32_t incl = b < nchunks ? chunk_last[b] : -1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = max(incl, u);
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int32_t before = s_carry;
    for (int i = 0; i < warp; ++i) before = max(before, s_warp[i]);
    const int32_t up = __shfl_up_sync(0xffffffffu, incl, 1);
    const int32_t excl = max(before, lane == 0 ? -1 : up);
    if (b < nchunks) chunk_pre[b] = excl;
    __syncthreads();
    if (tid == 1023) s_carry = max(before, incl);
    __syncthreads();
  }
  if (tid == 0) chunk_pre[nchunks] = s_carry;
}


__global__ void map_fill_kernel(int64_t w, int64_t n, const int32_t* __restrict__ crd,
                                const int32_t* __restrict__ last_empty,
                                const int32_t* __restrict__ chunk_pre,
                                unsigned long long* __restrict__ map, int64_t nchunks) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < w;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = ldg(crd + s);
    if (c < 0 || c >= n) continue;
    const int64_t b = s / kMapChunk;
    int64_t pe = ldg(chunk_pre + b);                                  // last empty before chunk b
    if (s > b * kMapChunk) pe = max64(pe, (int64_t)ldg(last_empty + s - 1));
    int64_t run;                                                      // occupied slots before s
    if (pe >= 0) {
      run = s - 1 - pe;
    } else {
      const int64_t g = ldg(chunk_pre + nchunks);                     // last empty overall
      run = g >= 0 ? s - 1 - (g - w) : w - 1;                         // wrap, or no empty slot
    }
    int64_t d = s - (int64_t)c % w;
    if (d < 0) d += w;
    if (d <= run)
      atomicMin(map + c, ((unsigned long long)d << 32) | (unsigned long long)(uint32_t)s);
  }
}

}  // namespace sl

using namespace sl;

extern "C" size_t sl_hashed_slot_map_workspace_bytes(int64_t n, int64_t w) {
  const int64_t nchunks = (w + kMapChunk - 1) / kMapChunk;
  return (size_t)n * 8 + (size_t)w * 4 + (size_t)(2 * nchunks + 1) * 4 + 512;
}

// Workspace layout: [map u64 x n][last_empty i32 x w][chunk_last x nchunks][chunk_pre x nchunks+1]
extern "C" int sl_hashed_slot_map(int64_t n, int64_t w, const int32_t* crd, void* ws,
                                  size_t ws_bytes, void* stream) {
  if (n < 0 || w <= 0 || !crd) return SL_ERR_INVALID;
  if (w > INT32_MAX || n > INT32_MAX) return SL_ERR_RANGE;
  if (!ws || ws_bytes < sl_hashed_slot_map_workspace_bytes(n, w)) return SL_ERR_WORKSPACE;
  cudaStream_t s = sl_host::as_stream(stream);
  const int64_t nchunks = (w + kMapChunk - 1) / kMapChunk;
  char* p = static_cast<char*>(ws);
  unsigned long long* map = reinterpret_cast<unsigned long long*>(p);
  int32_t* last_empty = reinterpret_cast<int32_t*>(p + (size_t)n * 8);
  int32_t* chunk_last = last_empty + w;
  int32_t* chunk_pre = chunk_last + nchunks;
  const int sms = sl_host::sm_count();
  hash_runs_kernel<<<(int)nchunks, kMapChunk, 0, s>>>(w, crd, last_empty, chunk_last, map, n);
  hash_chunk_scan_kernel<<<1, 1024, 0, s>>>(nchunks, chunk_last, chunk_pre);
  map_fill_kernel<<<min(sl_host::ceil_div(w, 256), 8 * sms), 256, 0, s>>>(
      w, n, crd, last_empty, chunk_pre, map, nchunks);
  return sl_host::launch_status();
}

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
