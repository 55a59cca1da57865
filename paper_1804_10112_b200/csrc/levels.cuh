// levels.cuh — device-side level functions with the reference's semantics.
//
// Each struct is one level kind of reference pkg/src/sparselevels/levels.py,
// with its capability set expressed as static traits (levels.py:35-41) and
// its access functions as inlined device code — the paper's "inline level
// functions".  Kernels compose these; the batched
// sl_level_query entry point (abi.cu) replays the reference's level-function
// unit tests (pkg/tests/test_levels.py) through them.
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace sl {

constexpr int32_t kEmpty = -1;  // levels.py:43 EMPTY

struct Bounds { int64_t lo, hi; };
struct PosFound { int64_t pos; bool found; };
struct CoordFound { int64_t coord; bool found; };

// Dense: value iteration, locate, insert (levels.py:218-219, 229-230, 268-269, 289-290).
struct DenseLevel {
  static constexpr bool kValueIter = true, kPosIter = false, kLocate = true, kInsert = true,
                        kAppend = false;
  int64_t n;
  SL_DEV Bounds coord_bounds(int64_t /*prefix_last*/) const { return {0, n}; }
  SL_DEV PosFound coord_access(int64_t parent_pos, int64_t c) const { return {parent_pos * n + c, true}; }
  SL_DEV PosFound locate(int64_t parent_pos, int64_t c) const { return {parent_pos * n + c, true}; }
  SL_DEV int64_t size(int64_t parent_size) const { return parent_size * n; }
};

// Range: value iteration only (levels.py:220-222, 229-230).
struct RangeLevel {
  static constexpr bool kValueIter = true, kPosIter = false, kLocate = false, kInsert = false,
                        kAppend = false;
  int64_t n, m;
  const int32_t* offset;
  SL_DEV Bounds coord_bounds(int64_t prefix_last) const {
    const int64_t off = offset[prefix_last];
    const int64_t lo = off < 0 ? -off : 0;
    const int64_t hi = n < m - off ? n : m - off;
    return {lo, hi};
  }
  SL_DEV PosFound coord_access(int64_t parent_pos, int64_t c) const { return {parent_pos * n + c, true}; }
};

// Compressed: position iteration, append (levels.py:239-240, 251-252, 201-202).
struct CompressedLevel {
  static constexpr bool kValueIter = false, kPosIter = true, kLocate = false, kInsert = false,
                        kAppend = true;
  const int32_t* pos;
  const int32_t* crd;
  int32_t crd_stride, crd_base;
  SL_DEV Bounds pos_bounds(int64_t parent_pos) const { return {pos[parent_pos], pos[parent_pos + 1]}; }
  SL_DEV CoordFound pos_access(int64_t p, int64_t /*prefix_last*/) const {
    return {crd[p * crd_stride + crd_base], true};
  }
};

// Singleton: branchless position iteration, append (levels.py:241-242, 251-252).
struct SingletonLevel {
  static constexpr bool kValueIter = false, kPosIter = true, kLocate = false, kInsert = false,
                        kAppend = true;
  const int32_t* crd;
  int32_t crd_stride, crd_base;
  SL_DEV Bounds pos_bounds(int64_t parent_pos) const { return {parent_pos, parent_pos + 1}; }
  SL_DEV CoordFound pos_access(int64_t p, int64_t /*prefix_last*/) const {
    return {crd[p * crd_stride + crd_base], true};
  }
};

// Offset: branchless position iteration; the governing diagonal is recovered
// from the position, d = p / range_n (levels.py:241-242, 253-256).
struct OffsetLevel {
  static constexpr bool kValueIter = false, kPosIter = true, kLocate = false, kInsert = false,
                        kAppend = false;
  const int32_t* offset;
  int64_t range_n;
  SL_DEV Bounds pos_bounds(int64_t parent_pos) const { return {parent_pos, parent_pos + 1}; }
  SL_DEV CoordFound pos_access(int64_t p, int64_t prefix_last) const {
    return {prefix_last + offset[p / range_n], true};
  }
};

// Hashed: position iteration (found = crd != -1), locate by linear probing,
// insert (levels.py:243-244, 257-259, 270-280, 291-292, 320-332).
struct HashedLevel {
  static constexpr bool kValueIter = false, kPosIter = true, kLocate = true, kInsert = true,
                        kAppend = false;
  const int32_t* crd;
  int64_t w;
  SL_DEV Bounds pos_bounds(int64_t parent_pos) const { return {parent_pos * w, (parent_pos + 1) * w}; }
  SL_DEV CoordFound pos_access(int64_t p, int64_t /*prefix_last*/) const {
    const int32_t c = crd[p];
    return {c, c != kEmpty};
  }
  // Scalar probe: identical step order to levels.py:273-280.
  SL_DEV PosFound locate(int64_t parent_pos, int64_t c) const {
    const int64_t base = parent_pos * w;
    const int64_t home = c % w;
    for (int64_t step = 0; step < w; ++step) {
      int64_t s = home + step;
      if (s >= w) s -= w;
      const int64_t p = base + s;
      const int32_t v = ldg(crd + p);
      if (v == c) return {p, true};
      if (v == kEmpty) return {-1, false};
    }
    return {-1, false};
  }
  // Cooperative probe by a tile of G lanes (G divides 32; lanes of the tile
  // are `lane0 .. lane0+G-1` of the calling warp, `mask` their membership).
  // Round r probes steps [r*G, r*G+G); the answer is the lowest step that holds
  // the coordinate or an empty slot — the first hit of the sequential probe.
  template <int G>
  SL_DEV PosFound locate_coop(int64_t parent_pos, int64_t c, int tile_lane, unsigned mask) const {
    const int64_t base = parent_pos * w;
    const int64_t home = c % w;
    for (int64_t step0 = 0; step0 < w; step0 += G) {
      const int64_t step = step0 + tile_lane;
      int32_t v = 0;  // lanes past the segment width see "neither"
      int64_t p = -1;
      if (step < w) {
        int64_t s = home + step;
        if (s >= w) s -= w;
        p = base + s;
        v = ldg(crd + p);
      }
      const bool hit = step < w && v == c;
      const bool stop = step < w && (v == c || v == kEmpty);
      const unsigned ballot = __ballot_sync(mask, stop);
      const unsigned tile_bits = G == 32 ? ballot : (ballot >> (threadIdx.x & 31 & ~(G - 1))) & ((1u << G) - 1u);
      if (tile_bits) {
        const int first = __ffs(tile_bits) - 1;
        const int src = (threadIdx.x & 31 & ~(G - 1)) + first;
        const int64_t pf = __shfl_sync(mask, p, src, 32);
        const bool hf = __shfl_sync(mask, hit ? 1 : 0, src, 32) != 0;
        return hf ? PosFound{pf, true} : PosFound{-1, false};
      }
    }
    return {-1, false};
  }
  SL_DEV int64_t size(int64_t parent_size) const { return parent_size * w; }
};

}  // namespace sl
