// tma.cuh — 1D bulk async copies (cp.async.bulk, the TMA's linear mode) and
// mbarrier helpers for sm_100a.  The streaming kernels move their index and
// value arrays global -> shared with these: one elected thread issues a few
// large copies, the copy engine keeps them in flight (no registers held), and
// the consumer threads wait on an mbarrier's transaction count.
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace sl {

SL_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// shared-space loads/stores by 32-bit shared address (no generic->shared
// conversion per access)
SL_DEV int32_t lds32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
SL_DEV void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

SL_DEV void sts64(uint32_t a, uint32_t v0, uint32_t v1) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(a), "r"(v0), "r"(v1) : "memory");
}

SL_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

// Make mbarrier.init visible to the async (TMA) proxy.
SL_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Order this thread's generic-proxy shared-memory accesses before later
// async-proxy (bulk copy) writes into the same buffer.
SL_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

SL_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

SL_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

SL_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Named barrier over `nthreads` threads (a consumer warp-group), id >= 1.
// Bulk prefetch of [p, p + n) elements into L2 (cp.async.bulk.prefetch.L2,
// one instruction; the range is widened to whole 16-byte granules, which
// stay inside the allocation's 16-byte-aligned extent)
template <typename T>
SL_DEV void prefetch_l2(const T* p, int64_t n) {
  if (n <= 0) return;
  const uintptr_t lo = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t hi = (reinterpret_cast<uintptr_t>(p + n) + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(hi - lo))
               : "memory");
}

SL_DEV void group_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Bulk copy `bytes` (multiple of 16, both addresses 16-byte aligned) from
// global to shared; completion is signalled on `bar` as transaction bytes.
// Tagged L2 evict-first: streamed operands are read once.
SL_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy_evict_first())
      : "memory");
}

// Same, default L2 policy (for reused operands such as x windows).
SL_DEV void bulk_g2s_keep(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Copy the element range [lo, hi) of a global array into smem so that element
// e lands at smem_base[e - lo0], where lo0 = lo rounded down to 16 bytes.
// Bulk copies cover the 16-byte-aligned interior; the (< 16-byte) head and
// tail are loaded by `lane` threads with plain loads (the caller syncs).
// Returns the bulk transaction bytes issued (0 if the range is tiny).
// `elected` must be true for exactly one thread.
template <typename T>
struct BulkRange {
  int64_t lo0;        // first element staged at smem index 0
  uint32_t tx_bytes;  // bytes the mbarrier must expect
  int64_t blo, bhi;   // bulk-copied element range
};

template <typename T>
SL_DEV BulkRange<T> plan_range(const T* g, int64_t lo, int64_t hi) {
  constexpr int64_t per16 = 16 / sizeof(T);
  const uintptr_t base = reinterpret_cast<uintptr_t>(g);
  // element index whose address is 16-byte aligned at or after lo / before hi
  const int64_t mis = (int64_t)((base / sizeof(T)) % per16);   // base misalignment in elements
  auto align_up = [&](int64_t e) { return ((e + mis + per16 - 1) / per16) * per16 - mis; };
  auto align_dn = [&](int64_t e) { return ((e + mis) / per16) * per16 - mis; };
  BulkRange<T> r;
  r.lo0 = align_dn(lo);
  r.blo = align_up(lo);
  r.bhi = align_dn(hi);
  if (r.bhi < r.blo) r.bhi = r.blo;
  r.tx_bytes = (uint32_t)((r.bhi - r.blo) * sizeof(T));
  return r;
}

template <typename T>
SL_DEV void issue_range(const T* g, const BulkRange<T>& r, T* s, uint64_t* bar) {
  if (r.tx_bytes) bulk_g2s(s + (r.blo - r.lo0), g + r.blo, r.tx_bytes, bar);
}

// plain loads of the unaligned head [lo, blo) and tail [bhi, hi)
template <typename T>
SL_DEV void edge_loads(const T* g, const BulkRange<T>& r, int64_t lo, int64_t hi, T* s, int tid,
                       int nthreads) {
  const int64_t nh = r.blo - lo < hi - lo ? r.blo - lo : hi - lo;
  for (int64_t e = tid; e < nh; e += nthreads) s[lo + e - r.lo0] = g[lo + e];
  const int64_t t0 = r.bhi > lo ? r.bhi : lo;
  for (int64_t e = t0 + tid; e < hi; e += nthreads)
    if (e >= r.blo) s[e - r.lo0] = g[e];
}

// Constant-time version for callers whose ranges are known to be short at the
// ends: the unaligned head and tail each hold fewer than 16/sizeof(T)
// elements, loaded by threads [0, head) and [64, 64 + tail) (blockDim >= 96).
template <typename T>
SL_DEV void edge_loads_small(const T* g, const BulkRange<T>& r, int64_t lo, int64_t hi, T* s,
                             int tid) {
  const int nh = (int)(min64(r.blo, hi) - lo);
  if (tid < nh) s[lo + tid - r.lo0] = g[lo + tid];
  const int64_t t0 = max64(r.bhi, lo) > min64(r.blo, hi) ? max64(r.bhi, lo) : min64(r.blo, hi);
  const int nt = (int)(hi - t0);
  const int k = tid - 64;
  if (k >= 0 && k < nt) s[t0 + k - r.lo0] = g[t0 + k];
}

// 32-bit versions for element ranges below 2^31 (the A+B tiles): the same
// placement, with shifts and masks instead of 64-bit divisions (the staging
// arithmetic was ~8% of the A+B count pass's instructions).
struct BulkRange32 {
  int32_t lo0, blo, bhi;
  uint32_t tx_bytes;
};

template <typename T>
SL_DEV BulkRange32 plan_range32(const T* g, int32_t lo, int32_t hi) {
  constexpr int32_t per16 = 16 / sizeof(T);
  const int32_t mis = (int32_t)((reinterpret_cast<uintptr_t>(g) / sizeof(T)) & (per16 - 1));
  BulkRange32 r;
  r.lo0 = ((lo + mis) & ~(per16 - 1)) - mis;
  r.blo = ((lo + mis + per16 - 1) & ~(per16 - 1)) - mis;
  r.bhi = ((hi + mis) & ~(per16 - 1)) - mis;
  if (r.bhi < r.blo) r.bhi = r.blo;
  r.tx_bytes = (uint32_t)(r.bhi - r.blo) * (uint32_t)sizeof(T);
  return r;
}

// Whole 16-byte granules covering [lo, hi): no plain edge loads at all.  The
// granules at the ends hold elements outside the range (garbage in the
// stage, never read); each granule holds at least one element of the range,
// so no read leaves the array's pages.
template <typename T>
SL_DEV BulkRange32 plan_granules32(const T* g, int32_t lo, int32_t hi) {
  constexpr int32_t per16 = 16 / sizeof(T);
  const int32_t mis = (int32_t)((reinterpret_cast<uintptr_t>(g) / sizeof(T)) & (per16 - 1));
  BulkRange32 r;
  r.lo0 = ((lo + mis) & ~(per16 - 1)) - mis;
  r.blo = r.lo0;
  r.bhi = hi > lo ? ((hi + mis + per16 - 1) & ~(per16 - 1)) - mis : r.lo0;
  r.tx_bytes = (uint32_t)(r.bhi - r.blo) * (uint32_t)sizeof(T);
  return r;
}

template <typename T>
SL_DEV void issue_range32(const T* g, const BulkRange32& r, T* s, uint64_t* bar) {
  if (r.tx_bytes) bulk_g2s(s + (r.blo - r.lo0), g + r.blo, r.tx_bytes, bar);
}

template <typename T>
SL_DEV void edge_loads_small32(const T* g, const BulkRange32& r, int32_t lo, int32_t hi, T* s,
                               int tid) {
  const int32_t hb = min(r.blo, hi);
  if (tid < hb - lo) s[lo + tid - r.lo0] = g[lo + tid];
  const int32_t t0 = max(max(r.bhi, lo), hb);
  const int k = tid - 64;
  if (k >= 0 && k < hi - t0) s[t0 + k - r.lo0] = g[t0 + k];
}

}  // namespace sl
