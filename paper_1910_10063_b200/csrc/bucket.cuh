// bucket.cuh -- key-range bucketing of scattered tail updates.
//
// Histogram and group-by updates for cold keys scatter over counter arrays
// far larger than L2 (2^26 u32 counters = 256 MiB), so one global atomic per
// cold row read-modify-writes a whole HBM line.  Instead, cold rows are
// appended (warp-aggregated) to per-key-range buckets -- sequential streams
// that L2 write-combines -- and a second kernel folds each bucket in shared
// memory, where its key range fits, then updates the global counters with
// plain coalesced read-modify-writes (each bucket owns its key range).
#pragma once
#include "skx_internal.cuh"

namespace skx {

// Warp-collective (every lane of the warp must call it, `active` or not):
// appends each active lane's `v` to bucket `b`.  Lanes of one bucket claim
// consecutive slots with one atomic.  Returns false for a lane whose slot
// fell past `cap` (the caller must then apply that update another way).
template <typename T>
__device__ __forceinline__ bool bucket_append(uint32_t b, bool active, T v,
                                              unsigned int* __restrict__ cursors,
                                              T* __restrict__ buf, uint64_t cap) {
  const uint32_t key = active ? b : 0xFFFFFFFFu;
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(peers) - 1;
  unsigned int base = 0;
  if (active && lane == leader) base = atomicAdd(&cursors[b], (unsigned int)__popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (!active) return true;
  const uint64_t pos = (uint64_t)base + __popc(peers & lanemask_lt());
  if (pos >= cap) return false;
  buf[(uint64_t)b * cap + pos] = v;
  return true;
}

}  // namespace skx
