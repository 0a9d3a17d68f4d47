// k_lookback.cuh -- decoupled look-back over streams (single-pass event
// offsets).  Each stream publishes its event count as soon as it is known
// (AGG) and its inclusive prefix once its own look-back resolved (INC); a
// successor sums predecessor aggregates 32 at a time (one status word per
// lane) until it meets an INC.  Streams are claimed in order through a global
// ticket, and a warp only ever waits on smaller tickets, so the protocol cannot
// deadlock.  Status words: flag in bits 62-63, value in bits 0-61.
#pragma once

#include "wgpf_dev.cuh"

namespace wgpf {

constexpr unsigned long long LB_AGG = 1ull << 62;
constexpr unsigned long long LB_INC = 2ull << 62;
constexpr unsigned long long LB_VAL = (1ull << 62) - 1;

__device__ __forceinline__ void lb_store(unsigned long long* p,
                                         unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long lb_load(
    const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Exclusive prefix of stream s (warp-collective; every lane returns it).
// Publishes AGG(count) first, INC(prefix + count) at the end.
__device__ inline unsigned long long lb_prefix(unsigned long long* status,
                                               uint64_t s,
                                               unsigned long long count) {
  const uint32_t lane = lane_id();
  if (s == 0) {
    if (lane == 0) lb_store(&status[0], LB_INC | count);
    __syncwarp();
    return 0;
  }
  if (lane == 0) lb_store(&status[s], LB_AGG | count);
  unsigned long long acc = 0;
  int64_t p = (int64_t)s - 1;  // next predecessor to inspect
  for (;;) {
    const int64_t q = p - (int64_t)lane;
    unsigned long long w = q >= 0 ? lb_load(&status[q]) : LB_INC;  // virtual INC 0 before stream 0
    const uint32_t not_ready = __ballot_sync(0xffffffffu, (w >> 62) == 0);
    const uint32_t inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
    // first INC lane (closest predecessor with an inclusive prefix)
    const uint32_t first_inc = inc ? __ffs(inc) - 1u : 32u;
    const uint32_t need = first_inc < 32 ? ((2u << first_inc) - 1u) : 0xffffffffu;
    if (not_ready & need) {  // some required predecessor not published yet
      __nanosleep(32);
      continue;
    }
    unsigned long long v = (lane <= first_inc) ? (w & LB_VAL) : 0ull;
    v = warp_sum(v);
    acc += v;
    if (first_inc < 32) break;
    p -= 32;
  }
  if (lane == 0) lb_store(&status[s], LB_INC | (acc + count));
  __syncwarp();
  return acc;
}

}  // namespace wgpf
