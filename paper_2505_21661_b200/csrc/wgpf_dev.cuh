// wgpf_dev.cuh -- device-side shared definitions of the P2 kernels.
//
// Layout in HBM of one replay call:
//   body      KPFT body: per stream {16 B header, slots * 8 B}, uniform stride
//   counts    u32[S]   events per stream (pass 1)
//   zpos      i32[S]   last chronological position with clamped depth 0
//   sflag     u32[S]   per-stream routing flags (fast / general)
//   offsets   u64[S]   exclusive scan of counts
//   events    wgpf_event[E]  (32 B, reference order)
//   stats     per label class: count, sum, min, max, first key, 64 bins
#pragma once

#include <cstdint>

#include "wgpf_format.h"

namespace wgpf {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kClassBits = 24;

// ---- per-stream routing flags (sflag) --------------------------------------
constexpr uint32_t SF_GENERAL = 1u;     // needs the thread-per-stream path
constexpr uint32_t SF_DECODE_ERR = 2u;  // decode error: no events
constexpr uint32_t SF_INVALID = 4u;     // single-stack count was wrong
constexpr uint32_t SF_WARP = 8u;        // warp-per-stream kernel (deep / wide)
constexpr uint32_t SF_DEEP = 16u;       // (with SF_WARP) fits the deep thread-per-
                                        // stream kernel (k_tpsd.cuh)

// ---- status block (device, read back once per call) ------------------------
struct DevStatus {
  unsigned long long decode_err;   // min over streams: (stream << 2) | code
  unsigned long long pair_err;     // min: (stream << 32) | chronological pos
  unsigned long long warn[4];      // dropped, tails, flagged, malformed
  unsigned long long n_general;    // streams routed to the general path
  unsigned long long invalid;      // single-stack invalid streams seen
  unsigned long long total_events; // scan total
  unsigned long long overflow;     // events beyond the caller capacity
  unsigned long long synth_overflow; // out-of-table class table full
  unsigned long long cap_mismatch;   // streams whose capacity != plan
  unsigned long long pad[4];
};
constexpr unsigned long long kNoErr = ~0ull;
constexpr uint32_t DEC_CAP = 1, DEC_FLUSH = 2, DEC_ZERO = 3;

// ---- plan tables -------------------------------------------------------------
struct DevPlan {
  uint64_t slots;      // plan.slots_per_warp_group
  uint32_t strategy;   // WGPF_STRATEGY_*
  uint32_t T;          // table labels
  uint32_t K;          // dense label classes (distinct table labels)
  uint32_t n_synth_wait;
  const uint32_t* class_of;   // [2^19] region id -> class (>= K: synthetic)
  const uint32_t* wait_class; // [K] class of label + ".wait" or kNone
  const uint8_t* is_marker;   // [K]
  const uint32_t* synth_wait_id;  // sorted out-of-table ids whose
  const uint32_t* synth_wait_cls; //   "region#<id>.wait" is a table label
};

// ---- statistics --------------------------------------------------------------
// Slot s < K: dense class s.  Slot K + h: open-addressed entry h of the
// synthetic-class table (key in hkey[h]).
struct DevStats {
  unsigned long long* count;
  unsigned long long* sum;
  unsigned long long* min;
  unsigned long long* max;
  unsigned long long* first; // min over (stream << 25 | k << 1 | kind)
  unsigned long long* hist;  // [slot * 64 + bin]
  uint32_t* hkey;            // [H]
  uint32_t K;
  uint32_t H;
};

__host__ __device__ inline unsigned long long first_key(uint64_t stream,
                                                        uint64_t k,
                                                        uint32_t kind) {
  return ((unsigned long long)stream << 25) | ((unsigned long long)k << 1) |
         kind;
}

__device__ inline uint32_t hist_bin(uint64_t d) {
  if (d < 4u) return (uint32_t)d;
  uint32_t k = 63u - (uint32_t)__clzll((long long)d);
  uint32_t b = 2u * k + (uint32_t)((d >> (k - 1u)) & 1u);
  return b < WGPF_HIST_BINS ? b : WGPF_HIST_BINS - 1u;
}

// hist_bin for durations below 2^32 (bin <= 63 without clamping): for
// d >= 2, 2k + bit k-1 of d (k = floor(log2 d)) is the float's exponent and
// top mantissa bit under round-toward-zero.
__device__ __forceinline__ uint32_t hist_bin32(uint32_t d) {
  const uint32_t b = (__float_as_uint(__uint2float_rz(d)) >> 22) - 254u;
  return d < 2u ? d : b;
}

// Slot of a class in the stats arrays (inserting synthetic classes).
__device__ inline int stats_slot(const DevStats& st, uint32_t cls,
                                 unsigned long long* overflow) {
  if (cls < st.K) return (int)cls;
  uint32_t h = (cls * 0x9E3779B1u) & (st.H - 1u);
  for (uint32_t i = 0; i < st.H; ++i) {
    uint32_t j = (h + i) & (st.H - 1u);
    uint32_t prev = atomicCAS(&st.hkey[j], kNone, cls);
    if (prev == kNone || prev == cls) return (int)(st.K + j);
  }
  atomicAdd(overflow, 1ull);
  return -1;
}

__device__ inline void stats_add_global(const DevStats& st, int slot,
                                        uint64_t d, unsigned long long key) {
  if (slot < 0) return;
  atomicAdd(&st.count[slot], 1ull);
  atomicAdd(&st.sum[slot], (unsigned long long)d);
  atomicMin(&st.min[slot], (unsigned long long)d);
  atomicMax(&st.max[slot], (unsigned long long)d);
  atomicMin(&st.first[slot], key);
  atomicAdd(&st.hist[(uint64_t)slot * WGPF_HIST_BINS + hist_bin(d)], 1ull);
}

// 64-bit shared-memory add / min without the CAS loops the compiler emits
// for 64-bit shared atomics: the add goes to the two 32-bit halves (each
// adder whose low-word add wraps carries exactly one into the high word), the
// min is skipped when the current value is already smaller (first-event keys
// only shrink early in a kernel).  Results are read after a barrier.
__device__ __forceinline__ void sadd64(unsigned long long* p, unsigned long long v) {
  uint32_t* w = reinterpret_cast<uint32_t*>(p);
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(w, lo);
  const uint32_t up = hi + ((uint32_t)(old + lo) < old ? 1u : 0u);
  if (up) atomicAdd(w + 1, up);
}
__device__ __forceinline__ void smin64(unsigned long long* p, unsigned long long v) {
  if (v < *reinterpret_cast<volatile unsigned long long*>(p)) atomicMin(p, v);
}

// Per-CTA shared-memory accumulators for dense classes < kSmemClasses.
constexpr uint32_t kSmemClasses = 64;
struct SmemStats {
  unsigned long long count[kSmemClasses];
  unsigned long long sum[kSmemClasses];
  unsigned long long first[kSmemClasses];
  uint32_t min[kSmemClasses];
  uint32_t max[kSmemClasses];
  uint32_t hist[kSmemClasses * WGPF_HIST_BINS];
};

__device__ inline void smem_stats_init(SmemStats& s) {
  for (uint32_t i = threadIdx.x; i < kSmemClasses; i += blockDim.x) {
    s.count[i] = 0;
    s.sum[i] = 0;
    s.first[i] = ~0ull;
    s.min[i] = 0xFFFFFFFFu;
    s.max[i] = 0;
  }
  for (uint32_t i = threadIdx.x; i < kSmemClasses * WGPF_HIST_BINS;
       i += blockDim.x)
    s.hist[i] = 0;
}

__device__ inline void smem_stats_flush(const SmemStats& s, const DevStats& st) {
  const uint32_t kc = st.K < kSmemClasses ? st.K : kSmemClasses;
  for (uint32_t c = threadIdx.x; c < kc; c += blockDim.x) {
    if (s.count[c] == 0) continue;
    atomicAdd(&st.count[c], s.count[c]);
    atomicAdd(&st.sum[c], s.sum[c]);
    atomicMin(&st.min[c], (unsigned long long)s.min[c]);
    atomicMax(&st.max[c], (unsigned long long)s.max[c]);
    atomicMin(&st.first[c], s.first[c]);
  }
  for (uint32_t i = threadIdx.x; i < kc * WGPF_HIST_BINS; i += blockDim.x)
    if (s.hist[i]) atomicAdd(&st.hist[i], (unsigned long long)s.hist[i]);
}

// Single event into the CTA accumulators (dense) or global (synthetic / wide).
__device__ inline void stats_add_one(SmemStats& s, const DevStats& st,
                                     uint32_t cls, uint64_t d,
                                     unsigned long long key,
                                     unsigned long long* overflow) {
  if (cls < kSmemClasses && cls < st.K) {
    sadd64(&s.count[cls], 1ull);
    sadd64(&s.sum[cls], (unsigned long long)d);
    atomicMin(&s.min[cls], (uint32_t)d);
    atomicMax(&s.max[cls], (uint32_t)d);
    smin64(&s.first[cls], key);
    atomicAdd(&s.hist[cls * WGPF_HIST_BINS + hist_bin(d)], 1u);
  } else {
    stats_add_global(st, stats_slot(st, cls, overflow), d, key);
  }
}

// ---- plan lookups ------------------------------------------------------------
__device__ inline uint32_t class_of(const DevPlan& p, uint32_t rid) {
  return p.class_of[rid];
}

__device__ inline bool class_is_marker(const DevPlan& p, uint32_t cls) {
  return cls < p.K && p.is_marker[cls];
}

// class of label(rid) + ".wait", or kNone
__device__ inline uint32_t wait_class_of(const DevPlan& p, uint32_t rid,
                                         uint32_t cls) {
  if (cls < p.K) return p.wait_class[cls];
  uint32_t lo = 0, hi = p.n_synth_wait;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (p.synth_wait_id[mid] < rid) lo = mid + 1; else hi = mid;
  }
  return (lo < p.n_synth_wait && p.synth_wait_id[lo] == rid)
             ? p.synth_wait_cls[lo]
             : kNone;
}

// ---- shared memory through 32-bit addresses ----------------------------------
// (hot loops: a generic pointer into dynamic shared memory makes the compiler
// rematerialise the shared window base at every access site)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}
// One 32-byte event with a single 256-bit store (STG.E.ENL2.256, sm_100):
// a full L2 sector per lane instead of two 16-byte halves.
__device__ __forceinline__ void stg256(void* p, uint4 a, uint4 b) {
  asm volatile("st.global.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p),
               "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z),
               "r"(b.w)
               : "memory");
}

// predicated form (no branch around the store; the operands are computed
// unconditionally)
__device__ __forceinline__ void stg256_if(bool q, uint64_t p, uint4 a, uint4 b) {
  asm volatile(
      "{ .reg .pred q; setp.ne.b32 q, %0, 0; @q st.global.v8.u32 [%1], {%2, %3, %4, %5, %6, "
      "%7, %8, %9}; }" ::"r"((uint32_t)q),
      "l"(p), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
      : "memory");
}
__device__ __forceinline__ uint64_t opaque_u64(uint64_t x) {
  uint64_t y;
  asm("mov.b64 %0, %1;" : "=l"(y) : "l"(x));
  return y;
}

// a value the compiler cannot see through (so it is not rematerialised)
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
  uint32_t y;
  asm("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ void sts16_if(bool p, uint32_t a, uint32_t v) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q st.shared.u16 [%1], %2; }" ::"r"(
                   (uint32_t)p),
               "r"(a), "h"((uint16_t)v)
               : "memory");
}
__device__ __forceinline__ void sts32_if(bool p, uint32_t a, uint32_t v) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q st.shared.u32 [%1], %2; }" ::"r"(
                   (uint32_t)p),
               "r"(a), "r"(v)
               : "memory");
}
__device__ __forceinline__ void sts64_if(bool p, uint32_t a, uint2 v) {
  asm volatile(
      "{ .reg .pred q; setp.ne.b32 q, %0, 0; @q st.shared.v2.u32 [%1], {%2, %3}; }" ::"r"(
          (uint32_t)p),
      "r"(a), "r"(v.x), "r"(v.y)
      : "memory");
}
__device__ __forceinline__ void sts128_if(bool p, uint32_t a, uint4 v) {
  asm volatile(
      "{ .reg .pred q; setp.ne.b32 q, %0, 0; @q st.shared.v4.u32 [%1], {%2, %3, %4, %5}; }" ::"r"(
          (uint32_t)p),
      "r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
      : "memory");
}
// (lo, hi) += d as one 64-bit add (add.cc / addc)
__device__ __forceinline__ void add64_u32(uint32_t& lo, uint32_t& hi, uint32_t d) {
  asm("add.cc.u32 %0, %0, %2; addc.u32 %1, %1, 0;" : "+r"(lo), "+r"(hi) : "r"(d));
}
__device__ __forceinline__ void red_add_if(bool p, uint32_t a, uint32_t v) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q red.shared.add.u32 [%1], %2; }" ::"r"(
                   (uint32_t)p),
               "r"(a), "r"(v)
               : "memory");
}

__device__ __forceinline__ void red_add(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// ---- warp helpers --------------------------------------------------------------
__device__ inline uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ inline uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ inline uint32_t lanemask_le() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}
__device__ inline uint32_t lanemask_gt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_gt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ inline T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace wgpf
