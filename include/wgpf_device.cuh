// wgpf_device.cuh -- P1: the device-side instrumentation runtime (header only,
// sm_100a).  The B200 realisation of the reference's lowered record ops:
//
//   InitOp        Engine::step Init        wgprof/vgpu.hpp:216-219  (index in a register)
//   ReadCounter   Engine::step ReadCounter wgprof/vgpu.hpp:220-223  (clock captured first)
//   StoreCounter  Engine::exec_store       wgprof/vgpu.hpp:240-273  (tag, slot = writes % cap)
//   FinalizeOp    Engine::image            wgprof/vgpu.hpp:136-148  (copy-out of the buffer)
//   buffer plan   BufferPlan::base_offset  wgprof/lower.hpp:57-64   (disjoint per-stream slots)
//   record tag    ProfileRecord::make      wgprof/trace.hpp:68-78
//
// Layout.  The CTA's profile buffer lives in shared memory in exactly the KPFT
// body layout the decoder reads (include/wgpf_format.h): per stream a 16-byte
// header then `cap` 8-byte slots.  Finalize copies it to HBM at
//   profile_mem + blockIdx_linear * streams_per_cta * (16 + 8 * cap)
// with 16-byte vector stores, so the device buffer *is* a KPFT body and a v1/v2
// header in front of it makes a reference-readable image (wgpf_collect /
// oracle tests).
//
// Recording.  One stream per warp (granularity warp) or per warp group.  The
// write index is a warp-uniform register; one lane performs the store
// (collaborative store): clock read, tag/address arithmetic,
// predicated STS.64, index increment -- no atomics, no branches.  Power-of-two
// capacities wrap with a mask; other capacities with a compare-and-reset
// slot register (lower.hpp:263-270 allows any divisor).
//
// Clock.  `%clock` (SR_CLOCKLO, 32-bit, per-SM cycles) as the payload, like the
// reference's 32-bit capture (vgpu.hpp:259); the decoder's unwrap restores
// 64-bit monotone time per stream.  A per-CTA side record keeps SM id and
// %globaltimer / %clock64 at init and finalize for cross-CTA alignment.
#pragma once

#include <cstdint>

#include "wgpf_format.h"

namespace wgpf_dev {

__device__ __forceinline__ uint32_t clock32() {
  uint32_t c;
  asm volatile("mov.u32 %0, %%clock;" : "=r"(c)::"memory");
  return c;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}

__device__ __forceinline__ uint32_t smid() {
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Per-CTA side record (optional): 32 bytes.
struct CtaTiming {
  uint32_t smid;
  uint32_t streams;
  uint64_t gt_start;   // %globaltimer at init (ns)
  uint64_t gt_end;     // %globaltimer at finalize (ns)
  uint32_t clk_start;  // %clock at init
  uint32_t clk_end;    // %clock at finalize
};

constexpr uint32_t kStreamHdr = WGPF_STREAM_HDR_BYTES;

// Bytes of shared memory the profile buffer needs per CTA.
__host__ __device__ constexpr uint32_t smem_bytes(uint32_t streams_per_cta,
                                                  uint32_t cap) {
  return streams_per_cta * (kStreamHdr + 8u * cap);
}

// Bytes of HBM the flushed buffers need for a grid.
__host__ __device__ constexpr uint64_t profile_bytes(uint64_t ctas,
                                                     uint32_t streams_per_cta,
                                                     uint32_t cap) {
  return ctas * streams_per_cta * (uint64_t)(kStreamHdr + 8u * cap);
}

// signature_for (vgpu.hpp:39-45) packed as trace.hpp:42-46 (wave slot 5 bits,
// SIMD 4 bits, pipe 3 bits): the tag's low 12 bits for stream `wg`
__host__ __device__ constexpr uint32_t signature_for(uint32_t wg) {
  return (wg % 32u) | (((wg / 32u) % 16u) << 5) | (((wg / 512u) % 8u) << 9);
}

__host__ __device__ constexpr uint32_t make_tag(bool start, uint32_t region,
                                                uint32_t sig = 0) {
  return (start ? WGPF_START_FLAG : 0u) | (region << 12) | (sig & WGPF_SIGNATURE_MASK);
}

// One recording stream (a warp or a warp group).  kPow2: capacity is a power
// of two (mask wrap); otherwise compare-and-reset.
template <bool kPow2 = true>
struct Recorder {
  uint32_t base;   // shared address of this stream's slot 0
  uint32_t mask;   // cap - 1 (kPow2) / cap (else)
  uint32_t writes; // total writes (record_count)
  uint32_t slot;   // current slot (non-pow2 only)
  bool leader;     // the lane that stores

  // InitOp: smem_buf = the CTA's buffer, stream = this warp's stream index in
  // the CTA.  Index state lives in registers (vgpu.hpp:216-219).
  __device__ __forceinline__ void init(void* smem_buf, uint32_t stream,
                                       uint32_t cap, bool is_leader) {
    const uint32_t b = smem_addr(smem_buf) + stream * (kStreamHdr + 8u * cap);
    base = b + kStreamHdr;
    mask = kPow2 ? cap - 1u : cap;
    writes = 0;
    slot = 0;
    leader = is_leader;
  }

  // ReadCounter + StoreCounter.  The clock is read before anything else
  // (vgpu.hpp:220-223, the reference charges the record cost after capture).
  template <bool kStart>
  __device__ __forceinline__ void record(uint32_t region, uint32_t sig = 0) {
    const uint32_t clk = clock32();
    put(make_tag(kStart, region, sig), clk);
  }

  __device__ __forceinline__ void start(uint32_t region, uint32_t sig = 0) {
    record<true>(region, sig);
  }
  __device__ __forceinline__ void end(uint32_t region, uint32_t sig = 0) {
    record<false>(region, sig);
  }

  // END(end_region) immediately followed by START(start_region): the two
  // RecordOps of a scope boundary (wait -> issue, issue -> next wait) share
  // one clock capture -- same records, half the critical-path cost there.
  __device__ __forceinline__ void mark(uint32_t end_region, uint32_t start_region,
                                       uint32_t sig = 0) {
    const uint32_t clk = clock32();
    put(make_tag(false, end_region, sig), clk);
    put(make_tag(true, start_region, sig), clk);
  }

  // StoreCounter: slot writes % cap (circular) -- vgpu.hpp:240-273
  __device__ __forceinline__ void put(uint32_t tag, uint32_t clk) {
    uint32_t s;
    if constexpr (kPow2) {
      s = writes & mask;
    } else {
      s = slot;
      slot = (slot + 1u == mask) ? 0u : slot + 1u;
    }
    const uint32_t addr = base + 8u * s;
    if (leader)
      asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(tag),
                   "r"(clk)
                   : "memory");
    ++writes;
  }

  // Stream header (done by the leader before the CTA flush).
  __device__ __forceinline__ void close(uint32_t block_index,
                                        uint32_t stream_id, uint32_t cap) {
    if (leader) {
      const uint32_t h = base - kStreamHdr;
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(h),
                   "r"(block_index), "r"(stream_id), "r"(writes), "r"(cap)
                   : "memory");
    }
  }
};

// The uninstrumented twin (strip_profiling, lower.hpp:303-314): the same
// kernel source compiled with NullRecorder records nothing and costs nothing,
// which is how T_vanilla of the overhead metric is measured.
struct NullRecorder {
  __device__ __forceinline__ void init(void*, uint32_t, uint32_t, bool) {}
  template <bool kStart>
  __device__ __forceinline__ void record(uint32_t, uint32_t = 0) {}
  __device__ __forceinline__ void start(uint32_t, uint32_t = 0) {}
  __device__ __forceinline__ void end(uint32_t, uint32_t = 0) {}
  __device__ __forceinline__ void mark(uint32_t, uint32_t, uint32_t = 0) {}
  __device__ __forceinline__ void close(uint32_t, uint32_t, uint32_t) {}
};

// ---- the instrumentation pass, as source-level helpers ---------------------
// The reference inserts RecordOps into its IR (instrument.hpp:163-244): a
// start/end pair around a synchronous region, and around every async launch /
// wait pair the four-record pattern (insert_async_pattern, :145-153; doc
// :14-25): S(X) immediately before the launch, E(X) immediately before the
// wait, S(X.wait) E(X.wait) immediately after it -- replay derives the wait
// interval as CLK2 - CLK1.  On B200 the launch is a TMA copy or a
// tcgen05.mma + commit and the wait an mbarrier phase wait; these helpers
// place the records at exactly those points so a kernel is instrumented by
// wrapping its issue and wait sites (auto_async), not by hand-placed records.

// RAII sync scope: S(region) now, E(region) when the scope closes.
template <class Rec>
struct Scope {
  Rec& rec;
  uint32_t region;
  __device__ __forceinline__ Scope(Rec& r, uint32_t id) : rec(r), region(id) {
    rec.start(region);
  }
  __device__ __forceinline__ ~Scope() { rec.end(region); }
};

// One async operation X (region ids x and x_wait = the "X.wait" label):
//   AsyncOp op(rec, x, xw);  op.launch([&]{ issue });  ... ;  op.wait([&]{ wait });
template <class Rec>
struct AsyncOp {
  Rec& rec;
  uint32_t x, xw;
  __device__ __forceinline__ AsyncOp(Rec& r, uint32_t x_, uint32_t xw_)
      : rec(r), x(x_), xw(xw_) {}
  // S(X) immediately before the launch
  template <class F>
  __device__ __forceinline__ void launch(F&& issue) {
    rec.start(x);
    issue();
  }
  // E(X) immediately before the wait; S(X.wait) E(X.wait) right after it
  template <class F>
  __device__ __forceinline__ void wait(F&& block) {
    rec.end(x);
    block();
    rec.start(xw);
    rec.end(xw);
  }
};

// launch and wait back to back (a producer that waits for its own copy)
template <class Rec, class L, class W>
__device__ __forceinline__ void async_region(Rec& rec, uint32_t x, uint32_t xw, L&& issue,
                                             W&& block) {
  AsyncOp<Rec> op(rec, x, xw);
  op.launch(issue);
  op.wait(block);
}

// FinalizeOp: after every stream of the CTA has closed (barrier), copy the
// CTA's buffer to HBM with 16-byte vector stores by all participating threads
// (coalesced; the buffer is a contiguous KPFT body segment).
__device__ __forceinline__ void flush(const void* smem_buf, void* profile_mem,
                                      uint64_t cta_linear, uint32_t bytes,
                                      uint32_t tid, uint32_t nthreads) {
  const uint4* src = reinterpret_cast<const uint4*>(smem_buf);
  uint4* dst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(profile_mem) +
                                        cta_linear * (uint64_t)bytes);
  for (uint32_t i = tid; i < bytes / 16u; i += nthreads) dst[i] = src[i];
}

}  // namespace wgpf_dev
