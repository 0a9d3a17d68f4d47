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
#include <type_traits>

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

static_assert(sizeof(CtaTiming) == sizeof(wgpf_cta_timing), "CtaTiming layout");

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

// Debug-mode pairing validation (the device form of validate_record_pairing,
// instrument.hpp:60-105): error codes of the first violation a stream meets.
// The 64-bit error word is stream << 32 | code << 24 | region, combined with
// atomicMin so the lowest stream's first violation wins (the reference checks
// wg 0 first); wgpf_collect turns it into the reference's message.
enum : uint32_t {
  kVErrEndMismatch = 1,       // record end "X" does not match the innermost open start
  kVErrPairCrossesLoop = 2,   // record pair "X" crosses a loop boundary
  kVErrStartCrossesLoop = 3,  // record start "X" crosses a loop boundary
  kVErrNeverClosed = 4,       // record start "X" is never closed
};
constexpr uint32_t kVDepth = 32;  // open scopes a validating recorder tracks

struct NoValidate {};
struct Validate {
  uint32_t stk[kVDepth];  // region | loop depth << 24
  uint32_t top;           // open scopes
  uint32_t depth;         // loop depth
  uint32_t stream;        // global stream index (error key)
  unsigned long long* err;
  bool failed;
};

// One recording stream (a warp or a warp group).
//   kPow2      capacity is a power of two (mask wrap); otherwise compare-and-reset
//   kFlush     BufferStrategy::Flush: slots are never overwritten; writes past the
//              capacity are counted (record_count > capacity), which wgpf_collect
//              reports as the reference's capacity-error (vgpu.hpp:261-265)
//   kValidate  debug mode: check the pairing rules of instrument.hpp:60-105 as the
//              records execute (loops marked with wgpf_dev::Loop)
template <bool kPow2 = true, bool kFlush = false, bool kValidate = false>
struct Recorder {
  uint32_t base;   // shared address of this stream's slot 0
  uint32_t mask;   // cap - 1 (kPow2) / cap (else)
  uint32_t writes; // total writes (record_count)
  uint32_t slot;   // current slot (non-pow2 circular only)
  uint32_t sig;    // signature bits stamped into every tag (0, signature_for,
                   // or the loop index -- LoweringConfig, lower.hpp:44-52)
  bool leader;     // the lane that stores
  std::conditional_t<kValidate, Validate, NoValidate> v;

  // InitOp: smem_buf = the CTA's buffer, stream = this warp's stream index in
  // the CTA.  Index state lives in registers (vgpu.hpp:216-219).
  __device__ __forceinline__ void init(void* smem_buf, uint32_t stream,
                                       uint32_t cap, bool is_leader) {
    const uint32_t b = smem_addr(smem_buf) + stream * (kStreamHdr + 8u * cap);
    base = b + kStreamHdr;
    mask = kPow2 ? cap - 1u : cap;
    writes = 0;
    slot = 0;
    sig = 0;
    leader = is_leader;
  }

  // debug mode: where violations go (global stream index, error word)
  __device__ __forceinline__ void validate_into(unsigned long long* err,
                                                uint32_t global_stream) {
    if constexpr (kValidate) {
      v.top = 0;
      v.depth = 0;
      v.stream = global_stream;
      v.err = err;
      v.failed = false;
    }
  }

  // signature_bits_enabled: the stream's hardware-id signature (vgpu.hpp:245-246)
  __device__ __forceinline__ void hw_signature(uint32_t stream_id) {
    sig = signature_for(stream_id);
  }
  // iteration_signature: the innermost loop's iteration index (vgpu.hpp:247-251)
  __device__ __forceinline__ void iteration(uint32_t i) { sig = i & WGPF_SIGNATURE_MASK; }

  // ReadCounter + StoreCounter.  The clock is read before anything else
  // (vgpu.hpp:220-223, the reference charges the record cost after capture).
  template <bool kStart>
  __device__ __forceinline__ void record(uint32_t region) {
    const uint32_t clk = clock32();
    check<kStart>(region);
    put(make_tag(kStart, region, sig), clk);
  }
  template <bool kStart>
  __device__ __forceinline__ void record(uint32_t region, uint32_t sig_bits) {
    const uint32_t clk = clock32();
    check<kStart>(region);
    put(make_tag(kStart, region, sig_bits), clk);
  }

  __device__ __forceinline__ void start(uint32_t region) { record<true>(region); }
  __device__ __forceinline__ void end(uint32_t region) { record<false>(region); }
  __device__ __forceinline__ void start(uint32_t region, uint32_t s) {
    record<true>(region, s);
  }
  __device__ __forceinline__ void end(uint32_t region, uint32_t s) {
    record<false>(region, s);
  }

  // END(end_region) immediately followed by START(start_region): the two
  // RecordOps of a scope boundary (wait -> issue, issue -> next wait) share
  // one clock capture -- same records, half the critical-path cost there.
  __device__ __forceinline__ void mark(uint32_t end_region, uint32_t start_region) {
    const uint32_t clk = clock32();
    check<false>(end_region);
    put(make_tag(false, end_region, sig), clk);
    check<true>(start_region);
    put(make_tag(true, start_region, sig), clk);
  }

  // StoreCounter: slot writes % cap (circular) -- vgpu.hpp:240-273
  __device__ __forceinline__ void put(uint32_t tag, uint32_t clk) {
    uint32_t s;
    bool keep = leader;
    if constexpr (kFlush) {
      s = writes;
      keep = keep && (kPow2 ? writes <= mask : writes < mask);
    } else if constexpr (kPow2) {
      s = writes & mask;
    } else {
      s = slot;
      slot = (slot + 1u == mask) ? 0u : slot + 1u;
    }
    const uint32_t addr = base + 8u * s;
    if (keep)
      asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(tag),
                   "r"(clk)
                   : "memory");
    ++writes;
  }

  // Stream header (done by the leader before the CTA flush).  Two 8-byte
  // stores: with an odd capacity the per-stream stride 16 + 8 * cap is only
  // 8-byte aligned.
  __device__ __forceinline__ void close(uint32_t block_index,
                                        uint32_t stream_id, uint32_t cap) {
    if constexpr (kValidate) {
      if (v.top && !v.failed) fail(kVErrNeverClosed, v.stk[v.top - 1] & 0xFFFFFFu);
    }
    if (leader) {
      const uint32_t h = base - kStreamHdr;
      asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(h), "r"(block_index),
                   "r"(stream_id)
                   : "memory");
      asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(h + 8u), "r"(writes),
                   "r"(cap)
                   : "memory");
    }
  }

  // ---- debug-mode pairing checks (instrument.hpp:60-105) ------------------
  __device__ __forceinline__ void fail(uint32_t code, uint32_t region) {
    if constexpr (kValidate) {
      v.failed = true;
      if (leader && v.err)
        atomicMin(v.err, ((unsigned long long)v.stream << 32) |
                             ((unsigned long long)code << 24) | region);
    }
  }
  template <bool kStart>
  __device__ __forceinline__ void check(uint32_t region) {
    if constexpr (kValidate) {
      if (v.failed) return;
      if (kStart) {
        if (v.top == kVDepth) {  // deeper than tracked: stop validating
          v.failed = true;
          return;
        }
        v.stk[v.top++] = region | (v.depth << 24);
      } else {
        const uint32_t t = v.top ? v.stk[v.top - 1] : ~0u;
        if (!v.top || (t & 0xFFFFFFu) != region) {
          fail(kVErrEndMismatch, region);
        } else if ((t >> 24) != v.depth) {
          fail(kVErrPairCrossesLoop, region);
        } else {
          --v.top;
        }
      }
    }
  }
  // loop boundaries (wgpf_dev::Loop): the end of an iteration is the
  // reference's LoopEnd -- a start opened at this depth must be closed by then
  __device__ __forceinline__ void loop_begin() {
    if constexpr (kValidate) ++v.depth;
  }
  __device__ __forceinline__ void loop_iteration_end() {
    if constexpr (kValidate) {
      if (!v.failed && v.top && (v.stk[v.top - 1] >> 24) == v.depth)
        fail(kVErrStartCrossesLoop, v.stk[v.top - 1] & 0xFFFFFFu);
    }
  }
  __device__ __forceinline__ void loop_end() {
    if constexpr (kValidate) {
      loop_iteration_end();
      --v.depth;
    }
  }
};

// An instrumented loop: stamps the iteration index into the signature bits
// when the recorder runs in iteration-signature mode (the caller sets it with
// iteration(); the outer loop's index comes back when the loop ends,
// vgpu.hpp:247-251 uses the innermost loop), and marks the loop boundaries for
// debug-mode validation.
//   { wgpf_dev::Loop<Rec> L(rec, iter_sig);  for (i...) { L.next(i); ... } }
template <class Rec>
struct Loop {
  Rec& rec;
  uint32_t saved;
  bool stamp;
  bool first = true;
  __device__ __forceinline__ Loop(Rec& r, bool iteration_signature)
      : rec(r), saved(r.sig), stamp(iteration_signature) {
    rec.loop_begin();
  }
  __device__ __forceinline__ void next(uint32_t i) {
    if (!first) rec.loop_iteration_end();
    first = false;
    if (stamp) rec.iteration(i);
  }
  __device__ __forceinline__ ~Loop() {
    rec.loop_end();
    rec.sig = saved;
  }
};

// The uninstrumented twin (strip_profiling, lower.hpp:303-314): the same
// kernel source compiled with NullRecorder records nothing and costs nothing,
// which is how T_vanilla of the overhead metric is measured.
struct NullRecorder {
  uint32_t sig = 0;
  __device__ __forceinline__ void init(void*, uint32_t, uint32_t, bool) {}
  __device__ __forceinline__ void validate_into(unsigned long long*, uint32_t) {}
  __device__ __forceinline__ void hw_signature(uint32_t) {}
  __device__ __forceinline__ void iteration(uint32_t) {}
  template <bool kStart>
  __device__ __forceinline__ void record(uint32_t, uint32_t = 0) {}
  __device__ __forceinline__ void start(uint32_t, uint32_t = 0) {}
  __device__ __forceinline__ void end(uint32_t, uint32_t = 0) {}
  __device__ __forceinline__ void mark(uint32_t, uint32_t) {}
  __device__ __forceinline__ void close(uint32_t, uint32_t, uint32_t) {}
  __device__ __forceinline__ void loop_begin() {}
  __device__ __forceinline__ void loop_iteration_end() {}
  __device__ __forceinline__ void loop_end() {}
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

// Back-to-back scopes on one stream: the phases of a warp-specialised
// pipeline loop (wait -> issue -> wait -> ...).  to(r) closes the open scope
// and opens r; the destructor closes the last one.  kShare: the END / START
// pair at each boundary shares one clock capture (Recorder::mark), otherwise
// every RecordOp captures its own.  Either way the records are exactly the
// hand-placed start/end pairs of instrument.hpp:163-244's sync regions.
// In a loop, name the phase each boundary closes and end every iteration
// with iteration_end(), so every tag is an immediate:
//   Chain<Rec, share> ch(rec);
//   for (k...) {
//     ch.to(WAIT, ISSUE);  wait();  ch.to(ISSUE, WAIT);  issue();
//     ch.iteration_end();
//   }                                   // ~Chain: end(ISSUE) if still open
template <class Rec, bool kShare>
struct Chain {
  Rec& rec;
  uint32_t cur = 0;
  bool open = false;
  __device__ __forceinline__ explicit Chain(Rec& r) : rec(r) {}
  __device__ __forceinline__ void to(uint32_t region) { to(region, cur); }
  // prev: the phase the caller knows is open here (it must equal the open
  // one) -- a constant at the call site, so the END tag is an immediate
  // even where the open phase is loop-carried
  __device__ __forceinline__ void to(uint32_t region, uint32_t prev) {
    if (!open) {
      rec.start(region);
    } else if constexpr (kShare) {
      rec.mark(prev, region);
    } else {
      rec.end(prev);
      rec.start(region);
    }
    cur = region;
    open = true;
  }
  __device__ __forceinline__ void close() {
    if (open) rec.end(cur);
    open = false;
  }
  // end of one loop iteration: with separate captures the iteration's last
  // phase closes here (a loop body then starts with nothing open, and every
  // tag is an immediate); with shared captures it stays open so the next
  // iteration's first boundary shares its capture
  __device__ __forceinline__ void iteration_end() {
    if constexpr (!kShare) close();
  }
  __device__ __forceinline__ ~Chain() { close(); }
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
// CTA's buffer to HBM with vector stores by all participating threads
// (coalesced; the buffer is a contiguous KPFT body segment).  16-byte stores
// when the segment size is a multiple of 16 (even capacities or an even
// stream count), else 8-byte stores (the segment, and its HBM offset, are
// then only 8-byte aligned).
__device__ __forceinline__ void flush(const void* smem_buf, void* profile_mem,
                                      uint64_t cta_linear, uint32_t bytes,
                                      uint32_t tid, uint32_t nthreads) {
  uint8_t* dst8 = static_cast<uint8_t*>(profile_mem) + cta_linear * (uint64_t)bytes;
  if ((bytes & 15u) == 0) {
    const uint4* src = reinterpret_cast<const uint4*>(smem_buf);
    uint4* dst = reinterpret_cast<uint4*>(dst8);
    for (uint32_t i = tid; i < bytes / 16u; i += nthreads) dst[i] = src[i];
  } else {
    const uint2* src = reinterpret_cast<const uint2*>(smem_buf);
    uint2* dst = reinterpret_cast<uint2*>(dst8);
    for (uint32_t i = tid; i < bytes / 8u; i += nthreads) dst[i] = src[i];
  }
}

// FinalizeOp on the bulk-copy engine: after the CTA's barrier one thread
// hands the whole buffer (a contiguous KPFT body segment) to cp.async.bulk
// (shared -> global) and waits for it; the other threads are free at once.
// Needs a 16-byte aligned segment of a multiple of 16 bytes (even capacities
// or an even stream count, and a 16-byte aligned profile_mem), else falls
// back to flush().  The records were written through the generic proxy, so
// the copy (async proxy) is preceded by a proxy fence.
__device__ __forceinline__ void flush_bulk(const void* smem_buf, void* profile_mem,
                                           uint64_t cta_linear, uint32_t bytes, uint32_t tid,
                                           uint32_t nthreads) {
  uint8_t* dst = static_cast<uint8_t*>(profile_mem) + cta_linear * (uint64_t)bytes;
  if ((bytes & 15u) != 0 || (reinterpret_cast<uintptr_t>(dst) & 15u) != 0) {
    flush(smem_buf, profile_mem, cta_linear, bytes, tid, nthreads);
    return;
  }
  if (tid == 0 && bytes) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_addr(smem_buf)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

}  // namespace wgpf_dev

// ---- the C-style device API of SURVEY.md 8(b) ------------------------------
// wgpf_init / wgpf_record / wgpf_finalize over a power-of-two circular
// Recorder (the state is the caller's register-resident wgpf_recorder):
//   InitOp      wgpf_init(r, smem_base, slots, warp_id)
//   RecordOp    wgpf_record_op(r, start, region) (ReadCounter + StoreCounter;
//               wgpf_record is the 8-byte record type of wgpf_format.h)
//   FinalizeOp  wgpf_finalize(r, ...)           (header, barrier, bulk flush)
typedef wgpf_dev::Recorder<true> wgpf_recorder;
__device__ __forceinline__ void wgpf_init(wgpf_recorder& r, void* smem_base, uint32_t slots,
                                          uint32_t warp_id) {
  r.init(smem_base, warp_id, slots, (threadIdx.x & 31u) == 0u);
}
__device__ __forceinline__ void wgpf_record_op(wgpf_recorder& r, bool start, uint32_t region) {
  if (start)
    r.start(region);
  else
    r.end(region);
}
// every thread of the CTA calls it (it contains the CTA barrier)
__device__ __forceinline__ void wgpf_finalize(wgpf_recorder& r, const void* smem_base,
                                              void* profile_mem, uint32_t block_index,
                                              uint32_t warp_id, uint32_t slots,
                                              uint32_t streams_per_cta) {
  r.close(block_index, warp_id, slots);
  __syncthreads();
  wgpf_dev::flush_bulk(smem_base, profile_mem, block_index,
                       wgpf_dev::smem_bytes(streams_per_cta, slots), threadIdx.x, blockDim.x);
}
