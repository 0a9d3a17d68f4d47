// p1_selftest.cu -- P1 device runtime exercised by known scope programs.
//
// wgpf_p1_selftest: every warp of every CTA runs the same scope program
// (nested sync scopes, the reference's 4-record async pattern
// instrument.hpp:14-25, a loop) through wgpf_dev::Recorder, then the CTA
// flushes its shared-memory buffer to HBM as a KPFT body.  The tests decode
// that body with the reference (oracle/_ref) and the CPU oracle and check the
// per-stream tag sequence against the program's store log (vgpu.hpp:269-271).
//
// wgpf_p1_record_cost: cycles per record op -- the same loop with and without
// records, timed per warp with %clock64 (PAPER.md:798 reports 33 cycles on
// H100).
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "wgpf_device.cuh"

// signature_for packs MachineConfig::signature_for (vgpu.hpp:39-45) as
// Signature::packed (trace.hpp:42-46); tests/test_models.py checks the same
// formula against the reference
static_assert(wgpf_dev::signature_for(0) == 0u, "");
static_assert(wgpf_dev::signature_for(33) == (1u | (1u << 5)), "");
static_assert(wgpf_dev::signature_for(4095) == (31u | (15u << 5) | (7u << 9)), "");
static_assert(wgpf_dev::signature_for(4096) == 0u, "");

namespace {

constexpr uint32_t R_KERNEL = 0, R_OUTER = 1, R_INNER = 2, R_ASYNC = 3,
                   R_ASYNC_WAIT = 4;

__device__ __forceinline__ uint32_t busy(uint32_t x, uint32_t n) {
  for (uint32_t i = 0; i < n; ++i) x = x * 1664525u + 1013904223u;
  return x;
}

// kAuto: the same program instrumented through the pass helpers
// (wgpf_dev::Scope / AsyncOp) instead of hand-placed records -- the store log
// must be identical.
template <bool kPow2, bool kAuto = false>
__global__ void k_selftest(uint8_t* profile, uint32_t cap, uint32_t iters,
                           uint32_t* sink, wgpf_dev::CtaTiming* timing) {
  extern __shared__ __align__(16) uint8_t buf[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t nwarps = blockDim.x >> 5;
  const uint64_t cta = blockIdx.x;
  if (threadIdx.x == 0 && timing) {
    timing[cta].smid = wgpf_dev::smid();
    timing[cta].streams = nwarps;
    timing[cta].gt_start = wgpf_dev::globaltimer();
    timing[cta].clk_start = wgpf_dev::clock32();
  }
  wgpf_dev::Recorder<kPow2> rec;
  rec.init(buf, warp, cap, lane == 0);
  uint32_t x = threadIdx.x + 7u * blockIdx.x;
  if constexpr (kAuto) {
    using Rec = wgpf_dev::Recorder<kPow2>;
    wgpf_dev::Scope<Rec> kernel(rec, R_KERNEL);
    for (uint32_t it = 0; it < iters; ++it) {
      {
        wgpf_dev::Scope<Rec> outer(rec, R_OUTER);
        x = busy(x, 16 + (it & 3));
        wgpf_dev::Scope<Rec> inner(rec, R_INNER);
        x = busy(x, 8 + warp);
      }
      wgpf_dev::AsyncOp<Rec> op(rec, R_ASYNC, R_ASYNC_WAIT);
      op.launch([&] { x = busy(x, 4); });
      op.wait([&] { x = busy(x, 32); });
    }
  } else {
  rec.start(R_KERNEL);
  for (uint32_t it = 0; it < iters; ++it) {
    rec.start(R_OUTER);
    x = busy(x, 16 + (it & 3));
    rec.start(R_INNER);
    x = busy(x, 8 + warp);
    rec.end(R_INNER);
    rec.end(R_OUTER);
    rec.start(R_ASYNC);  // S(X) before the launch
    x = busy(x, 4);
    rec.end(R_ASYNC);    // E(X) before the wait
    x = busy(x, 32);     // the wait
    rec.start(R_ASYNC_WAIT);
    rec.end(R_ASYNC_WAIT);
  }
  rec.end(R_KERNEL);
  }
  rec.close((uint32_t)cta, warp, cap);
  __syncthreads();
  const uint32_t bytes = wgpf_dev::smem_bytes(nwarps, cap);
  wgpf_dev::flush(buf, profile, cta, bytes, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0 && timing) {
    timing[cta].gt_end = wgpf_dev::globaltimer();
    timing[cta].clk_end = wgpf_dev::clock32();
  }
  if (x == 0xFFFFFFFFu) sink[0] = x;
}

// The selftest program through the C-style device API (wgpf_init /
// wgpf_record / wgpf_finalize): the same records as k_selftest.
__global__ void k_selftest_capi(uint8_t* profile, uint32_t cap, uint32_t iters,
                                uint32_t* sink) {
  extern __shared__ __align__(16) uint8_t buf[];
  const uint32_t warp = threadIdx.x >> 5;
  wgpf_recorder rec;
  wgpf_init(rec, buf, cap, warp);
  uint32_t x = threadIdx.x + 7u * blockIdx.x;
  wgpf_record_op(rec, true, R_KERNEL);
  for (uint32_t it = 0; it < iters; ++it) {
    wgpf_record_op(rec, true, R_OUTER);
    x = busy(x, 16 + (it & 3));
    wgpf_record_op(rec, true, R_INNER);
    x = busy(x, 8 + warp);
    wgpf_record_op(rec, false, R_INNER);
    wgpf_record_op(rec, false, R_OUTER);
    wgpf_record_op(rec, true, R_ASYNC);
    x = busy(x, 4);
    wgpf_record_op(rec, false, R_ASYNC);
    x = busy(x, 32);
    wgpf_record_op(rec, true, R_ASYNC_WAIT);
    wgpf_record_op(rec, false, R_ASYNC_WAIT);
  }
  wgpf_record_op(rec, false, R_KERNEL);
  wgpf_finalize(rec, buf, profile, blockIdx.x, warp, cap, blockDim.x >> 5);
  if (x == 0xFFFFFFFFu) sink[0] = x;
}

// Per-warp cycle cost of N record ops inside an ALU loop.
template <bool kRecord>
__global__ void k_record_cost(uint32_t n, uint64_t* cycles, uint32_t* sink) {
  extern __shared__ __align__(16) uint8_t buf[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  wgpf_dev::Recorder<true> rec;
  rec.init(buf, warp, 256, lane == 0);
  uint32_t x = threadIdx.x;
  __syncwarp();
  const uint64_t t0 = clock64();
  for (uint32_t i = 0; i < n; ++i) {
    if constexpr (kRecord) rec.start(1);
    x = x * 1664525u + 1013904223u;
    if constexpr (kRecord) rec.end(1);
    x = x * 1664525u + 1013904223u;
  }
  __syncwarp();
  const uint64_t t1 = clock64();
  if (lane == 0) cycles[blockIdx.x * (blockDim.x >> 5) + warp] = t1 - t0;
  if (x == 0xFFFFFFFFu) sink[0] = x;
}

// FinalizeOp cost: cycles from the CTA barrier after the last record to the
// end of the copy-out of a `bytes` profile buffer (per CTA, all CTAs of the
// grid flushing at once, as at the end of an instrumented kernel): 16-B
// vector stores by every thread (kBulk = false) or one cp.async.bulk by one
// thread (kBulk = true).
template <bool kBulk>
__global__ void k_flush_cost(uint8_t* profile, uint32_t bytes, uint64_t* cycles) {
  extern __shared__ __align__(16) uint8_t buf[];
  for (uint32_t i = threadIdx.x; i < bytes / 4u; i += blockDim.x)
    reinterpret_cast<uint32_t*>(buf)[i] = i * 2654435761u + blockIdx.x;
  __syncthreads();
  const uint64_t t0 = clock64();
  if constexpr (kBulk)
    wgpf_dev::flush_bulk(buf, profile, blockIdx.x, bytes, threadIdx.x, blockDim.x);
  else
    wgpf_dev::flush(buf, profile, blockIdx.x, bytes, threadIdx.x, blockDim.x);
  __syncthreads();
  const uint64_t t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// ---- scope-program interpreter ------------------------------------------------
// Runs a lowered scope program (p1.lower_scopes -> p1.program_encoding): warp
// w of every CTA executes body w -- START / END record ops, loops, ALU busy
// work -- through Recorder<kPow2, kFlush, kValidate>, with the loop boundaries
// and iteration signatures of wgpf_dev::Loop (the interpreter keeps its own
// loop stack, so it calls the Recorder's loop hooks directly, exactly as Loop
// does).  The vGPU analogue is Engine::step over a lowered body
// (vgpu.hpp:206-238, LoopBegin / LoopEnd :366-381).
constexpr uint32_t kProgLoops = 8;

template <bool kPow2, bool kFlush, bool kValidate>
__global__ void k_program(uint8_t* profile, uint32_t cap, const uint2* ops,
                          const uint32_t* body_off, uint32_t sig_mode,
                          unsigned long long* verr, uint32_t* sink) {
  extern __shared__ __align__(16) uint8_t buf[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t nwarps = blockDim.x >> 5;
  const uint32_t bytes = wgpf_dev::smem_bytes(nwarps, cap);
  // deterministic images: unwritten slots read as zero (as the vGPU's)
  for (uint32_t i = threadIdx.x; i < bytes / 8u; i += blockDim.x)
    reinterpret_cast<uint2*>(buf)[i] = make_uint2(0, 0);
  __syncthreads();
  wgpf_dev::Recorder<kPow2, kFlush, kValidate> rec;
  rec.init(buf, warp, cap, lane == 0);
  rec.validate_into(verr, blockIdx.x * nwarps + warp);
  if (sig_mode == 1) rec.hw_signature(warp);
  const uint2* b = ops + body_off[warp];
  const uint32_t n = body_off[warp + 1] - body_off[warp];
  uint32_t lpc[kProgLoops], lrem[kProgLoops], lit[kProgLoops], lsig[kProgLoops];
  uint32_t top = 0;
  uint32_t x = threadIdx.x + 7u * blockIdx.x;
  for (uint32_t pc = 0; pc < n;) {
    const uint2 o = b[pc];
    switch (o.x) {
      case 0:
        rec.start(o.y);
        ++pc;
        break;
      case 1:
        rec.end(o.y);
        ++pc;
        break;
      case 2:  // LoopBegin
        lpc[top] = pc + 1;
        lrem[top] = o.y;
        lit[top] = 0;
        lsig[top] = rec.sig;
        ++top;
        rec.loop_begin();
        if (sig_mode == 2) rec.iteration(0);
        ++pc;
        break;
      case 3: {  // LoopEnd
        const uint32_t t = top - 1;
        if (--lrem[t] > 0) {
          rec.loop_iteration_end();
          ++lit[t];
          if (sig_mode == 2) rec.iteration(lit[t]);
          pc = lpc[t];
        } else {
          rec.loop_end();
          rec.sig = lsig[t];
          --top;
          ++pc;
        }
        break;
      }
      default:
        x = busy(x, o.y);
        ++pc;
        break;
    }
  }
  rec.close(blockIdx.x, warp, cap);
  __syncthreads();
  wgpf_dev::flush(buf, profile, blockIdx.x, bytes, threadIdx.x, blockDim.x);
  if (x == 0xFFFFFFFFu) sink[0] = x;
}

// ---- loop-entry cost (vgpu.hpp:366-369; "+5 instructions") -------
// n entries of an inner loop of `trips` iterations (a runtime value: not
// unrolled), with or without a START/END pair in the inner body.  Per-warp
// cycles T(n, trips) = n (E + trips B): two runs, (n, 1) and (n / 2, 2), give
// the per-entry cost E = 2 (T(n, 1) - T(n / 2, 2)) / n, and the
// instrumentation's loop-entry cost is E(records) - E(no records).
template <bool kRecord>
__global__ void k_loop_entry(uint32_t n, uint32_t trips, uint64_t* cycles,
                             uint32_t* sink) {
  extern __shared__ __align__(16) uint8_t buf[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  wgpf_dev::Recorder<true> rec;
  rec.init(buf, warp, 256, lane == 0);
  uint32_t x = threadIdx.x;
  __syncwarp();
  const uint64_t t0 = clock64();
  for (uint32_t e = 0; e < n; ++e) {
#pragma unroll 1
    for (uint32_t i = 0; i < trips; ++i) {
      if constexpr (kRecord) rec.start(1);
      x = x * 1664525u + 1013904223u;
      if constexpr (kRecord) rec.end(1);
    }
    x ^= e;
  }
  __syncwarp();
  const uint64_t t1 = clock64();
  if (lane == 0) cycles[blockIdx.x * (blockDim.x >> 5) + warp] = t1 - t0;
  if (x == 0xFFFFFFFFu) sink[0] = x;
}

// ---- per-scope timing accuracy (2 % relative error) ---------------
// Every warp runs `scopes` scopes back to back, each a dependent chain of
// `chain` integer multiply-adds (deterministic latency, nothing to overlap);
// instrumented, each scope is one START / END pair.  Ground truth: the same
// kernel uninstrumented, timed by CUDA events at two scope counts -- the
// slope is the true per-scope time.  The record-derived scope durations
// (decoded, sync-corrected) are converted to ns with the SM clock rate of the
// CtaTiming side records.
// chase != null: the scope is a chain of dependent global loads through a
// random cycle (memory-latency scopes, L2 misses) instead of integer MADs.
template <bool kInstr>
__global__ void k_accuracy(uint8_t* profile, uint32_t cap, uint32_t scopes, uint32_t chain,
                           wgpf_dev::CtaTiming* timing, const uint32_t* chase,
                           uint32_t chase_mask, uint32_t* sink) {
  extern __shared__ __align__(16) uint8_t buf[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t nwarps = blockDim.x >> 5;
  if (threadIdx.x == 0 && timing) {
    timing[blockIdx.x].smid = wgpf_dev::smid();
    timing[blockIdx.x].streams = nwarps;
    timing[blockIdx.x].gt_start = wgpf_dev::globaltimer();
    timing[blockIdx.x].clk_start = wgpf_dev::clock32();
  }
  std::conditional_t<kInstr, wgpf_dev::Recorder<true>, wgpf_dev::NullRecorder> rec;
  rec.init(buf, warp, cap, lane == 0);
  uint32_t x = threadIdx.x + 1u, a = 1664525u + (blockIdx.x & 1u);
  if (chase) x = (x * 2654435761u + blockIdx.x * 40503u) & chase_mask;
  for (uint32_t s = 0; s < scopes; ++s) {
    rec.start(0);
    if (chase) {
      for (uint32_t i = 0; i < chain; ++i) x = __ldcg(chase + x);
    } else {
#pragma unroll 4
      for (uint32_t i = 0; i < chain; ++i) x = x * a + 1013904223u;
    }
    rec.end(0);
  }
  if constexpr (kInstr) {
    rec.close(blockIdx.x, warp, cap);
    __syncthreads();
    wgpf_dev::flush(buf, profile, blockIdx.x, wgpf_dev::smem_bytes(nwarps, cap), threadIdx.x,
                    blockDim.x);
  } else {
    __syncthreads();
  }
  // (the uninstrumented kernel keeps the CTA timing too: its cycles between
  // two scope counts are the ground truth in the SM's own clock)
  if (threadIdx.x == 0 && timing) {
    timing[blockIdx.x].gt_end = wgpf_dev::globaltimer();
    timing[blockIdx.x].clk_end = wgpf_dev::clock32();
  }
  if (x == 0xFFFFFFFFu) sink[0] = x;
}

}  // namespace

extern "C" int wgpf_p1_accuracy(uint32_t ctas, uint32_t warps, uint32_t scopes,
                                uint32_t chain, int instr, void* d_profile, uint32_t cap,
                                void* d_timing, const void* d_chase, uint32_t chase_mask,
                                void* stream) {
  const uint32_t* chase = static_cast<const uint32_t*>(d_chase);
  static uint32_t* sink = nullptr;
  if (!sink) cudaMalloc(&sink, 4);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (instr) {
    if (!cap || (cap & (cap - 1)) || cap < 2 * scopes) return 11;
    const uint32_t smem = wgpf_dev::smem_bytes(warps, cap);
    cudaFuncSetAttribute(k_accuracy<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_accuracy<true><<<ctas, warps * 32, smem, st>>>(static_cast<uint8_t*>(d_profile), cap,
                                                     scopes, chain,
                                                     static_cast<wgpf_dev::CtaTiming*>(d_timing),
                                                     chase, chase_mask, sink);
  } else {
    k_accuracy<false><<<ctas, warps * 32, 0, st>>>(
        nullptr, cap, scopes, chain, static_cast<wgpf_dev::CtaTiming*>(d_timing), chase,
        chase_mask, sink);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}

template <bool P, bool F, bool V>
static int launch_program(void* d_profile, uint32_t ctas, uint32_t nb, uint32_t cap,
                          uint32_t sig_mode, const void* ops, const void* offs,
                          void* verr, cudaStream_t st, uint32_t* sink) {
  const uint32_t smem = wgpf_dev::smem_bytes(nb, cap);
  cudaFuncSetAttribute(k_program<P, F, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  k_program<P, F, V><<<ctas, nb * 32, smem, st>>>(
      static_cast<uint8_t*>(d_profile), cap, static_cast<const uint2*>(ops),
      static_cast<const uint32_t*>(offs), sig_mode,
      static_cast<unsigned long long*>(verr), sink);
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}

// runs a lowered scope program (see k_program); d_verr: the 64-bit error word
// of debug-mode recorders (initialised to ~0 by the caller), or null
extern "C" int wgpf_p1_run_program(void* d_profile, uint32_t ctas, uint32_t n_bodies,
                                   uint32_t cap, int flush, int validate,
                                   uint32_t sig_mode, const void* d_ops,
                                   const void* d_offs, void* d_verr, void* stream) {
  static uint32_t* sink = nullptr;
  if (!sink) cudaMalloc(&sink, 4);
  if (!cap || !n_bodies || n_bodies > 32) return 11;
  if (validate && !d_verr) return 11;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool pow2 = !(cap & (cap - 1));
  const int k = (pow2 ? 1 : 0) | (flush ? 2 : 0) | (validate ? 4 : 0);
#define WGPF_PROG(P, F, V)                                                     \
  launch_program<P, F, V>(d_profile, ctas, n_bodies, cap, sig_mode, d_ops, d_offs, \
                          d_verr, st, sink)
  switch (k) {
    case 0: return WGPF_PROG(false, false, false);
    case 1: return WGPF_PROG(true, false, false);
    case 2: return WGPF_PROG(false, true, false);
    case 3: return WGPF_PROG(true, true, false);
    case 4: return WGPF_PROG(false, false, true);
    case 5: return WGPF_PROG(true, false, true);
    case 6: return WGPF_PROG(false, true, true);
    default: return WGPF_PROG(true, true, true);
  }
#undef WGPF_PROG
}

extern "C" int wgpf_p1_loop_entry(uint32_t n, uint32_t trips, uint32_t warps,
                                  int record, void* d_cycles, void* stream) {
  static uint32_t* sink = nullptr;
  if (!sink) cudaMalloc(&sink, 4);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint32_t smem = wgpf_dev::smem_bytes(warps, 256);
  auto* cyc = static_cast<uint64_t*>(d_cycles);
  if (record) {
    cudaFuncSetAttribute(k_loop_entry<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    k_loop_entry<true><<<1, warps * 32, smem, st>>>(n, trips, cyc, sink);
  } else {
    k_loop_entry<false><<<1, warps * 32, smem, st>>>(n, trips, cyc, sink);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}

// the selftest program through the C-style device API (pow2 caps)
extern "C" int wgpf_p1_selftest_capi(void* d_profile, uint32_t ctas, uint32_t warps_per_cta,
                                     uint32_t cap, uint32_t iters, void* stream) {
  static uint32_t* sink = nullptr;
  if (!sink) cudaMalloc(&sink, 4);
  if (!cap || (cap & (cap - 1))) return 11;
  const uint32_t smem = wgpf_dev::smem_bytes(warps_per_cta, cap);
  cudaFuncSetAttribute(k_selftest_capi, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_selftest_capi<<<ctas, warps_per_cta * 32, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<uint8_t*>(d_profile), cap, iters, sink);
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}

// the selftest program instrumented through the pass helpers (pow2 caps)
extern "C" int wgpf_p1_selftest_auto(void* d_profile, uint32_t ctas,
                                     uint32_t warps_per_cta, uint32_t cap,
                                     uint32_t iters, void* stream) {
  static uint32_t* sink = nullptr;
  if (!sink) cudaMalloc(&sink, 4);
  if (!cap || (cap & (cap - 1))) return 11;
  const uint32_t smem = wgpf_dev::smem_bytes(warps_per_cta, cap);
  cudaFuncSetAttribute(k_selftest<true, true>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_selftest<true, true><<<ctas, warps_per_cta * 32, smem,
                           reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<uint8_t*>(d_profile), cap, iters, sink, nullptr);
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}

extern "C" int wgpf_p1_selftest(void* d_profile, uint32_t ctas,
                                uint32_t warps_per_cta, uint32_t cap,
                                uint32_t iters, void* d_timing, void* stream) {
  static uint32_t* sink = nullptr;
  if (!sink) cudaMalloc(&sink, 4);
  const uint32_t smem = wgpf_dev::smem_bytes(warps_per_cta, cap);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool pow2 = cap && !(cap & (cap - 1));
  if (pow2) {
    cudaFuncSetAttribute(k_selftest<true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_selftest<true><<<ctas, warps_per_cta * 32, smem, st>>>(
        static_cast<uint8_t*>(d_profile), cap, iters, sink,
        static_cast<wgpf_dev::CtaTiming*>(d_timing));
  } else {
    cudaFuncSetAttribute(k_selftest<false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_selftest<false><<<ctas, warps_per_cta * 32, smem, st>>>(
        static_cast<uint8_t*>(d_profile), cap, iters, sink,
        static_cast<wgpf_dev::CtaTiming*>(d_timing));
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}

// cycles[warps] out; returns 0 on success.  record != 0 selects the
// instrumented loop.
extern "C" int wgpf_p1_record_cost(uint32_t n, uint32_t warps, int record,
                                   void* d_cycles, void* stream) {
  static uint32_t* sink = nullptr;
  if (!sink) cudaMalloc(&sink, 4);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint32_t smem = wgpf_dev::smem_bytes(warps, 256);
  if (record) {
    cudaFuncSetAttribute(k_record_cost<true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_record_cost<true><<<1, warps * 32, smem, st>>>(
        n, static_cast<uint64_t*>(d_cycles), sink);
  } else {
    k_record_cost<false><<<1, warps * 32, smem, st>>>(
        n, static_cast<uint64_t*>(d_cycles), sink);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}

// cycles[ctas] out (see k_flush_cost); bytes a multiple of 16.
extern "C" int wgpf_p1_flush_cost(uint32_t ctas, uint32_t threads, uint32_t bytes, int bulk,
                                  void* d_profile, void* d_cycles, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto* kfn = bulk ? k_flush_cost<true> : k_flush_cost<false>;
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  kfn<<<ctas, threads, bytes, st>>>(static_cast<uint8_t*>(d_profile), bytes,
                                    static_cast<uint64_t*>(d_cycles));
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}
