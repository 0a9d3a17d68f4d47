// k_count.cuh -- pass 1 of replay_image: per-stream decode checks, event
// counts and fast-path routing, one warp per stream, coalesced tag reads.
//
// decode_image (trace.hpp:222-251): capacity must equal the plan (:227-231),
// a flush stream may not claim more records than slots (:238-240), circular
// streams start at record_count % capacity (:243-246).
//
// Event count.  Every matched END yields one interval and every interval one
// event (a consumed wait marker cannot be malformed because unwrapped clocks
// are monotone, trace.hpp:262-269 + :455), so events = #END - dropped_heads.
// Under single-stack nesting (which the instrumentation pass guarantees,
// instrument.hpp:60-105, and which every suffix of a properly nested stream
// keeps) dropped_heads = -min(0, min_t Q(t)) with Q the running
// #START - #END.  Pass 2 verifies the single-stack assumption and reroutes any
// stream that violates it (SF_INVALID) to an exact recount.
//
// Routing: the thread-per-stream kernel (k_tps.cuh) takes streams with
// region ids < tps_regions and nesting <= tps_depth; other fast streams are
// listed for the warp-per-stream kernel (SF_WARP).
// Routing to the general path (SF_GENERAL): region ids >= fast_regions,
// nesting deeper than kMaxDepth, or a wait-marker START after z (below) that
// is not closed by the very next record (pass 2 could not decide whether it
// is ever closed).
//
// z = the last chronological position where the clamped depth
// D(t) = Q(t) - min(0, min_{k<=t} Q(k)) is 0: every START at or before z is
// closed later.
#pragma once

#include <type_traits>

#include "wgpf_dev.cuh"
#include "k_window.cuh"

namespace wgpf {

struct CountArgs {
  const uint8_t* body;
  uint64_t stride;      // 16 + 8 * plan.slots
  uint64_t n_streams;
  DevPlan plan;
  uint32_t* counts;
  int32_t* zpos;
  uint32_t* sflag;
  DevStatus* status;
  uint32_t fast_regions; // region ids below this may take the fast path
  uint32_t max_depth;    // nesting the fast path holds in shared memory
  uint32_t force_general;
  uint32_t tps_regions;  // thread-per-stream path: region ids below this
  uint32_t tps_depth;    //   and nesting up to this (0: path disabled)
  uint32_t deep_regions; // deep thread-per-stream path (SF_DEEP): ids below
  uint32_t deep_depth;   //   this, nesting up to this (0: path disabled)
  unsigned long long* warp_list;  // SF_WARP streams (not SF_DEEP)
  unsigned long long* warp_len;
  unsigned long long* deep_list;  // SF_WARP | SF_DEEP streams
  unsigned long long* deep_len;
  uint32_t wide_regions; // wide thread-per-stream path (k_tpsd<kWide>): the
  uint32_t wide_depth;   //   rest of the warp list with ids below this and
                         //   nesting up to this (0: path disabled)
  unsigned long long* wide_list;  // SF_WARP | SF_DEEP streams of the wide path
  unsigned long long* wide_len;
  uint32_t tma;          // k_count_tps: the body's tensor map is valid
  uint32_t list_general; // no thread-per-stream emit kernel (every stream is
                         // listed): SF_GENERAL streams go to the warp list
                         // too, whose kernel hands them to the general path
  uint64_t list_base;    // index of stream 0 of this body in the call's
                         // stream arrays (overlapped chunks): list entries
                         // and decode-error positions are call-global
};

__global__ void __launch_bounds__(256) k_count_fast(CountArgs a) {
  __shared__ uint8_t marker_region[256];
  for (uint32_t r = threadIdx.x; r < 256; r += blockDim.x)
    marker_region[r] =
        r < a.fast_regions ? class_is_marker(a.plan, a.plan.class_of[r]) : 0;
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint32_t le = lanemask_le();
  for (uint64_t s = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
       s < a.n_streams; s += warps) {
    const uint8_t* base = a.body + s * a.stride;
    const uint4 h = *reinterpret_cast<const uint4*>(base);  // 16-B header
    const uint32_t cnt = h.z, cap = h.w;
    uint32_t code = 0;
    if ((uint64_t)cap != a.plan.slots)
      code = DEC_CAP;
    else if (cnt > cap)
      code = a.plan.strategy == WGPF_STRATEGY_FLUSH ? DEC_FLUSH
                                                    : (cap == 0 ? DEC_ZERO : 0);
    if (code) {
      if (lane == 0) {
        a.counts[s] = 0;
        a.zpos[s] = -1;
        a.sflag[s] = SF_DECODE_ERR;
        atomicMin(&a.status->decode_err, ((unsigned long long)s << 2) | code);
        if (code == DEC_CAP) atomicAdd(&a.status->cap_mismatch, 1ull);
      }
      continue;
    }
    const uint32_t n = cnt <= cap ? cnt : cap;
    const uint32_t start = cnt <= cap ? 0u : cnt % cap;
    const uint32_t* tags = reinterpret_cast<const uint32_t*>(base + 16);
    int32_t q_in = 0;     // Q before the chunk
    int32_t run_min = 0;  // min(0, min Q so far)
    int32_t max_d = 0;
    uint32_t n_end = 0;
    int32_t z = -1;
    int64_t last_bad = -1;
    bool wide = false;
    bool tps_out = false;  // region id beyond the thread-per-stream tables
    bool deep_out = false; // region id beyond the deep kernel's tables
    bool wide_out = false; // region id beyond the wide kernel's tables
    bool prev_end = false;       // record c-1 is an END
    uint32_t pend_rid = kNone;   // lane-31 marker START awaiting its END
    auto chunk = [&](uint32_t c, uint32_t tag) {
      const uint32_t i = c + lane;
      const bool valid = i < n;
      const uint32_t rid = (tag >> 12) & (WGPF_MAX_REGIONS - 1u);
      const bool st = valid && (tag & WGPF_START_FLAG);
      const bool en = valid && !(tag & WGPF_START_FLAG);
      const bool in_range = rid < a.fast_regions;
      wide |= valid && !in_range;
      tps_out |= valid && rid >= a.tps_regions;
      deep_out |= valid && rid >= a.deep_regions;
      wide_out |= valid && rid >= a.wide_regions;
      const uint32_t smk = __ballot_sync(0xffffffffu, st);
      const uint32_t emk = __ballot_sync(0xffffffffu, en);
      const int32_t q = q_in + (int32_t)__popc(smk & le) - (int32_t)__popc(emk & le);
      const int32_t cmin = __reduce_min_sync(0xffffffffu, valid ? q : INT32_MAX);
      uint32_t zm;
      int32_t d;
      if (cmin >= run_min) {
        zm = __ballot_sync(0xffffffffu, valid && q == run_min);
        d = q - run_min;
      } else {  // a new running minimum inside the chunk: prefix-min scan
        int32_t pm = valid ? q : INT32_MAX;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, pm, o);
          if ((int)lane >= o) pm = min(pm, y);
        }
        const int32_t rm = min(run_min, pm);
        zm = __ballot_sync(0xffffffffu, valid && q == rm);
        d = q - rm;
        run_min = min(run_min, cmin);
      }
      max_d = max(max_d, __reduce_max_sync(0xffffffffu, valid ? d : 0));
      if (zm) z = (int32_t)(c + 31u - __clz(zm));
      // wait-marker STARTs right after an END that the next record does not
      // close (conservative: the marker class test is done in pass 2)
      // (the shuffle runs on every lane; selecting afterwards keeps the warp
      // converged -- a shuffle inside a lane-divergent ternary deadlocks)
      const uint32_t pe_up = __shfl_up_sync(0xffffffffu, (uint32_t)en, 1);
      const bool pe = lane == 0 ? prev_end : (bool)pe_up;
      const uint32_t t1 = __shfl_down_sync(0xffffffffu, tag, 1);
      const bool mk_start = st && pe && in_range && marker_region[rid];
      const bool closed_next = (lane < 31) && (i + 1 < n) &&
                               !(t1 & WGPF_START_FLAG) &&
                               ((t1 >> 12) & (WGPF_MAX_REGIONS - 1u)) == rid;
      const uint32_t bm = __ballot_sync(0xffffffffu, mk_start && !closed_next && lane < 31);
      if (pend_rid != kNone) {  // lane 31 of the previous chunk
        const uint32_t t0 = __shfl_sync(0xffffffffu, tag, 0);
        const bool ok0 = n > c && !(t0 & WGPF_START_FLAG) &&
                         ((t0 >> 12) & (WGPF_MAX_REGIONS - 1u)) == pend_rid;
        if (!ok0) last_bad = max(last_bad, (int64_t)c - 1);
      }
      if (bm) last_bad = max(last_bad, (int64_t)(c + 31u - __clz(bm)));
      const uint32_t p31 = __shfl_sync(0xffffffffu, (mk_start && lane == 31) ? rid : kNone, 31);
      pend_rid = p31;
      prev_end = __shfl_sync(0xffffffffu, (uint32_t)en, 31);
      n_end += __popc(emk);
      q_in += (int32_t)__popc(smk) - (int32_t)__popc(emk);
    };
    // 8 chunks (256 records) of tags in flight per warp, then process
    constexpr uint32_t G = 8;
    for (uint32_t c0 = 0; c0 < n; c0 += 32 * G) {
      uint32_t tg[G];
#pragma unroll
      for (uint32_t k = 0; k < G; ++k) {
        const uint32_t i = c0 + 32 * k + lane;
        uint32_t slot = start + i;
        if (slot >= cap) slot -= cap;
        tg[k] = i < n ? __ldg(tags + 2ull * slot) : 0u;
      }
#pragma unroll
      for (uint32_t k = 0; k < G; ++k)
        if (c0 + 32 * k < n) chunk(c0 + 32 * k, tg[k]);
    }
    if (pend_rid != kNone) last_bad = max(last_bad, (int64_t)n - 1);
    wide = __any_sync(0xffffffffu, wide);
    tps_out = __any_sync(0xffffffffu, tps_out);
    deep_out = __any_sync(0xffffffffu, deep_out);
    wide_out = __any_sync(0xffffffffu, wide_out);
    if (lane == 0) {
      a.counts[s] = n_end - (uint32_t)(-run_min);
      a.zpos[s] = z;
      const bool general = wide || a.force_general ||
                           max_d > (int32_t)a.max_depth || last_bad > (int64_t)z;
      const bool warp = a.tps_depth != 0 && !general && (tps_out || max_d > (int32_t)a.tps_depth);
      const bool deep = warp && !deep_out && max_d <= (int32_t)a.deep_depth;
      const bool wide = warp && !deep && !wide_out && max_d <= (int32_t)a.wide_depth;
      a.sflag[s] = general ? SF_GENERAL
                           : (warp ? (SF_WARP | (deep || wide ? SF_DEEP : 0u)) : 0u);
      if (warp && deep)
        a.deep_list[atomicAdd(a.deep_len, 1ull)] = s;
      else if (wide)
        a.wide_list[atomicAdd(a.wide_len, 1ull)] = s;
      else if (warp || (general && a.list_general))
        a.warp_list[atomicAdd(a.warp_len, 1ull)] = s;
    }
  }
}


// Thread-per-stream pass 1 (same outputs as k_count_fast): lane l of a warp
// owns stream 32 b + l and walks its records sequentially, windows staged in
// shared memory (k_window.cuh).  Used when the capacity is even and at most
// kTpsMaxSlots (the record windows need 16-B chunk alignment).
//
// Two instantiations: the stand-alone pass (kCountWarps warps per CTA, as
// many CTAs as fit) and the co-resident one of the overlapped replay
// (capi.cu replay_overlapped): one warp per CTA at <= 64 registers, two CTAs
// per SM, small enough to run beside the emit kernel's CTA on every SM, so
// pass 1 of chunk k+1 uses the issue slots and DRAM bandwidth that k_tps of
// chunk k leaves idle.
#ifndef WGPF_COUNT_WARPS
#define WGPF_COUNT_WARPS 4
#endif
constexpr uint32_t kCountWarps = WGPF_COUNT_WARPS;
constexpr uint32_t kCountW = 16;  // records per window: 128-B runs per stream
#ifndef WGPF_COUNT_UNROLL
#define WGPF_COUNT_UNROLL 16
#endif
constexpr int kCountUnroll = WGPF_COUNT_UNROLL;
#ifndef WGPF_COUNT_MINB
#define WGPF_COUNT_MINB 4  // launch bound: 4 CTAs per SM -> <= 128 registers (ptxas
                           // then picks 96: 20 warps / SM; unbounded it took 118 and
                           // 16 warps: config 4 1.67 -> 1.61 ms, config 5 1.97 -> 1.88)
#endif
constexpr uint32_t kCountMinBlocks = WGPF_COUNT_MINB;
#ifndef WGPF_COUNT_CO_UNROLL
#define WGPF_COUNT_CO_UNROLL 8
#endif
constexpr int kCountCoUnroll = WGPF_COUNT_CO_UNROLL;
#ifndef WGPF_COUNT_CO_CTAS
#define WGPF_COUNT_CO_CTAS 2  // co-resident pass-1 CTAs (one warp each) per SM
#endif
constexpr uint32_t kCountCoCtas = WGPF_COUNT_CO_CTAS;
#ifndef WGPF_COUNT_CO_MINB
#define WGPF_COUNT_CO_MINB 32  // launch bound: 32 one-warp CTAs per SM -> <= 64 registers
#endif
constexpr uint32_t kCountCoMinBlocks = WGPF_COUNT_CO_MINB;
using CountWin = RecWindowsT<kCountW>;

// tm: the body as a TMA tensor with box {CountWin::kTpsPitch / 4, 32};
// tm_tail: the same without L2 promotion, for windows within 256 B of the
// streams' last records (promotion there would pull the unused slots)
template <uint32_t kWarps, int kUnroll, uint32_t kMinBlocks>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks)
    k_count_tps(CountArgs a, const __grid_constant__ CUtensorMap tm,
                const __grid_constant__ CUtensorMap tm_tail) {
  __shared__ uint8_t marker_region[256];
  __shared__ __align__(128) uint8_t recbuf[kWarps][2 * 32 * CountWin::kTpsPitch];
  __shared__ __align__(8) unsigned long long wbar[kWarps][2];
  for (uint32_t r = threadIdx.x; r < 256; r += blockDim.x)
    marker_region[r] =
        r < a.fast_regions ? class_is_marker(a.plan, a.plan.class_of[r]) : 0;
  __syncthreads();
  uint32_t mbits = 0;  // marker regions among ids < 32
  for (uint32_t r = 0; r < 32; ++r) mbits |= (uint32_t)marker_region[r] << r;
  const uint32_t FULL = 0xffffffffu;
  const uint32_t lane = lane_id();
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t cap = (uint32_t)a.plan.slots;
  CountWin win;
  win.init(recbuf[w], lane, a.stride, cap);
  const uint32_t s_bar = smem_addr(&wbar[w][0]);  // + 8 * buffer
  const uint32_t s_buf = smem_addr(recbuf[w]);
  if (a.tma && lane == 0) {
    win_bar_init(s_bar);
    win_bar_init(s_bar + 8u);
    win_bar_fence();
  }
  __syncwarp();
  uint32_t bphase = 0;
  const uint64_t wstep = (uint64_t)gridDim.x * kWarps;
  for (uint64_t b = (uint64_t)blockIdx.x * kWarps + w; b * 32 < a.n_streams;
       b += wstep) {
    const uint64_t s = b * 32 + lane;
    const bool live = s < a.n_streams;
    uint4 h = make_uint4(0u, 0u, 0u, cap);
    if (live) h = *reinterpret_cast<const uint4*>(a.body + s * a.stride);
    const uint32_t cnt = h.z, hcap = h.w;
    // decode_image checks (trace.hpp:227-240)
    uint32_t code = 0;
    if (live) {
      if (hcap != cap)
        code = DEC_CAP;
      else if (cnt > hcap)
        code = a.plan.strategy == WGPF_STRATEGY_FLUSH ? DEC_FLUSH : (hcap == 0 ? DEC_ZERO : 0);
      if (code) {
        a.counts[s] = 0;
        a.zpos[s] = -1;
        a.sflag[s] = SF_DECODE_ERR;
        atomicMin(&a.status->decode_err, ((unsigned long long)(s + a.list_base) << 2) | code);
        if (code == DEC_CAP) atomicAdd(&a.status->cap_mismatch, 1ull);
      }
    }
    const bool act = live && !code;
    const uint32_t n = act ? (cnt <= cap ? cnt : cap) : 0u;
    const uint32_t start = act && cnt > cap ? cnt % cap : 0u;
    const uint32_t nmax = __reduce_max_sync(FULL, n);
    if (nmax == 0) {
      if (act) {
        a.counts[s] = 0;
        a.zpos[s] = -1;
        a.sflag[s] = a.force_general ? SF_GENERAL : 0u;
      }
      continue;
    }
    const bool tmab = a.tma && __all_sync(FULL, start == 0u);
    const uint32_t ntail = __reduce_min_sync(FULL, act ? n : 0xFFFFFFFFu);
    auto issue = [&](uint32_t bs, uint32_t c0) {
      if (tmab) {
        if (lane == 0)
          win_tma(s_buf + bs * (32u * CountWin::kTpsPitch),
                  c0 + CountWin::kTpsPitch / 8u + 32u <= ntail ? &tm : &tm_tail,
                  s_bar + 8u * bs, (int)(4u + 2u * c0), (int)(b * 32),
                  32u * CountWin::kTpsPitch);
      } else {
        win.issue(bs, c0);
      }
    };
    if (!tmab) win.begin(a.body + b * 32 * a.stride, start, n);
    const uint2* slots = reinterpret_cast<const uint2*>(a.body + (act ? s : 0) * a.stride + 16);
    uint32_t t0 = 0, t1 = 0;  // tags of records i, i+1
    if (n > 0) t0 = slots[start].x;
    if (n > 1) t1 = slots[start + 1 < cap ? start + 1 : start + 1 - cap].x;
    issue(0, 2);
    cp_async_commit();
    int32_t q = 0, run_min = 0, max_d = 0, z = -1, last_bad = -1;
    uint32_t maxrid = 0;  // region-id range: fast / thread-per-stream routing
    bool prev_end = false;
    // kFull: positions i, i+1 exist on every lane -- no bounds predicates
    auto step = [&](auto full, uint32_t i, uint32_t t2) {
      constexpr bool kFull = decltype(full)::value;
      const bool valid = kFull || i < n;
      const bool isS = (int32_t)t0 < 0;
      const uint32_t rid = (t0 >> 12) & (WGPF_MAX_REGIONS - 1u);
      maxrid = valid ? max(maxrid, rid) : maxrid;
      q += valid ? 2 * (int32_t)(t0 >> 31) - 1 : 0;  // START +1, END -1
      run_min = min(run_min, q);
      const int32_t d = q - run_min;
      z = (valid && d == 0) ? (int32_t)i : z;
      max_d = max(max_d, d);
      // a wait-marker START right after an END that the next record does
      // not close: only z can tell whether it is ever closed
      uint32_t mk;
      if (rid < 32u)
        mk = (mbits >> rid) & 1u;
      else
        mk = rid < a.fast_regions ? marker_region[rid & 255u] : 0u;
      const bool mk_start = valid && isS && prev_end && mk;
      const bool closed_next = (kFull || i + 1 < n) && (int32_t)t1 >= 0 &&
                               ((t1 >> 12) & (WGPF_MAX_REGIONS - 1u)) == rid;
      last_bad = (mk_start && !closed_next) ? (int32_t)i : last_bad;
      prev_end = valid && !isS;
      t0 = t1;
      t1 = t2;
    };
    const uint32_t nmin = __reduce_min_sync(FULL, act ? n : 0u);
    for (uint32_t w0 = 0; w0 < nmax; w0 += kCountW) {
      const uint32_t bsel = (w0 / kCountW) & 1u;
      if (w0 + kCountW < nmax) issue(bsel ^ 1u, w0 + kCountW + 2u);
      if (tmab) {
        win_wait(s_bar + 8u * bsel, (bphase >> bsel) & 1u);
        bphase ^= 1u << bsel;
      } else {
        cp_async_commit();
        cp_async_wait1();
      }
      __syncwarp();
      const uint2* rec = win.lane_records(bsel, lane, start);
      if (w0 + kCountW + 1u <= nmin) {
#pragma unroll kUnroll
        for (uint32_t j = 0; j < kCountW; ++j) step(std::true_type{}, w0 + j, rec[j].x);
      } else {
#pragma unroll 1
        for (uint32_t j = 0; j < kCountW; ++j) step(std::false_type{}, w0 + j, rec[j].x);
      }
      __syncwarp();
    }
    // #START + #END = n and #START - #END = q
    const uint32_t n_end = (n - (uint32_t)q) >> 1;
    const bool wide = n && maxrid >= a.fast_regions;
    const bool tps_out = n && maxrid >= a.tps_regions;
    bool to_deep = false, to_warp = false, to_wide = false;
    if (act) {
      a.counts[s] = n_end - (uint32_t)(-run_min);
      a.zpos[s] = z;
      const bool general = wide || a.force_general || max_d > (int32_t)a.max_depth ||
                           last_bad > z;
      const bool warp = a.tps_depth != 0 && !general &&
                        (tps_out || max_d > (int32_t)a.tps_depth);
      const bool deep = warp && !(n && maxrid >= a.deep_regions) &&
                        max_d <= (int32_t)a.deep_depth;
      const bool wide = warp && !deep && !(n && maxrid >= a.wide_regions) &&
                        max_d <= (int32_t)a.wide_depth;
      a.sflag[s] = general ? SF_GENERAL
                           : (warp ? (SF_WARP | (deep || wide ? SF_DEEP : 0u)) : 0u);
      to_deep = warp && deep;
      to_wide = wide;
      to_warp = (warp && !deep && !wide) || (general && a.list_general);
    }
    // warp-aggregated appends: one atomic per warp, the batch's listed
    // streams stay consecutive and in stream order (coalesced window copies
    // in the list kernels)
    const uint32_t lt = lanemask_lt();
    const uint32_t dm = __ballot_sync(FULL, to_deep);
    if (dm) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(a.deep_len, (unsigned long long)__popc(dm));
      base = __shfl_sync(FULL, base, 0);
      if (to_deep) a.deep_list[base + __popc(dm & lt)] = s + a.list_base;
    }
    const uint32_t vm = __ballot_sync(FULL, to_wide);
    if (vm) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(a.wide_len, (unsigned long long)__popc(vm));
      base = __shfl_sync(FULL, base, 0);
      if (to_wide) a.wide_list[base + __popc(vm & lt)] = s + a.list_base;
    }
    const uint32_t wm = __ballot_sync(FULL, to_warp);
    if (wm) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(a.warp_len, (unsigned long long)__popc(wm));
      base = __shfl_sync(FULL, base, 0);
      if (to_warp) a.warp_list[base + __popc(wm & lt)] = s + a.list_base;
    }
  }
}

}  // namespace wgpf
