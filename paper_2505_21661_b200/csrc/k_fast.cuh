// k_fast.cuh -- pass 2 of replay_image, warp-cooperative: one warp per
// stream, 32 chronological records per step (lane t holds record c + t).
//
// Per step, with ballots / shuffles / match.any instead of a sequential
// stack walk:
//   unwrap_clock (trace.hpp:257-272)  u = hi:v where hi counts the mod-2^32
//       wraps, i.e. ballot(v_t < v_{t-1}) prefix popcounts.
//   pair_records (trace.hpp:294-346)  clamped depth D from ballot prefix
//       counts; a START opens level D, an END closes level D_before; the END's
//       partner is the last START at the same level: match.any on the level,
//       highest START lane below, else the per-level table in shared memory
//       (carried across steps).  The partner's region must equal the END's
//       (single-stack nesting); otherwise the stream is recounted exactly.
//       Iteration numbers: lanes of a region meet through a shared bit mask
//       (atomicOr) + per-region counters.
//   replay (trace.hpp:398-487)  sync correction, wait markers (the marker
//       START at end_pos + 1, closed either immediately or because it lies at
//       or before the stream's last zero-depth position z from pass 1),
//       orphans (staged in a per-warp HBM scratch, written last).
//   region_stats (pipeline.hpp:114-133) + histograms: per-lane register
//       accumulators flushed on a class change, one shared histogram
//       increment per event; per-CTA totals flushed to HBM at exit.
// Events are written at offsets from the pass-1 scan, coalesced per step.
#pragma once

#include "wgpf_dev.cuh"

namespace wgpf {

constexpr uint32_t kFastRegions = 256;  // region ids handled by the fast path
constexpr uint32_t kMaxDepth = 64;      // nesting levels in shared memory
constexpr uint32_t kFastWarps = 8;      // warps per CTA

struct FastArgs {
  const uint8_t* body;
  uint64_t stride;
  uint64_t n_streams;
  uint64_t stream_base;
  DevPlan plan;
  DevStats stats;
  DevStatus* status;
  const uint32_t* counts;
  const int32_t* zpos;
  uint32_t* sflag;
  const uint64_t* offsets;
  wgpf_event* events;
  uint64_t events_cap;
  uint64_t record_cost;
  wgpf_event* orphan_scratch;  // per warp: (cap / 2 + 1) events
  uint32_t cap;
  uint32_t fast_regions;
  uint32_t no_stats;
  unsigned long long* general_list;  // streams left for the general path
  unsigned long long* general_len;
  // list mode: only the streams list[0 .. *list_len) (pass 1's SF_WARP
  // streams; the thread-per-stream kernel handles the rest)
  const unsigned long long* list;
  const unsigned long long* list_len;
  uint32_t tps_regions;  // k_tps: region ids in its tables
  uint32_t tma;          // k_tps: the tensor map of the body is valid
  unsigned long long* batch_ctr;  // k_tps: dynamic batch counter (zeroed)
  uint32_t group;        // k_tps: streams per block W (lane l of batch (j, w)
                         // takes stream (32 j + l) W + w; 1 = consecutive)
  uint32_t list_general; // list kernels hand their SF_GENERAL entries to the
                         // general path (no k_tps pass to collect them)
  unsigned long long* deep_rep;  // k_tpsd: per-CTA count / sum / histogram
                                 // replicas (zeroed; summed by k_deep_reduce)
  uint64_t list_base;    // k_tps over one chunk of the call's streams
                         // (overlapped replay): general-list entries are
                         // call-global stream indices
};

struct LevelEntry {  // last START seen at a nesting level
  uint32_t lo;       // low 32 bits of the unwrapped clock (= raw payload)
  uint32_t hi;       // high bits
  uint32_t pos;      // chronological position
  uint32_t info;     // region | consumable << 31
};

struct FastSmem {
  SmemStats st;
  uint32_t cinfo[kFastRegions];  // class | marker << 31
  uint32_t wcls[kFastRegions];   // class of label + ".wait" (or kNone)
  LevelEntry lvl[kFastWarps][kMaxDepth];
  uint32_t cnt[kFastWarps][kFastRegions];
  uint32_t rmask[kFastWarps][kFastRegions];  // lanes ending a region this step
  unsigned long long warn[4];
  unsigned long long bar[kFastWarps][2];  // staging mbarriers (kStage)
};

// Staging: each warp double-buffers whole streams (header + slots) in shared
// memory; lane 0 issues the next stream's TMA bulk copy (cp.async.bulk,
// completion on an mbarrier) before the current one is processed, so every
// warp keeps one stream-sized read in flight.
__device__ inline void stage_issue(unsigned long long* bar, void* dst,
                                   const void* src, uint32_t bytes) {
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
      "[%1], %2, [%3];" ::"r"(d),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(b)
      : "memory");
}

__device__ inline void stage_wait(unsigned long long* bar, uint32_t parity) {
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}

__device__ inline void store_event(wgpf_event* dst, uint64_t st, uint64_t en,
                                   uint32_t region, uint32_t it, uint32_t blk,
                                   uint32_t wg) {
  stg256(dst, make_uint4((uint32_t)st, (uint32_t)(st >> 32), (uint32_t)en, (uint32_t)(en >> 32)),
         make_uint4(region, it, blk, wg));
}

// Group-aggregated statistics update for one event per participating lane.
__device__ inline void fast_stats(FastSmem& sm, const DevStats& st,
                                  DevStatus* status, bool part, uint32_t cls,
                                  uint32_t d, unsigned long long key) {
  // Warp-uniform loop over the distinct classes present (and, per class, the
  // distinct histogram bins): only full-mask ballots / shuffles / reductions,
  // which stay on the converged fast path (a reduction over a match.any
  // group mask lowers to a serialised WARPSYNC.COLLECTIVE loop).
  const uint32_t FULL = 0xffffffffu;
  const uint32_t bin = hist_bin(d);
  const uint32_t lane = lane_id();
  uint32_t rem = __ballot_sync(FULL, part);
  while (rem) {
    const uint32_t ld = __ffs(rem) - 1u;  // lowest lane: smallest event index
    const uint32_t c = __shfl_sync(FULL, cls, ld);
    const bool mine = part && cls == c;
    const uint32_t m = __ballot_sync(FULL, mine);
    const uint32_t lo = __reduce_add_sync(FULL, mine ? (d & 0xFFFFu) : 0u);
    const uint32_t hi = __reduce_add_sync(FULL, mine ? (d >> 16) : 0u);
    const uint32_t mn = __reduce_min_sync(FULL, mine ? d : 0xFFFFFFFFu);
    const uint32_t mx = __reduce_max_sync(FULL, mine ? d : 0u);
    const bool dense = c < kSmemClasses && c < st.K;
    int slot = -1;
    if (lane == ld) {
      const uint32_t n = __popc(m);
      const unsigned long long sum =
          (unsigned long long)lo + ((unsigned long long)hi << 16);
      if (dense) {
        sadd64(&sm.st.count[c], (unsigned long long)n);
        sadd64(&sm.st.sum[c], sum);
        atomicMin(&sm.st.min[c], mn);
        atomicMax(&sm.st.max[c], mx);
        smin64(&sm.st.first[c], key);
      } else {
        slot = stats_slot(st, c, &status->synth_overflow);
        if (slot >= 0) {
          atomicAdd(&st.count[slot], (unsigned long long)n);
          atomicAdd(&st.sum[slot], sum);
          atomicMin(&st.min[slot], (unsigned long long)mn);
          atomicMax(&st.max[slot], (unsigned long long)mx);
          atomicMin(&st.first[slot], key);
        }
      }
    }
    slot = __shfl_sync(FULL, slot, ld);
    uint32_t hb = m;
    while (hb) {
      const uint32_t bl = __ffs(hb) - 1u;
      const uint32_t b = __shfl_sync(FULL, bin, bl);
      const uint32_t mb = __ballot_sync(FULL, mine && bin == b);
      if (lane == bl) {
        if (dense)
          atomicAdd(&sm.st.hist[c * WGPF_HIST_BINS + b], (uint32_t)__popc(mb));
        else if (slot >= 0)
          atomicAdd(&st.hist[(uint64_t)slot * WGPF_HIST_BINS + b],
                    (unsigned long long)__popc(mb));
      }
      hb &= ~mb;
    }
    rem &= ~m;
  }
}

// Per-lane register accumulator for one label class: events reaching a lane
// mostly repeat their class (periodic scope patterns), so count / sum / min /
// max / first key accumulate in registers and reach shared memory only when
// the lane's class changes (and once at kernel exit).
struct LaneAcc {
  uint32_t cls, cnt, mn, mx;
  unsigned long long sum, first;
};

__device__ inline void acc_init(LaneAcc& a) {
  a.cls = kNone;
  a.cnt = 0;
}

__device__ inline void acc_flush(LaneAcc& a, FastSmem& sm, const DevStats& st,
                                 DevStatus* status) {
  if (!a.cnt) return;
  if (a.cls < kSmemClasses && a.cls < st.K) {
    sadd64(&sm.st.count[a.cls], (unsigned long long)a.cnt);
    sadd64(&sm.st.sum[a.cls], a.sum);
    atomicMin(&sm.st.min[a.cls], a.mn);
    atomicMax(&sm.st.max[a.cls], a.mx);
    smin64(&sm.st.first[a.cls], a.first);
  } else {
    const int slot = stats_slot(st, a.cls, &status->synth_overflow);
    if (slot >= 0) {
      atomicAdd(&st.count[slot], (unsigned long long)a.cnt);
      atomicAdd(&st.sum[slot], a.sum);
      atomicMin(&st.min[slot], (unsigned long long)a.mn);
      atomicMax(&st.max[slot], (unsigned long long)a.mx);
      atomicMin(&st.first[slot], a.first);
    }
  }
  a.cnt = 0;
}

// One event per participating lane: register accumulators per class (flushed
// on a class change), one shared histogram increment.
__device__ inline void lane_stats(LaneAcc& a, FastSmem& sm, const DevStats& st,
                                  DevStatus* status, bool part, uint32_t cls,
                                  uint32_t d, unsigned long long key) {
  if (!part) return;
  const uint32_t bin = hist_bin(d);
  // one shared increment per event (same-address increments of a warp are
  // aggregated by the hardware; match.any grouping cost more than it saved)
  if (cls < kSmemClasses && cls < st.K) {
    atomicAdd(&sm.st.hist[cls * WGPF_HIST_BINS + bin], 1u);
  } else {
    const int slot = stats_slot(st, cls, &status->synth_overflow);
    if (slot >= 0)
      atomicAdd(&st.hist[(uint64_t)slot * WGPF_HIST_BINS + bin], 1ull);
  }
  if (cls != a.cls) {
    acc_flush(a, sm, st, status);
    a.cls = cls;
    a.sum = 0;
    a.mn = 0xFFFFFFFFu;
    a.mx = 0;
    a.first = key;
  }
  ++a.cnt;
  a.first = min(a.first, key);
  a.sum += d;
  a.mn = min(a.mn, d);
  a.mx = max(a.mx, d);
}

// Shared-memory bytes of k_fast_emit<kStage> (staging: 2 buffers per warp).
__host__ __device__ inline uint32_t fast_stage_stride(uint64_t stride) {
  return (uint32_t)((stride + 127) & ~127ull);
}
__host__ inline size_t fast_smem_bytes(bool stage, uint64_t stride) {
  size_t b = (sizeof(FastSmem) + 127) & ~size_t(127);
  if (stage) b += (size_t)kFastWarps * 2 * fast_stage_stride(stride);
  return b;
}

template <bool kStage>
__global__ void __launch_bounds__(kFastWarps * 32) k_fast_emit(FastArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  FastSmem& sm = *reinterpret_cast<FastSmem*>(smem_raw);
  const uint32_t lane = lane_id();
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t sstride = fast_stage_stride(a.stride);
  uint8_t* stage = smem_raw + ((sizeof(FastSmem) + 127) & ~size_t(127)) +
                   (size_t)w * 2 * sstride;
  if (kStage && lane == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(&sm.bar[w][b]))));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!a.no_stats) smem_stats_init(sm.st);
  for (uint32_t r = threadIdx.x; r < kFastRegions; r += blockDim.x) {
    uint32_t ci = kNone, wc = kNone;
    if (r < a.fast_regions) {
      const uint32_t c = a.plan.class_of[r];
      ci = c | (class_is_marker(a.plan, c) ? 0x80000000u : 0u);
      wc = c < a.plan.K ? a.plan.wait_class[c] : kNone;
    }
    sm.cinfo[r] = ci;
    sm.wcls[r] = wc;
  }
  if (threadIdx.x < 4) sm.warn[threadIdx.x] = 0;
  __syncthreads();
  const bool abort_all = a.status->decode_err != kNoErr;
  LevelEntry* lvl = sm.lvl[w];
  uint32_t* cnt = sm.cnt[w];
  uint32_t* rmask = sm.rmask[w];
  for (uint32_t r = lane; r < kFastRegions; r += 32) rmask[r] = 0u;
  const uint64_t gw = (uint64_t)blockIdx.x * kFastWarps + w;
  wgpf_event* orphans = a.orphan_scratch + gw * (a.cap / 2 + 1);
  const uint32_t lt = lanemask_lt(), le = lanemask_le();
  const uint64_t cost = a.record_cost;
  uint32_t w_drop = 0, w_tail = 0, w_flag = 0, w_mal = 0;
  LaneAcc acc_e, acc_w;  // exec / orphan events, wait events
  acc_init(acc_e);
  acc_init(acc_w);

  const uint64_t wstep = (uint64_t)gridDim.x * kFastWarps;
  const uint64_t n_iter = a.list ? *a.list_len : a.n_streams;
  auto sid = [&](uint64_t t) -> uint64_t { return a.list ? a.list[t] : t; };
  uint32_t sbuf = 0, sphase = 0;  // staging buffer in use, parity bits
  if (kStage && !abort_all && lane == 0 && gw < n_iter)
    stage_issue(&sm.bar[w][0], stage, a.body + sid(gw) * a.stride, (uint32_t)a.stride);
  for (uint64_t t = gw; !abort_all && t < n_iter; t += wstep) {
    const uint64_t s = sid(t);
    if constexpr (kStage) {
      // prefetch the warp's next stream into the other buffer
      __syncwarp();
      if (lane == 0 && t + wstep < n_iter)
        stage_issue(&sm.bar[w][sbuf ^ 1], stage + (sbuf ^ 1) * sstride,
                    a.body + sid(t + wstep) * a.stride, (uint32_t)a.stride);
      stage_wait(&sm.bar[w][sbuf], (sphase >> sbuf) & 1u);
      sphase ^= 1u << sbuf;
    }
    const uint8_t* base =
        kStage ? stage + sbuf * sstride : a.body + s * a.stride;
    if constexpr (kStage) sbuf ^= 1;
    const uint32_t flag = a.sflag[s];
    if (flag & (SF_DECODE_ERR | SF_GENERAL)) {
      if ((flag & SF_GENERAL) && lane == 0 && (!a.list || a.list_general)) {
        const unsigned long long k = atomicAdd(a.general_len, 1ull);
        a.general_list[k] = s;
      }
      continue;
    }
    const uint4 h = *reinterpret_cast<const uint4*>(base);
    const uint32_t cntw = h.z, cap = h.w;
    const uint32_t n = cntw <= cap ? cntw : cap;
    const uint32_t start = cntw <= cap ? 0u : cntw % cap;
    const uint32_t blk = h.x, wg = h.y;
    const int32_t z = a.zpos[s];
    const uint32_t want = a.counts[s];
    const uint64_t off = a.offsets[s];
    const uint64_t gs = s + a.stream_base;
    const uint2* slots = reinterpret_cast<const uint2*>(base + 16);
    for (uint32_t r = lane; r < a.fast_regions; r += 32) cnt[r] = 0;

    auto load = [&](uint32_t c) -> uint2 {
      const uint32_t i = c + lane;
      if (i >= n) return make_uint2(0u, 0u);
      uint32_t slot = start + i;
      if (slot >= cap) slot -= cap;
      return slots[slot];
    };

    uint2 rc = load(0);
    uint32_t hi = 0, vprev = 0;  // unwrap carry
    int32_t D = 0;               // clamped depth before the chunk
    uint64_t kb = 0;             // base events emitted
    uint32_t n_orph = 0;
    bool prev_end_matched = false;  // record c-1 is a matched END
    uint32_t prev_rid = 0;          //   its region
    bool bad = false;
    __syncwarp();

    for (uint32_t c = 0; c < n; c += 32) {
      __syncwarp();                   // level / counter tables of chunk c-32
      const uint2 rn = load(c + 32);  // prefetch the next chunk
      const uint32_t i = c + lane;
      const bool valid = i < n;
      const uint32_t tag = rc.x, v = rc.y;
      const bool st = valid && (tag & WGPF_START_FLAG);
      const bool en = valid && !(tag & WGPF_START_FLAG);
      const uint32_t rid = (tag >> 12) & (WGPF_MAX_REGIONS - 1u);

      // ---- unwrap ---------------------------------------------------------
      uint32_t vp = __shfl_up_sync(0xffffffffu, v, 1);
      if (lane == 0) vp = vprev;
      const uint32_t wm = __ballot_sync(0xffffffffu, valid && v < vp);
      const uint32_t my_hi = hi + __popc(wm & le);

      // ---- clamped depth --------------------------------------------------
      const uint32_t smk = __ballot_sync(0xffffffffu, st);
      const uint32_t emk = __ballot_sync(0xffffffffu, en);
      const int32_t q = D + (int32_t)__popc(smk & le) - (int32_t)__popc(emk & le);
      const int32_t cmin = __reduce_min_sync(0xffffffffu, valid ? q : INT32_MAX);
      int32_t dafter = q;
      if (cmin < 0) {
        int32_t pm = valid ? q : INT32_MAX;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, pm, o);
          if ((int)lane >= o) pm = min(pm, y);
        }
        dafter = q - min(0, pm);
      }
      int32_t dbefore = __shfl_up_sync(0xffffffffu, dafter, 1);
      if (lane == 0) dbefore = D;
      const bool mend = en && dbefore > 0;  // matched END
      const bool dropped = en && dbefore == 0;
      const uint32_t L = st ? (uint32_t)dafter : (uint32_t)dbefore;  // level

      // ---- consumable flag of this START (prev record is a matched,
      //      non-marker END whose wait class is this START's class) --------
      const bool pm_prev_raw = __shfl_up_sync(0xffffffffu, (uint32_t)mend, 1);
      const uint32_t prid_raw = __shfl_up_sync(0xffffffffu, rid, 1);
      const bool prev_m = lane == 0 ? prev_end_matched : pm_prev_raw;
      const uint32_t prid = lane == 0 ? prev_rid : prid_raw;
      const uint32_t my_info = sm.cinfo[valid ? rid : 0];
      bool consumable = false;
      if (st && prev_m && i > 0) {
        const uint32_t pinfo = sm.cinfo[prid];
        consumable = !(pinfo & 0x80000000u) &&
                     sm.wcls[prid] == (my_info & 0x7FFFFFFFu);
      }

      // ---- partner START: same level, highest START lane below ------------
      // (match.any only when the step has both STARTs and matched ENDs: with
      // no matched END, START levels strictly increase, so each START is the
      // last at its level and no END has a partner inside the step)
      const uint32_t key = (st || mend) ? L : (0x80000000u | lane);
      uint32_t grp = 1u << lane;
      if (smk != 0u && __any_sync(0xffffffffu, mend))
        grp = __match_any_sync(0xffffffffu, key);
      const uint32_t cand = grp & smk & lt;
      const uint32_t src = cand ? 31u - __clz(cand) : lane;
      const uint32_t s_v = __shfl_sync(0xffffffffu, v, src);
      const uint32_t s_hi = __shfl_sync(0xffffffffu, my_hi, src);
      const uint32_t s_info = __shfl_sync(
          0xffffffffu, rid | (consumable ? 0x80000000u : 0u), src);
      uint32_t p_lo = s_v, p_hi = s_hi, p_pos = c + src, p_info = s_info;
      if (mend && !cand) {
        const LevelEntry e = lvl[L - 1];
        p_lo = e.lo;
        p_hi = e.hi;
        p_pos = e.pos;
        p_info = e.info;
      }
      __syncwarp();
      if (st && !(grp & smk & lanemask_gt())) {
        LevelEntry e;
        e.lo = v;
        e.hi = my_hi;
        e.pos = i;
        e.info = rid | (consumable ? 0x80000000u : 0u);
        lvl[L - 1] = e;
      }

      // ---- validation (single-stack nesting) and the 2^32 check ----------
      const uint64_t u = ((uint64_t)my_hi << 32) | v;
      const uint64_t su = ((uint64_t)p_hi << 32) | p_lo;
      const bool mism = mend && (p_info & 0x7FFFFFFFu) != rid;
      const bool too_long = mend && !mism && (u - su) >= (1ull << 32);
      if (__any_sync(0xffffffffu, mism)) {
        if (lane == 0) {
          atomicAdd(&a.status->invalid, 1ull);
          a.sflag[s] = flag | SF_INVALID;
        }
        bad = true;
        break;
      }
      if (__any_sync(0xffffffffu, too_long)) {
        const uint32_t fm = __ballot_sync(0xffffffffu, too_long);
        if (lane == 0)
          atomicMin(&a.status->pair_err,
                    ((unsigned long long)gs << 32) | (c + __ffs(fm) - 1u));
        bad = true;
        break;
      }

      // ---- iteration numbers per region id --------------------------------
      // lanes of a region find each other through a shared bit mask (one
      // shared atomicOr each) instead of match.any
      if (mend) atomicOr(&rmask[rid], 1u << lane);
      __syncwarp();
      const uint32_t rgrp = mend ? rmask[rid] : 0u;
      uint32_t it = 0;
      if (mend) it = cnt[rid] + __popc(rgrp & lt);
      __syncwarp();
      if (mend && !(rgrp & lt)) {
        cnt[rid] += __popc(rgrp);
        rmask[rid] = 0u;
      }

      // ---- replay -----------------------------------------------------------
      const uint32_t cls = my_info & 0x7FFFFFFFu;
      const bool is_mk = (my_info & 0x80000000u) != 0u;
      const bool base_ev = mend && !is_mk;
      // look-ahead records i+1, i+2 (next lanes or the next chunk)
      const uint32_t t1 = __shfl_down_sync(0xffffffffu, tag, 1);
      const uint32_t v1 = __shfl_down_sync(0xffffffffu, v, 1);
      const uint32_t t2 = __shfl_down_sync(0xffffffffu, tag, 2);
      const uint32_t n0t = __shfl_sync(0xffffffffu, rn.x, 0);
      const uint32_t n0v = __shfl_sync(0xffffffffu, rn.y, 0);
      const uint32_t n1t = __shfl_sync(0xffffffffu, rn.x, 1);
      const uint32_t nt1 = lane == 31 ? n0t : t1;
      const uint32_t nv1 = lane == 31 ? n0v : v1;
      const uint32_t nt2 = lane == 31 ? n1t : (lane == 30 ? n0t : t2);
      bool consumed = false;
      if (base_ev && i + 1 < n && (nt1 & WGPF_START_FLAG)) {
        const uint32_t r1 = (nt1 >> 12) & (WGPF_MAX_REGIONS - 1u);
        const uint32_t i1 = sm.cinfo[r1];
        if ((i1 & 0x80000000u) && sm.wcls[rid] == (i1 & 0x7FFFFFFFu)) {
          const bool closes_next =
              i + 2 < n && !(nt2 & WGPF_START_FLAG) &&
              ((nt2 >> 12) & (WGPF_MAX_REGIONS - 1u)) == r1;
          consumed = (int64_t)(i + 1) <= (int64_t)z || closes_next;
        }
      }
      const bool orphan = mend && is_mk && !(p_info & 0x80000000u);
      const uint32_t bm = __ballot_sync(0xffffffffu, base_ev);
      const uint32_t cm = __ballot_sync(0xffffffffu, consumed);
      const uint64_t kpos = kb + __popc(bm & lt) + __popc(cm & lt);
      kb += __popc(bm) + __popc(cm);

      uint32_t e_dur = 0, w_dur = 0;
      uint32_t wc = kNone;
      if (base_ev) {
        const uint64_t meas = u - su;
        const uint64_t ovh = cost * (uint64_t)(i - p_pos);
        const uint64_t corr = meas >= ovh ? meas - ovh : 0;
        e_dur = (uint32_t)corr;
        const uint64_t idx = off + kpos;
        if (a.events) {
          if (idx < a.events_cap)
            store_event(a.events + idx, su, su + corr, rid | WGPF_EV_CORRECTED,
                        it, blk, wg);
          else
            atomicAdd(&a.status->overflow, 1ull);
        }
        if (consumed) {
          const uint32_t r1 = (nt1 >> 12) & (WGPF_MAX_REGIONS - 1u);
          wc = sm.cinfo[r1] & 0x7FFFFFFFu;
          const uint32_t h1 = my_hi + (nv1 < v ? 1u : 0u);
          const uint64_t u1 = ((uint64_t)h1 << 32) | nv1;
          const uint64_t wd = u1 - u;
          const bool corr_w = wd > cost;
          w_flag += !corr_w;
          w_dur = (uint32_t)wd;
          if (a.events) {
            if (idx + 1 < a.events_cap)
              store_event(a.events + idx + 1, u, u1,
                          r1 | WGPF_EV_WAIT | (corr_w ? WGPF_EV_CORRECTED : 0u),
                          it, blk, wg);
            else
              atomicAdd(&a.status->overflow, 1ull);
          }
        }
      }
      // orphans -> per-warp scratch, written after all base events
      const uint32_t om = __ballot_sync(0xffffffffu, orphan);
      if (orphan) {
        wgpf_event e;
        e.start = su;
        e.end = u;
        e.region = rid;
        e.iteration = it;
        e.block_index = blk;
        e.warp_group = wg;
        orphans[n_orph + __popc(om & lt)] = e;
      }
      n_orph += __popc(om);
      w_drop += dropped;

      if (!a.no_stats) {
        lane_stats(acc_e, sm, a.stats, a.status, base_ev, cls, e_dur,
                   first_key(gs, kpos, 0u));
        if (__any_sync(0xffffffffu, consumed))
          lane_stats(acc_w, sm, a.stats, a.status, consumed, wc, w_dur,
                     first_key(gs, kpos + 1, 1u));
      }

      // ---- carries ----------------------------------------------------------
      const uint32_t vm = __ballot_sync(0xffffffffu, valid);
      const uint32_t last = 31u - __clz(vm);
      hi += __popc(wm);
      vprev = __shfl_sync(0xffffffffu, v, last);
      D = __shfl_sync(0xffffffffu, dafter, last);
      prev_end_matched = __shfl_sync(0xffffffffu, (uint32_t)mend, last);
      prev_rid = __shfl_sync(0xffffffffu, rid, last);
      rc = rn;
    }
    if (bad) continue;
    if (kb + n_orph != want) {  // cannot happen for single-stack streams
      if (lane == 0) {
        atomicAdd(&a.status->invalid, 1ull);
        a.sflag[s] = flag | SF_INVALID;
      }
      continue;
    }
    __syncwarp();
    // orphans after all base events (trace.hpp:469-485)
    for (uint32_t j = lane; j < ((n_orph + 31u) & ~31u); j += 32) {
      const bool ok = j < n_orph;
      wgpf_event e;
      if (ok) e = orphans[j];
      const uint64_t idx = off + kb + j;
      if (ok && a.events) {
        if (idx < a.events_cap)
          store_event(a.events + idx, e.start, e.end, e.region, e.iteration,
                      blk, wg);
        else
          atomicAdd(&a.status->overflow, 1ull);
      }
      if (!a.no_stats) {
        const uint32_t ci = ok ? sm.cinfo[e.region] & 0x7FFFFFFFu : 0u;
        lane_stats(acc_e, sm, a.stats, a.status, ok, ci,
                   ok ? (uint32_t)(e.end - e.start) : 0u,
                   first_key(gs, kb + j, 0u));
      }
    }
    w_mal += n_orph;
    w_tail += (uint32_t)D;
  }
  if (!a.no_stats) {
    acc_flush(acc_e, sm, a.stats, a.status);
    acc_flush(acc_w, sm, a.stats, a.status);
  }
  // warnings: w_drop / w_flag are per lane, w_tail / w_mal per warp (lane 0)
  const unsigned long long d = warp_sum((unsigned long long)w_drop);
  const unsigned long long f = warp_sum((unsigned long long)w_flag);
  if (lane == 0) {
    if (d) atomicAdd(&sm.warn[0], d);
    if (w_tail) atomicAdd(&sm.warn[1], (unsigned long long)w_tail);
    if (f) atomicAdd(&sm.warn[2], f);
    if (w_mal) atomicAdd(&sm.warn[3], (unsigned long long)w_mal);
  }
  __syncthreads();
  if (threadIdx.x < 4 && sm.warn[threadIdx.x])
    atomicAdd(&a.status->warn[threadIdx.x], sm.warn[threadIdx.x]);
  if (!a.no_stats) smem_stats_flush(sm.st, a.stats);
}

}  // namespace wgpf
