// k_tps.cuh -- pass 2 of replay_image, thread-per-stream: one lane per
// stream, 32 streams per warp advancing in lockstep over chronological
// positions.  This is the main path for shallow streams (nesting <= kTpsDepth,
// region ids < kTpsRegions, <= kTpsClasses label classes); deeper or wider
// streams take the warp-per-stream kernel (k_fast.cuh), irregular ones the
// exact general path (k_general.cuh).
//
// Same algorithm as the reference, sequential per stream:
//   unwrap_clock (trace.hpp:257-272)   hi += (v < v_prev)
//   pair_records (trace.hpp:294-346)   one stack per stream in shared memory;
//       pass 1 guarantees depth <= kTpsDepth; an END whose stack top has
//       another region breaks the single-stack assumption, and a duration
//       >= 2^32 is the reference's pair error (trace.hpp:330-336): both mark
//       the stream SF_INVALID -> exact recount and re-emit on the general
//       path, which reports the error.
//   replay (trace.hpp:398-487)          sync correction, wait markers decided
//       with the look-ahead records i+1, i+2 and pass 1's z, orphans last.
//   region_stats (pipeline.hpp:114-133) lane-private count / min / max / sum
//       per class in shared memory (no atomics); the first-event key per warp
//       (a shared atomicMin when a lane meets a class for the first time).
//
// Scheduling.  A batch is one warp index w of 32 consecutive blocks (lane l
// <- stream (32 j + l) W + w, W streams per block, host-detected): the lanes
// run the same record-type sequence, the walk's branches are warp-uniform,
// and an all-START step does nothing but the push.  Batches beyond the first
// grid-wide round come from a global counter (dynamic load balance).
//
// Data movement.  Records: the warp stages 8-record windows (+2 look-ahead)
// of its 32 streams in shared memory, double buffered: one 3-D TMA box per
// window when every stream of the batch starts at slot 0, else cp.async
// (16-B chunks; chunk k of the window of stream l is copied by a fixed lane,
// so one instruction covers a few contiguous lines).  Lanes read records in
// 16-B pairs (conflict-free at the 80-B lane pitch).  Events: each lane stores its 32-B events straight
// to HBM (one 256-bit store per event, a full L2 sector; a stream's events are contiguous, so
// L2 completes each line before write-back).  Measured against staging the
// events in shared-memory rings with a warp-cooperative coalesced flush, the
// direct stores are faster (the flush costs more issue slots than the
// scattered stores cost the LSU), and per-lane TMA bulk stores serialise (the
// bulk-copy instruction takes uniform operands).
// The step is written predicated with 32-bit timing arithmetic (a pair whose
// duration reaches 2^32 is an error, so every emitted duration fits); errors
// are recorded per lane and handled after the stream (the stack depth stays
// within pass 1's bound whatever the regions, so a lane can keep going).
// Histograms: one per-CTA table, one shared atomic per event (lanes without
// an event add into a spare word: no branch); a class's count is the sum of
// its bins.
#pragma once

#include <type_traits>

#include "k_fast.cuh"
#include "k_window.cuh"

namespace wgpf {

#ifndef WGPF_TPS_UNROLL
#define WGPF_TPS_UNROLL 4
#endif
constexpr int kTpsUnroll = WGPF_TPS_UNROLL;  // full steps unrolled per window
constexpr int kTpsPairUnroll = kTpsUnroll / 2;  // (record pairs)
#ifndef WGPF_TPS_WARPS
#define WGPF_TPS_WARPS 15  // measured: 15 -> 5.10 ms, 16 -> 5.38 (8 B spills at 128 regs), 14 -> 5.22
#endif
constexpr uint32_t kTpsMaxWarps = WGPF_TPS_WARPS;     // warps per CTA (<=)
constexpr uint32_t kTpsDepth = 8;                     // stack entries per lane
constexpr uint32_t kTpsRegions = 32;                  // region ids < this
constexpr uint32_t kTpsClasses = 16;                  // dense classes held
// stack entry: the START's region id stays where the record tag has it
// (bits 12..16), so an END compares it with one xor
constexpr uint32_t kStkRid = (kTpsRegions - 1u) << 12;

struct TpsWarpSmem {
  uint8_t rec[2][32 * kTpsPitch];    // record windows
#ifdef WGPF_STK_EMPTY
  // row -1: what an empty stack reads (never written; its value is not used).
  // Default: row -1 is the last 256 B of rec[1], read but unused -- the
  // dedicated row (for compute-sanitizer racecheck, which reports the read
  // against the window's TMA write) costs 2.8 % (emit 5.27 vs 5.13 ms)
  uint2 stk_empty[32];
#endif
  uint2 stk[kTpsDepth][32];          // {lo clock, pos | rid<<12 | cons<<17 | hi<<18}
  wgpf_event orph[32];               // one orphan per lane (more: SF_INVALID)
  unsigned long long bar[2];         // TMA windows: one mbarrier per buffer
};

struct TpsCtaSmem {
  uint32_t info[kTpsRegions];  // class | marker<<8 | wait class<<16 (0xFF none)
  unsigned long long warn[4];
};

// Per-warp dynamic tables (R = region ids in use, K = classes):
//   a     uint4 [K][32]       {min, max, sum lo, sum hi} per class and lane
//   first u64 [K]             first-event key (per warp: shared atomicMin
//                             when a lane meets a class for the first time,
//                             i.e. while its min is still the initial ~0)
//   cnt   u16 [R][32]         iteration counters
// and per CTA hist u32 [K][64]; a class's event count is the sum of its bins.
struct TpsTables {
  uint4* a;
  unsigned long long* first;
  uint16_t* cnt;
};

__host__ __device__ inline size_t tps_align(size_t b) { return (b + 127) & ~size_t(127); }
__host__ __device__ inline size_t tps_tables_bytes(uint32_t K, uint32_t R) {
  return tps_align((size_t)K * 32 * 16 + (size_t)K * 8 + (size_t)R * 64);
}
__host__ __device__ inline TpsTables tps_tables(uint8_t* p, uint32_t K, uint32_t R) {
  TpsTables t;
  t.a = reinterpret_cast<uint4*>(p);
  t.first = reinterpret_cast<unsigned long long*>(p + (size_t)K * 32 * 16);
  t.cnt = reinterpret_cast<uint16_t*>(p + (size_t)K * 32 * 16 + (size_t)K * 8);
  return t;
}
__host__ __device__ inline size_t tps_hist_bytes(uint32_t K) {
  return tps_align((size_t)K * WGPF_HIST_BINS * 4 + 4);  // + a spare word
}
__host__ inline size_t tps_smem_bytes(uint32_t K, uint32_t R, uint32_t warps) {
  return tps_align(sizeof(TpsCtaSmem)) + tps_hist_bytes(K) +
         warps * (tps_align(sizeof(TpsWarpSmem)) + tps_tables_bytes(K, R));
}
// warps per CTA that fit the shared memory of one SM (one CTA per SM)
__host__ inline uint32_t tps_warps(uint32_t K, uint32_t R, size_t smem_limit) {
  uint32_t w = kTpsMaxWarps;
  while (w > 1 && tps_smem_bytes(K, R, w) > smem_limit) --w;
  return w;
}

// kEmit: events materialised; kStats: statistics.
// tm: the body as a TMA tensor (a.tma != 0), see k_window.cuh; tm_tail: the
// same without L2 promotion, for windows within 256 B of the streams' end
template <bool kEmit, bool kStats>
__global__ void __launch_bounds__(kTpsMaxWarps * 32, 1)
    k_tps(FastArgs a, const __grid_constant__ CUtensorMap tm,
          const __grid_constant__ CUtensorMap tm_tail) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  TpsCtaSmem& cs = *reinterpret_cast<TpsCtaSmem*>(smem_raw);
  const uint32_t lane = lane_id();
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t nw = blockDim.x >> 5;
  const uint32_t K = a.plan.K;
  const uint32_t R = a.tps_regions;
  uint32_t* const hist = reinterpret_cast<uint32_t*>(smem_raw + tps_align(sizeof(TpsCtaSmem)));
  uint8_t* const wbase0 = smem_raw + tps_align(sizeof(TpsCtaSmem)) + tps_hist_bytes(K);
  TpsWarpSmem& ws = *reinterpret_cast<TpsWarpSmem*>(wbase0 + w * tps_align(sizeof(TpsWarpSmem)));
  uint8_t* const tb0 = wbase0 + nw * tps_align(sizeof(TpsWarpSmem));
  const TpsTables tb = tps_tables(tb0 + w * tps_tables_bytes(K, R), K, R);
  constexpr bool stats = kStats;
  constexpr bool emit = kEmit;
  for (uint32_t c = 0; c < K; ++c) tb.a[c * 32 + lane] = make_uint4(0xFFFFFFFFu, 0u, 0u, 0u);
  for (uint32_t c = lane; c < K; c += 32) tb.first[c] = ~0ull;
  for (uint32_t i = threadIdx.x; i < K * WGPF_HIST_BINS; i += blockDim.x) hist[i] = 0;
  for (uint32_t r = threadIdx.x; r < kTpsRegions; r += blockDim.x) {
    uint32_t inf = 0xFFFFFFFFu;
    if (r < a.fast_regions) {
      const uint32_t c = a.plan.class_of[r];
      const uint32_t wc = c < K ? a.plan.wait_class[c] : kNone;
      inf = (c & 0xFFu) | (class_is_marker(a.plan, c) ? 0x100u : 0u) |
            ((wc < K ? wc : 0xFFu) << 16);
    }
    cs.info[r] = inf;
  }
  if (threadIdx.x < 4) cs.warn[threadIdx.x] = 0;
  const uint32_t s_bar = smem_addr(&ws.bar[0]);  // + 8 * buffer
  if (a.tma && lane == 0) {
    win_bar_init(s_bar);
    win_bar_init(s_bar + 8u);
    win_bar_fence();
  }
  uint32_t bphase = 0;  // parity of each buffer's next completion (bit = buffer)
  __syncthreads();
  const bool abort_all = a.status->decode_err != kNoErr;
  const uint32_t FULL = 0xffffffffu;
  const uint32_t lt = lanemask_lt();
  const uint32_t cost = (uint32_t)a.record_cost;  // host: < 2^21 on this path
  const uint32_t cap = a.cap;
  uint32_t w_drop = 0, w_tail = 0, w_flag = 0, w_mal = 0, w_ovf = 0;

  // Lane mapping.  The streams of one block are its warps' (or warp
  // groups'), W of them, in image order; warps of the traced kernel with the
  // same index run the same program, so a batch takes one warp index w of 32
  // consecutive blocks: lane l <- stream (32 j + l) W + w.  The lanes then
  // walk identical record-type sequences and the walk's branches are warp-
  // uniform.  (Any mapping gives the same results: events go to pass 1's
  // offsets, and a lane still meets its streams in increasing order.)
  const uint32_t W = a.group;
  const uint64_t n_blocks = a.n_streams / W;  // (host: W divides n_streams)
  const uint64_t n_batches = W * ((n_blocks + 31) / 32);

  // 32-bit shared addresses of the hot tables (this lane's column)
  // (opaque: kept in registers instead of being rebuilt from the CTA's
  // shared window base at every use)
  const uint32_t s_info = opaque_u32(smem_addr(cs.info));
  const uint32_t s_hist = opaque_u32(smem_addr(hist));
  const uint32_t s_hist_spare = opaque_u32(smem_addr(hist + K * WGPF_HIST_BINS));
  const uint32_t s_stk = smem_addr(&ws.stk[0][lane]);    // + 256 * level
  const uint32_t s_cnt = smem_addr(tb.cnt + lane);        // + 64 * region
  const uint32_t s_a = smem_addr(tb.a + lane);            // + 512 * class
  const uint32_t s_orph = smem_addr(&ws.orph[lane]);

  const uint64_t wstep = (uint64_t)gridDim.x * nw;
  // Batches: the first gridDim.x * nw statically, then dynamically from a
  // global counter (the next index is fetched at the top of each batch, so
  // the atomic's latency hides behind the walk): warps finish together
  // whatever the per-batch work (producer / consumer warp indices differ).
  unsigned long long nxt = 0;
  for (uint64_t b = (uint64_t)blockIdx.x * nw + w; !abort_all && b < n_batches;
       b = wstep + __shfl_sync(FULL, nxt, 0)) {
    if (lane == 0) nxt = atomicAdd(a.batch_ctr, 1ull);
    const uint64_t jb = b / W;                 // batch of 32 blocks
    const uint32_t wi = (uint32_t)(b - jb * W);  // warp index within them
    const uint64_t s0 = jb * 32 * W + wi;      // lane 0's stream
    const uint64_t s = s0 + (uint64_t)lane * W;
    const uint32_t flag = jb * 32 + lane < n_blocks ? a.sflag[s] : SF_DECODE_ERR;
    if (flag & SF_GENERAL) {
      const unsigned long long k = atomicAdd(a.general_len, 1ull);
      a.general_list[k] = s + a.list_base;
    }
    const bool act = !(flag & (SF_DECODE_ERR | SF_GENERAL | SF_WARP));
    const uint8_t* sbase = a.body + (act ? s : 0) * a.stride;
    uint4 h = make_uint4(0u, 0u, 0u, cap);
    if (act) h = *reinterpret_cast<const uint4*>(sbase);
    const uint32_t n = act ? (h.z <= cap ? h.z : cap) : 0u;
    const uint32_t start = h.z <= cap ? 0u : h.z % cap;
    const uint32_t nmax = __reduce_max_sync(FULL, n);
    if (nmax == 0) continue;
    const uint32_t blk = h.x, wg = h.y;
    const int32_t z = act ? a.zpos[s] : -1;
    const uint32_t want = act ? a.counts[s] : 0u;
    const uint64_t off = act ? a.offsets[s] : 0ull;
    const uint64_t gs = s + a.stream_base;
    const unsigned long long gkey = (unsigned long long)gs << 25;
    const uint2* slots = reinterpret_cast<const uint2*>(sbase + 16);
    for (uint32_t r = 0; r < R; ++r) tb.cnt[r * 32 + lane] = 0;

    // one TMA box per window when every stream of the batch starts at slot 0
    const bool tmab = a.tma && __all_sync(FULL, start == 0u);
    const uint32_t s_buf = smem_addr(ws.rec[0]);
    // cp.async window state only for batches that need it (its ~35
    // registers are dead in the TMA walk)
    RecWindows win;
    if (!tmab) {
      win.init(ws.rec[0], lane, a.stride * W, cap);  // lanes W streams apart
      win.begin(a.body + s0 * a.stride, start, n);
    }
    // WGPF_TAIL_SEL: windows whose rows end within 256 B (32 records) of the
    // shortest stream's last record without L2 promotion (it would pull
    // unused slots).  Measured on config 4: emit 5.38 vs 5.13 ms without the
    // per-window map selection (tm_tail is then unused here)
#ifdef WGPF_TAIL_SEL
    const uint32_t ntail = __reduce_min_sync(FULL, act ? n : 0xFFFFFFFFu);
#endif
    auto issue = [&](uint32_t bs, uint32_t c0) {
      if (tmab) {
        if (lane == 0)
          win_tma3(s_buf + bs * (32u * kTpsPitch),
#ifdef WGPF_TAIL_SEL
                   c0 + kTpsPitch / 8u + 32u <= ntail ? &tm : &tm_tail,
#else
                   &tm,
#endif
                   s_bar + 8u * bs,
                   (int)(4u + 2u * c0), (int)wi, (int)(jb * 32), 32u * kTpsPitch);
      } else {
        win.issue(bs, c0);
      }
    };

    uint2 r0 = make_uint2(0u, 0u), r1 = make_uint2(0u, 0u);
    if (n > 0) r0 = slots[start];
    if (n > 1) r1 = slots[start + 1 < cap ? start + 1 : start + 1 - cap];
    uint32_t inf0 = cs.info[(r0.x >> 12) & (kTpsRegions - 1u)];
    issue(0, 2);
    cp_async_commit();

    // stack top as a shared address: row sp-1 of the lane's column; the
    // empty stack points one row below (stk_empty: read, never written, and
    // only used when an END has a partner)
    const uint32_t s_stk0 = s_stk - 256u;
    uint32_t hi = 0, vprev = 0, stop = s_stk0;
    uint32_t pw = 0xFFu;  // wait class of the previous record if it was a
                          // matched base END, else none
    uint32_t kw = 0;      // events of this stream written
    uint32_t n_orph = 0;
    bool broken = false;  // single-stack nesting broken or a pair >= 2^32:
                          // the exact general path redoes the stream

    // events of this stream that fit the caller's buffer (events <= records,
    // so a stream ending inside the capacity needs no per-store check)
    const uint32_t lim = off + n <= a.events_cap
                             ? 0xFFFFFFFFu
                             : (off < a.events_cap ? (uint32_t)(a.events_cap - off) : 0u);
    const uint64_t ev0 = opaque_u64(reinterpret_cast<uint64_t>(a.events + (act ? off : 0ull)));
    auto put = [&](bool p, uint32_t k, uint32_t slo, uint32_t shi, uint32_t elo,
                   uint32_t ehi, uint32_t region, uint32_t it) {
      // (events past lim are counted once at the stream end: kw - lim)
      stg256_if(p & (k < lim), ev0 + 32ull * k, make_uint4(slo, shi, elo, ehi),
                make_uint4(region, it, blk, wg));
    };
    // one event of class cls (predicated on p): lane-private min / max / sum,
    // per-warp first key, CTA histogram (which also gives the count).  A lane
    // meets its events in key order, so the first-key atomic fires while the
    // lane's min is still ~0 (again only if every duration so far was
    // 2^32-1: a larger key, which the min leaves alone).
    auto lstat = [&](bool p, uint32_t cls, uint32_t d, uint32_t kpos, uint32_t kind) {
      const uint32_t c = p ? cls : 0u;
      const uint32_t ea = s_a + c * 512u;
      uint4 x = lds128(ea);
      if (p && x.x == 0xFFFFFFFFu) atomicMin(&tb.first[c], gkey | (kpos << 1) | kind);
      x.x = min(x.x, d);
      x.y = max(x.y, d);
      add64_u32(x.z, x.w, d);
      sts128_if(p, ea, x);
      // (unpredicated: lanes without an event count into a spare word past
      // the table -- no branch around the shared atomic)
      red_add(p ? s_hist + 4u * (c * WGPF_HIST_BINS + hist_bin32(d)) : s_hist_spare, 1u);
    };
    // kFull: positions i .. i+2 exist on every lane (the bulk of the walk):
    // no per-record bounds predicates
    auto step = [&](auto full, uint32_t i, uint2 r2) {
      constexpr bool kFull = decltype(full)::value;
      const bool valid = kFull || i < n;
      const uint32_t tag = r0.x, v = r0.y;
      const bool isS = (int32_t)tag < 0;
      const bool st = valid && isS;
      const bool en = valid && !isS;
      const uint32_t rid = (tag >> 12) & (kTpsRegions - 1u);
      const uint32_t inf = inf0;
      const uint32_t r1id = (r1.x >> 12) & (kTpsRegions - 1u);
      const uint32_t i1 = lds32(s_info + 4u * r1id);
      if constexpr (kFull) {
        // every lane at a START (grouped lanes run the same program): a push
        // is all that happens -- no event, no statistics, no wait marker
        if (__all_sync(FULL, isS)) {
          hi += v < vprev ? 1u : 0u;
          vprev = v;
          sts64_if(true, stop + 256u,
                   make_uint2(v, i | (tag & kStkRid) | ((pw == (inf & 0xFFu) ? 1u : 0u) << 17) |
                                     (hi << 18)));
          stop += 256u;
          pw = 0xFFu;
          inf0 = i1;
          r0 = r1;
          r1 = r2;
          return;
        }
      }
      hi += (valid && v < vprev) ? 1u : 0u;
      vprev = valid ? v : vprev;
      // ---- stack ------------------------------------------------------------
      const uint2 e = lds64(stop);
      const bool nonempty = stop != s_stk0;
      const bool mend = en && nonempty;
      w_drop += (en && !nonempty) ? 1u : 0u;
      // Dead predicated stores are skipped by warp votes (grouped lanes: a
      // general step is mostly all-END, wait events and orphans are rare).
      // Measured on config 4 with all three votes: emit 5.06 vs 5.12 ms (one
      // or two of them alone: no gain or slower -- the schedule changes)
      if (__any_sync(FULL, st))
      sts64_if(st, stop + 256u,
               make_uint2(v, i | (tag & kStkRid) | ((pw == (inf & 0xFFu) ? 1u : 0u) << 17) |
                                 (hi << 18)));
      stop = stop + (st ? 256u : 0u) - (mend ? 256u : 0u);
      const uint32_t shi = e.y >> 18;
      const uint32_t meas = v - e.x;  // low 32 bits of u - su
      const bool dhi = hi != shi + (v < e.x ? 1u : 0u);
      const bool mism = mend && ((e.y ^ tag) & kStkRid) != 0u;
      const bool tlong = mend && !mism && dhi;
      broken |= mism || tlong;
      const bool ok = mend && !mism && !tlong;
      // (rows exist for region ids < R; positions past the stream end hold
      // arbitrary tags, so clamp -- the value is only used when ok)
      const uint32_t ca = s_cnt + 64u * (kFull ? rid : min(rid, R - 1u));
      const uint32_t it = lds16(ca);
      sts16_if(ok, ca, it + 1u);
      const bool is_mk = (inf & 0x100u) != 0u;
      const bool base = ok && !is_mk;
      const bool orphan = ok && is_mk && !((e.y >> 17) & 1u);
      // ---- exec event: sync correction ---------------------------------------
      const uint32_t dpos = i - (e.y & 2047u);
      // dpos < 2^11 and cost < 2^21 (host): the product fits 32 bits
      const uint32_t ovh = cost * dpos;
      const uint32_t corr = ovh > meas ? 0u : meas - ovh;
      // ---- wait marker START at i+1 -------------------------------------------
      const bool cclose = (kFull || i + 2 < n) && (int32_t)r2.x >= 0 &&
                          ((r2.x >> 12) & (kTpsRegions - 1u)) == r1id;
      const bool consumed = base && (kFull || i + 1 < n) && (int32_t)r1.x < 0 &&
                            (i1 & 0x100u) && (inf >> 16) == (i1 & 0xFFu) &&
                            ((int32_t)(i + 1) <= z || cclose);
      const uint32_t wd = r1.y - v;  // consecutive records: u1 - u < 2^32
      const bool corr_w = wd > cost;
      w_flag += (consumed && !corr_w) ? 1u : 0u;
      const uint32_t kpos = kw;
      if constexpr (emit) {
        const uint32_t elo = e.x + corr;
        put(base, kw, e.x, shi, elo, shi + (elo < corr ? 1u : 0u), rid | WGPF_EV_CORRECTED,
            it);
        if (__any_sync(FULL, consumed))
        put(consumed, kw + 1u, v, hi, r1.y, hi + (r1.y < v ? 1u : 0u),
            r1id | WGPF_EV_WAIT | (corr_w ? WGPF_EV_CORRECTED : 0u), it);
      }
      kw += (base ? 1u : 0u) + (consumed ? 1u : 0u);
      pw = base ? (inf >> 16) : 0xFFu;
      // orphan marker interval (written after the base events): keep one
      if (__any_sync(FULL, orphan && n_orph == 0)) {
      sts128_if(orphan && n_orph == 0, s_orph, make_uint4(e.x, shi, v, hi));
      sts64_if(orphan && n_orph == 0, s_orph + 16u, make_uint2(rid, it));  // (block, wg: registers)
      }
      n_orph += orphan ? 1u : 0u;
      if constexpr (stats) {
        lstat(base, inf & 0xFFu, corr, kpos, 0u);
        if (__any_sync(FULL, consumed)) lstat(consumed, i1 & 0xFFu, wd, kpos + 1u, 1u);
      }
      inf0 = i1;
      r0 = r1;
      r1 = r2;
    };

    const uint32_t nmin = __reduce_min_sync(FULL, act ? n : 0u);
    const bool even_start = __all_sync(FULL, (start & 1u) == 0u);
    // the window loop, specialised for TMA batches (the bulk: unrolled steps)
    // and cp.async batches (wrapped circular streams: steps not unrolled)
    auto walk = [&](auto tma_tag) {
      constexpr bool kTma = decltype(tma_tag)::value;
      for (uint32_t w0 = 0; w0 < nmax; w0 += kTpsW) {
        const uint32_t bsel = (w0 / kTpsW) & 1u;
        if (w0 + kTpsW < nmax) issue(bsel ^ 1u, w0 + kTpsW + 2u);
        if constexpr (kTma) {
          win_wait(s_bar + 8u * bsel, (bphase >> bsel) & 1u);
          bphase ^= 1u << bsel;
        } else {
          cp_async_commit();
          cp_async_wait1();
        }
        __syncwarp();
        const uint2* myrec =
            kTma ? reinterpret_cast<const uint2*>(ws.rec[bsel] + lane * kTpsPitch)
                 : win.lane_records(bsel, lane, start);
        // records in 16-B pairs when starts are even: one conflict-free
        // LDS.128 per two steps (8-B loads at the 80-B lane pitch hit 4-way
        // bank conflicts)
        const uint4* myrec2 = reinterpret_cast<const uint4*>(myrec);
        if (w0 + kTpsW + 2u <= nmin) {
          if constexpr (kTma) {
#pragma unroll kTpsPairUnroll
            for (uint32_t j = 0; j < kTpsW; j += 2) {
              const uint4 q = myrec2[j / 2];
              step(std::true_type{}, w0 + j, make_uint2(q.x, q.y));
              step(std::true_type{}, w0 + j + 1, make_uint2(q.z, q.w));
            }
          } else if (even_start) {
#pragma unroll 1
            for (uint32_t j = 0; j < kTpsW; j += 2) {
              const uint4 q = myrec2[j / 2];
              step(std::true_type{}, w0 + j, make_uint2(q.x, q.y));
              step(std::true_type{}, w0 + j + 1, make_uint2(q.z, q.w));
            }
          } else {
#pragma unroll 1
            for (uint32_t j = 0; j < kTpsW; ++j) step(std::true_type{}, w0 + j, myrec[j]);
          }
        } else {
#pragma unroll 1
          for (uint32_t j = 0; j < kTpsW; ++j) step(std::false_type{}, w0 + j, myrec[j]);
        }
        __syncwarp();
      }
    };
    if (tmab)
      walk(std::true_type{});
    else
      walk(std::false_type{});
    // stream end: the orphan after the base events, final writes, checks
    const bool bad = broken || n_orph > 1;
    const bool po = act && !bad && n_orph == 1;
    if (__any_sync(FULL, po)) {
      const wgpf_event o = ws.orph[lane];
      if (emit)
        put(po, kw, (uint32_t)o.start, (uint32_t)(o.start >> 32), (uint32_t)o.end,
            (uint32_t)(o.end >> 32), o.region, o.iteration);
      if (stats)
        lstat(po, cs.info[o.region & 31u] & 0xFFu, (uint32_t)(o.end - o.start), kw, 0u);
      kw += po ? 1u : 0u;
    }
    w_ovf += act && kw > lim ? kw - lim : 0u;
    if (act) {
      // exact recount + re-emit on the general path, which also reports the
      // reference's pair error (trace.hpp:330-336) if there is one
      if (bad || kw != want) {
        atomicAdd(&a.status->invalid, 1ull);  // exact recount
        a.sflag[s] = flag | SF_INVALID;
      }
      if (!bad) {
        w_mal += n_orph;
        w_tail += (stop - s_stk0) >> 8;
      }
    }
  }
  // lane-private stats -> global; warnings
  const unsigned long long d = warp_sum((unsigned long long)w_drop);
  const unsigned long long f = warp_sum((unsigned long long)w_flag);
  const unsigned long long t = warp_sum((unsigned long long)w_tail);
  const unsigned long long m = warp_sum((unsigned long long)w_mal);
  const unsigned long long ov = warp_sum((unsigned long long)w_ovf);
  if (lane == 0 && ov) atomicAdd(&a.status->overflow, ov);
  if (lane == 0) {
    if (d) atomicAdd(&cs.warn[0], d);
    if (t) atomicAdd(&cs.warn[1], t);
    if (f) atomicAdd(&cs.warn[2], f);
    if (m) atomicAdd(&cs.warn[3], m);
  }
  if (stats) {
    for (uint32_t c = 0; c < K; ++c) {
      const uint4 x = tb.a[c * 32 + lane];
      // (no event: min ~0 and max 0; an event of 2^32-1 cycles has max ~0)
      if (!__any_sync(FULL, x.x != 0xFFFFFFFFu || x.y != 0u)) continue;
      const unsigned long long sum =
          warp_sum(((unsigned long long)x.w << 32) | x.z);
      const uint32_t mn = __reduce_min_sync(FULL, x.x);
      const uint32_t mx = __reduce_max_sync(FULL, x.y);
      const unsigned long long fk = tb.first[c];
      if (lane == 0) {
        atomicAdd(&a.stats.sum[c], sum);
        atomicMin(&a.stats.min[c], (unsigned long long)mn);
        atomicMax(&a.stats.max[c], (unsigned long long)mx);
        atomicMin(&a.stats.first[c], fk);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 4 && cs.warn[threadIdx.x])
    atomicAdd(&a.status->warn[threadIdx.x], cs.warn[threadIdx.x]);
  if (stats) {  // CTA histograms -> global; counts = bin sums
    for (uint32_t i = threadIdx.x; i < K * WGPF_HIST_BINS; i += blockDim.x) {
      if (hist[i]) atomicAdd(&a.stats.hist[i], (unsigned long long)hist[i]);
    }
    for (uint32_t c = w; c < K; c += nw) {
      const unsigned long long cnt = warp_sum(
          (unsigned long long)hist[c * WGPF_HIST_BINS + lane] + hist[c * WGPF_HIST_BINS + 32 + lane]);
      if (lane == 0 && cnt) atomicAdd(&a.stats.count[c], cnt);
    }
  }
}

}  // namespace wgpf
