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
//       another region breaks the single-stack assumption -> SF_INVALID
//       (exact recount); durations >= 2^32 -> pair error (trace.hpp:330-336).
//   replay (trace.hpp:398-487)          sync correction, wait markers decided
//       with the look-ahead records i+1, i+2 and pass 1's z, orphans last.
//   region_stats (pipeline.hpp:114-133) lane-private count / min / max / sum /
//       first key per class in shared memory (no atomics), histogram through
//       match.any groups and one shared atomic per group.
//
// Data movement.  Records: the warp stages 16-record windows of its 32 streams
// in shared memory with cp.async (16-B chunks, double buffered; chunk k of the
// window of stream l is copied by a fixed lane, so one instruction covers a
// few contiguous lines).  Events: each lane stages 4 events (128 B) in shared
// memory and writes them with one TMA bulk store (cp.async.bulk, bulk_group),
// double buffered.  Per record a lane executes ~1 shared load; per event two
// 16-B shared stores and a quarter of a bulk store.
#pragma once

#include "k_fast.cuh"

namespace wgpf {

constexpr uint32_t kTpsMaxWarps = 8;                  // warps per CTA (<=)
constexpr uint32_t kTpsW = 16;                        // records per window
constexpr uint32_t kTpsChunks = (kTpsW + 2) / 2;      // 16-B chunks per window
constexpr uint32_t kTpsPitch = 16 * kTpsChunks;       // bytes per lane window
constexpr uint32_t kTpsDepth = 16;                    // stack entries per lane
constexpr uint32_t kTpsRegions = 32;                  // region ids < this
constexpr uint32_t kTpsClasses = 16;                  // dense classes held
constexpr uint32_t kTpsEvb = 4;                       // events per buffer
constexpr uint32_t kTpsEvPitch = 32 * kTpsEvb + 16;   // padded: no conflicts
constexpr uint32_t kTpsMaxSlots = 2046;               // pos / hi in 11+15 bits

struct TpsWarpSmem {
  uint8_t rec[2][32 * kTpsPitch];    // record windows
  uint8_t evb[2][32 * kTpsEvPitch];  // event staging
  uint2 stk[kTpsDepth][32];          // {lo clock, pos | rid<<11 | cons<<16 | hi<<17}
  uint16_t cnt[kTpsRegions][32];     // iteration counters
  wgpf_event orph[32];               // one orphan per lane (more: SF_INVALID)
};

struct TpsCtaSmem {
  uint32_t info[kTpsRegions];  // class | marker<<8 | wait class<<16 (0xFF none)
  unsigned long long warn[4];
  uint32_t hist[kTpsClasses * WGPF_HIST_BINS];
};

// Lane-private stats of one warp, [class][lane]: {count, min, max, sum lo},
// sum hi, first key.
struct TpsLaneStats {
  uint4* a;
  uint32_t* hi;
  unsigned long long* first;
};

__host__ __device__ inline size_t tps_align(size_t b) { return (b + 127) & ~size_t(127); }
__host__ __device__ inline size_t tps_lane_stats_bytes(uint32_t K) {
  return tps_align((size_t)K * 32 * (16 + 4 + 8));
}
__host__ inline size_t tps_smem_bytes(uint32_t K, uint32_t warps) {
  return tps_align(sizeof(TpsCtaSmem)) +
         warps * (tps_align(sizeof(TpsWarpSmem)) + tps_lane_stats_bytes(K));
}
// warps per CTA that fit the shared memory of one SM (one CTA per SM)
__host__ inline uint32_t tps_warps(uint32_t K, size_t smem_limit) {
  uint32_t w = kTpsMaxWarps;
  while (w > 1 && tps_smem_bytes(K, w) > smem_limit) --w;
  return w;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc,
                                           uint32_t bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile(
      "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
      "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ssrc))), "r"(bytes)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(kTpsMaxWarps * 32, 1) k_tps(FastArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  TpsCtaSmem& cs = *reinterpret_cast<TpsCtaSmem*>(smem_raw);
  const uint32_t lane = lane_id();
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t K = a.plan.K;
  const uint32_t nw = blockDim.x >> 5;
  TpsWarpSmem& ws = *reinterpret_cast<TpsWarpSmem*>(
      smem_raw + tps_align(sizeof(TpsCtaSmem)) + w * tps_align(sizeof(TpsWarpSmem)));
  uint8_t* lsb = smem_raw + tps_align(sizeof(TpsCtaSmem)) +
                 nw * tps_align(sizeof(TpsWarpSmem)) +
                 w * tps_lane_stats_bytes(K);
  TpsLaneStats ls;
  ls.a = reinterpret_cast<uint4*>(lsb);
  ls.hi = reinterpret_cast<uint32_t*>(lsb + (size_t)K * 32 * 16);
  ls.first = reinterpret_cast<unsigned long long*>(lsb + (size_t)K * 32 * 20);
  const bool stats = !a.no_stats;
  for (uint32_t c = 0; c < K; ++c) {
    ls.a[c * 32 + lane] = make_uint4(0u, 0xFFFFFFFFu, 0u, 0u);
    ls.hi[c * 32 + lane] = 0;
    ls.first[c * 32 + lane] = ~0ull;
  }
  for (uint32_t i = threadIdx.x; i < K * WGPF_HIST_BINS; i += blockDim.x) cs.hist[i] = 0;
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
  __syncthreads();
  const bool abort_all = a.status->decode_err != kNoErr;
  const uint32_t FULL = 0xffffffffu;
  const uint32_t lt = lanemask_lt();
  const uint64_t cost = a.record_cost;
  const uint32_t cap = a.cap;
  uint32_t w_drop = 0, w_tail = 0, w_flag = 0, w_mal = 0;
  uint32_t ebuf = 0;  // event staging buffer in use

  // static chunk assignment of the record windows: chunk k of this lane is
  // part pk of stream lane slk
  uint32_t slk[kTpsChunks], pk[kTpsChunks];
#pragma unroll
  for (uint32_t k = 0; k < kTpsChunks; ++k) {
    const uint32_t q = k * 32 + lane;
    slk[k] = q / kTpsChunks;
    pk[k] = q - slk[k] * kTpsChunks;
  }

  const uint64_t wstep = (uint64_t)gridDim.x * nw;
  for (uint64_t b = (uint64_t)blockIdx.x * nw + w; !abort_all && b * 32 < a.n_streams;
       b += wstep) {
    const uint64_t s = b * 32 + lane;
    const uint32_t flag = s < a.n_streams ? a.sflag[s] : SF_DECODE_ERR;
    if (flag & SF_GENERAL) {
      const unsigned long long k = atomicAdd(a.general_len, 1ull);
      a.general_list[k] = s;
    }
    const bool act = !(flag & (SF_DECODE_ERR | SF_GENERAL | SF_WARP));
    const uint8_t* sbase = a.body + (act ? s : 0) * a.stride;
    uint4 h = make_uint4(0u, 0u, 0u, cap);
    if (act) h = *reinterpret_cast<const uint4*>(sbase);
    uint32_t n = act ? (h.z <= cap ? h.z : cap) : 0u;
    const uint32_t start = h.z <= cap ? 0u : h.z % cap;
    const uint32_t nmax = __reduce_max_sync(FULL, n);
    if (nmax == 0) continue;
    const uint32_t blk = h.x, wg = h.y;
    const int32_t z = act ? a.zpos[s] : -1;
    const uint32_t want = act ? a.counts[s] : 0u;
    const uint64_t off = act ? a.offsets[s] : 0ull;
    const uint64_t gs = s + a.stream_base;
    const uint2* slots = reinterpret_cast<const uint2*>(sbase + 16);
#pragma unroll
    for (uint32_t r = 0; r < kTpsRegions; ++r) ws.cnt[r][lane] = 0;

    // window sources: physical (even) slot of chunk k for window c0 = 2
    uint32_t wp[kTpsChunks], wlim[kTpsChunks];
    const uint8_t* wsrc[kTpsChunks];
#pragma unroll
    for (uint32_t k = 0; k < kTpsChunks; ++k) {
      const uint32_t st_k = __shfl_sync(FULL, start, slk[k]);
      wlim[k] = __shfl_sync(FULL, n, slk[k]);
      uint32_t p = st_k + 2u;
      if (p >= cap) p -= cap;
      p = (p & ~1u) + 2u * pk[k];
      if (p >= cap) p -= cap;
      wp[k] = p;
      wsrc[k] = a.body + (b * 32 + slk[k]) * a.stride + 16;
    }
    auto issue = [&](uint32_t bsel, uint32_t c0) {
      uint8_t* dst = ws.rec[bsel];
#pragma unroll
      for (uint32_t k = 0; k < kTpsChunks; ++k) {
        if (c0 < wlim[k])
          cp_async16(dst + slk[k] * kTpsPitch + 16u * pk[k], wsrc[k] + 8ull * wp[k]);
        wp[k] += kTpsW;
        if (wp[k] >= cap) wp[k] -= cap;
      }
    };
    const uint32_t shift = start & 1u;
    const uint8_t* myrec0 = ws.rec[0] + lane * kTpsPitch + 8u * shift;

    uint2 r0 = make_uint2(0u, 0u), r1 = make_uint2(0u, 0u);
    if (n > 0) r0 = slots[start];
    if (n > 1) r1 = slots[start + 1 < cap ? start + 1 : start + 1 - cap];
    issue(0, 2);
    cp_async_commit();

    uint32_t hi = 0, vprev = 0, sp = 0;
    uint32_t pw = 0xFFu;  // wait class of the previous record if it was a
                          // matched base END, else none
    uint64_t kb = 0;      // base events emitted
    uint32_t fill = 0;    // events in the staging buffer
    uint64_t eb = off;    // event index of the buffer's first event
    uint32_t n_orph = 0;
    uint8_t* const evl0 = ws.evb[0] + lane * kTpsEvPitch;  // + ebuf * buffer

    auto flush = [&]() {
      if (!fill) return;
      const uint64_t room = eb < a.events_cap ? a.events_cap - eb : 0ull;
      const uint32_t m = (uint64_t)fill <= room ? fill : (uint32_t)room;
      if (m) bulk_store(a.events + eb, evl0 + ebuf * (32u * kTpsEvPitch), 32u * m);
      if (m < fill) atomicAdd(&a.status->overflow, (unsigned long long)(fill - m));
      ebuf ^= 1u;
      bulk_wait_read1();  // the buffer switched to is free again
      eb += fill;
      fill = 0;
    };
    auto stage = [&](uint64_t st, uint64_t en, uint32_t region, uint32_t it) {
      uint4* p = reinterpret_cast<uint4*>(evl0 + ebuf * (32u * kTpsEvPitch) + 32u * fill);
      p[0] = make_uint4((uint32_t)st, (uint32_t)(st >> 32), (uint32_t)en,
                        (uint32_t)(en >> 32));
      p[1] = make_uint4(region, it, blk, wg);
      if (++fill == kTpsEvb) flush();
    };
    auto lstat = [&](uint32_t cls, uint32_t d, unsigned long long key) {
      uint4* e = ls.a + cls * 32 + lane;
      uint4 x = *e;
      if (x.x == 0) ls.first[cls * 32 + lane] = key;
      x.x += 1;
      x.y = min(x.y, d);
      x.z = max(x.z, d);
      const uint32_t sm = x.w + d;
      if (sm < d) ls.hi[cls * 32 + lane] += 1;
      x.w = sm;
      *e = x;
    };
    auto lhist = [&](bool part, uint32_t cls, uint32_t d) {
      const uint32_t bin = hist_bin(d);
      const uint32_t key = part ? ((cls << 6) | bin) : (0xFC000000u | lane);
      const uint32_t grp = __match_any_sync(FULL, key);
      if (part && !(grp & lt)) atomicAdd(&cs.hist[(cls << 6) | bin], (uint32_t)__popc(grp));
    };

    for (uint32_t w0 = 0; w0 < nmax; w0 += kTpsW) {
      const uint32_t bsel = (w0 / kTpsW) & 1u;
      if (w0 + kTpsW < nmax) issue(bsel ^ 1u, w0 + kTpsW + 2u);
      cp_async_commit();
      cp_async_wait1();
      __syncwarp();
      const uint8_t* myrec = myrec0 + bsel * (32 * kTpsPitch);
#pragma unroll 4
      for (uint32_t j = 0; j < kTpsW; ++j) {
        const uint32_t i = w0 + j;
        const uint2 r2 = *reinterpret_cast<const uint2*>(myrec + 8u * j);
        const bool valid = i < n;
        const uint32_t tag = r0.x, v = r0.y;
        const bool st = valid && (tag & WGPF_START_FLAG);
        const bool en = valid && !(tag & WGPF_START_FLAG);
        const uint32_t rid = (tag >> 12) & (kTpsRegions - 1u);
        const uint32_t inf = cs.info[rid];
        hi += (valid && v < vprev) ? 1u : 0u;
        if (valid) vprev = v;
        const uint32_t cls = inf & 0xFFu;
        bool base_ev = false, consumed = false;
        uint32_t e_dur = 0, w_dur = 0, wc = 0;
        uint64_t kpos = kb;
        if (st) {
          const uint32_t cons = (pw == cls) ? 1u : 0u;
          ws.stk[sp][lane] = make_uint2(v, i | (rid << 11) | (cons << 16) | (hi << 17));
          ++sp;
        }
        uint32_t npw = 0xFFu;
        if (en) {
          if (sp == 0) {
            ++w_drop;
          } else {
            --sp;
            const uint2 e = ws.stk[sp][lane];
            const uint32_t p_rid = (e.y >> 11) & 31u;
            const uint64_t u = ((uint64_t)hi << 32) | v;
            const uint64_t su = ((uint64_t)(e.y >> 17) << 32) | e.x;
            if (p_rid != rid) {  // not single-stack: exact recount
              atomicAdd(&a.status->invalid, 1ull);
              a.sflag[s] = flag | SF_INVALID;
              n = 0;
            } else if (u - su >= (1ull << 32)) {
              atomicMin(&a.status->pair_err, ((unsigned long long)gs << 32) | i);
              n = 0;
            } else {
              const uint32_t it = ws.cnt[rid][lane];
              ws.cnt[rid][lane] = (uint16_t)(it + 1u);
              if (!(inf & 0x100u)) {  // base scope: exec event
                base_ev = true;
                const uint64_t meas = u - su;
                const uint64_t ovh = cost * (uint64_t)(i - (e.y & 2047u));
                const uint64_t corr = meas >= ovh ? meas - ovh : 0ull;
                e_dur = (uint32_t)corr;
                if (a.events) stage(su, su + corr, rid | WGPF_EV_CORRECTED, it);
                ++kb;
                npw = inf >> 16;
                // wait marker START at i+1, closed (z or the next record)
                if (i + 1 < n && (r1.x & WGPF_START_FLAG)) {
                  const uint32_t r1id = (r1.x >> 12) & (kTpsRegions - 1u);
                  const uint32_t i1 = cs.info[r1id];
                  if ((i1 & 0x100u) && (inf >> 16) == (i1 & 0xFFu)) {
                    const bool closes_next = i + 2 < n && !(r2.x & WGPF_START_FLAG) &&
                                             ((r2.x >> 12) & (kTpsRegions - 1u)) == r1id;
                    if ((int64_t)(i + 1) <= (int64_t)z || closes_next) {
                      consumed = true;
                      wc = i1 & 0xFFu;
                      const uint32_t h1 = hi + (r1.y < v ? 1u : 0u);
                      const uint64_t u1 = ((uint64_t)h1 << 32) | r1.y;
                      const uint64_t wd = u1 - u;
                      const bool corr_w = wd > cost;
                      w_flag += corr_w ? 0u : 1u;
                      w_dur = (uint32_t)wd;
                      if (a.events)
                        stage(u, u1, r1id | WGPF_EV_WAIT | (corr_w ? WGPF_EV_CORRECTED : 0u),
                              it);
                      ++kb;
                    }
                  }
                }
              } else if (!((e.y >> 16) & 1u)) {  // orphan marker interval
                if (n_orph == 0) {
                  wgpf_event& o = ws.orph[lane];
                  o.start = su;
                  o.end = u;
                  o.region = rid;
                  o.iteration = it;
                  o.block_index = blk;
                  o.warp_group = wg;
                  n_orph = 1;
                } else {  // more than one: exact recount
                  atomicAdd(&a.status->invalid, 1ull);
                  a.sflag[s] = flag | SF_INVALID;
                  n = 0;
                }
              }
            }
          }
        }
        pw = npw;
        if (stats) {
          if (__any_sync(FULL, base_ev)) {
            if (base_ev) lstat(cls, e_dur, first_key(gs, kpos, 0u));
            lhist(base_ev, cls, e_dur);
          }
          if (__any_sync(FULL, consumed)) {
            if (consumed) lstat(wc, w_dur, first_key(gs, kpos + 1, 1u));
            lhist(consumed, wc, w_dur);
          }
        }
        r0 = r1;
        r1 = r2;
      }
      __syncwarp();
    }
    // stream end: orphans after the base events, flush, checks
    const bool ok = act && n != 0;
    if (ok && n_orph) {
      const wgpf_event o = ws.orph[lane];
      if (a.events) stage(o.start, o.end, o.region, o.iteration);
    }
    if (stats) {
      const bool po = ok && n_orph;
      const uint32_t oc = po ? cs.info[ws.orph[lane].region & 31u] & 0xFFu : 0u;
      const uint32_t od = po ? (uint32_t)(ws.orph[lane].end - ws.orph[lane].start) : 0u;
      if (__any_sync(FULL, po)) {
        if (po) lstat(oc, od, first_key(gs, kb, 0u));
        lhist(po, oc, od);
      }
    }
    flush();
    if (ok) {
      if (kb + n_orph != want) {
        atomicAdd(&a.status->invalid, 1ull);
        a.sflag[s] = flag | SF_INVALID;
      }
      w_mal += n_orph;
      w_tail += sp;
    }
  }
  bulk_wait_all();
  // lane-private stats -> CTA -> global
  const unsigned long long d = warp_sum((unsigned long long)w_drop);
  const unsigned long long f = warp_sum((unsigned long long)w_flag);
  const unsigned long long t = warp_sum((unsigned long long)w_tail);
  const unsigned long long m = warp_sum((unsigned long long)w_mal);
  if (lane == 0) {
    if (d) atomicAdd(&cs.warn[0], d);
    if (t) atomicAdd(&cs.warn[1], t);
    if (f) atomicAdd(&cs.warn[2], f);
    if (m) atomicAdd(&cs.warn[3], m);
  }
  if (stats) {
    for (uint32_t c = 0; c < K; ++c) {
      const uint4 x = ls.a[c * 32 + lane];
      const unsigned long long cnt = warp_sum((unsigned long long)x.x);
      if (cnt == 0) continue;
      const unsigned long long sum = warp_sum(
          ((unsigned long long)ls.hi[c * 32 + lane] << 32) | x.w);
      const uint32_t mn = __reduce_min_sync(FULL, x.y);
      const uint32_t mx = __reduce_max_sync(FULL, x.z);
      unsigned long long fk = ls.first[c * 32 + lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) fk = min(fk, __shfl_xor_sync(FULL, fk, o));
      if (lane == 0) {
        atomicAdd(&a.stats.count[c], cnt);
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
  if (stats)
    for (uint32_t i = threadIdx.x; i < K * WGPF_HIST_BINS; i += blockDim.x)
      if (cs.hist[i]) atomicAdd(&a.stats.hist[i], (unsigned long long)cs.hist[i]);
}

}  // namespace wgpf
