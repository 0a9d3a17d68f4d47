// k_general.cuh -- the exact, general replay path: one thread per stream.
//
// Used for streams the warp-cooperative fast path does not take (region ids
// outside the dense table, nesting that is not single-stack, deep nesting,
// wait markers it cannot decide), for exact recounts, and for everything
// under WGPF_F_FORCE_GENERAL.  It restates, per stream:
//   pair_records  trace.hpp:294-346  (per-region stacks, iteration numbers,
//                                     dropped heads / truncated tails, 2^32)
//   replay        trace.hpp:398-487  (sync correction, wait markers, orphans)
// with scratch in HBM: unwrapped clocks, per-region LIFO threaded through a
// prev-START array, an open-addressed region table, and the intervals.
#pragma once

#include "wgpf_dev.cuh"

namespace wgpf {

struct GenArgs {
  const uint8_t* body;
  uint64_t stride;
  uint64_t n_streams;
  uint64_t stream_base;   // global index of stream 0 of this call
  DevPlan plan;
  DevStats stats;
  DevStatus* status;
  uint32_t* counts;
  uint32_t* sflag;
  const uint64_t* offsets;
  wgpf_event* events;     // may be null (stats only)
  uint64_t events_cap;
  uint64_t record_cost;
  // work list: streams list[first .. first + n) (list == null: identity)
  const uint64_t* list;
  const unsigned long long* list_len; // device count when list is used
  uint64_t first;
  uint64_t batch;
  // scratch (per batch slot)
  uint8_t* scratch;
  uint64_t scratch_stride;
  uint32_t cap;           // plan slots (max stream length)
  uint32_t hm_size;       // power of two >= 2 * cap
  uint32_t no_stats;
};

struct HmEntry {
  uint32_t region;
  int32_t head;
  uint32_t completed;
  uint32_t depth;
};

struct GenIv {
  uint64_t start, end;
  uint32_t sp, ep;
  uint32_t region;  // | 0x80000000 when consumed
  uint32_t iteration;
};

struct GenScratch {
  uint64_t* uc;
  uint32_t* prev;
  int32_t* sidx;
  HmEntry* hm;
  GenIv* iv;
};

__device__ inline GenScratch gen_scratch(const GenArgs& a, uint64_t slot) {
  uint8_t* p = a.scratch + slot * a.scratch_stride;
  GenScratch s;
  s.uc = reinterpret_cast<uint64_t*>(p);
  p += 8ull * a.cap;
  s.hm = reinterpret_cast<HmEntry*>(p);
  p += 16ull * a.hm_size;
  s.iv = reinterpret_cast<GenIv*>(p);
  p += 32ull * (a.cap / 2 + 1);
  s.prev = reinterpret_cast<uint32_t*>(p);
  p += 4ull * a.cap;
  s.sidx = reinterpret_cast<int32_t*>(p);
  return s;
}

__host__ inline uint64_t gen_scratch_bytes(uint32_t cap, uint32_t hm) {
  uint64_t b = 8ull * cap + 16ull * hm + 32ull * (cap / 2 + 1) + 8ull * cap;
  return (b + 255) & ~255ull;
}

__device__ inline HmEntry* hm_get(HmEntry* hm, uint32_t size, uint32_t rid) {
  uint32_t h = (rid * 0x9E3779B1u) & (size - 1u);
  for (;;) {
    HmEntry* e = &hm[h];
    if (e->region == rid) return e;
    if (e->region == kNone) {
      e->region = rid;
      e->head = -1;
      e->completed = 0;
      e->depth = 0;
      return e;
    }
    h = (h + 1u) & (size - 1u);
  }
}

// Pairs one stream.  Returns the number of intervals; on a >= 2^32 interval
// records the error and returns kNone.
__device__ inline uint32_t gen_pair(const GenArgs& a, uint64_t s,
                                    const GenScratch& sc, bool keep,
                                    uint32_t* dropped, uint32_t* tails,
                                    uint32_t* n_out) {
  const uint8_t* base = a.body + s * a.stride;
  const uint4 h = *reinterpret_cast<const uint4*>(base);
  const uint32_t cnt = h.z, cap = h.w;
  const uint32_t n = cnt <= cap ? cnt : cap;
  const uint32_t start = cnt <= cap ? 0u : cnt % cap;
  *n_out = n;
  for (uint32_t i = 0; i < a.hm_size; ++i) sc.hm[i].region = kNone;
  const uint2* slots = reinterpret_cast<const uint2*>(base + 16);
  uint64_t cur = 0;
  uint32_t vprev = 0, n_iv = 0, drop = 0;
  for (uint32_t pos = 0; pos < n; ++pos) {
    uint32_t slot = start + pos;
    if (slot >= cap) slot -= cap;
    const uint2 r = slots[slot];
    cur = pos == 0 ? (uint64_t)r.y : cur + (uint32_t)(r.y - vprev);
    vprev = r.y;
    sc.uc[pos] = cur;
    if (keep) sc.sidx[pos] = -1;
    const uint32_t rid = (r.x >> 12) & (WGPF_MAX_REGIONS - 1u);
    HmEntry* e = hm_get(sc.hm, a.hm_size, rid);
    if (r.x & WGPF_START_FLAG) {
      sc.prev[pos] = (uint32_t)e->head;
      e->head = (int32_t)pos;
      e->depth++;
    } else {
      if (e->head < 0) {
        ++drop;
        continue;
      }
      const uint32_t sp = (uint32_t)e->head;
      e->head = (int32_t)sc.prev[sp];
      e->depth--;
      const uint32_t it = e->completed++;
      const uint64_t st = sc.uc[sp];
      if (cur - st >= (1ull << 32)) {
        atomicMin(&a.status->pair_err,
                  ((unsigned long long)(s + a.stream_base) << 32) | pos);
        return kNone;
      }
      if (keep) {
        GenIv v;
        v.start = st;
        v.end = cur;
        v.sp = sp;
        v.ep = pos;
        v.region = rid;
        v.iteration = it;
        sc.iv[n_iv] = v;
        sc.sidx[sp] = (int32_t)n_iv;
      }
      ++n_iv;
    }
  }
  uint32_t t = 0;
  for (uint32_t i = 0; i < a.hm_size; ++i)
    if (sc.hm[i].region != kNone) t += sc.hm[i].depth;
  *dropped = drop;
  *tails = t;
  return n_iv;
}

__device__ inline uint64_t gen_stream_of(const GenArgs& a, uint64_t k) {
  return a.list ? a.list[k] : k;
}

__global__ void __launch_bounds__(128) k_general_count(GenArgs a) {
  const uint64_t n_work = a.list ? *a.list_len : a.n_streams;
  const uint64_t slot = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t k = a.first + slot;
  if (slot >= a.batch || k >= n_work) return;
  const uint64_t s = gen_stream_of(a, k);
  if (a.sflag[s] & SF_DECODE_ERR) return;
  uint32_t dropped, tails, n;
  const uint32_t c = gen_pair(a, s, gen_scratch(a, slot), false, &dropped,
                              &tails, &n);
  a.counts[s] = c == kNone ? 0u : c;
}

__global__ void __launch_bounds__(128) k_general_emit(GenArgs a) {
  __shared__ SmemStats sst;
  __shared__ unsigned long long swarn[4];
  if (!a.no_stats) smem_stats_init(sst);
  if (threadIdx.x < 4) swarn[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t n_work = a.list ? *a.list_len : a.n_streams;
  const uint64_t slot = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t k = a.first + slot;
  uint32_t w_drop = 0, w_tail = 0, w_flag = 0, w_mal = 0;
  if (slot < a.batch && k < n_work && a.status->decode_err == kNoErr) {
    const uint64_t s = gen_stream_of(a, k);
    const GenScratch sc = gen_scratch(a, slot);
    uint32_t n;
    const uint32_t n_iv = (a.sflag[s] & SF_DECODE_ERR)
                              ? kNone
                              : gen_pair(a, s, sc, true, &w_drop, &w_tail, &n);
    if (n_iv != kNone && n_iv != a.counts[s]) {
      atomicAdd(&a.status->invalid, 1ull);
      a.sflag[s] |= SF_INVALID;
    } else if (n_iv != kNone) {
      const uint64_t off = a.offsets[s];
      const uint64_t gs = s + a.stream_base;
      const uint4 h = *reinterpret_cast<const uint4*>(a.body + s * a.stride);
      const uint32_t blk = h.x, wg = h.y;
      const uint64_t cost = a.record_cost;
      uint64_t kk = 0;
      auto emit = [&](uint64_t st, uint64_t en, uint32_t rid, uint32_t flags,
                      uint32_t it, uint32_t cls) {
        const uint64_t idx = off + kk;
        if (a.events) {
          if (idx < a.events_cap) {
            wgpf_event ev;
            ev.start = st;
            ev.end = en;
            ev.region = rid | flags;
            ev.iteration = it;
            ev.block_index = blk;
            ev.warp_group = wg;
            a.events[idx] = ev;
          } else {
            atomicAdd(&a.status->overflow, 1ull);
          }
        }
        if (!a.no_stats)
          stats_add_one(sst, a.stats, cls, en - st,
                        first_key(gs, kk, (flags & WGPF_EV_WAIT) ? 1u : 0u),
                        &a.status->synth_overflow);
        ++kk;
      };
      for (uint32_t i = 0; i < n_iv; ++i) {
        GenIv v = sc.iv[i];
        if (v.region & 0x80000000u) continue;  // consumed
        const uint32_t cls = class_of(a.plan, v.region);
        if (class_is_marker(a.plan, cls)) continue;
        const uint64_t inside = (uint64_t)(v.ep - v.sp);
        const uint64_t overhead = cost * inside;
        const uint64_t measured = v.end - v.start;
        emit(v.start, v.start + (measured >= overhead ? measured - overhead : 0),
             v.region, WGPF_EV_CORRECTED, v.iteration, cls);
        sc.iv[i].region = v.region | 0x80000000u;
        if (v.ep + 1u >= n) continue;
        const int32_t m = sc.sidx[v.ep + 1u];
        if (m < 0) continue;
        const GenIv mv = sc.iv[m];
        const uint32_t mrid = mv.region & 0x7FFFFFFFu;
        const uint32_t mcls = class_of(a.plan, mrid);
        if (!class_is_marker(a.plan, mcls)) continue;
        if (mcls != wait_class_of(a.plan, v.region, cls)) continue;
        sc.iv[m].region = mrid | 0x80000000u;
        // wait = [CLK1 = base end, CLK2 = marker start]; never malformed
        // because unwrapped clocks are monotone (trace.hpp:455-458).
        const uint64_t ws = v.end, we = mv.start;
        const bool corr = we - ws > cost;
        if (!corr) ++w_flag;
        emit(ws, we, mrid, WGPF_EV_WAIT | (corr ? WGPF_EV_CORRECTED : 0u),
             v.iteration, mcls);
      }
      for (uint32_t i = 0; i < n_iv; ++i) {  // orphan markers (:469-485)
        const GenIv v = sc.iv[i];
        if (v.region & 0x80000000u) continue;
        const uint32_t cls = class_of(a.plan, v.region);
        if (!class_is_marker(a.plan, cls)) continue;
        emit(v.start, v.end, v.region, 0u, v.iteration, cls);
        ++w_mal;
      }
    }
  }
  // block-reduced warnings
  const unsigned long long d = warp_sum((unsigned long long)w_drop);
  const unsigned long long t = warp_sum((unsigned long long)w_tail);
  const unsigned long long f = warp_sum((unsigned long long)w_flag);
  const unsigned long long m = warp_sum((unsigned long long)w_mal);
  if (lane_id() == 0) {
    if (d) atomicAdd(&swarn[0], d);
    if (t) atomicAdd(&swarn[1], t);
    if (f) atomicAdd(&swarn[2], f);
    if (m) atomicAdd(&swarn[3], m);
  }
  __syncthreads();
  if (threadIdx.x < 4 && swarn[threadIdx.x])
    atomicAdd(&a.status->warn[threadIdx.x], swarn[threadIdx.x]);
  if (!a.no_stats) smem_stats_flush(sst, a.stats);
}

}  // namespace wgpf
