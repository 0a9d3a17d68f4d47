// k_misc.cuh -- device kernels behind the reference's unit-level entry
// points (unwrap_clock, pair_records, replay on caller intervals,
// decode_image).  replay_image is the hot path; these serve the same API
// surface for single streams.
#pragma once

#include "k_general.cuh"
#include "wgpf_dev.cuh"

namespace wgpf {

// unwrap_clock (trace.hpp:257-272): u[i] = hi_i << 32 | v[i] where hi_i is
// the number of k <= i with v[k] < v[k-1] (each gap < 2^32 carries at most
// once).  Pass A flags wraps, a scan counts them, pass B combines.
__global__ void k_unwrap_flags(const uint32_t* v, uint64_t n, uint32_t* f) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    f[i] = (i > 0 && v[i] < v[i - 1]) ? 1u : 0u;
}

__global__ void k_unwrap_combine(const uint32_t* v, const uint64_t* hi,
                                 uint64_t n, uint64_t* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (hi[i] << 32) | v[i];
}

// decode_image on a validated body: chronological records of stream s at
// offset off[s] (one warp per stream, coalesced).
__global__ void k_decode_records(const uint8_t* body, uint64_t stride,
                                 uint64_t n_streams, const uint64_t* off,
                                 wgpf_record* out) {
  const uint32_t lane = lane_id();
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t s = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
       s < n_streams; s += warps) {
    const uint8_t* base = body + s * stride;
    const uint4 h = *reinterpret_cast<const uint4*>(base);
    const uint32_t cnt = h.z, cap = h.w;
    const uint32_t n = cnt <= cap ? cnt : cap;
    const uint32_t start = cnt <= cap ? 0u : cnt % cap;
    const uint2* slots = reinterpret_cast<const uint2*>(base + 16);
    for (uint32_t i = lane; i < n; i += 32) {
      uint32_t slot = start + i;
      if (slot >= cap) slot -= cap;
      const uint2 r = slots[slot];
      out[off[s] + i] = wgpf_record{r.x, r.y};
    }
  }
}

__global__ void k_decode_counts(const uint8_t* body, uint64_t stride,
                                uint64_t n_streams, uint64_t* n_out,
                                wgpf_decoded_stream* ds) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
       s < n_streams; s += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 h = *reinterpret_cast<const uint4*>(body + s * stride);
    const uint32_t n = h.z <= h.w ? h.z : h.w;
    n_out[s] = n;
    ds[s].block_index = h.x;
    ds[s].warp_group = h.y;
    ds[s].dropped_records = h.z > h.w ? h.z - h.w : 0u;
    ds[s].pad = 0;
    ds[s].count = n;
  }
}

// pair_records on one stream: the general per-region pairing, intervals out
// in END order.
__global__ void k_pair_one(GenArgs a, wgpf_interval* out, uint32_t* info) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const GenScratch sc = gen_scratch(a, 0);
  uint32_t dropped = 0, tails = 0, n;
  const uint32_t n_iv = gen_pair(a, 0, sc, true, &dropped, &tails, &n);
  info[0] = n_iv;
  info[1] = dropped;
  info[2] = tails;
  if (n_iv == kNone) return;
  for (uint32_t i = 0; i < n_iv; ++i) {
    const GenIv v = sc.iv[i];
    wgpf_interval o;
    o.region_id = v.region;
    o.iteration = v.iteration;
    o.start = v.start;
    o.end = v.end;
    o.start_pos = v.sp;
    o.end_pos = v.ep;
    out[i] = o;
  }
}

// replay (trace.hpp:398-487) on caller-built intervals of one stream.  The
// marker index (std::map<start_pos, index>, :405-410; later entries win) is a
// linear probe here: unit-level entry point, n = one stream's intervals.
__global__ void k_replay_one(const wgpf_interval* iv, uint64_t n, DevPlan plan,
                             uint32_t block, uint32_t wg, uint64_t cost,
                             uint8_t* consumed, wgpf_event* out,
                             unsigned long long* info) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  uint64_t k = 0, flagged = 0, malformed = 0;
  for (uint64_t i = 0; i < n; ++i) consumed[i] = 0;
  auto is_mk = [&](uint64_t i) {
    return class_is_marker(plan, plan.class_of[iv[i].region_id & (WGPF_MAX_REGIONS - 1u)]);
  };
  for (uint64_t i = 0; i < n; ++i) {
    if (consumed[i] || is_mk(i)) continue;
    const wgpf_interval a = iv[i];
    const uint64_t inside = a.end_pos - a.start_pos;
    const uint64_t overhead = cost * inside;
    const uint64_t measured = a.end - a.start;
    wgpf_event ev{a.start, a.start + (measured >= overhead ? measured - overhead : 0),
                  a.region_id | WGPF_EV_CORRECTED, a.iteration, block, wg};
    out[k++] = ev;
    consumed[i] = 1;
    int64_t m = -1;
    for (uint64_t j = 0; j < n; ++j)
      if (is_mk(j) && iv[j].start_pos == a.end_pos + 1) m = (int64_t)j;
    if (m < 0) continue;
    const uint32_t rid = a.region_id & (WGPF_MAX_REGIONS - 1u);
    const uint32_t mrid = iv[m].region_id & (WGPF_MAX_REGIONS - 1u);
    if (plan.class_of[mrid] != wait_class_of(plan, rid, plan.class_of[rid]))
      continue;
    consumed[m] = 1;
    const uint64_t ws = a.end, we = iv[m].start;
    if (we < ws) {
      ++malformed;
      continue;
    }
    const bool corr = we - ws > cost;
    flagged += !corr;
    out[k++] = wgpf_event{ws, we,
                          iv[m].region_id | WGPF_EV_WAIT |
                              (corr ? WGPF_EV_CORRECTED : 0u),
                          a.iteration, block, wg};
  }
  for (uint64_t i = 0; i < n; ++i) {
    if (consumed[i] || !is_mk(i)) continue;
    out[k++] = wgpf_event{iv[i].start, iv[i].end, iv[i].region_id,
                          iv[i].iteration, block, wg};
    ++malformed;
  }
  info[0] = k;
  info[1] = flagged;
  info[2] = malformed;
}

}  // namespace wgpf
