// k_stats.cuh -- region_stats finalisation (pipeline.hpp:114-133), the
// bit-exact mean recurrence, stats over arbitrary event arrays, and the
// multi-GPU export / merge of packed per-label tables.
#pragma once

#include "wgpf_dev.cuh"

namespace wgpf {

// warp_group of each label's first event: the first key holds the global
// stream index; this rank owns streams [base, base + n).
__global__ void k_resolve_first(DevStats st, uint32_t n_slots,
                                const uint8_t* body, uint64_t stride,
                                uint64_t stream_base, uint64_t n_streams,
                                unsigned long long* first_wg) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_slots || st.count[i] == 0) return;
  const uint64_t gs = st.first[i] >> 25;
  if (gs < stream_base || gs - stream_base >= n_streams) return;
  const uint4 h =
      *reinterpret_cast<const uint4*>(body + (gs - stream_base) * stride);
  first_wg[i] = h.y;
}

// region_stats over an event array (device).  Block-local shared-memory
// accumulation, first key = event index (<< 1 | kind); wg from the event.
__global__ void __launch_bounds__(256) k_event_stats(const wgpf_event* ev,
                                                     uint64_t n, DevPlan plan,
                                                     DevStats st,
                                                     DevStatus* status) {
  __shared__ SmemStats sst;
  smem_stats_init(sst);
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const wgpf_event e = ev[i];
    const uint32_t rid = e.region & WGPF_EV_REGION_MASK;
    const uint32_t cls = plan.class_of[rid];
    const unsigned long long key =
        ((unsigned long long)i << 1) | ((e.region & WGPF_EV_WAIT) ? 1u : 0u);
    const uint64_t d = e.end - e.start;
    if (d >> 32) {  // durations beyond 32 bits: global, 64-bit path
      stats_add_global(st, stats_slot(st, cls, &status->synth_overflow), d,
                       key);
    } else {
      stats_add_one(sst, st, cls, d, key, &status->synth_overflow);
    }
  }
  __syncthreads();
  smem_stats_flush(sst, st);
}

__global__ void k_event_first_wg(const wgpf_event* ev, DevStats st,
                                 uint32_t n_slots,
                                 unsigned long long* first_wg) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_slots || st.count[i] == 0) return;
  first_wg[i] = ev[st.first[i] >> 1].warp_group;
}

// Exact mean: the reference's recurrence mean = (mean * count + d) /
// (count + 1) in IEEE double, round-to-nearest, no contraction, over the
// label's durations in global event order (u32 count as the reference).
// seg[c] .. seg[c+1] index the class-sorted (stable) durations.
__global__ void k_exact_mean(const uint32_t* sorted_cls,
                             const unsigned long long* dur, uint64_t n,
                             const DevStats st, uint32_t n_slots,
                             double* mean_out, const int* slot_of_class_dense) {
  // one thread per slot: binary search the segment of its class
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_slots) return;
  mean_out[i] = 0.0;
  if (st.count[i] == 0) return;
  const uint32_t cls = i < st.K ? i : st.hkey[i - st.K];
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (sorted_cls[mid] < cls) lo = mid + 1; else hi = mid;
  }
  double mean = 0.0;
  uint32_t count = 0;
  for (uint64_t k = lo; k < n && sorted_cls[k] == cls; ++k) {
    const double prod = __dmul_rn(mean, (double)count);
    const double num = __dadd_rn(prod, (double)dur[k]);
    mean = __ddiv_rn(num, (double)(uint32_t)(count + 1u));
    ++count;
  }
  mean_out[i] = mean;
  (void)slot_of_class_dense;
}

__global__ void k_event_class_dur(const wgpf_event* ev, uint64_t n,
                                  DevPlan plan, uint32_t* cls_out,
                                  unsigned long long* dur_out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const wgpf_event e = ev[i];
    cls_out[i] = plan.class_of[e.region & WGPF_EV_REGION_MASK];
    dur_out[i] = e.end - e.start;
  }
}

// ---- packed export / merge ----------------------------------------------------
// Per slot, 70 u64: count, sum, min, max, first, first_wg, hist[64]; slot
// order = dense classes then the synthetic hash table, whose keys follow as
// H u64 (class or ~0).
constexpr uint32_t kPackedPerSlot = 70;

__global__ void k_stats_pack(DevStats st, uint32_t n_slots,
                             const unsigned long long* first_wg,
                             unsigned long long* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_slots) {
    unsigned long long* o = out + (uint64_t)i * kPackedPerSlot;
    o[0] = st.count[i];
    o[1] = st.sum[i];
    o[2] = st.min[i];
    o[3] = st.max[i];
    o[4] = st.first[i];
    o[5] = first_wg[i];
    for (uint32_t b = 0; b < WGPF_HIST_BINS; ++b)
      o[6 + b] = st.hist[(uint64_t)i * WGPF_HIST_BINS + b];
  }
  if (i < st.H)
    out[(uint64_t)n_slots * kPackedPerSlot + i] = st.hkey[i];
}

// Pass 1: accumulate every rank's table into this context (keys of the
// synthetic part are matched by class).
__global__ void k_stats_merge(DevStats st, uint32_t n_slots,
                              const unsigned long long* in, uint32_t n_ranks,
                              DevStatus* status) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t per = (uint64_t)n_slots * kPackedPerSlot + st.H;
  if (gid >= (uint64_t)n_ranks * n_slots) return;
  const uint32_t r = (uint32_t)(gid / n_slots), i = (uint32_t)(gid % n_slots);
  const unsigned long long* rb = in + r * per;
  const unsigned long long* o = rb + (uint64_t)i * kPackedPerSlot;
  if (o[0] == 0) return;
  int slot = (int)i;
  if (i >= st.K) {
    const uint32_t cls = (uint32_t)rb[(uint64_t)n_slots * kPackedPerSlot + (i - st.K)];
    slot = stats_slot(st, cls, &status->synth_overflow);
    if (slot < 0) return;
  }
  atomicAdd(&st.count[slot], o[0]);
  atomicAdd(&st.sum[slot], o[1]);
  atomicMin(&st.min[slot], o[2]);
  atomicMax(&st.max[slot], o[3]);
  atomicMin(&st.first[slot], o[4]);
  for (uint32_t b = 0; b < WGPF_HIST_BINS; ++b)
    if (o[6 + b]) atomicAdd(&st.hist[(uint64_t)slot * WGPF_HIST_BINS + b], o[6 + b]);
}

// Pass 2: the warp_group of the winning first key.
__global__ void k_stats_merge_wg(DevStats st, uint32_t n_slots,
                                 const unsigned long long* in, uint32_t n_ranks,
                                 unsigned long long* first_wg) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t per = (uint64_t)n_slots * kPackedPerSlot + st.H;
  if (gid >= (uint64_t)n_ranks * n_slots) return;
  const uint32_t r = (uint32_t)(gid / n_slots), i = (uint32_t)(gid % n_slots);
  const unsigned long long* rb = in + r * per;
  const unsigned long long* o = rb + (uint64_t)i * kPackedPerSlot;
  if (o[0] == 0) return;
  int slot = (int)i;
  if (i >= st.K) {
    const uint32_t cls = (uint32_t)rb[(uint64_t)n_slots * kPackedPerSlot + (i - st.K)];
    slot = -1;
    for (uint32_t h = 0; h < st.H; ++h)
      if (st.hkey[h] == cls) slot = (int)(st.K + h);
    if (slot < 0) return;
  }
  if (st.first[slot] == o[4]) first_wg[slot] = o[5];
}

}  // namespace wgpf
