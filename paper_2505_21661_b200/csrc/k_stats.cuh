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
// RN(num / n) for num >= 0, n >= 1 an integer below 2^53, from the
// reciprocal y = RN(1 / n) (computed off the recurrence's critical path):
// Markstein's correction q1 = q0 + r y with the exact FMA residual, then a
// check that the exact quotient lies strictly inside q1's rounding interval
// (the residual of q1, exact, against n times half the neighbouring gaps;
// every product is exact: n < 2^53 times a power of two); a tie or a miss
// takes the IEEE division.  Bit-identical to __ddiv_rn, ~5 dependent FP64
// operations instead of the division's long sequence.
__device__ __forceinline__ double div_rn_by_int(double num, double n, double y) {
  const double q0 = __dmul_rn(num, y);
  const double r0 = __fma_rn(-q0, n, num);
  const double q1 = __fma_rn(r0, y, q0);
  if (q1 <= 0.0) return num == 0.0 ? 0.0 : __ddiv_rn(num, n);
  const double r1 = __fma_rn(-q1, n, num);  // n (x - q1), exact
  const long long b = __double_as_longlong(q1);
  const double up = __longlong_as_double(b + 1) - q1;    // gap above q1
  const double down = q1 - __longlong_as_double(b - 1);  // gap below q1
  if (r1 < 0.5 * up * n && -r1 < 0.5 * down * n) return q1;
  return __ddiv_rn(num, n);
}

// The reference's mean recurrence (pipeline.hpp:129): mean = (mean * count +
// d) / (count + 1) in IEEE double, round-to-nearest, no contraction, over the
// label's durations in global event order (u32 count as the reference).  One
// thread per class: the segment of its class in the class-sorted (stable)
// durations is found first, so the loop's loads and reciprocals do not wait
// on the recurrence.
// One CTA per class.  The recurrence is one thread's serial chain, so the
// rest of the CTA feeds it: warps 1-3 stream the class's durations from HBM
// and compute the per-step constants -- d as a double and y = RN(1 / (count
// + 1)) -- into a double-buffered shared-memory ring, one chunk ahead of the
// consumer (thread 0), which then only runs the chain: 5 dependent FP64
// operations per event (prod, num, the Markstein quotient q1), with the
// quotient's exactness check beside it (ILP) rather than on it.  A block of
// kB steps with a failed check (a tie or a miss, rare) is redone with the
// checked division (div_rn_by_int) from the block's start.
constexpr uint32_t kEmChunk = 1024;  // events per ring chunk
constexpr uint32_t kEmThreads = 128;
__global__ void __launch_bounds__(kEmThreads) k_exact_mean(
    const uint32_t* sorted_cls, const unsigned long long* dur, uint64_t n, const DevStats st,
    uint32_t n_slots, double* mean_out, const int* slot_of_class_dense) {
  (void)slot_of_class_dense;
  __shared__ double2 ring[2][kEmChunk];  // {y, d}
  __shared__ unsigned long long seg[2];
  const uint32_t i = blockIdx.x;
  const uint32_t tid = threadIdx.x;
  if (i >= n_slots) return;
  if (st.count[i] == 0) {
    if (tid == 0) mean_out[i] = 0.0;
    return;
  }
  if (tid == 0) {
    const uint32_t cls = i < st.K ? i : st.hkey[i - st.K];
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (sorted_cls[mid] < cls) lo = mid + 1; else hi = mid;
    }
    uint64_t end = lo, top = n;
    while (end < top) {
      const uint64_t mid = (end + top) >> 1;
      if (sorted_cls[mid] <= cls) end = mid + 1; else top = mid;
    }
    seg[0] = lo;
    seg[1] = end;
  }
  __syncthreads();
  const uint64_t lo = seg[0], len = seg[1] - seg[0];
  const uint64_t chunks = (len + kEmChunk - 1) / kEmChunk;
  // producers: warps 1..3 fill chunk q of the ring
  auto fill = [&](uint64_t q) {
    const uint64_t base = q * kEmChunk;
    const uint32_t m = (uint32_t)(len - base < kEmChunk ? len - base : kEmChunk);
    double2* r = ring[q & 1];
    for (uint32_t j = tid - 32u; j < m; j += kEmThreads - 32u) {
      const uint32_t c = (uint32_t)(base + j);  // the u32 count before this event
      r[j] = make_double2(__drcp_rn((double)(uint32_t)(c + 1u)),
                          (double)__ldg(dur + lo + base + j));
    }
  };
  if (tid >= 32) fill(0);
  __syncthreads();
  double mean = 0.0;
  uint32_t count = 0;
  for (uint64_t q = 0; q < chunks; ++q) {
    if (tid >= 32) {
      if (q + 1 < chunks) fill(q + 1);
    } else if (tid == 0) {
      const double2* r = ring[q & 1];
      const uint32_t m = (uint32_t)(len - q * kEmChunk < kEmChunk ? len - q * kEmChunk : kEmChunk);
      constexpr uint32_t kB = 16;
      uint32_t j0 = 0;
      for (; j0 + kB <= m; j0 += kB) {
        double2 v[kB];
#pragma unroll
        for (uint32_t j = 0; j < kB; ++j) v[j] = r[j0 + j];
        double mm = mean;
        bool ok = true;
#pragma unroll
        for (uint32_t j = 0; j < kB; ++j) {
          const uint32_t c = count + j;
          const double m1 = (double)(uint32_t)(c + 1u), y = v[j].x;
          const double prod = __dmul_rn(mm, (double)c);
          const double num = __dadd_rn(prod, v[j].y);
          const double q0 = __dmul_rn(num, y);
          const double r0 = __fma_rn(-q0, m1, num);
          const double q1 = __fma_rn(r0, y, q0);
          const double r1 = __fma_rn(-q1, m1, num);
          const long long bb = __double_as_longlong(q1);
          const double up = __longlong_as_double(bb + 1) - q1;
          const double down = q1 - __longlong_as_double(bb - 1);
          // (bitwise, not short-circuit: predicated compares, no branches
          // beside the chain)
          const bool zero = num == 0.0;
          const bool good = (q1 > 0.0) & (r1 < 0.5 * up * m1) & (-r1 < 0.5 * down * m1);
          ok = ok & ((zero & (q1 == 0.0)) | (!zero & good));
          mm = q1;
        }
        if (!ok) {
          mm = mean;
          for (uint32_t j = 0; j < kB; ++j) {
            const uint32_t c = count + j;
            const double m1 = (double)(uint32_t)(c + 1u);
            mm = div_rn_by_int(__dadd_rn(__dmul_rn(mm, (double)c), v[j].y), m1, v[j].x);
          }
        }
        mean = mm;
        count += kB;
      }
      for (uint32_t j = j0; j < m; ++j) {
        const double m1 = (double)(uint32_t)(count + 1u);
        const double prod = __dmul_rn(mean, (double)count);
        mean = div_rn_by_int(__dadd_rn(prod, r[j].y), m1, r[j].x);
        ++count;
      }
    }
    __syncthreads();
  }
  if (tid == 0) mean_out[i] = mean;
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
