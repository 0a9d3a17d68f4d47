// k_cp.cuh -- K6: interval-overlap analysis on the GPU.
//
// analyze_critical_path (perfmodel.hpp:317-501): stages = label classes of
// the events (Exec events of ".wait" labels skipped, :323-328), each sorted
// by iteration (:332-335; ties by event index), steady window drops the first
// and last instance when >= 3 (:338-342), mean = llround(sum / n) (:350-351).
// Program-order gating (:364-385) is O(n^2) in the reference; here the steady
// events are sorted by (gate key, end) and each event binary-searches the
// window end in [start - theta, start + theta] (close(), :357-360), scanning
// it from the largest end down for the first e != f with e.start <= f.start
// and breaking end ties by the smaller label (:379-381) -- identical results
// in O(n log n).  Barrier edges (:387-406) test "exists e in src with
// close(e.end, f.start)" by binary search over src ends.  The label-graph fold
// and the max-weight simple cycle (:408-499) run on the host (tiny graph).
//
// Role overlap counters (this framework's definition, oracle/wgpf_oracle.h
// wgpo_overlap): per block, |union| of Exec intervals per role (producer /
// consumer warp groups), |intersection| = |U0| + |U1| - |U0 u U1|, span and
// bubbles; union lengths by a segmented max-scan over (key, start)-sorted
// intervals.
#pragma once

#include "wgpf_dev.cuh"

namespace wgpf {

// class key per event (kNone for dropped events) + iteration
__global__ void k_cp_prep(const wgpf_event* ev, uint64_t n, DevPlan plan,
                          uint32_t* cls_key) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const wgpf_event e = ev[i];
    const uint32_t cls = plan.class_of[e.region & WGPF_EV_REGION_MASK];
    const bool drop = !(e.region & WGPF_EV_WAIT) && class_is_marker(plan, cls);
    cls_key[i] = drop ? kNone : cls;
  }
}

// key = rank(cls) << 32 | iteration  (rank: label order of the class)
__global__ void k_cp_rank_key(const wgpf_event* ev, const uint32_t* cls_key,
                              uint64_t n, const uint32_t* uniq,
                              const uint32_t* rank_of, uint32_t n_uniq,
                              unsigned long long* key, uint64_t* idx) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = cls_key[i];
    uint32_t r = 0xFFFFFFFFu;
    if (c != kNone) {
      uint32_t lo = 0, hi = n_uniq;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (uniq[mid] < c) lo = mid + 1; else hi = mid;
      }
      r = rank_of[lo];
    }
    key[i] = ((unsigned long long)r << 32) | ev[i].iteration;
    idx[i] = i;
  }
}

// steady entries: stage id, and sort keys for the gating / barrier searches
struct CpEntry {
  uint64_t start, end;
  uint64_t gkey;   // gate key (warp_group or block << 32 | warp_group)
  uint32_t stage;
  uint32_t pad;
};

__global__ void k_cp_gather(const wgpf_event* ev, const uint64_t* sorted_idx,
                            const uint64_t* win_lo, const uint64_t* win_hi,
                            const uint64_t* out_off, uint32_t n_stages,
                            int gate_by_block, CpEntry* out,
                            unsigned long long* stage_sum) {
  const uint32_t s = blockIdx.y;
  if (s >= n_stages) return;
  const uint64_t lo = win_lo[s], hi = win_hi[s];
  unsigned long long acc = 0;
  for (uint64_t k = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < hi;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const wgpf_event e = ev[sorted_idx[k]];
    CpEntry c;
    c.start = e.start;
    c.end = e.end;
    c.gkey = gate_by_block ? (((uint64_t)e.block_index << 32) | e.warp_group)
                           : (uint64_t)e.warp_group;
    c.stage = s;
    c.pad = 0;
    out[out_off[s] + (k - lo)] = c;
    acc += e.end - e.start;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0 && acc) atomicAdd(&stage_sum[s], acc);
}

__device__ inline bool cp_close(uint64_t pred_end, uint64_t succ_start,
                                uint64_t theta) {
  const uint64_t lo = pred_end > theta ? pred_end - theta : 0;
  return succ_start >= lo && succ_start <= pred_end + theta;
}

// Program-order gating.  `by_end` = all entries sorted by (gkey, end);
// `pos_of` maps an entry (index in `all`) to its position in by_end so e != f
// can be tested.  bind[gate_stage * S + f_stage] += 1.
__global__ void k_cp_gate(const CpEntry* all, uint64_t n_all,
                          const CpEntry* by_end, const uint64_t* by_end_src,
                          uint64_t theta, uint32_t S,
                          unsigned long long* bind) {
  for (uint64_t fi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; fi < n_all;
       fi += (uint64_t)gridDim.x * blockDim.x) {
    const CpEntry f = all[fi];
    const uint64_t lo_end = f.start > theta ? f.start - theta : 0;
    const uint64_t hi_end = f.start + theta;
    // last position with (gkey, end) <= (f.gkey, hi_end)
    uint64_t lo = 0, hi = n_all;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      const CpEntry& m = by_end[mid];
      if (m.gkey < f.gkey || (m.gkey == f.gkey && m.end <= hi_end))
        lo = mid + 1;
      else
        hi = mid;
    }
    int64_t best = -1;
    uint64_t best_end = 0;
    uint32_t best_stage = 0;
    for (uint64_t p = lo; p-- > 0;) {
      const CpEntry& e = by_end[p];
      if (e.gkey != f.gkey || e.end < lo_end) break;
      if (best >= 0 && e.end < best_end) break;  // past the max-end group
      if (by_end_src[p] == fi || e.start > f.start) continue;
      if (!cp_close(e.end, f.start, theta)) continue;
      if (best < 0 || e.stage < best_stage) {
        best = (int64_t)p;
        best_end = e.end;
        best_stage = e.stage;
      }
    }
    if (best >= 0)
      atomicAdd(&bind[(uint64_t)best_stage * S + f.stage], 1ull);
  }
}

// Barrier edge src -> dst: count dst steady events f having some src event
// e with close(e.end, f.start).  src_ends sorted ascending.
__global__ void k_cp_barrier(const CpEntry* dst, uint64_t n_dst,
                             const uint64_t* src_ends, uint64_t n_src,
                             uint64_t theta, unsigned long long* counter) {
  unsigned long long acc = 0;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_dst;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = dst[k].start;
    // any e.end in [s - theta, s + theta] (close() with clamp at 0)
    const uint64_t lo_end = s > theta ? s - theta : 0;
    uint64_t lo = 0, hi = n_src;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (src_ends[mid] < lo_end) lo = mid + 1; else hi = mid;
    }
    if (lo < n_src && cp_close(src_ends[lo], s, theta)) ++acc;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0 && acc) atomicAdd(counter, acc);
}

__global__ void k_cp_ends(const CpEntry* e, uint64_t n, uint64_t* ends) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    ends[i] = e[i].end;
}

// ---- role overlap -------------------------------------------------------------
// Per Exec event with a role: up to two interval copies keyed by
// (block, set) with set 0 = role 0, 1 = role 1, 2 = roles 0+1.
__global__ void k_ov_expand(const wgpf_event* ev, uint64_t n,
                            const uint8_t* role_of_wg, uint32_t n_roles,
                            unsigned long long* key, uint64_t* s_out,
                            uint64_t* e_out, unsigned long long* span_lo,
                            unsigned long long* span_hi, uint64_t n_blocks) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const wgpf_event e = ev[i];
    if (e.block_index < n_blocks) {
      atomicMin(&span_lo[e.block_index], (unsigned long long)e.start);
      atomicMax(&span_hi[e.block_index], (unsigned long long)e.end);
    }
    uint32_t r = 2;
    if (!(e.region & WGPF_EV_WAIT) && e.warp_group < n_roles && e.end > e.start)
      r = role_of_wg[e.warp_group];
    const bool in = r < 2;
    const unsigned long long b = (unsigned long long)e.block_index << 2;
    key[2 * i] = in ? (b | r) : ~0ull;
    key[2 * i + 1] = in ? (b | 2u) : ~0ull;
    s_out[2 * i] = s_out[2 * i + 1] = e.start;
    e_out[2 * i] = e_out[2 * i + 1] = e.end;
  }
}

// Sorted by (key, start): union length per key.  Sequential over a key's
// run in one thread is fine for the per-CTA sizes here; runs are found by
// scanning from every run head.
__global__ void k_ov_union(const unsigned long long* key, const uint64_t* st,
                           const uint64_t* en, uint64_t n,
                           unsigned long long* out /* [blocks*4] */) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (key[i] == ~0ull) continue;
    if (i > 0 && key[i - 1] == key[i]) continue;  // not a run head
    uint64_t total = 0, cs = st[i], ce = en[i];
    uint64_t j = i + 1;
    for (; j < n && key[j] == key[i]; ++j) {
      if (st[j] <= ce) {
        if (en[j] > ce) ce = en[j];
      } else {
        total += ce - cs;
        cs = st[j];
        ce = en[j];
      }
    }
    total += ce - cs;
    atomicAdd(&out[key[i]], (unsigned long long)total);
  }
}

__global__ void k_iota_u64(uint64_t* a, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = i;
}

__global__ void k_gather_u64(const uint64_t* src, const uint64_t* perm,
                             uint64_t n, uint64_t* dst) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}

// gate keys of entries taken in the order `perm`
__global__ void k_cp_gkeys(const CpEntry* e, const uint64_t* perm, uint64_t n,
                           uint64_t* gk) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    gk[i] = e[perm[i]].gkey;
}

__global__ void k_cp_permute(const CpEntry* e, const uint64_t* perm, uint64_t n,
                             CpEntry* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = e[perm[i]];
}

__global__ void k_ov_maxblock(const wgpf_event* ev, uint64_t n,
                              unsigned long long* mx) {
  unsigned long long m = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)ev[i].block_index);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0) atomicMax(mx, m);
}

}  // namespace wgpf
