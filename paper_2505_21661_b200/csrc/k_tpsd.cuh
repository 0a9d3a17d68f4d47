// k_tpsd.cuh -- pass 2 of replay_image for DEEP and WIDE streams, thread per
// stream.  Same algorithm and outputs as k_tps (k_tps.cuh documents the
// reference mapping: unwrap_clock trace.hpp:257-272, pair_records :294-346,
// replay :398-487, region_stats pipeline.hpp:114-133); two geometries
// (DeepGeom below): the deep list (nesting <= 64, region ids < 64; config 5:
// 64 nested scopes, 64 labels) and the wide list (nesting <= 32, region ids
// < 256: plans with up to 256 labels).  What changes against k_tps:
//
//   * stacks.  The kernel is latency-bound (a lane's walk is a serial chain),
//     so warps per SM are what it runs on, and shared memory is what limits
//     them: the stack is split into a u32 clock row and a meta row of
//     {position (9 bits) | region | consumable} (u16 deep, u32 wide), and
//     the clock's high word is not stored at all: a pair's wrap count is read
//     off the positions of the lane's last two clock wraps (a duration
//     reaches 2^32 iff two wraps lie after the START, or one and the END's
//     low word is not below the START's).  Iteration counters are u8 (a
//     region completes at most cap / 2 <= 256 times), record windows 4
//     positions (+2) wide, three buffers: 12 warps per SM deep, 10 wide.
//   * statistics cannot be lane-private for 64+ classes.  Streams of a trace
//     usually advance in lockstep (same scope program, same wrap position),
//     so a warp's events of one step mostly share a class: then one lane
//     applies the warp's redux-reduced min / max to the CTA table with
//     fire-and-forget shared reductions and the sum and the match.any-
//     aggregated histogram bins to this CTA's replica rows in HBM with
//     fire-and-forget global reductions (k_deep_reduce adds the replicas;
//     counts are the bin sums); otherwise each lane updates the tables with
//     atomics.  First-event keys skip their reductions once the batch's
//     smallest stream has met the class.
//   * kMarkers = false (no ".wait" labels in the plan) compiles out the
//     consumed-wait / orphan-marker machinery of replay.
//   * record windows: one 2-D TMA box per window when the warp's 32 list
//     entries are 32 consecutive streams with one even start slot and the
//     window does not cross the circular wrap (config 5: all but one window
//     per stream), else 16-B cp.async chunks.  Lanes read records in 16-B
//     pairs when the start is even (conflict-free LDS.128 at the 48-B pitch).
//
// It runs over pass 1's deep and wide lists (SF_WARP | SF_DEEP, not
// general); the warp-per-stream kernel (k_fast.cuh) takes pass 1's warp
// list (the rest).  Capacities up to kDeepMaxSlots (positions in 9 bits).
#pragma once

#include <type_traits>

#include "k_tps.cuh"

namespace wgpf {

// Geometry.  kWide = false (the deep list): nesting <= 64, region ids < 64,
// u16 stack meta {position (9) | region (6) | consumable (1)}.  kWide = true
// (the wide list, plans with up to 256 region labels): nesting <= 32, region
// ids < 256, u32 meta {position (9) | region (8) | consumable (1)}; the
// iteration counters (u8 per region and lane) grow to 8 KB per warp and the
// CTA tables to 256 classes, the stack halves: 10 warps per SM.
template <bool kWide>
struct DeepGeom {
  static constexpr uint32_t kDepth = kWide ? 32u : 64u;
  static constexpr uint32_t kRegions = kWide ? 256u : 64u;
  static constexpr uint32_t kClasses = kWide ? 256u : kSmemClasses;
  using Meta = std::conditional_t<kWide, uint32_t, uint16_t>;
  static constexpr uint32_t kMetaRid = (kRegions - 1u) << 9;  // region bits of the meta
  static constexpr uint32_t kCons = kWide ? 17u : 15u;         // consumable bit
};
constexpr uint32_t kDeepDepth = DeepGeom<false>::kDepth;
constexpr uint32_t kDeepRegions = DeepGeom<false>::kRegions;
constexpr uint32_t kWideDepth = DeepGeom<true>::kDepth;
constexpr uint32_t kWideRegions = DeepGeom<true>::kRegions;
constexpr uint32_t kDeepMaxSlots = 512;  // stack positions in 9 bits
#ifndef WGPF_DEEP_W
#define WGPF_DEEP_W 4
#endif
constexpr uint32_t kDeepW = WGPF_DEEP_W;  // positions per record window
#ifndef WGPF_DEEP_P48
// exact-pitch windows: a lane row holds exactly the window's kDeepW records
// (odd starts copy records with 8-B cp.async instead of an extra 16-B chunk);
// measured on config 5: 6.37 vs 6.42 ms with the 48-B rows (WGPF_DEEP_P48),
// and the 1.5 KB it frees per warp buys nothing -- 13 warps: 6.47 ms
constexpr uint32_t kDeepChunks = kDeepW / 2;
constexpr uint32_t kDeepPitch = 8 * kDeepW;  // 32 B
#endif
// Swizzled window rows.  At the 32-B pitch a lane's 16-B pair reads are
// 2-way bank conflicted (lanes l and l + 4 of a quarter warp hit the same
// banks: 8 wavefronts per LDS.128 instead of 4, ncu: 24 % excess shared
// wavefronts).  The rows are stored with the two 16-B chunks of a row
// swapped when address bit 7 is set (the TMA's SWIZZLE_32B pattern, bit 4 ^=
// bit 7), which the cp.async fills and the reads follow: conflict-free.
#if !defined(WGPF_DEEP_P48) && !defined(WGPF_DEEP_NO_SWZ) && WGPF_DEEP_W == 4
#define WGPF_DEEP_SWZ 1
constexpr CUtensorMapSwizzle kDeepSwizzle = CU_TENSOR_MAP_SWIZZLE_32B;
#else
constexpr CUtensorMapSwizzle kDeepSwizzle = CU_TENSOR_MAP_SWIZZLE_NONE;
#endif
// byte offset of 16-B chunk c in the window row at shared address row
__device__ __forceinline__ uint32_t deep_chunk(uint32_t row, uint32_t c) {
#ifdef WGPF_DEEP_SWZ
  return 16u * (c ^ ((row >> 7) & 1u));
#else
  return 16u * c;
#endif
}
#ifdef WGPF_DEEP_P48
constexpr uint32_t kDeepChunks = WinGeom<kDeepW>::kChunks;
constexpr uint32_t kDeepPitch = WinGeom<kDeepW>::kPitch;  // 48 B: 12 words
#endif
#ifndef WGPF_DEEP_WARPS
#define WGPF_DEEP_WARPS 12
#endif
constexpr uint32_t kDeepWarps = WGPF_DEEP_WARPS;
#ifndef WGPF_DEEP_UNROLL
#define WGPF_DEEP_UNROLL 2  // record pairs per full-step loop iteration (measured: 2 > 1 by 1 %)
#endif
constexpr int kDeepUnroll = WGPF_DEEP_UNROLL;

#ifndef WGPF_DEEP_BUFS
#define WGPF_DEEP_BUFS 3
#endif
constexpr uint32_t kDeepBufs = WGPF_DEEP_BUFS;  // record windows: 2 or 3 (1 / 2 ahead)

template <bool kWide>
struct DeepWarpSmem {
  using G = DeepGeom<kWide>;
  uint8_t rec[kDeepBufs][32 * kDeepPitch];  // record windows
  uint32_t lo_empty[32];                    // row -1 of each stack array: what
  uint32_t stk_lo[G::kDepth][32];           //   an empty stack reads (never
  typename G::Meta meta_empty[32];          //   written; the value is unused)
  typename G::Meta stk_meta[G::kDepth][32]; // START clock (low word);
                                            // position | region | consumable
  uint8_t cnt[G::kRegions][32];             // iteration counters
  uint32_t seen[G::kClasses / 32];          // (kWide) first-key classes met
  unsigned long long bar[kDeepBufs];        // TMA windows: one mbarrier per buffer
};

// Per CTA only what needs a shared reduction: min / max (native u32 shared
// reductions) and the first-event key.  Sums and histogram bins go to this
// CTA's own replica of the table in global memory (kDeepRep u64 per class:
// [unused], sum, 64 bins; a class's count is the sum of its bins) with
// fire-and-forget global reductions
// (native u64 in L2; a 64-bit shared add would be a CAS loop), aggregated per
// warp first; k_deep_reduce sums the replicas afterwards.  Per-CTA replicas
// keep SMs off each other's L2 lines (one shared table: 40 % slower), and
// moving the 16-KB histogram out of shared memory buys warps.
constexpr uint32_t kDeepRep = 2 + WGPF_HIST_BINS;
template <bool kWide>
struct DeepCtaSmem {
  using G = DeepGeom<kWide>;
  unsigned long long first[G::kClasses];
  uint32_t min[G::kClasses];
  uint32_t max[G::kClasses];
  uint32_t info[G::kRegions];  // class | marker<<8 | wait class<<16
  unsigned long long warn[4];
};

__host__ __device__ inline size_t deep_smem_bytes(uint32_t warps, bool wide = false) {
  return wide ? tps_align(sizeof(DeepCtaSmem<true>)) +
                    warps * tps_align(sizeof(DeepWarpSmem<true>))
              : tps_align(sizeof(DeepCtaSmem<false>)) +
                    warps * tps_align(sizeof(DeepWarpSmem<false>));
}
__host__ inline uint32_t deep_warps(size_t smem_limit, bool wide = false) {
  uint32_t w = kDeepWarps;
  while (w > 1 && deep_smem_bytes(w, wide) > smem_limit) --w;
  return w;
}
// per-CTA replica rows of the statistics (k_tpsd / k_deep_reduce)
__host__ __device__ inline uint32_t deep_classes(bool wide) {
  return wide ? DeepGeom<true>::kClasses : DeepGeom<false>::kClasses;
}

__device__ __forceinline__ uint32_t lds8(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts8_if(bool p, uint32_t a, uint32_t v) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q st.shared.u8 [%1], %2; }" ::"r"(
                   (uint32_t)p),
               "r"(a), "h"((uint16_t)v)
               : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((uint16_t)v) : "memory");
}
// stack meta rows: u16 (deep) or u32 (wide)
template <class M>
__device__ __forceinline__ uint32_t lds_meta(uint32_t a) {
  if constexpr (sizeof(M) == 2) return lds16(a); else return lds32(a);
}
template <class M>
__device__ __forceinline__ void sts_meta(uint32_t a, uint32_t v) {
  if constexpr (sizeof(M) == 2) sts16(a, v); else sts32(a, v);
}
template <class M>
__device__ __forceinline__ void sts_meta_if(bool p, uint32_t a, uint32_t v) {
  if constexpr (sizeof(M) == 2) sts16_if(p, a, v); else sts32_if(p, a, v);
}
__device__ __forceinline__ void red_gadd64(unsigned long long* a, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void red_min32(uint32_t a, uint32_t v) {
  asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_max32(uint32_t a, uint32_t v) {
  asm volatile("red.shared.max.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// tm: the body as a 2-D TMA tensor {stride / 4, n_streams}, box
// {kDeepPitch / 4, 32} (a.tma != 0).
// kMarkers: the plan has wait-marker labels ("X.wait").  Without them no
// record can be a consumed wait or an orphan marker (replay,
// trace.hpp:421-485, only pairs a base with a ".wait" class), so that
// machinery -- about a fifth of an END step -- is compiled out.
// kWide: the geometry above (DeepGeom).
template <bool kEmit, bool kStats, bool kMarkers, bool kWide>
__global__ void __launch_bounds__(kDeepWarps * 32, 1)
    k_tpsd(FastArgs a, const __grid_constant__ CUtensorMap tm) {
  using G = DeepGeom<kWide>;
  using CtaS = DeepCtaSmem<kWide>;
  using WarpS = DeepWarpSmem<kWide>;
  constexpr uint32_t kMS = sizeof(typename G::Meta) / 2u;  // meta row scale
  extern __shared__ __align__(128) uint8_t smem_raw[];
  CtaS& cs = *reinterpret_cast<CtaS*>(smem_raw);
  const uint32_t lane = lane_id();
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t nw = blockDim.x >> 5;
  const uint32_t K = a.plan.K;
  WarpS& ws = *reinterpret_cast<WarpS*>(smem_raw + tps_align(sizeof(CtaS)) +
                                        w * tps_align(sizeof(WarpS)));
  constexpr bool stats = kStats;
  constexpr bool emit = kEmit;
  for (uint32_t c = threadIdx.x; c < G::kClasses; c += blockDim.x) {
    cs.first[c] = ~0ull;
    cs.min[c] = 0xFFFFFFFFu;
    cs.max[c] = 0u;
  }
  for (uint32_t r = threadIdx.x; r < G::kRegions; r += blockDim.x) {
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
    for (uint32_t k = 0; k < kDeepBufs; ++k) win_bar_init(s_bar + 8u * k);
    win_bar_fence();
  }
  uint32_t bphase = 0;  // parity of each buffer's next TMA completion
  __syncthreads();
  const bool abort_all = a.status->decode_err != kNoErr;
  const uint32_t FULL = 0xffffffffu;
  const uint32_t cost = (uint32_t)a.record_cost;  // host: < 2^21 on this path
  const uint32_t cap = a.cap;
  uint32_t w_drop = 0, w_tail = 0, w_flag = 0, w_mal = 0, w_ovf = 0;

  const uint32_t s_info = opaque_u32(smem_addr(cs.info));
  const uint32_t s_lo = smem_addr(&ws.stk_lo[0][lane]);      // + 128 * level
  const uint32_t s_meta = smem_addr(&ws.stk_meta[0][lane]);  // + 64 kMS * level
  const uint32_t s_cnt = smem_addr(&ws.cnt[0][lane]);        // + 32 * region
  const uint32_t s_cnt_all = smem_addr(&ws.cnt[0][0]);
  const uint32_t s_min = opaque_u32(smem_addr(cs.min));
  const uint32_t s_max = opaque_u32(smem_addr(cs.max));
  // one orphan per lane, in global scratch (rare)
  wgpf_event* const orph = a.orphan_scratch + ((size_t)blockIdx.x * nw + w) * 32u + lane;
  const uint32_t s_rec = smem_addr(ws.rec[0]);
  const uint64_t n_list = *a.list_len;

  // this CTA's replica of the count / sum / histogram table
  unsigned long long* const rep = a.deep_rep + (size_t)blockIdx.x * G::kClasses * kDeepRep;
  const uint32_t s_seen = smem_addr(ws.seen);  // (kWide)
  // First-event keys.  Keys are (stream, event index): a lane meets its
  // keys in increasing order and the batch's smallest stream (lane `lmin`)
  // beats every other lane.  So once a warp-uniform step of class c has had
  // lmin participate, no later event of class c in this batch can lower the
  // minimum: `wseen` (warp-uniform, bit c) skips the key reductions then.
  unsigned long long wseen = 0;
  uint32_t lmin = 0;
  // one event per participating lane into the statistics
  auto wstat = [&](bool p, uint32_t cls, uint32_t d, unsigned long long key) {
    const uint32_t pm = __ballot_sync(FULL, p);
    if (pm == 0) return;
    // one class for every participating lane?  (two independent reductions)
    const uint32_t c0 = __reduce_min_sync(FULL, p ? cls : 0xFFFFFFFFu);
    const bool uni = c0 == __reduce_max_sync(FULL, p ? cls : 0u);
    const uint32_t leader = __ffs(pm) - 1u;
    // histogram bin: lanes with the same bin aggregate into one reduction
    const uint32_t bin = hist_bin32(d);
    if (uni && c0 < G::kClasses && c0 < K) {
      unsigned long long* const rc = rep + c0 * kDeepRep;  // this class's replica row
      const uint32_t dd = p ? d : 0u;
      const uint32_t mn = __reduce_min_sync(FULL, p ? d : 0xFFFFFFFFu);
      const uint32_t mx = __reduce_max_sync(FULL, dd);
      // the sum: one 32-bit reduction when 32 x max cannot carry out, else
      // two 16-bit halves
      unsigned long long sum;
      if (mx < (1u << 27)) {
        sum = __reduce_add_sync(FULL, dd);
      } else {
        const uint32_t slo = __reduce_add_sync(FULL, dd & 0xFFFFu);
        const uint32_t shi = __reduce_add_sync(FULL, dd >> 16);
        sum = (unsigned long long)slo + ((unsigned long long)shi << 16);
      }
      const uint32_t same = __match_any_sync(FULL, p ? bin : 0xFFFFFFFFu);
      bool seen;
      if constexpr (kWide)  // (lane 0's view of the warp's table, broadcast)
        seen = (__shfl_sync(FULL, lds32(s_seen + 4u * (c0 >> 5)), 0) >> (c0 & 31u)) & 1u;
      else
        seen = (wseen >> c0) & 1ull;
      if (!seen) {
        // smallest 64-bit first-event key of the participating lanes
        const unsigned long long cur_first =
            *reinterpret_cast<volatile unsigned long long*>(&cs.first[c0]);
        const uint32_t khi = __reduce_min_sync(FULL, p ? (uint32_t)(key >> 32) : 0xFFFFFFFFu);
        const bool cand = p && (uint32_t)(key >> 32) == khi;
        const uint32_t klo = __reduce_min_sync(FULL, cand ? (uint32_t)key : 0xFFFFFFFFu);
        const unsigned long long fk = ((unsigned long long)khi << 32) | klo;
        if (lane == leader && fk < cur_first) atomicMin(&cs.first[c0], fk);
        if ((pm >> lmin) & 1u) {
          if constexpr (kWide) {
            if (lane == 0)
              sts32(s_seen + 4u * (c0 >> 5), lds32(s_seen + 4u * (c0 >> 5)) | (1u << (c0 & 31u)));
          } else {
            wseen |= 1ull << c0;
          }
        }
      }
      if (lane == leader) {
        // fire-and-forget reductions: nothing comes back to wait for (the
        // count is the sum of the histogram bins, k_deep_reduce)
        red_gadd64(rc + 1u, sum);
        red_min32(s_min + 4u * c0, mn);
        red_max32(s_max + 4u * c0, mx);
      }
      if (p && lane == __ffs(same) - 1u) red_gadd64(rc + 2u + bin, (unsigned long long)__popc(same));
    } else if (p) {
      if (cls < G::kClasses && cls < K) {
        red_gadd64(rep + cls * kDeepRep + 1u, (unsigned long long)d);
        red_gadd64(rep + cls * kDeepRep + 2u + bin, 1ull);
        red_min32(s_min + 4u * cls, d);
        red_max32(s_max + 4u * cls, d);
        smin64(&cs.first[cls], key);
      } else {
        stats_add_global(a.stats, stats_slot(a.stats, cls, &a.status->synth_overflow), d,
                         key);
      }
    }
  };

  const uint64_t wstep = (uint64_t)gridDim.x * nw;
  for (uint64_t b = (uint64_t)blockIdx.x * nw + w; !abort_all && b * 32 < n_list; b += wstep) {
    const uint64_t li = b * 32 + lane;
    const uint64_t s = li < n_list ? a.list[li] : 0ull;
    const uint32_t flag = li < n_list ? a.sflag[s] : SF_DECODE_ERR;
    if ((flag & SF_GENERAL) && a.list_general) {
      // (a re-emit after an exact recount: the stream is the general path's)
      const unsigned long long k = atomicAdd(a.general_len, 1ull);
      a.general_list[k] = s;
    }
    const bool act = (flag & SF_DEEP) && !(flag & (SF_DECODE_ERR | SF_GENERAL));
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
    const unsigned long long gkey = (unsigned long long)(s + a.stream_base) << 25;
    {
      // lane of the batch's smallest active stream (first-key shortcut)
      const uint32_t shi_ = __reduce_min_sync(FULL, act ? (uint32_t)(s >> 32) : 0xFFFFFFFFu);
      const uint32_t slo_ =
          __reduce_min_sync(FULL, act && (uint32_t)(s >> 32) == shi_ ? (uint32_t)s : 0xFFFFFFFFu);
      lmin = __ffs(__ballot_sync(FULL, act && s == (((uint64_t)shi_ << 32) | slo_))) - 1u;
      wseen = 0;
      if (kWide && lane < G::kClasses / 32u) sts32(s_seen + 4u * lane, 0u);
    }
    const uint2* slots = reinterpret_cast<const uint2*>(sbase + 16);
    // iteration counters: the warp clears its 2 KB table with 16-B stores
#pragma unroll
    for (uint32_t k = lane; k < G::kRegions * 32u / 16u; k += 32)
      sts128_if(true, s_cnt_all + 16u * k, make_uint4(0u, 0u, 0u, 0u));
    __syncwarp();

    // TMA windows: the warp's list entries are 32 consecutive streams with
    // one even start slot (config 5: every batch)
    const uint32_t s32 = (uint32_t)s;
    const uint32_t s_first = __shfl_sync(FULL, s32, 0);
    const uint32_t st0 = __shfl_sync(FULL, start, 0);
    const bool tmab = a.tma && __all_sync(FULL, act && s32 == s_first + lane &&
                                                    start == st0 && (start & 1u) == 0u);
    // cp.async windows: chunk k of this lane copies part (q % C) of the
    // window of batch slot q / C, q = 32 k + lane; that slot's stream from
    // its lane.  wst[k]: that stream's start slot (the chunk's physical slot
    // for a window is computed when a window needs cp.async -- one per
    // stream on config 5, at the circular wrap)
    uint32_t wst[kDeepChunks];
    const uint8_t* srck[kDeepChunks];  // slots of chunk k's stream (null: none)
    const uint32_t live = act ? 1u : 0u;
#pragma unroll
    for (uint32_t k = 0; k < kDeepChunks; ++k) {
      const uint32_t q = k * 32u + lane, sl = q / kDeepChunks;
      wst[k] = __shfl_sync(FULL, start, sl);
      const uint32_t ss = __shfl_sync(FULL, s32, sl);
      srck[k] = __shfl_sync(FULL, live, sl) ? a.body + (uint64_t)ss * a.stride + 16 : nullptr;
    }
    uint32_t tma_buf = 0;  // bit b: buffer b's window came by TMA
    auto issue = [&](uint32_t bsel, uint32_t c0) {
      // (physical slot of the window's first position: even on this path)
      uint32_t p = st0 + c0;
      p = p >= cap ? p - cap : p;
      if (tmab && p + kDeepW <= cap) {
        if (lane == 0)
          win_tma(s_rec + bsel * (32 * kDeepPitch), &tm, s_bar + 8u * bsel,
                  (int)(4u + 2u * p), (int)s_first, 32u * kDeepPitch);
        tma_buf |= 1u << bsel;
      } else {
        tma_buf &= ~(1u << bsel);
#pragma unroll
        for (uint32_t k = 0; k < kDeepChunks; ++k) {
          const uint32_t q = k * 32u + lane, sl = q / kDeepChunks, part = q % kDeepChunks;
#ifndef WGPF_DEEP_P48
          // records c0 + 2 part, + 1 of the window: one 16-B chunk at an
          // even physical slot, else two 8-B records (the second may wrap)
          uint32_t p = wst[k] + c0 + 2u * part;
          p = p >= cap ? p - cap : p;
          p = p >= cap ? p - cap : p;
          const uint32_t row = s_rec + bsel * (32 * kDeepPitch) + sl * kDeepPitch;
          const uint32_t dst = row + deep_chunk(row, part);
          if (srck[k]) {
            if ((p & 1u) == 0u) {
              cp_async16(dst, srck[k] + 8u * p);
            } else {
              const uint32_t p1 = p + 1u == cap ? 0u : p + 1u;
              cp_async8(dst, srck[k] + 8u * p);
              cp_async8(dst + 8u, srck[k] + 8u * p1);
            }
          }
#else
          // the even physical slot at or below (start + c0) mod cap, + part
          uint32_t p = wst[k] + c0;
          p = p >= cap ? p - cap : p;  // (c0 < cap + 2: one subtraction
          p = p >= cap ? p - cap : p;  //  may not suffice)
          p = (p & ~1u) + 2u * part;
          p = p >= cap ? p - cap : p;
          if (srck[k])
            cp_async16(s_rec + bsel * (32 * kDeepPitch) + sl * kDeepPitch + 16u * part,
                       srck[k] + 8u * p);
#endif
        }
      }
    };

    uint2 r0 = make_uint2(0u, 0u), r1 = make_uint2(0u, 0u);
    if (n > 0) r0 = slots[start];
    if (n > 1) r1 = slots[start + 1 < cap ? start + 1 : start + 1 - cap];
    uint32_t inf0 = cs.info[(r0.x >> 12) & (G::kRegions - 1u)];
    // kDeepBufs - 1 windows in flight ahead of the walk
    issue(0, 2);
    cp_async_commit();
    if (kDeepBufs == 3) {
      if (kDeepW < nmax) issue(1, 2 + kDeepW);
      cp_async_commit();
    }

    // stack top: offset 64 * level (meta) / 128 * level (clock); empty = -64
    // (reads row -1 of each array: lo_empty / meta_empty, never written, used
    // only when an END has a partner)
    int32_t tp = -64;
    uint32_t hi = 0, vprev = 0;
    uint32_t w_last = 0, w_prev = 0;  // positions of the last two clock wraps
    uint32_t pw = 0xFFu;
    uint32_t kw = 0;
    uint32_t n_orph = 0;
    bool broken = false;
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
    auto step = [&](auto full, uint32_t i, uint2 r2) {
      constexpr bool kFull = decltype(full)::value;
      const bool valid = kFull || i < n;
      const uint32_t tag = r0.x, v = r0.y;
      const bool isS = (int32_t)tag < 0;
      const bool st = valid && isS;
      const bool en = valid && !isS;
      const uint32_t rid = (tag >> 12) & (G::kRegions - 1u);
      const uint32_t inf = inf0;
      const uint32_t r1id = (r1.x >> 12) & (G::kRegions - 1u);
      const uint32_t i1 = lds32(s_info + 4u * r1id);
      const bool wrap = valid && v < vprev;
      const uint32_t meta_new =
          i | ((tag >> 3) & G::kMetaRid) |
          ((kMarkers && pw == (inf & 0xFFu) ? 1u : 0u) << G::kCons);
      if constexpr (kFull) {
        // every lane at a START (the streams of a trace run the same program
        // from the same wrap position): a push is all that happens
        if (__all_sync(FULL, isS)) {
          hi += wrap ? 1u : 0u;
          w_prev = wrap ? w_last : w_prev;
          w_last = wrap ? i : w_last;
          vprev = v;
          tp += 64;
          sts32(s_lo + 2 * tp, v);
          sts_meta<typename G::Meta>(s_meta + kMS * tp, meta_new);
          pw = 0xFFu;
          inf0 = i1;
          r0 = r1;
          r1 = r2;
          return;
        }
      }
      hi += wrap ? 1u : 0u;
      w_prev = wrap ? w_last : w_prev;
      w_last = wrap ? i : w_last;
      vprev = valid ? v : vprev;
      const uint32_t elo = lds32(s_lo + 2 * tp);
      const uint32_t em = lds_meta<typename G::Meta>(s_meta + kMS * tp);
      const bool nonempty = tp >= 0;
      const bool mend = en && nonempty;
      w_drop += (en && !nonempty) ? 1u : 0u;
      sts32_if(st, s_lo + 2 * (tp + 64), v);
      sts_meta_if<typename G::Meta>(st, s_meta + kMS * (tp + 64), meta_new);
      tp += (st ? 64 : 0) - (mend ? 64 : 0);
      const uint32_t spos = em & 511u;
      const uint32_t meas = v - elo;  // low 32 bits of u - su
      // the pair spans >= 2^32 cycles iff two clock wraps lie after the
      // START, or one and the END's low word is not below the START's
      const bool tl = w_prev > spos || (w_last > spos && v >= elo);
      const bool mism = mend && ((em ^ (tag >> 3)) & G::kMetaRid) != 0u;
      const bool tlong = mend && !mism && tl;
      broken |= mism || tlong;
      const bool ok = mend && !mism && !tlong;
      const uint32_t shi = hi - (v < elo ? 1u : 0u);
      const uint32_t ca = s_cnt + 32u * rid;
      const uint32_t it = lds8(ca);
      sts8_if(ok, ca, it + 1u);
      const bool is_mk = kMarkers && (inf & 0x100u) != 0u;
      const bool base = ok && !is_mk;
      const bool orphan = kMarkers && ok && is_mk && !((em >> G::kCons) & 1u);
      const uint32_t dpos = i - spos;
      const uint32_t ovh = cost * dpos;
      const uint32_t corr = ovh > meas ? 0u : meas - ovh;
      const bool cclose = (kFull || i + 2 < n) && (int32_t)r2.x >= 0 &&
                          ((r2.x >> 12) & (G::kRegions - 1u)) == r1id;
      const bool consumed = kMarkers && base && (kFull || i + 1 < n) && (int32_t)r1.x < 0 &&
                            (i1 & 0x100u) && (inf >> 16) == (i1 & 0xFFu) &&
                            ((int32_t)(i + 1) <= z || cclose);
      const uint32_t wd = r1.y - v;
      const bool corr_w = wd > cost;
      w_flag += (consumed && !corr_w) ? 1u : 0u;
      const uint32_t kpos = kw;
      if constexpr (emit) {
        const uint32_t eend = elo + corr;
        put(base, kw, elo, shi, eend, shi + (eend < corr ? 1u : 0u), rid | WGPF_EV_CORRECTED,
            it);
        if constexpr (kMarkers)
          put(consumed, kw + 1u, v, hi, r1.y, hi + (r1.y < v ? 1u : 0u),
              r1id | WGPF_EV_WAIT | (corr_w ? WGPF_EV_CORRECTED : 0u), it);
      }
      kw += (base ? 1u : 0u) + (consumed ? 1u : 0u);
      pw = base ? (inf >> 16) : 0xFFu;
      if (orphan && n_orph == 0)
        *orph = wgpf_event{(uint64_t)elo | ((uint64_t)shi << 32), (uint64_t)v | ((uint64_t)hi << 32),
                           rid, it, 0u, 0u};
      n_orph += orphan ? 1u : 0u;
      if constexpr (stats) {
        wstat(base, inf & 0xFFu, corr, gkey | (kpos << 1));
        if constexpr (kMarkers)
          if (__any_sync(FULL, consumed))
            wstat(consumed, i1 & 0xFFu, wd, gkey | ((kpos + 1u) << 1) | 1u);
      }
      inf0 = i1;
      r0 = r1;
      r1 = r2;
    };

    const uint32_t nmin = __reduce_min_sync(FULL, act ? n : 0u);
    const bool even_start = __all_sync(FULL, (start & 1u) == 0u);
    uint32_t bsel = 0, bnext = kDeepBufs - 1u;  // window k's buffer: k % kDeepBufs
    constexpr uint32_t ahead = (kDeepBufs - 1u) * kDeepW;
    for (uint32_t w0 = 0; w0 < nmax; w0 += kDeepW) {
      if (w0 + ahead < nmax) issue(bnext, w0 + ahead + 2u);
      cp_async_commit();
      if (kDeepBufs == 3)
        cp_async_wait2();
      else
        cp_async_wait1();
      if ((tma_buf >> bsel) & 1u) {
        win_wait(s_bar + 8u * bsel, (bphase >> bsel) & 1u);
        bphase ^= 1u << bsel;
      }
      __syncwarp();
#ifndef WGPF_DEEP_P48
      const uint2* myrec = reinterpret_cast<const uint2*>(ws.rec[bsel] + lane * kDeepPitch);
      constexpr bool kPairs = true;  // rows are 16-B aligned for any start
#ifdef WGPF_DEEP_SWZ
      const uint32_t myrow = s_rec + bsel * (32 * kDeepPitch) + lane * kDeepPitch;
      const uint32_t msw = (myrow >> 7) & 1u;  // chunks of this row swapped
      // record j of the window (chunk j / 2, half j % 2)
      const uint8_t* const myrowp = ws.rec[bsel] + lane * kDeepPitch;
      auto rec_at = [&](uint32_t j) {
        return *reinterpret_cast<const uint2*>(myrowp + 16u * ((j >> 1) ^ msw) + 8u * (j & 1u));
      };
#else
      auto rec_at = [&](uint32_t j) { return myrec[j]; };
#endif
#else
      const uint2* myrec = reinterpret_cast<const uint2*>(
          ws.rec[bsel] + lane * kDeepPitch + 8u * (start & 1u));
      const bool kPairs = even_start;
      auto rec_at = [&](uint32_t j) { return myrec[j]; };
#endif
      if (w0 + kDeepW + 2u <= nmin) {
        if (kPairs) {
          // 16-B record pairs: one conflict-free LDS.128 per two steps
          const uint4* myrec2 = reinterpret_cast<const uint4*>(myrec);
#pragma unroll kDeepUnroll
          for (uint32_t j = 0; j < kDeepW; j += 2) {
#ifdef WGPF_DEEP_SWZ
            const uint4 q = *reinterpret_cast<const uint4*>(myrowp + 16u * ((j >> 1) ^ msw));
#else
            const uint4 q = myrec2[j / 2];
#endif
            step(std::true_type{}, w0 + j, make_uint2(q.x, q.y));
            step(std::true_type{}, w0 + j + 1, make_uint2(q.z, q.w));
          }
        } else {
#pragma unroll 1
          for (uint32_t j = 0; j < kDeepW; ++j) step(std::true_type{}, w0 + j, rec_at(j));
        }
      } else {
#pragma unroll 1
        for (uint32_t j = 0; j < kDeepW; ++j) step(std::false_type{}, w0 + j, rec_at(j));
      }
      __syncwarp();
      bsel = bsel == kDeepBufs - 1u ? 0u : bsel + 1u;
      bnext = bnext == kDeepBufs - 1u ? 0u : bnext + 1u;
    }
    const bool bad = broken || n_orph > 1;
    const bool po = act && !bad && n_orph == 1;
    if (__any_sync(FULL, po)) {
      const wgpf_event o = po ? *orph : wgpf_event{};
      if (emit)
        put(po, kw, (uint32_t)o.start, (uint32_t)(o.start >> 32), (uint32_t)o.end,
            (uint32_t)(o.end >> 32), o.region, o.iteration);
      if (stats)
        wstat(po, cs.info[o.region & (G::kRegions - 1u)] & 0xFFu,
              (uint32_t)(o.end - o.start), gkey | (kw << 1));
      kw += po ? 1u : 0u;
    }
    w_ovf += act && kw > lim ? kw - lim : 0u;
    if (act) {
      if (bad || kw != want) {
        atomicAdd(&a.status->invalid, 1ull);
        a.sflag[s] = flag | SF_INVALID;
      }
      if (!bad) {
        w_mal += n_orph;
        w_tail += (uint32_t)(tp + 64) >> 6;
      }
    }
  }
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
  __syncthreads();
  if (threadIdx.x < 4 && cs.warn[threadIdx.x])
    atomicAdd(&a.status->warn[threadIdx.x], cs.warn[threadIdx.x]);
  if (stats) {  // the CTA's min / max / first keys into the global table
    const uint32_t kc = K < G::kClasses ? K : G::kClasses;
    for (uint32_t c = threadIdx.x; c < kc; c += blockDim.x) {
      if (cs.min[c] == 0xFFFFFFFFu && cs.max[c] == 0u && cs.first[c] == ~0ull) continue;
      atomicMin(&a.stats.min[c], (unsigned long long)cs.min[c]);
      atomicMax(&a.stats.max[c], (unsigned long long)cs.max[c]);
      atomicMin(&a.stats.first[c], cs.first[c]);
    }
  }
}

// Sums the per-CTA replicas of the deep kernel into the global table.
// classes: the replica rows per CTA (deep_classes)
__global__ void k_deep_reduce(const unsigned long long* rep, uint32_t ctas, uint32_t K,
                              DevStats st, uint32_t classes) {
  const uint32_t kc = K < classes ? K : classes;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < kc * kDeepRep;
       i += gridDim.x * blockDim.x) {
    unsigned long long t = 0;
    for (uint32_t b = 0; b < ctas; ++b) t += rep[(size_t)b * classes * kDeepRep + i];
    if (!t) continue;
    const uint32_t c = i / kDeepRep, f = i % kDeepRep;
    if (f == 0)
      continue;  // (unused: counts are the bin sums, below)
    else if (f == 1)
      atomicAdd(&st.sum[c], t);
    else {
      atomicAdd(&st.hist[c * WGPF_HIST_BINS + (f - 2)], t);
      atomicAdd(&st.count[c], t);  // a class's count is the sum of its bins
    }
  }
}

}  // namespace wgpf
