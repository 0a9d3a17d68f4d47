// k_window.cuh -- record windows of the thread-per-stream kernels (k_tps,
// k_count_tps): a warp owns 32 consecutive streams (lane l = stream l) and
// walks them in lockstep over chronological positions.  Records reach shared
// memory in windows of kTpsW positions per stream, double buffered, with
// cp.async 16-B chunks.  Chunk k of the window of stream l is copied by a
// fixed lane (q = k * 32 + lane -> stream q / kTpsChunks, part q % kTpsChunks),
// so one copy instruction covers a few contiguous runs of the body.
//
// Circular streams start at physical slot `start` (trace.hpp:243-246); a
// window for chronological position c0 starts at the even physical slot at or
// below (start + c0) mod cap, so 16-B chunks never straddle the wrap (the
// capacity is even on this path) and the lane reads its records at offset
// (start & 1) in its window.
#pragma once

#include <cuda.h>  // CUtensorMap

#include "wgpf_dev.cuh"

namespace wgpf {

// records per window: kW (template); the emit kernel uses kTpsW
template <uint32_t kW>
struct WinGeom {
  static constexpr uint32_t kChunks = (kW + 2) / 2;  // 16-B chunks per window
  static constexpr uint32_t kPitch = 16 * kChunks;   // bytes per lane window
};
constexpr uint32_t kTpsW = 8;
constexpr uint32_t kTpsChunks = WinGeom<kTpsW>::kChunks;
constexpr uint32_t kTpsPitch = WinGeom<kTpsW>::kPitch;
constexpr uint32_t kTpsMaxSlots = 2046;               // even; pos fits 11 bits

__device__ __forceinline__ void cp_async16(uint32_t sdst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t sdst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sdst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait2() {
  asm volatile("cp.async.wait_group 2;" ::: "memory");
}

template <uint32_t kW = kTpsW>
struct RecWindowsT {
  static constexpr uint32_t kTpsW = kW;
  static constexpr uint32_t kTpsChunks = WinGeom<kW>::kChunks;
  static constexpr uint32_t kTpsPitch = WinGeom<kW>::kPitch;
  uint32_t slk[kTpsChunks];                  // static chunk assignment:
  uint32_t sdst[kTpsChunks];                 //   stream, shared destination
  uint32_t wp[kTpsChunks], wlim[kTpsChunks]; // physical slot, stream length
  const uint8_t* src[kTpsChunks];            // slots of chunk k's stream
  uint64_t stride;
  uint32_t cap;
  uint8_t* buf;                              // [2][32 * kTpsPitch]
  uint32_t pk2[kTpsChunks];                  // 2 * part (slots)

  __device__ __forceinline__ void init(uint8_t* smem, uint32_t lane,
                                       uint64_t stride_, uint32_t cap_) {
    buf = smem;
    stride = stride_;
    cap = cap_;
    const uint32_t b0 = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
#pragma unroll
    for (uint32_t k = 0; k < kTpsChunks; ++k) {
      const uint32_t q = k * 32 + lane;
      slk[k] = q / kTpsChunks;
      const uint32_t part = q - slk[k] * kTpsChunks;
      pk2[k] = 2u * part;
      sdst[k] = b0 + slk[k] * kTpsPitch + 16u * part;
    }
  }
  // streams of this batch: body of the warp's first stream, this lane's
  // stream start slot and length; first window at c0 = 2 (records 0 and 1
  // are loaded directly)
  __device__ __forceinline__ void begin(const uint8_t* batch_body,
                                        uint32_t start, uint32_t n) {
#pragma unroll
    for (uint32_t k = 0; k < kTpsChunks; ++k) {
      src[k] = batch_body + 16 + (uint64_t)slk[k] * stride;
      const uint32_t st_k = __shfl_sync(0xffffffffu, start, slk[k]);
      wlim[k] = __shfl_sync(0xffffffffu, n, slk[k]);
      uint32_t p = st_k + 2u;
      if (p >= cap) p -= cap;
      p = (p & ~1u) + pk2[k];
      if (p >= cap) p -= cap;
      wp[k] = p;
    }
  }
  // copy the window of chronological positions [c0, c0 + kTpsW) of all 32
  // streams into buffer bsel (windows are issued in order, c0 += kTpsW)
  __device__ __forceinline__ void issue(uint32_t bsel, uint32_t c0) {
    const uint32_t boff = bsel * (32 * kTpsPitch);
#pragma unroll
    for (uint32_t k = 0; k < kTpsChunks; ++k) {
      if (c0 < wlim[k]) cp_async16(sdst[k] + boff, src[k] + 8u * wp[k]);
      wp[k] += kTpsW;
      if (wp[k] >= cap) wp[k] -= cap;
    }
  }
  // this lane's records in buffer bsel
  __device__ __forceinline__ const uint2* lane_records(uint32_t bsel, uint32_t lane,
                                                       uint32_t start) const {
    return reinterpret_cast<const uint2*>(buf + bsel * (32 * kTpsPitch) +
                                          lane * kTpsPitch + 8u * (start & 1u));
  }
};
using RecWindows = RecWindowsT<kTpsW>;

// ---- TMA windows ---------------------------------------------------------------
// When all 32 streams of a batch start at slot 0 (flush plans, and circular
// streams that never wrapped), the window of positions [c0, c0 + kW + 2) of
// the 32 streams is one 2-D box of the body -- 32 rows (streams) x kPitch
// bytes at byte 16 + 8 c0 -- in exactly the per-lane layout above: one TMA
// load by one lane instead of kChunks cp.async per lane.  The host encodes
// the body as a u32 tensor {stride / 4, n_streams}, box {kPitch / 4, 32};
// bytes past a row's end are zero-filled (positions >= n, never used).
__device__ __forceinline__ void win_bar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void win_bar_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// (one lane) expect `bytes` on bar and start the box load at (x, y)
__device__ __forceinline__ void win_tma(uint32_t dst, const CUtensorMap* m, uint32_t bar,
                                        int x, int y, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
// 3-D form: the body as {stride / 4, W, n_blocks} (streams of a block
// innermost), box {kPitch / 4, 1, 32}: one warp index of 32 blocks
__device__ __forceinline__ void win_tma3(uint32_t dst, const CUtensorMap* m, uint32_t bar,
                                         int x, int y, int z, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void win_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WIN_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WIN_WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

}  // namespace wgpf
