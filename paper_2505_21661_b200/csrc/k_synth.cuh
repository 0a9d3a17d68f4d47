// k_synth.cuh -- K7: synthetic KPFT bodies of SURVEY.md 8(d) configs 4 and 5
// written straight into HBM (bench workload; the CPU restatement is
// oracle/synth.py and tests/test_synth.py checks them bit for bit).
//
// One warp per stream.  splitmix64 is counter based, so draw k of stream s is
// mix(seed_s + (k + 1) * gamma) and every lane computes its own draw; clocks
// are a warp inclusive scan (mod 2^32) of the gaps.
#pragma once

#include "wgpf_dev.cuh"

namespace wgpf {

__device__ inline uint64_t splitmix_draw(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ inline uint32_t warp_incl_scan_u32(uint32_t x) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if ((int)lane >= o) x += y;
  }
  return x;
}

__device__ inline uint32_t mixed_tag(uint32_t warp, uint32_t i) {
  if (warp < 4) {
    const uint32_t L = ((i >> 2) & 1u) ? 2u : 0u;
    const uint32_t ph = i & 3u;
    const uint32_t region = L + (ph >= 2 ? 1u : 0u);
    const bool start = ph == 0 || ph == 2;
    return (start ? WGPF_START_FLAG : 0u) | (region << 12);
  }
  const uint32_t j = i & 7u;
  return j < 4 ? (WGPF_START_FLAG | ((4u + j) << 12)) : ((4u + (7u - j)) << 12);
}

__device__ inline uint32_t nested_tag(uint32_t w) {
  const uint32_t j = w & 127u;
  return j < 64 ? (WGPF_START_FLAG | (j << 12)) : ((127u - j) << 12);
}

constexpr uint32_t kSynthCap = 256;
constexpr uint32_t kNestedWrites = 1000;

__global__ void __launch_bounds__(256) k_synth(uint8_t* body, uint32_t shape,
                                               uint64_t stream0,
                                               uint64_t n_streams,
                                               uint64_t n_long) {
  const uint32_t lane = lane_id();
  const uint64_t stride = 16ull + 8ull * kSynthCap;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t s = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
       s < n_streams; s += warps) {
    const uint64_t gs = stream0 + s;
    const uint64_t seed = 0x5EEDull ^ gs;
    uint8_t* base = body + s * stride;
    uint2* slots = reinterpret_cast<uint2*>(base + 16);
    const uint32_t warp = (uint32_t)(gs & 15u);
    uint32_t count, writes;
    if (shape == 0) {
      count = gs < n_long ? 222u : 221u;
      writes = count;
    } else {
      count = kNestedWrites;
      writes = kNestedWrites;
    }
    if (lane == 0)
      *reinterpret_cast<uint4*>(base) =
          make_uint4((uint32_t)(gs >> 4), warp, count, kSynthCap);
    uint32_t carry = 0;
    const uint32_t total = shape == 0 ? kSynthCap : writes;
    for (uint32_t c = 0; c < total; c += 32) {
      const uint32_t i = c + lane;
      const bool live = i < writes;
      uint32_t val = 0;
      if (live) {
        const uint64_t z = splitmix_draw(seed, i);
        if (i == 0) {
          val = (uint32_t)z;
        } else {
          const uint64_t mod =
              (shape == 0 && warp < 4 && (i & 3u) == 2u) ? 4000ull : 200ull;
          val = (uint32_t)(1ull + z % mod);
        }
      }
      const uint32_t clock = carry + warp_incl_scan_u32(val);
      carry = __shfl_sync(0xffffffffu, clock, 31);
      if (shape == 0) {
        slots[i] = live ? make_uint2(mixed_tag(warp, i), clock) : make_uint2(0, 0);
      } else if (live && i >= writes - kSynthCap) {
        slots[i % kSynthCap] = make_uint2(nested_tag(i), clock);
      }
    }
  }
}

}  // namespace wgpf
