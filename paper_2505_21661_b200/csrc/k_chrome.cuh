// k_chrome.cuh -- export_chrome_trace (trace.hpp:493-511) on the GPU: the
// reference's Chrome Trace JSON (nlohmann ordered_json dump(2)) of an event
// array in HBM, byte-identical to the host writer (capi_chrome.inc).
//
// Two passes over the events, one thread per event: k_chrome_len computes
// each event's text length (label, pid, tid, ts, dur, iteration, kind,
// corrected, separator), a device-wide exclusive scan places the texts, and
// k_chrome_write formats each event into a per-warp shared-memory buffer (the
// 32 texts of a warp are contiguous in the output) that the warp then copies
// out with coalesced byte stores.  Numbers: include/wgpf_grisu2.h (the
// reference JSON library's Grisu2 + layout), shared with the host writer.
#pragma once

#include "wgpf_dev.cuh"
#include "wgpf_grisu2.h"

namespace wgpf {

// escaped label texts ("..." with quotes) of region ids < n_labels
struct ChromeLabels {
  const char* text;
  const uint32_t* off;  // [n_labels + 1]
  uint32_t n_labels;
};

constexpr uint32_t kChromeMaxEvent = 512;  // bytes of one event's text (host
                                           // checks labels <= kChromeMaxLabel)
constexpr uint32_t kChromeMaxLabel = 200;  // 190 fixed + 200 + 111 numbers <= 512
constexpr uint32_t kChromeWarps = 2;

// the fixed text between the fields
#define WGPF_CH_A "    {\n      \"name\": "
#define WGPF_CH_B ",\n      \"ph\": \"X\",\n      \"pid\": "
#define WGPF_CH_C ",\n      \"tid\": "
#define WGPF_CH_D ",\n      \"ts\": "
#define WGPF_CH_E ",\n      \"dur\": "
#define WGPF_CH_F ",\n      \"args\": {\n        \"iteration\": "
#define WGPF_CH_G ",\n        \"kind\": "
#define WGPF_CH_H ",\n        \"corrected\": "
#define WGPF_CH_I "\n      }\n    }"

__device__ __forceinline__ uint32_t dec_len(uint64_t v) {
  uint32_t n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

template <uint32_t N>
__device__ __forceinline__ char* put_lit(char* o, const char (&s)[N]) {
#pragma unroll
  for (uint32_t i = 0; i + 1 < N; ++i) o[i] = s[i];
  return o + (N - 1);
}

// event text -> o (or only its length when o == nullptr)
__device__ uint32_t chrome_event(char* o, const wgpf_event& e, uint64_t i, uint64_t n,
                                 double cpu, const ChromeLabels& lab) {
  char ts[32], du[32];
  const uint32_t rid = e.region & WGPF_EV_REGION_MASK;
  const int lts = wgpf_json::format_double(ts, __ddiv_rn(__ull2double_rn(e.start), cpu));
  const int ldu =
      wgpf_json::format_double(du, __ddiv_rn(__ull2double_rn(e.end - e.start), cpu));
  const bool wait = (e.region & WGPF_EV_WAIT) != 0;
  const bool corr = (e.region & WGPF_EV_CORRECTED) != 0;
  const bool last = i + 1 == n;
  uint32_t llab;
  if (rid < lab.n_labels)
    llab = lab.off[rid + 1] - lab.off[rid];
  else
    llab = 9 + dec_len(rid);  // "region#<id>" with quotes
  const uint32_t len = (sizeof(WGPF_CH_A) - 1) + llab + (sizeof(WGPF_CH_B) - 1) +
                       dec_len(e.block_index) + (sizeof(WGPF_CH_C) - 1) +
                       dec_len(e.warp_group) + (sizeof(WGPF_CH_D) - 1) + lts +
                       (sizeof(WGPF_CH_E) - 1) + ldu + (sizeof(WGPF_CH_F) - 1) +
                       dec_len(e.iteration) + (sizeof(WGPF_CH_G) - 1) + 6 +
                       (sizeof(WGPF_CH_H) - 1) + (corr ? 4 : 5) +
                       (sizeof(WGPF_CH_I) - 1) + (last ? 1 : 2);
  if (!o) return len;
  o = put_lit(o, WGPF_CH_A);
  if (rid < lab.n_labels) {
    for (uint32_t k = lab.off[rid]; k < lab.off[rid + 1]; ++k) *o++ = lab.text[k];
  } else {
    o = put_lit(o, "\"region#");
    o += wgpf_json::format_u64(o, rid);
    *o++ = '"';
  }
  o = put_lit(o, WGPF_CH_B);
  o += wgpf_json::format_u64(o, e.block_index);
  o = put_lit(o, WGPF_CH_C);
  o += wgpf_json::format_u64(o, e.warp_group);
  o = put_lit(o, WGPF_CH_D);
  for (int k = 0; k < lts; ++k) *o++ = ts[k];
  o = put_lit(o, WGPF_CH_E);
  for (int k = 0; k < ldu; ++k) *o++ = du[k];
  o = put_lit(o, WGPF_CH_F);
  o += wgpf_json::format_u64(o, e.iteration);
  o = put_lit(o, WGPF_CH_G);
  o = wait ? put_lit(o, "\"wait\"") : put_lit(o, "\"exec\"");
  o = put_lit(o, WGPF_CH_H);
  o = corr ? put_lit(o, "true") : put_lit(o, "false");
  o = put_lit(o, WGPF_CH_I);
  if (last) {
    *o++ = '\n';
  } else {
    *o++ = ',';
    *o++ = '\n';
  }
  return len;
}

__global__ void k_chrome_len(const wgpf_event* ev, uint64_t n, double cpu,
                             ChromeLabels lab, uint32_t* len) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    len[i] = chrome_event(nullptr, ev[i], i, n, cpu, lab);
}

// off: exclusive scan of len (bytes before each event, from the first event)
__global__ void __launch_bounds__(kChromeWarps * 32)
    k_chrome_write(const wgpf_event* ev, uint64_t n, double cpu, ChromeLabels lab,
                   const uint64_t* off, char* out) {
  __shared__ char buf[kChromeWarps][32 * kChromeMaxEvent];
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  const uint64_t warps = (uint64_t)gridDim.x * kChromeWarps;
  for (uint64_t b = (uint64_t)blockIdx.x * kChromeWarps + w; b * 32 < n; b += warps) {
    const uint64_t i0 = b * 32, i = i0 + lane;
    const uint64_t base = off[i0];
    uint32_t rel = 0, mine = 0;
    if (i < n) {
      rel = (uint32_t)(off[i] - base);
      mine = chrome_event(buf[w] + rel, ev[i], i, n, cpu, lab);
    }
    const uint32_t total = __reduce_max_sync(0xffffffffu, rel + mine);
    __syncwarp();
    char* dst = out + base;
    for (uint32_t k = lane; k < total; k += 32) dst[k] = buf[w][k];
    __syncwarp();
  }
}

}  // namespace wgpf
