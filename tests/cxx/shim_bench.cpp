// Drop-in C++ path, end to end: what a reference user's program does after
// swapping <wgprof/...> for "wgprof_b200.hpp" -- raw KPFT
// bytes in a pageable std::vector -> deserialize_image -> replay_image ->
// region_stats, value semantics throughout (one TimelineEvent with a
// std::string label per event).  The input is a slice of the synthetic
// config-4 trace (generated on the device by wgpf_synth_body and copied into
// the vector, outside the timed region).  Prints one JSON object.
//
//   shim_bench <streams> [reps]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#include "wgprof_b200.hpp"

using namespace wgprof;
using clk = std::chrono::steady_clock;

static double secs(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : (1u << 19);
  const int reps = argc > 2 ? std::atoi(argv[2]) : 3;
  const uint64_t cap = 256, stride = 16 + 8 * cap;
  const std::vector<std::string> labels = {"TMA0", "TMA0.wait", "TMA1", "TMA1.wait",
                                           "MMA",  "MMA.k",     "EPI",  "EPI.st"};
  // the raw trace: KPFT v2 header + body (v1 holds at most 65,535 streams; the
  // drop-in's deserialize_image reads the framework's v2 container as well)
  std::vector<std::uint8_t> raw(16 + n * stride);
  {
    wgpf_ctx* c = b200::ctx();
    void* d = nullptr;
    if (cudaMalloc(&d, n * stride) != cudaSuccess) return 2;
    b200::set_plan(cap, BufferStrategy::Flush, labels);
    b200::check(wgpf_synth_body(c, d, WGPF_SYNTH_MIXED, 0, n, n / 2));
    cudaMemcpy(raw.data() + 16, d, n * stride, cudaMemcpyDeviceToHost);
    cudaFree(d);
    const char hdr[8] = {'K', 'P', 'F', 'T', 2, 0, 0, 0};
    std::memcpy(raw.data(), hdr, 8);
    std::memcpy(raw.data() + 8, &n, 8);
  }
  BufferPlan plan{cap, BufferStrategy::Flush, labels};
  double best_total = 1e30, best_deser = 0, best_replay = 0, best_stats = 0;
  uint64_t records = 0, events = 0;
  for (int r = 0; r < reps + 1; ++r) {
    const auto t0 = clk::now();
    GlobalTraceImage img = deserialize_image(raw);
    const auto t1 = clk::now();
    TraceReplay tr = replay_image(img, plan, 33);
    const auto t2 = clk::now();
    auto st = region_stats(tr.events);
    const auto t3 = clk::now();
    records = 0;
    for (const auto& s : img.streams) records += std::min(s.record_count, s.slot_capacity);
    events = tr.events.size();
    if (r > 0 && secs(t0, t3) < best_total) {
      best_total = secs(t0, t3);
      best_deser = secs(t0, t1);
      best_replay = secs(t1, t2);
      best_stats = secs(t2, t3);
    }
    if (st.empty()) return 3;
  }
  // breakdown of region_stats: label packing on the host, the GPU statistics
  // with the reference's exact mean recurrence, and without it (sum / count)
  double t_pack = 0, t_exact = 0, t_fast = 0;
  {
    GlobalTraceImage img = deserialize_image(raw);
    TraceReplay tr = replay_image(img, plan, 33);
    const auto a = clk::now();
    std::vector<std::string> table;
    auto ev = b200::pack_events(tr.events, table);
    const auto b = clk::now();
    b200::set_plan(0, BufferStrategy::Flush, table);
    std::vector<wgpf_region_stat> st(table.size() + 1);
    std::uint32_t ns = 0;
    b200::check(wgpf_region_stats(b200::ctx(), ev.data(), tr.events.size(), 0,
                                  WGPF_F_EXACT_MEAN, st.data(), (uint32_t)st.size(), &ns));
    const auto c = clk::now();
    b200::check(wgpf_region_stats(b200::ctx(), ev.data(), tr.events.size(), 0, 0, st.data(),
                                  (uint32_t)st.size(), &ns));
    const auto d = clk::now();
    t_pack = secs(a, b);
    t_exact = secs(b, c);
    t_fast = secs(c, d);
  }
  std::printf("{\"pack_events_s\": %.6f, \"gpu_stats_exact_mean_s\": %.6f, "
              "\"gpu_stats_sum_over_count_s\": %.6f}\n", t_pack, t_exact, t_fast);
  std::printf(
      "{\"streams\": %llu, \"records\": %llu, \"events\": %llu, \"bytes\": %llu, "
      "\"seconds\": %.6f, \"records_per_s\": %.6e, \"deserialize_s\": %.6f, "
      "\"replay_image_s\": %.6f, \"region_stats_s\": %.6f}\n",
      (unsigned long long)n, (unsigned long long)records, (unsigned long long)events,
      (unsigned long long)raw.size(), best_total, records / best_total, best_deser,
      best_replay, best_stats);
  return 0;
}
