// End-to-end test of the drop-in C++ shim (include/wgprof_b200.hpp): the
// reference's own test cases (test_trace.cpp, test_replay.cpp), written
// against the reference signatures, run on the GPU through libwgpf.so.
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>

#include "wgprof_b200.hpp"

using namespace wgprof;

static int failures = 0;
#define CHECK(cond)                                                    \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

static std::vector<std::uint8_t> read_bytes(const std::string& p) {
  std::ifstream is(p, std::ios::binary);
  return std::vector<std::uint8_t>(std::istreambuf_iterator<char>(is), {});
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "tests/golden/fixtures";

  // test_trace.cpp:9-27
  CHECK(ProfileRecord::make(true, 3, 0, 1000).tag == 0x80003000u);
  CHECK(ProfileRecord::make(true, (1u << 19) - 1, 0xFFF, 0).tag == 0xFFFFFFFFu);
  bool threw = false;
  try {
    ProfileRecord::make(true, 1u << 19, 0, 0);
  } catch (const Error&) {
    threw = true;
  }
  CHECK(threw);

  // test_trace.cpp:82-105 circular decode
  {
    GlobalTraceImage img;
    TraceStream s;
    s.record_count = 6;
    s.slot_capacity = 4;
    s.slots = {ProfileRecord::make(true, 4, 0, 4), ProfileRecord::make(true, 5, 0, 5),
               ProfileRecord::make(true, 2, 0, 2), ProfileRecord::make(true, 3, 0, 3)};
    img.streams.push_back(s);
    BufferPlan plan;
    plan.slots_per_warp_group = 4;
    plan.strategy = BufferStrategy::Circular;
    auto d = decode_image(img, plan);
    CHECK(d.size() == 1 && d[0].dropped_records == 2);
    std::vector<std::uint32_t> r;
    for (auto& x : d[0].records) r.push_back(x.region_id());
    CHECK((r == std::vector<std::uint32_t>{2, 3, 4, 5}));
    CHECK(deserialize_image(serialize_image(img)) == img);
  }
  // test_trace.cpp:132-136 unwrap
  {
    auto u = unwrap_clock({0xFFFFFF00u, 0x00000100u});
    CHECK(u.size() == 2 && u[1] - u[0] == 0x200);
  }
  // test_trace.cpp:171-187 nested pairing
  {
    std::vector<ProfileRecord> st = {
        ProfileRecord::make(true, 0, 0, 10), ProfileRecord::make(true, 1, 0, 20),
        ProfileRecord::make(false, 1, 0, 30), ProfileRecord::make(false, 0, 0, 40)};
    auto res = pair_records(st, {"a", "b"});
    CHECK(res.intervals.size() == 2);
    CHECK(res.intervals[0].label == "b" && res.intervals[0].start == 20 &&
          res.intervals[0].end == 30);
    CHECK(res.intervals[1].label == "a" && res.intervals[1].start == 10 &&
          res.intervals[1].end == 40);
  }
  // test_replay.cpp:51-64 worked example
  {
    PairResult pairs;
    pairs.intervals.push_back({0, "G", 0, 10, 150, 0, 1});
    pairs.intervals.push_back({1, "G.wait", 0, 400, 410, 2, 3});
    auto rr = replay(pairs, 0, 0, 33);
    CHECK(rr.events.size() == 2);
    CHECK(rr.events[1].region == "G.wait" && rr.events[1].kind == EventKind::Wait &&
          rr.events[1].duration() == 250 && rr.events[1].corrected);
  }
  // test_replay.cpp:66-79 sync correction
  {
    PairResult pairs;
    pairs.intervals.push_back({1, "inner", 0, 40, 80, 1, 2});
    pairs.intervals.push_back({0, "outer", 0, 10, 176, 0, 3});
    auto rr = replay(pairs, 0, 0, 33);
    CHECK(rr.events.size() == 2 && rr.events[1].duration() == 166 - 33 - 2 * 33);
  }
  // fixtures (SURVEY.md Appendix B golden results)
  {
    auto img = deserialize_image(read_bytes(dir + "/simple.kpft"));
    BufferPlan plan;
    plan.slots_per_warp_group = 300;
    plan.strategy = BufferStrategy::Flush;
    plan.region_labels = {"Scale", "Matmul", "Matmul.wait"};
    auto tr = replay_image(img, plan, 33);
    CHECK(tr.events.size() == 150);
    auto st = region_stats(tr.events);
    CHECK(st.size() == 3);
    CHECK(st["Matmul"].count == 50 && st["Matmul"].mean == 600.0);
    CHECK(st["Matmul.wait"].kind == EventKind::Wait && st["Matmul.wait"].mean == 300.0);
    CHECK(st["Scale"].min == 2000 && st["Scale"].max == 2000);
  }
  {
    auto img = deserialize_image(read_bytes(dir + "/fa3_vanilla.kpft"));
    BufferPlan plan;
    plan.slots_per_warp_group = 64;
    plan.strategy = BufferStrategy::Circular;
    std::ifstream dev(dir + "/fa3_vanilla.dev");
    std::string line;
    std::getline(dev, line);
    while (std::getline(dev, line)) {
      auto p = line.find("region ");
      if (p == std::string::npos || line.find('"') == std::string::npos) continue;
      auto a = line.find('"'), b = line.rfind('"');
      plan.region_labels.push_back(line.substr(a + 1, b - a - 1));
    }
    auto tr = replay_image(img, plan, 33);
    CHECK(tr.events.size() == 128);
    auto st = region_stats(tr.events);
    CHECK(st["GEMM0.c0.wait"].count == 6);
    CHECK(st["GEMM0.c0.wait"].mean == 1127.8333333333333);  // non-integer (H1)
    CHECK(st["GEMM0.c0.wait"].min == 800 && st["GEMM0.c0.wait"].max == 1200);
    // export_chrome_trace: the reference's bytes (out/fa3_vanilla.json)
    auto js = export_chrome_trace(tr.events, 1000.0);
    auto want = read_bytes(dir + "/fa3_vanilla.json");
    CHECK(js == std::string(want.begin(), want.end()));
    // analyze_critical_path with the program's barrier edges (argv[2]:
    // "src<TAB>dst" lines, derived from fa3_vanilla.dev by the test driver)
    if (argc > 2) {
      std::vector<std::pair<std::string, std::string>> edges;
      std::ifstream ef(argv[2]);
      std::string el;
      while (std::getline(ef, el)) {
        auto t = el.find('\t');
        if (t != std::string::npos) edges.emplace_back(el.substr(0, t), el.substr(t + 1));
      }
      auto cp = analyze_critical_path(tr.events, edges);
      CHECK(cp.period == 4200);
      CHECK((cp.cycle == std::vector<std::string>{"GEMM1.c0", "GEMM1.c0.wait", "Load V0",
                                                  "Load V0.wait"}));
      // the stage graph feeds ws_latency: the unfolded cycle is its longest
      // path (perfmodel.hpp:479-491)
      CHECK(cp.graph.nodes.size() == cp.stage_mean.size());
      CHECK(cp.graph.edges.size() == cp.cycle.size() - 1);
      const WsResult ws = ws_latency(cp.graph);
      CHECK(ws.latency == cp.period);
      CHECK(ws.critical_path == cp.cycle);
    }
  }
  if (failures == 0) std::printf("ALL PASS\n");
  return failures ? 1 : 0;
}
