// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers straight from /root/reference
// (nothing is copied into this repo) and exposes a tiny extern "C" surface so
// that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg can run the reference's own CPU implementation of the
// trace post-processor.  The product (paper_2505_21661_b200/) never links or
// calls this library.
//
// Built by oracle/Makefile into oracle/_ref/libwgprof_ref.so with
//   -I/root/reference/proj/include -I/root/reference/proj/tests -I<nlohmann>
// The reference namespace is renamed (#define wgprof wgprof_ref) so that it
// can never clash with the drop-in's namespace.
//
// Reference entry points wrapped here:
//   deserialize_image  wgprof/trace.hpp:181     decode_image   trace.hpp:222
//   unwrap_clock       trace.hpp:257            pair_records   trace.hpp:294
//   replay             trace.hpp:398            replay_image   pipeline.hpp:66
//   region_stats       pipeline.hpp:114         analyze_critical_path perfmodel.hpp:317
//   run_pipeline/write_artifacts pipeline.hpp:248,271 (fixture regeneration)
//   testgen::random_program tests/support.hpp:26 (random replay programs)
//   swp_latency / ws_latency / roofline / overhead_model / load_stage_table
//                      perfmodel.hpp:44,97,180,196,202 (text in / text out)

#define wgprof wgprof_ref
#include "support.hpp"
#include "wgprof/config.hpp"
#include "wgprof/lower.hpp"
#include "wgprof/perfmodel.hpp"
#include "wgprof/pipeline.hpp"
#include "wgprof/trace.hpp"
#include "wgprof/vgpu.hpp"
#undef wgprof

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace R = wgprof_ref;

extern "C" {

// ---------------------------------------------------------------------------
// Common result plumbing.
// ---------------------------------------------------------------------------

struct ref_status {
  int code;           // 0 = ok, else 1 + ErrorKind (error.hpp:8-18); 100 = other
  char category[32];  // Error::category()
  char message[1024]; // Error::what()
};

struct ref_event {
  uint64_t start, end;
  uint32_t label; // index into the result's label list
  uint32_t iteration, block, wg;
  uint32_t kind;      // 0 exec, 1 wait
  uint32_t corrected; // 0/1
};

struct ref_stat {
  uint32_t label;
  uint32_t wg;
  uint32_t kind;
  uint32_t count;
  uint64_t min, max;
  double mean;
};

struct ref_replay_out {
  ref_status st;
  uint64_t n_events;
  ref_event* events;
  uint32_t n_labels;
  char* label_blob; // n_labels NUL-terminated strings back to back
  uint64_t label_blob_len;
  uint32_t dropped_heads, truncated_tails, flagged_preconditions,
      malformed_groups;
  uint32_t n_stats;
  ref_stat* stats; // region_stats order (std::map => sorted by label)
};

static void set_ok(ref_status* st) {
  st->code = 0;
  st->category[0] = 0;
  st->message[0] = 0;
}

static void set_err(ref_status* st, const R::Error& e) {
  st->code = 1 + static_cast<int>(e.kind());
  std::snprintf(st->category, sizeof st->category, "%s", e.category());
  std::snprintf(st->message, sizeof st->message, "%s", e.what());
}

static void set_other(ref_status* st, const std::exception& e) {
  st->code = 100;
  std::snprintf(st->category, sizeof st->category, "%s", "exception");
  std::snprintf(st->message, sizeof st->message, "%s", e.what());
}

static std::vector<std::string> split_blob(const char* blob, uint32_t n) {
  std::vector<std::string> out;
  out.reserve(n);
  const char* p = blob;
  for (uint32_t i = 0; i < n; ++i) {
    out.emplace_back(p);
    p += out.back().size() + 1;
  }
  return out;
}

struct LabelInterner {
  std::unordered_map<std::string, uint32_t> ids;
  std::vector<std::string> names;
  uint32_t id(const std::string& s) {
    auto it = ids.find(s);
    if (it != ids.end())
      return it->second;
    uint32_t v = static_cast<uint32_t>(names.size());
    ids.emplace(s, v);
    names.push_back(s);
    return v;
  }
  void export_to(ref_replay_out* out) const {
    out->n_labels = static_cast<uint32_t>(names.size());
    uint64_t len = 0;
    for (const auto& s : names)
      len += s.size() + 1;
    out->label_blob = static_cast<char*>(std::malloc(len ? len : 1));
    out->label_blob_len = len;
    char* p = out->label_blob;
    for (const auto& s : names) {
      std::memcpy(p, s.c_str(), s.size() + 1);
      p += s.size() + 1;
    }
  }
};

static R::BufferPlan make_plan(uint64_t slots, uint32_t strategy,
                               const char* label_blob, uint32_t n_labels) {
  R::BufferPlan plan;
  plan.slots_per_warp_group = slots;
  plan.strategy =
      strategy == 0 ? R::BufferStrategy::Circular : R::BufferStrategy::Flush;
  plan.region_labels = split_blob(label_blob, n_labels);
  return plan;
}

static void export_events(const std::vector<R::TimelineEvent>& evs,
                          LabelInterner& li, ref_replay_out* out) {
  out->n_events = evs.size();
  out->events = static_cast<ref_event*>(
      std::malloc(sizeof(ref_event) * (evs.size() ? evs.size() : 1)));
  for (size_t i = 0; i < evs.size(); ++i) {
    const auto& e = evs[i];
    ref_event& o = out->events[i];
    o.start = e.start;
    o.end = e.end;
    o.label = li.id(e.region);
    o.iteration = e.iteration;
    o.block = e.block_index;
    o.wg = e.warp_group;
    o.kind = e.kind == R::EventKind::Wait ? 1u : 0u;
    o.corrected = e.corrected ? 1u : 0u;
  }
}

static void export_stats(const std::vector<R::TimelineEvent>& evs,
                         LabelInterner& li, ref_replay_out* out) {
  auto stats = R::region_stats(evs);
  out->n_stats = static_cast<uint32_t>(stats.size());
  out->stats = static_cast<ref_stat*>(
      std::malloc(sizeof(ref_stat) * (stats.size() ? stats.size() : 1)));
  uint32_t k = 0;
  for (const auto& [label, rs] : stats) {
    ref_stat& s = out->stats[k++];
    s.label = li.id(label);
    s.wg = rs.warp_group;
    s.kind = rs.kind == R::EventKind::Wait ? 1u : 0u;
    s.count = rs.count;
    s.min = rs.min;
    s.max = rs.max;
    s.mean = rs.mean;
  }
}

void ref_free_replay(ref_replay_out* out) {
  std::free(out->events);
  std::free(out->label_blob);
  std::free(out->stats);
  out->events = nullptr;
  out->label_blob = nullptr;
  out->stats = nullptr;
}

// deserialize_image -> replay_image -> region_stats on raw KPFT bytes.
int ref_replay_kpft(const uint8_t* bytes, uint64_t n, uint64_t slots,
                    uint32_t strategy, const char* label_blob,
                    uint32_t n_labels, uint64_t record_cost,
                    ref_replay_out* out) {
  std::memset(out, 0, sizeof *out);
  set_ok(&out->st);
  try {
    std::vector<uint8_t> buf(bytes, bytes + n);
    R::BufferPlan plan = make_plan(slots, strategy, label_blob, n_labels);
    R::GlobalTraceImage img = R::deserialize_image(buf);
    R::TraceReplay tr = R::replay_image(img, plan, record_cost);
    LabelInterner li;
    export_events(tr.events, li, out);
    export_stats(tr.events, li, out);
    li.export_to(out);
    out->dropped_heads = tr.dropped_heads;
    out->truncated_tails = tr.truncated_tails;
    out->flagged_preconditions = tr.flagged_preconditions;
    out->malformed_groups = tr.malformed_groups;
  } catch (const R::Error& e) {
    set_err(&out->st, e);
  } catch (const std::exception& e) {
    set_other(&out->st, e);
  }
  return out->st.code;
}

// ---------------------------------------------------------------------------
// decode_image on raw KPFT bytes: chronological records per stream.
// ---------------------------------------------------------------------------

struct ref_decode_out {
  ref_status st;
  uint64_t n_streams;
  uint32_t* block;    // per stream
  uint32_t* wg;       // per stream
  uint32_t* dropped;  // per stream
  uint64_t* offset;   // per stream, into records (n_streams + 1 entries)
  uint64_t n_records;
  uint32_t* tags;
  uint32_t* payloads;
};

void ref_free_decode(ref_decode_out* o) {
  std::free(o->block);
  std::free(o->wg);
  std::free(o->dropped);
  std::free(o->offset);
  std::free(o->tags);
  std::free(o->payloads);
  std::memset(o, 0, sizeof *o);
}

int ref_decode_kpft(const uint8_t* bytes, uint64_t n, uint64_t slots,
                    uint32_t strategy, ref_decode_out* out) {
  std::memset(out, 0, sizeof *out);
  set_ok(&out->st);
  try {
    std::vector<uint8_t> buf(bytes, bytes + n);
    R::BufferPlan plan = make_plan(slots, strategy, "", 0);
    auto ds = R::decode_image(R::deserialize_image(buf), plan);
    out->n_streams = ds.size();
    size_t ns = ds.size() ? ds.size() : 1;
    out->block = static_cast<uint32_t*>(std::malloc(4 * ns));
    out->wg = static_cast<uint32_t*>(std::malloc(4 * ns));
    out->dropped = static_cast<uint32_t*>(std::malloc(4 * ns));
    out->offset = static_cast<uint64_t*>(std::malloc(8 * (ds.size() + 1)));
    uint64_t total = 0;
    for (size_t s = 0; s < ds.size(); ++s) {
      out->block[s] = ds[s].block_index;
      out->wg[s] = ds[s].warp_group;
      out->dropped[s] = ds[s].dropped_records;
      out->offset[s] = total;
      total += ds[s].records.size();
    }
    out->offset[ds.size()] = total;
    out->n_records = total;
    out->tags = static_cast<uint32_t*>(std::malloc(4 * (total ? total : 1)));
    out->payloads =
        static_cast<uint32_t*>(std::malloc(4 * (total ? total : 1)));
    uint64_t k = 0;
    for (const auto& d : ds)
      for (const auto& r : d.records) {
        out->tags[k] = r.tag;
        out->payloads[k] = r.payload;
        ++k;
      }
  } catch (const R::Error& e) {
    set_err(&out->st, e);
  } catch (const std::exception& e) {
    set_other(&out->st, e);
  }
  return out->st.code;
}

// unwrap_clock (trace.hpp:257).
void ref_unwrap_clock(const uint32_t* v, uint64_t n, uint64_t* out) {
  std::vector<uint32_t> in(v, v + n);
  auto u = R::unwrap_clock(in);
  std::memcpy(out, u.data(), 8 * n);
}

// ---------------------------------------------------------------------------
// pair_records (trace.hpp:294) on one chronological stream.
// ---------------------------------------------------------------------------

struct ref_interval {
  uint32_t region_id;
  uint32_t label;
  uint32_t iteration;
  uint32_t pad;
  uint64_t start, end, start_pos, end_pos;
};

struct ref_pair_out {
  ref_status st;
  uint64_t n;
  ref_interval* iv;
  uint32_t dropped_heads, truncated_tails;
  uint32_t n_labels;
  char* label_blob;
  uint64_t label_blob_len;
};

void ref_free_pair(ref_pair_out* o) {
  std::free(o->iv);
  std::free(o->label_blob);
  o->iv = nullptr;
  o->label_blob = nullptr;
}

int ref_pair_records(const uint32_t* tags, const uint32_t* payloads,
                     uint64_t n, const char* label_blob, uint32_t n_labels,
                     ref_pair_out* out) {
  std::memset(out, 0, sizeof *out);
  set_ok(&out->st);
  try {
    std::vector<R::ProfileRecord> stream(n);
    for (uint64_t i = 0; i < n; ++i) {
      stream[i].tag = tags[i];
      stream[i].payload = payloads[i];
    }
    auto table = split_blob(label_blob, n_labels);
    auto pr = R::pair_records(stream, table);
    LabelInterner li;
    out->n = pr.intervals.size();
    out->iv = static_cast<ref_interval*>(
        std::malloc(sizeof(ref_interval) * (out->n ? out->n : 1)));
    for (size_t i = 0; i < pr.intervals.size(); ++i) {
      const auto& a = pr.intervals[i];
      ref_interval& b = out->iv[i];
      b.region_id = a.region_id;
      b.label = li.id(a.label);
      b.iteration = a.iteration;
      b.pad = 0;
      b.start = a.start;
      b.end = a.end;
      b.start_pos = a.start_pos;
      b.end_pos = a.end_pos;
    }
    out->dropped_heads = pr.dropped_heads;
    out->truncated_tails = pr.truncated_tails;
    ref_replay_out tmp{};
    li.export_to(&tmp);
    out->n_labels = tmp.n_labels;
    out->label_blob = tmp.label_blob;
    out->label_blob_len = tmp.label_blob_len;
  } catch (const R::Error& e) {
    set_err(&out->st, e);
  } catch (const std::exception& e) {
    set_other(&out->st, e);
  }
  return out->st.code;
}

// replay (trace.hpp:398) on caller-built intervals (labels given by index
// into label_blob), as the reference's test_replay.cpp does.
int ref_replay_pairs(const ref_interval* iv, uint64_t n,
                     const char* label_blob, uint32_t n_labels,
                     uint32_t block, uint32_t wg, uint64_t record_cost,
                     ref_replay_out* out) {
  std::memset(out, 0, sizeof *out);
  set_ok(&out->st);
  try {
    auto names = split_blob(label_blob, n_labels);
    R::PairResult pr;
    for (uint64_t i = 0; i < n; ++i) {
      R::RawInterval r;
      r.region_id = iv[i].region_id;
      r.label = names.at(iv[i].label);
      r.iteration = iv[i].iteration;
      r.start = iv[i].start;
      r.end = iv[i].end;
      r.start_pos = iv[i].start_pos;
      r.end_pos = iv[i].end_pos;
      pr.intervals.push_back(std::move(r));
    }
    auto rr = R::replay(pr, block, wg, record_cost);
    LabelInterner li;
    export_events(rr.events, li, out);
    export_stats(rr.events, li, out);
    li.export_to(out);
    out->flagged_preconditions = rr.flagged_preconditions;
    out->malformed_groups = rr.malformed_groups;
  } catch (const R::Error& e) {
    set_err(&out->st, e);
  } catch (const std::exception& e) {
    set_other(&out->st, e);
  }
  return out->st.code;
}

// ---------------------------------------------------------------------------
// analyze_critical_path (perfmodel.hpp:317) on the replay of a KPFT image,
// with the barrier edges coming from the reference's .dev device program.
// ---------------------------------------------------------------------------

struct ref_cp_out {
  ref_status st;
  uint32_t n_cycle;
  char* cycle_blob; // NUL-separated labels
  uint64_t cycle_blob_len;
  uint64_t period;
  uint32_t n_nodes;
  char* node_blob; // NUL-separated labels (graph nodes, sorted)
  uint64_t node_blob_len;
  uint64_t* node_duration;
  uint32_t n_edges;
  uint32_t* edge_src;
  uint32_t* edge_dst;
  uint32_t n_barrier_edges;
  char* barrier_edge_blob; // src\0dst\0 pairs
  uint64_t barrier_edge_blob_len;
};

static char* make_blob(const std::vector<std::string>& v, uint64_t* len) {
  uint64_t l = 0;
  for (const auto& s : v)
    l += s.size() + 1;
  char* b = static_cast<char*>(std::malloc(l ? l : 1));
  char* p = b;
  for (const auto& s : v) {
    std::memcpy(p, s.c_str(), s.size() + 1);
    p += s.size() + 1;
  }
  *len = l;
  return b;
}

void ref_free_cp(ref_cp_out* o) {
  std::free(o->cycle_blob);
  std::free(o->node_blob);
  std::free(o->node_duration);
  std::free(o->edge_src);
  std::free(o->edge_dst);
  std::free(o->barrier_edge_blob);
  std::memset(o, 0, sizeof *o);
}

int ref_critical_path_kpft(const uint8_t* bytes, uint64_t n,
                           const char* dev_text, uint64_t record_cost,
                           uint64_t slack, int exclude_warmup,
                           ref_cp_out* out) {
  std::memset(out, 0, sizeof *out);
  set_ok(&out->st);
  try {
    std::vector<uint8_t> buf(bytes, bytes + n);
    R::DeviceProgram dp = R::parse_device_program(dev_text);
    R::TraceReplay tr =
        R::replay_image(R::deserialize_image(buf), dp.plan, record_cost);
    R::CriticalPathOptions opts;
    opts.slack_tolerance = slack;
    opts.exclude_warmup = exclude_warmup != 0;
    auto cp = R::analyze_critical_path(tr.events, dp, opts);
    out->n_cycle = static_cast<uint32_t>(cp.cycle.size());
    out->cycle_blob = make_blob(cp.cycle, &out->cycle_blob_len);
    out->period = cp.period;
    std::vector<std::string> nodes;
    for (const auto& nd : cp.graph.nodes)
      nodes.push_back(nd.label);
    out->n_nodes = static_cast<uint32_t>(nodes.size());
    out->node_blob = make_blob(nodes, &out->node_blob_len);
    out->node_duration = static_cast<uint64_t*>(
        std::malloc(8 * (nodes.size() ? nodes.size() : 1)));
    for (size_t i = 0; i < nodes.size(); ++i)
      out->node_duration[i] = cp.graph.nodes[i].duration;
    out->n_edges = static_cast<uint32_t>(cp.graph.edges.size());
    size_t ne = cp.graph.edges.size() ? cp.graph.edges.size() : 1;
    out->edge_src = static_cast<uint32_t*>(std::malloc(4 * ne));
    out->edge_dst = static_cast<uint32_t*>(std::malloc(4 * ne));
    for (size_t i = 0; i < cp.graph.edges.size(); ++i) {
      out->edge_src[i] = static_cast<uint32_t>(cp.graph.edges[i].first);
      out->edge_dst[i] = static_cast<uint32_t>(cp.graph.edges[i].second);
    }
    auto be = R::detail::barrier_edges(dp);
    std::vector<std::string> flat;
    for (const auto& [a, b] : be) {
      flat.push_back(a);
      flat.push_back(b);
    }
    out->n_barrier_edges = static_cast<uint32_t>(be.size());
    out->barrier_edge_blob = make_blob(flat, &out->barrier_edge_blob_len);
  } catch (const R::Error& e) {
    set_err(&out->st, e);
  } catch (const std::exception& e) {
    set_other(&out->st, e);
  }
  return out->st.code;
}

// ---------------------------------------------------------------------------
// Fixture regeneration (run_pipeline + write_artifacts + the .dev text).
// ---------------------------------------------------------------------------

int ref_run_fixture(const char* conf_path, const char* kir_path,
                    const char* out_prefix, ref_status* st) {
  set_ok(st);
  try {
    auto pc = R::make_pipeline_config(R::load_config(conf_path));
    pc.kernel_file = kir_path;
    const std::string p(out_prefix);
    pc.raw_trace_path = p + ".kpft";
    pc.chrome_trace_path = p + ".json";
    pc.replay_report_path = p + "_replay.json";
    pc.model_report_path = p + "_model.json";
    auto rr = R::run_pipeline(pc);
    R::write_artifacts(rr, pc);
    R::write_file(p + ".dev", R::print_device_program(rr.device));
    std::string meta = std::to_string(pc.machine.record_cost) + "\n";
    R::write_file(p + ".cost", meta);
  } catch (const R::Error& e) {
    set_err(st, e);
  } catch (const std::exception& e) {
    set_other(st, e);
  }
  return st->code;
}

// Random replay programs exactly as the reference's acceptance suite makes
// them (tests/support.hpp:26 random_program, test_acceptance.cpp:63-69
// lower_with, vgpu.hpp:424 simulate).  Writes the serialized image and the
// lowered device program text.
int ref_random_program_image(uint64_t seed, int index, int with_loop,
                             uint32_t num_wgs, uint32_t strategy,
                             uint64_t slots_total, const char* out_prefix,
                             ref_status* st) {
  set_ok(st);
  try {
    // num_wgs == 0 reproduces test_acceptance.cpp:108 ((i % 3) + 1 warp
    // groups); slots_total is per warp group (x num_wgs, :110-111).
    testgen::Rng rng(seed);
    R::KernelProgram p;
    for (int i = 0; i <= index; ++i)
      p = testgen::random_program(rng, with_loop != 0,
                                  num_wgs ? num_wgs : (uint32_t)(i % 3) + 1);
    R::LoweringConfig cfg;
    cfg.buffer_strategy =
        strategy == 0 ? R::BufferStrategy::Circular : R::BufferStrategy::Flush;
    cfg.buffer_slots_total = slots_total * p.num_warp_groups;
    auto dp = R::lower(p, cfg);
    auto sim = R::simulate(dp, R::MachineConfig{});
    const std::string pre(out_prefix);
    R::write_file(pre + ".kpft", R::serialize_image(sim.image));
    R::write_file(pre + ".dev", R::print_device_program(dp));
  } catch (const R::Error& e) {
    set_err(st, e);
  } catch (const std::exception& e) {
    set_other(st, e);
  }
  return st->code;
}

// lower() (lower.hpp:220-301) of a KIR text program (ir.hpp:540
// parse_program) under a LoweringConfig, and optionally simulate() it
// (vgpu.hpp:424).  Writes <out_prefix>.plan ("<slots>\n" then one region
// label per line, id order) and, when simulating, <out_prefix>.kpft (the
// vGPU's image) and <out_prefix>.log (the store log: per warp group one line
// of hex tags, vgpu.hpp:269-271).
int ref_lower_kir(const char* kir, uint32_t strategy, uint64_t slots_total,
                  int signature_bits, int iteration_signature, int global_buffer,
                  int simulate, const char* out_prefix, ref_status* st) {
  set_ok(st);
  try {
    auto p = R::parse_program(kir);
    R::LoweringConfig cfg;
    cfg.buffer_strategy =
        strategy == 0 ? R::BufferStrategy::Circular : R::BufferStrategy::Flush;
    cfg.buffer_slots_total = slots_total;
    cfg.signature_bits_enabled = signature_bits != 0;
    cfg.iteration_signature = iteration_signature != 0;
    cfg.buffer_type = global_buffer ? R::BufferType::Global : R::BufferType::Shared;
    auto dp = R::lower(p, cfg);
    const std::string pre(out_prefix);
    std::string plan = std::to_string(dp.plan.slots_per_warp_group) + "\n";
    for (const auto& l : dp.plan.region_labels) plan += l + "\n";
    R::write_file(pre + ".plan", plan);
    if (simulate) {
      auto sim = R::simulate(dp, R::MachineConfig{});
      R::write_file(pre + ".kpft", R::serialize_image(sim.image));
      std::string log;
      char hex[16];
      for (const auto& wg : sim.store_log) {
        for (const auto& r : wg) {
          snprintf(hex, sizeof hex, "%08x ", r.tag);
          log += hex;
        }
        log += "\n";
      }
      R::write_file(pre + ".log", log);
    }
  } catch (const R::Error& e) {
    set_err(st, e);
  } catch (const std::exception& e) {
    set_other(st, e);
  }
  return st->code;
}

// ---------------------------------------------------------------------------
// CPU baseline harness: the reference functions, unmodified, over disjoint
// <= 65535-stream KPFT v1 chunks, with harness-level parallelism over
// `nthreads` workers.  The timed region starts from raw
// KPFT bytes in RAM (each chunk's bytes are pre-built into a std::vector before
// the clock starts because the reference API takes a vector) and covers
// deserialize_image -> decode_image -> pair_records -> replay -> region_stats.
// ---------------------------------------------------------------------------

struct ref_bench_out {
  ref_status st;
  double seconds;
  uint64_t records; // surviving records decoded
  uint64_t events;
  uint64_t streams;
};

// body: a KPFT v2/v1 body (no file header), uniform stride 16 + 8*slots.
int ref_bench_replay(const uint8_t* body, uint64_t n_streams, uint64_t slots,
                     uint32_t strategy, const char* label_blob,
                     uint32_t n_labels, uint64_t record_cost,
                     uint64_t chunk_streams, int nthreads,
                     ref_bench_out* out) {
  std::memset(out, 0, sizeof *out);
  set_ok(&out->st);
  try {
    if (chunk_streams == 0 || chunk_streams > 0xFFFF)
      chunk_streams = 0xFFFF;
    const uint64_t stride = 16 + 8 * slots;
    std::vector<std::vector<uint8_t>> chunks;
    for (uint64_t s0 = 0; s0 < n_streams; s0 += chunk_streams) {
      uint64_t cnt = std::min<uint64_t>(chunk_streams, n_streams - s0);
      std::vector<uint8_t> b(8 + cnt * stride);
      std::memcpy(b.data(), "KPFT", 4);
      b[4] = 1;
      b[5] = 0;
      b[6] = static_cast<uint8_t>(cnt & 0xFF);
      b[7] = static_cast<uint8_t>((cnt >> 8) & 0xFF);
      std::memcpy(b.data() + 8, body + s0 * stride, cnt * stride);
      chunks.push_back(std::move(b));
    }
    R::BufferPlan plan = make_plan(slots, strategy, label_blob, n_labels);
    if (nthreads < 1)
      nthreads = 1;
    std::atomic<uint64_t> next{0}, recs{0}, evs{0};
    std::atomic<int> failed{0};
    std::string err_cat, err_msg;
    std::mutex mu;
    auto worker = [&]() {
      uint64_t r = 0, e = 0;
      for (;;) {
        uint64_t c = next.fetch_add(1);
        if (c >= chunks.size())
          break;
        try {
          auto img = R::deserialize_image(chunks[c]);
          for (const auto& d : R::decode_image(img, plan)) {
            auto pr = R::pair_records(d.records, plan.region_labels);
            auto rr = R::replay(pr, d.block_index, d.warp_group, record_cost);
            auto st = R::region_stats(rr.events);
            r += d.records.size();
            e += rr.events.size();
            (void)st;
          }
        } catch (const std::exception& ex) {
          std::lock_guard<std::mutex> g(mu);
          failed = 1;
          err_msg = ex.what();
        }
      }
      recs += r;
      evs += e;
    };
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ths;
    for (int i = 0; i < nthreads; ++i)
      ths.emplace_back(worker);
    for (auto& t : ths)
      t.join();
    auto t1 = std::chrono::steady_clock::now();
    out->seconds = std::chrono::duration<double>(t1 - t0).count();
    out->records = recs.load();
    out->events = evs.load();
    out->streams = n_streams;
    if (failed) {
      out->st.code = 100;
      std::snprintf(out->st.message, sizeof out->st.message, "%s",
                    err_msg.c_str());
    }
  } catch (const std::exception& e) {
    set_other(&out->st, e);
  }
  return out->st.code;
}

// export_chrome_trace (trace.hpp:493-511) of an event array in this
// framework's 32-byte layout (wgpf_event: start, end, region | WAIT<<31 |
// CORRECTED<<30, iteration, block, warp_group; label = labels[region] or
// "region#<id>", trace.hpp:302-306).  *out is malloc'ed (free with
// ref_free_text); returns the byte count, or -1 with st set.
struct ref_wgpf_event {
  uint64_t start, end;
  uint32_t region, iteration, block, wg;
};

int64_t ref_export_chrome(const ref_wgpf_event* ev, uint64_t n,
                          const char* label_blob, uint32_t n_labels,
                          double cycles_per_us, char** out, ref_status* st) {
  try {
    const auto labels = split_blob(label_blob, n_labels);
    std::vector<R::TimelineEvent> evs;
    evs.reserve(n);
    for (uint64_t i = 0; i < n; ++i) {
      R::TimelineEvent t;
      const uint32_t rid = ev[i].region & 0x3FFFFFFFu;
      t.region = rid < labels.size() ? labels[rid] : "region#" + std::to_string(rid);
      t.kind = (ev[i].region >> 31) ? R::EventKind::Wait : R::EventKind::Exec;
      t.corrected = ((ev[i].region >> 30) & 1u) != 0;
      t.start = ev[i].start;
      t.end = ev[i].end;
      t.iteration = ev[i].iteration;
      t.block_index = ev[i].block;
      t.warp_group = ev[i].wg;
      evs.push_back(std::move(t));
    }
    const std::string js = R::export_chrome_trace(evs, cycles_per_us);
    *out = static_cast<char*>(std::malloc(js.size() + 1));
    std::memcpy(*out, js.data(), js.size());
    set_ok(st);
    return static_cast<int64_t>(js.size());
  } catch (const R::Error& e) {
    set_err(st, e);
  } catch (const std::exception& e) {
    set_other(st, e);
  }
  return -1;
}

void ref_free_text(char* p) { std::free(p); }

// Analytic models.  Text protocol (tests/test_models.py):
//   in : one "swp <nwg> <npipe> <nloop>", "stage <name> <t_load> <t_comp>",
//        "node <label> <duration>", "edge <a> <b>", "roofline f t r b w",
//        "overhead v n c" per line; "table" + the rest of the text is a stage
//        table for load_stage_table.
//   out: "ok <result...>" or "err <kind> <message>".
// labels travel %-encoded (they may hold blanks): %XX -> byte
static std::string pct_dec(const std::string& s) {
  std::string o;
  for (size_t i = 0; i < s.size(); ++i) {
    if (s[i] == '%' && i + 2 < s.size()) {
      o.push_back(static_cast<char>(std::stoi(s.substr(i + 1, 2), nullptr, 16)));
      i += 2;
    } else {
      o.push_back(s[i]);
    }
  }
  return o;
}
static std::string pct_enc(const std::string& s) {
  static const char* hx = "0123456789ABCDEF";
  std::string o;
  for (unsigned char c : s) {
    if (c <= ' ' || c == '%' || c >= 0x7F) {
      o.push_back('%');
      o.push_back(hx[c >> 4]);
      o.push_back(hx[c & 15]);
    } else {
      o.push_back(static_cast<char>(c));
    }
  }
  return o;
}
static char* dup_text(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}
char* ref_models(const char* text) {
  std::string in(text);
  std::ostringstream out;
  try {
    if (in.rfind("table\n", 0) == 0) {
      std::istringstream is(in.substr(6));
      auto st = R::load_stage_table(is);
      out << "ok";
      for (const auto& x : st) out << " " << x.name << " " << x.t_load << " " << x.t_comp;
      return dup_text(out.str());
    }
    std::istringstream is(in);
    std::string kw;
    R::SwpInput swp;
    R::WsInput ws;
    bool is_swp = false, is_ws = false;
    while (is >> kw) {
      if (kw == "swp") {
        is >> swp.n_warp_groups >> swp.n_pipe_stages >> swp.n_loop;
        is_swp = true;
      } else if (kw == "stage") {
        R::SwpStage st;
        is >> st.name >> st.t_load >> st.t_comp;
        swp.stages.push_back(st);
      } else if (kw == "node") {
        R::WsNode nd;
        is >> nd.label >> nd.duration;
        nd.label = pct_dec(nd.label);
        ws.nodes.push_back(nd);
        is_ws = true;
      } else if (kw == "edge") {
        std::size_t a, b;
        is >> a >> b;
        ws.edges.emplace_back(a, b);
        is_ws = true;
      } else if (kw == "wsempty") {
        is_ws = true;
      } else if (kw == "roofline") {
        R::RooflineInput r;
        is >> r.flops >> r.throughput >> r.t_read >> r.bytes >> r.bandwidth;
        auto x = R::roofline(r);
        out << "ok " << x.compute_cycles << " " << x.memory_cycles;
        return dup_text(out.str());
      } else if (kw == "plan") {  // plan <regions> <nwg> <strategy 0|1> <cap> <n> <trips...>
        std::uint32_t regions, nwg;
        int strat;
        std::uint64_t cap, n;
        is >> regions >> nwg >> strat >> cap >> n;
        std::vector<std::uint64_t> trips(n);
        for (auto& t : trips) is >> t;
        auto pl = R::plan_slots(regions, trips, nwg,
                                strat ? R::BufferStrategy::Flush : R::BufferStrategy::Circular, cap);
        out << "ok " << pl.slots_per_warp_group;
        return dup_text(out.str());
      } else if (kw == "sig") {
        std::uint32_t wg;
        is >> wg;
        R::MachineConfig mc;
        out << "ok " << mc.signature_for(wg).packed();
        return dup_text(out.str());
      } else if (kw == "overhead") {
        R::OverheadInput o;
        is >> o.t_vanilla >> o.n_record >> o.cycle_record;
        out << "ok " << R::overhead_model(o);
        return dup_text(out.str());
      }
    }
    if (is_swp) {
      auto r = R::swp_latency(swp);
      out << "ok " << r.delta << " " << r.latency;
    } else if (is_ws) {
      auto r = R::ws_latency(ws);
      out << "ok " << r.latency;
      for (const auto& l : r.critical_path) out << " " << pct_enc(l);
    } else {
      out << "err none no model";
    }
  } catch (const R::Error& e) {
    out.str("");
    out << "err " << static_cast<int>(e.kind()) << " " << e.what();
  }
  return dup_text(out.str());
}

} // extern "C"
