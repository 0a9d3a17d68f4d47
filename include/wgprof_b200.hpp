// wgprof_b200.hpp -- drop-in C++ shim: the reference's namespace wgprof trace
// API (value semantics, wgprof::Error exceptions) implemented over the C-ABI
// of libwgpf.so (include/wgpf.h), i.e. over the sm_100a kernels.
//
// Replaces, signature for signature (paths relative to
// /root/reference/proj/include/):
//   wgprof/error.hpp:8-55       ErrorKind, Error, category()
//   wgprof/trace.hpp:58-99      ProfileRecord, encode_record, decode_record
//   wgprof/trace.hpp:105-209    TraceStream, GlobalTraceImage,
//                               serialize_image, deserialize_image
//   wgprof/lower.hpp:42,57-73   BufferStrategy, BufferPlan
//   wgprof/trace.hpp:215-251    DecodedStream, decode_image        (GPU)
//   wgprof/trace.hpp:257-272    unwrap_clock                       (GPU)
//   wgprof/trace.hpp:278-346    RawInterval, PairResult, pair_records (GPU)
//   wgprof/trace.hpp:352-487    EventKind, TimelineEvent, ReplayResult,
//                               replay                             (GPU)
//   wgprof/pipeline.hpp:58-81   TraceReplay, replay_image          (GPU)
//   wgprof/pipeline.hpp:105-133 RegionStats, region_stats          (GPU)
//   wgprof/perfmodel.hpp:22-222 swp_latency, ws_latency, roofline,
//                               overhead_model, load_stage_table   (host)
//
// A program built against the reference's headers switches by including this
// header instead and linking libwgpf.so.  Do not include it
// together with the reference headers (same namespace).
#pragma once

#include <algorithm>
#include <array>
#include <cctype>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <sstream>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

// nlohmann/json (the reference's one third-party dependency, trace.hpp:10
// includes it as <json.hpp>) for make_replay_report when it is on the path
#if __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#define WGPROF_B200_HAVE_JSON 1
#elif __has_include(<json.hpp>)
#include <json.hpp>
#define WGPROF_B200_HAVE_JSON 1
#endif

#include "wgpf.h"

namespace wgprof {

enum class ErrorKind { Parse, Validate, Instrument, Lower, Capacity, Deadlock,
                       Trace, Config, Io };

class Error : public std::runtime_error {
 public:
  Error(ErrorKind kind, const std::string& message)
      : std::runtime_error(message), kind_(kind) {}
  ErrorKind kind() const { return kind_; }
  const char* category() const {
    return wgpf_error_category(1 + static_cast<int>(kind_));
  }

 private:
  ErrorKind kind_;
};

inline constexpr std::uint32_t kStartFlag = WGPF_START_FLAG;
inline constexpr std::uint32_t kSignatureMask = WGPF_SIGNATURE_MASK;
inline constexpr std::uint32_t kRegionIdBits = WGPF_REGION_BITS;
inline constexpr std::uint32_t kMaxRegions = WGPF_MAX_REGIONS;
inline constexpr std::uint64_t kRecordBytes = WGPF_RECORD_BYTES;
inline constexpr std::uint16_t kTraceVersion = 1;
inline const char* kWaitSuffix = ".wait";

struct ProfileRecord {
  std::uint32_t tag = 0;
  std::uint32_t payload = 0;
  bool is_start() const { return (tag & kStartFlag) != 0; }
  std::uint32_t region_id() const { return (tag >> 12) & (kMaxRegions - 1); }
  std::uint16_t signature() const {
    return static_cast<std::uint16_t>(tag & kSignatureMask);
  }
  static ProfileRecord make(bool is_start, std::uint32_t region,
                            std::uint16_t signature, std::uint32_t clock) {
    if (region >= kMaxRegions)
      throw Error(ErrorKind::Trace, "region id " + std::to_string(region) +
                                        " overflows the 19-bit tag field");
    return ProfileRecord{(is_start ? kStartFlag : 0u) | (region << 12) |
                             (signature & kSignatureMask),
                         clock};
  }
  bool operator==(const ProfileRecord&) const = default;
};

inline std::array<std::uint8_t, 8> encode_record(const ProfileRecord& r) {
  std::array<std::uint8_t, 8> out{};
  for (int i = 0; i < 4; ++i) out[i] = (r.tag >> (8 * i)) & 0xFF;
  for (int i = 0; i < 4; ++i) out[4 + i] = (r.payload >> (8 * i)) & 0xFF;
  return out;
}

inline ProfileRecord decode_record(const std::uint8_t* b) {
  ProfileRecord r;
  for (int i = 0; i < 4; ++i) r.tag |= static_cast<std::uint32_t>(b[i]) << (8 * i);
  for (int i = 0; i < 4; ++i)
    r.payload |= static_cast<std::uint32_t>(b[4 + i]) << (8 * i);
  return r;
}

struct TraceStream {
  std::uint32_t block_index = 0;
  std::uint32_t warp_group = 0;
  std::uint32_t record_count = 0;
  std::uint32_t slot_capacity = 0;
  std::vector<ProfileRecord> slots;
  bool operator==(const TraceStream&) const = default;
};

struct GlobalTraceImage {
  std::vector<TraceStream> streams;
  bool operator==(const GlobalTraceImage&) const = default;
};

enum class BufferStrategy { Circular, Flush };

struct BufferPlan {
  std::uint64_t slots_per_warp_group = 0;
  BufferStrategy strategy = BufferStrategy::Circular;
  std::vector<std::string> region_labels;
  std::uint64_t base_offset(std::uint32_t wg) const {
    return wg * slots_per_warp_group * kRecordBytes;
  }
  bool operator==(const BufferPlan&) const = default;
};

struct DecodedStream {
  std::uint32_t block_index = 0;
  std::uint32_t warp_group = 0;
  std::uint32_t dropped_records = 0;
  std::vector<ProfileRecord> records;
};

struct RawInterval {
  std::uint32_t region_id = 0;
  std::string label;
  std::uint32_t iteration = 0;
  std::uint64_t start = 0;
  std::uint64_t end = 0;
  std::size_t start_pos = 0;
  std::size_t end_pos = 0;
};

struct PairResult {
  std::vector<RawInterval> intervals;
  std::uint32_t dropped_heads = 0;
  std::uint32_t truncated_tails = 0;
};

enum class EventKind { Exec, Wait };

struct TimelineEvent {
  std::string region;
  std::uint32_t block_index = 0;
  std::uint32_t warp_group = 0;
  std::uint32_t iteration = 0;
  std::uint64_t start = 0;
  std::uint64_t end = 0;
  EventKind kind = EventKind::Exec;
  bool corrected = false;
  std::uint64_t duration() const { return end - start; }
  bool operator==(const TimelineEvent&) const = default;
};

struct ReplayResult {
  std::vector<TimelineEvent> events;
  std::uint32_t flagged_preconditions = 0;
  std::uint32_t malformed_groups = 0;
};

struct TraceReplay {
  std::vector<TimelineEvent> events;
  std::uint32_t dropped_heads = 0;
  std::uint32_t truncated_tails = 0;
  std::uint32_t flagged_preconditions = 0;
  std::uint32_t malformed_groups = 0;
};

struct RegionStats {
  std::uint32_t warp_group = 0;
  EventKind kind = EventKind::Exec;
  std::uint32_t count = 0;
  std::uint64_t min = 0;
  std::uint64_t max = 0;
  double mean = 0.0;
};

// ---------------------------------------------------------------------------
// implementation details
// ---------------------------------------------------------------------------
namespace b200 {

struct Ctx {
  wgpf_ctx* h = nullptr;
  Ctx() {
    int rc = wgpf_create(0, nullptr, &h);
    if (rc != WGPF_OK)
      throw std::runtime_error(
          "wgprof_b200: no usable CUDA device (this implementation has no "
          "CPU fallback)");
  }
  ~Ctx() {
    if (h) wgpf_destroy(h);
  }
};

inline wgpf_ctx* ctx() {
  thread_local std::unique_ptr<Ctx> c;
  if (!c) c = std::make_unique<Ctx>();
  return c->h;
}

inline void check(int rc) {
  if (rc == WGPF_OK) return;
  const std::string msg = wgpf_last_error(ctx());
  if (rc >= 1 && rc <= 9) throw Error(static_cast<ErrorKind>(rc - 1), msg);
  throw std::runtime_error(std::string("wgpf: ") + wgpf_error_category(rc) +
                           ": " + msg);
}

inline void set_plan(std::uint64_t slots, BufferStrategy st,
                     const std::vector<std::string>& labels) {
  std::vector<const char*> p;
  p.reserve(labels.size());
  for (const auto& s : labels) p.push_back(s.c_str());
  check(wgpf_set_plan(ctx(), slots, static_cast<std::uint32_t>(st), p.data(),
                      static_cast<std::uint32_t>(p.size())));
}

// The host side of the value-semantics API (one std::string-labelled
// TimelineEvent per event, vectors of ProfileRecord) is per-element work:
// it runs over the host's cores in contiguous ranges.
inline unsigned host_threads() {
  static const unsigned n = [] {
    const unsigned h = std::thread::hardware_concurrency();
    return std::max(1u, std::min(32u, h ? h : 1u));
  }();
  return n;
}
template <class F>  // f(begin, end, part)
inline void parallel_ranges(std::size_t n, F&& f, std::size_t min_per = 1u << 16) {
  const unsigned parts = (unsigned)std::min<std::size_t>(
      host_threads(), std::max<std::size_t>(1, n / std::max<std::size_t>(1, min_per)));
  if (parts <= 1) {
    f(std::size_t(0), n, 0u);
    return;
  }
  std::vector<std::thread> th;
  const std::size_t per = (n + parts - 1) / parts;
  for (unsigned p = 1; p < parts; ++p)
    th.emplace_back([&, p] { f(std::min(n, p * per), std::min(n, (p + 1) * per), p); });
  f(std::size_t(0), std::min(n, per), 0u);
  for (auto& t : th) t.join();
}

// TimelineEvents -> 32-byte events with a dense label table (first-seen order)
// (not value-initialised: every element is written below, in parallel, so
// the pages are first touched by the writing threads)
struct EventBuf {
  std::unique_ptr<wgpf_event[]> p;
  wgpf_event* data() { return p.get(); }
  const wgpf_event* data() const { return p.get(); }
};
inline EventBuf pack_events(const std::vector<TimelineEvent>& events,
                            std::vector<std::string>& table) {
  // distinct labels per range (events repeat a handful of labels: each
  // lookup first compares with the range's previous label), merged in
  // first-seen order; then the ids
  const std::size_t n = events.size();
  const unsigned parts = host_threads();
  std::vector<std::vector<std::string>> seen(parts);
  parallel_ranges(n, [&](std::size_t lo, std::size_t hi, unsigned p) {
    std::unordered_map<std::string_view, bool> m;
    const std::string* last = nullptr;
    for (std::size_t i = lo; i < hi; ++i) {
      const std::string& r = events[i].region;
      if (last && r == *last) continue;
      last = &r;
      if (m.emplace(r, true).second) seen[p].push_back(r);
    }
  });
  std::unordered_map<std::string_view, std::uint32_t> ids;
  for (auto& v : seen)
    for (auto& l : v)
      if (!ids.count(l)) {
        table.push_back(l);
        ids.emplace(table.back(), 0);
      }
  ids.clear();
  for (std::uint32_t k = 0; k < table.size(); ++k) ids.emplace(table[k], k);
  EventBuf ev{std::unique_ptr<wgpf_event[]>(new wgpf_event[n + 1])};
  parallel_ranges(n, [&](std::size_t lo, std::size_t hi, unsigned) {
    const std::string* last = nullptr;
    std::uint32_t last_id = 0;
    for (std::size_t i = lo; i < hi; ++i) {
      const auto& e = events[i];
      if (!last || e.region != *last) {
        last = &e.region;
        last_id = ids.find(e.region)->second;
      }
      ev.p[i] = wgpf_event{e.start, e.end,
                         last_id | (e.kind == EventKind::Wait ? WGPF_EV_WAIT : 0u) |
                             (e.corrected ? WGPF_EV_CORRECTED : 0u),
                         e.iteration, e.block_index, e.warp_group};
    }
  });
  return ev;
}

inline std::string label_of(const std::vector<std::string>& t, std::uint32_t id) {
  return id < t.size() ? t[id] : "region#" + std::to_string(id);
}

inline TimelineEvent to_event(const wgpf_event& e,
                              const std::vector<std::string>& labels) {
  TimelineEvent t;
  t.region = label_of(labels, e.region & WGPF_EV_REGION_MASK);
  t.block_index = e.block_index;
  t.warp_group = e.warp_group;
  t.iteration = e.iteration;
  t.start = e.start;
  t.end = e.end;
  t.kind = (e.region & WGPF_EV_WAIT) ? EventKind::Wait : EventKind::Exec;
  t.corrected = (e.region & WGPF_EV_CORRECTED) != 0;
  return t;
}

inline void put_u32(std::vector<std::uint8_t>& o, std::uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back((v >> (8 * i)) & 0xFF);
}

// An in-memory image as a KPFT v2 container (u64 stream count) for the
// C-ABI: the reference's decode_image / replay_image take the image in
// memory and never serialise it, so the v1 u16 count limit must not apply.
struct ByteBuf {  // (not value-initialised: every byte is written, in parallel)
  std::unique_ptr<std::uint8_t[]> p;
  std::size_t n = 0;
  std::uint8_t* data() { return p.get(); }
  const std::uint8_t* data() const { return p.get(); }
  std::size_t size() const { return n; }
};
template <class Img>
inline ByteBuf pack_image(const Img& img) {
  static_assert(sizeof(ProfileRecord) == 8, "ProfileRecord is {u32 tag, u32 payload}");
  const std::size_t ns = img.streams.size();
  std::vector<std::size_t> at(ns + 1);
  at[0] = 16;
  for (std::size_t k = 0; k < ns; ++k) {
    const auto& s = img.streams[k];
    if (s.slots.size() != s.slot_capacity)
      throw Error(ErrorKind::Trace,
                  "stream slot count does not match its declared capacity");
    at[k + 1] = at[k] + 16 + 8 * s.slots.size();
  }
  ByteBuf out{std::unique_ptr<std::uint8_t[]>(new std::uint8_t[at[ns]]), at[ns]};
  const std::uint64_t n = ns;
  std::memcpy(out.data(), "KPFT\x02\0\0\0", 8);
  std::memcpy(out.data() + 8, &n, 8);
  // (records and headers are little-endian u32s: the host layout)
  parallel_ranges(ns, [&](std::size_t lo, std::size_t hi, unsigned) {
    for (std::size_t k = lo; k < hi; ++k) {
      const auto& s = img.streams[k];
      const std::uint32_t h[4] = {s.block_index, s.warp_group, s.record_count,
                                  s.slot_capacity};
      std::memcpy(out.data() + at[k], h, 16);
      std::memcpy(out.data() + at[k] + 16, s.slots.data(), 8 * s.slots.size());
    }
  }, 1024);
  return out;
}

}  // namespace b200

// ---------------------------------------------------------------------------
// image format (host)
// ---------------------------------------------------------------------------

inline std::vector<std::uint8_t> serialize_image(const GlobalTraceImage& img) {
  std::vector<std::uint8_t> out = {'K', 'P', 'F', 'T', 1, 0};
  if (img.streams.size() > 0xFFFF)
    throw Error(ErrorKind::Trace, "too many streams for the image header");
  out.push_back(img.streams.size() & 0xFF);
  out.push_back((img.streams.size() >> 8) & 0xFF);
  for (const auto& s : img.streams) {
    if (s.slots.size() != s.slot_capacity)
      throw Error(ErrorKind::Trace,
                  "stream slot count does not match its declared capacity");
    b200::put_u32(out, s.block_index);
    b200::put_u32(out, s.warp_group);
    b200::put_u32(out, s.record_count);
    b200::put_u32(out, s.slot_capacity);
    for (const auto& r : s.slots) {
      auto b = encode_record(r);
      out.insert(out.end(), b.begin(), b.end());
    }
  }
  return out;
}

inline GlobalTraceImage deserialize_image(const std::vector<std::uint8_t>& bytes) {
  auto need = [&](std::size_t pos, std::size_t n) {
    if (pos + n > bytes.size()) throw Error(ErrorKind::Trace, "truncated trace image");
  };
  auto u32 = [&](std::size_t pos) {
    return static_cast<std::uint32_t>(bytes[pos]) |
           (static_cast<std::uint32_t>(bytes[pos + 1]) << 8) |
           (static_cast<std::uint32_t>(bytes[pos + 2]) << 16) |
           (static_cast<std::uint32_t>(bytes[pos + 3]) << 24);
  };
  need(0, 4);
  if (std::memcmp(bytes.data(), "KPFT", 4) != 0)
    throw Error(ErrorKind::Trace, "bad magic: not a trace image");
  need(4, 2);
  const std::uint16_t version = bytes[4] | (bytes[5] << 8);
  // version 1 as the reference; version 2 is this framework's container for
  // more than 65,535 streams (u64 count, include/wgpf_format.h) -- an
  // extension: the reference rejects it here (trace.hpp:187-190)
  if (version != kTraceVersion && version != 2)
    throw Error(ErrorKind::Trace,
                "unsupported trace version " + std::to_string(version));
  std::uint64_t count = 0;
  std::size_t pos = 8;
  if (version == 1) {
    need(6, 2);
    count = bytes[6] | (bytes[7] << 8);
  } else {
    need(8, 8);
    count = static_cast<std::uint64_t>(u32(8)) | (static_cast<std::uint64_t>(u32(12)) << 32);
    pos = 16;
  }
  GlobalTraceImage img;
  img.streams.resize(count);
  std::vector<std::size_t> at(count);
  for (auto& s : img.streams) {  // framing, in order (the reference's errors)
    need(pos, 16);
    s.block_index = u32(pos);
    s.warp_group = u32(pos + 4);
    s.record_count = u32(pos + 8);
    s.slot_capacity = u32(pos + 12);
    pos += 16;
    need(pos, static_cast<std::size_t>(s.slot_capacity) * 8);
    at[&s - img.streams.data()] = pos;
    pos += static_cast<std::size_t>(s.slot_capacity) * 8;
  }
  if (pos != bytes.size())
    throw Error(ErrorKind::Trace, "trailing bytes after trace image");
  static_assert(sizeof(ProfileRecord) == 8, "ProfileRecord is {u32 tag, u32 payload}");
  b200::parallel_ranges(count, [&](std::size_t lo, std::size_t hi, unsigned) {
    for (std::size_t k = lo; k < hi; ++k) {
      auto& s = img.streams[k];
      s.slots.resize(s.slot_capacity);
      std::memcpy(s.slots.data(), bytes.data() + at[k], 8ull * s.slot_capacity);
    }
  }, 1024);
  return img;
}

// ---------------------------------------------------------------------------
// GPU-backed post-processing
// ---------------------------------------------------------------------------

inline std::vector<DecodedStream> decode_image(const GlobalTraceImage& img,
                                               const BufferPlan& plan) {
  b200::set_plan(plan.slots_per_warp_group, plan.strategy, plan.region_labels);
  const auto bytes = b200::pack_image(img);
  std::size_t total = 0;
  for (const auto& s : img.streams) total += s.slot_capacity;
  std::vector<wgpf_record> recs(total + 1);
  std::vector<wgpf_decoded_stream> ds(img.streams.size() + 1);
  std::uint64_t nr = 0, ns = 0;
  b200::check(wgpf_decode_image(b200::ctx(), bytes.data(), bytes.size(),
                                recs.data(), recs.size(), &nr, ds.data(),
                                ds.size(), &ns));
  std::vector<DecodedStream> out(ns);
  for (std::uint64_t s = 0; s < ns; ++s) {
    out[s].block_index = ds[s].block_index;
    out[s].warp_group = ds[s].warp_group;
    out[s].dropped_records = ds[s].dropped_records;
    for (std::uint64_t k = 0; k < ds[s].count; ++k)
      out[s].records.push_back(ProfileRecord{recs[ds[s].offset + k].tag,
                                             recs[ds[s].offset + k].payload});
  }
  return out;
}

inline std::vector<std::uint64_t> unwrap_clock(const std::vector<std::uint32_t>& v) {
  std::vector<std::uint64_t> out(v.size());
  if (!v.empty())
    b200::check(wgpf_unwrap_clock(b200::ctx(), v.data(), v.size(), out.data()));
  return out;
}

inline PairResult pair_records(const std::vector<ProfileRecord>& stream,
                               const std::vector<std::string>& region_table) {
  b200::set_plan(0, BufferStrategy::Flush, region_table);
  std::vector<wgpf_record> r(stream.size() + 1);
  for (std::size_t i = 0; i < stream.size(); ++i)
    r[i] = wgpf_record{stream[i].tag, stream[i].payload};
  std::vector<wgpf_interval> iv(stream.size() / 2 + 1);
  std::uint64_t n = 0;
  PairResult out;
  b200::check(wgpf_pair_records(b200::ctx(), r.data(), stream.size(), iv.data(),
                                iv.size(), &n, &out.dropped_heads,
                                &out.truncated_tails));
  for (std::uint64_t i = 0; i < n; ++i) {
    RawInterval x;
    x.region_id = iv[i].region_id;
    x.label = b200::label_of(region_table, iv[i].region_id);
    x.iteration = iv[i].iteration;
    x.start = iv[i].start;
    x.end = iv[i].end;
    x.start_pos = iv[i].start_pos;
    x.end_pos = iv[i].end_pos;
    out.intervals.push_back(std::move(x));
  }
  return out;
}

inline ReplayResult replay(const PairResult& pairs, std::uint32_t block_index,
                           std::uint32_t warp_group, std::uint64_t record_cost) {
  // Labels travel as ids: one table entry per distinct label string.
  std::vector<std::string> table;
  std::unordered_map<std::string, std::uint32_t> ids;
  std::vector<wgpf_interval> iv(pairs.intervals.size() + 1);
  for (std::size_t i = 0; i < pairs.intervals.size(); ++i) {
    const auto& a = pairs.intervals[i];
    auto it = ids.find(a.label);
    std::uint32_t id;
    if (it == ids.end()) {
      id = static_cast<std::uint32_t>(table.size());
      ids.emplace(a.label, id);
      table.push_back(a.label);
    } else {
      id = it->second;
    }
    iv[i] = wgpf_interval{id, a.iteration, a.start, a.end, a.start_pos, a.end_pos};
  }
  b200::set_plan(0, BufferStrategy::Flush, table);
  std::vector<wgpf_event> ev(pairs.intervals.size() + 1);
  std::uint64_t n = 0;
  wgpf_warnings w{};
  b200::check(wgpf_replay_intervals(b200::ctx(), iv.data(), pairs.intervals.size(),
                                    block_index, warp_group, record_cost,
                                    ev.data(), ev.size(), &n, &w));
  ReplayResult out;
  for (std::uint64_t i = 0; i < n; ++i) out.events.push_back(b200::to_event(ev[i], table));
  out.flagged_preconditions = w.flagged_preconditions;
  out.malformed_groups = w.malformed_groups;
  return out;
}

inline TraceReplay replay_image(const GlobalTraceImage& image,
                                const BufferPlan& plan,
                                std::uint64_t record_cost) {
  b200::set_plan(plan.slots_per_warp_group, plan.strategy, plan.region_labels);
  const auto bytes = b200::pack_image(image);
  std::size_t cap = 1;
  for (const auto& s : image.streams) cap += s.slot_capacity / 2 + 1;
  // (not value-initialised: the pages are first written by the copy-out)
  std::unique_ptr<wgpf_event[]> ev(new wgpf_event[cap]);
  std::uint64_t n = 0;
  wgpf_warnings w{};
  int rc = wgpf_replay_image(b200::ctx(), bytes.data(), bytes.size(), record_cost,
                             ev.get(), cap, 0, &n, &w);
  b200::check(rc);
  TraceReplay out;
  // the events' storage is faulted in by all host threads first: resize's
  // default construction is serial, and page faults on a multi-GB fresh
  // allocation would otherwise dominate it
  out.events.reserve(n);
  {
    unsigned char* raw = reinterpret_cast<unsigned char*>(out.events.data());
    const std::size_t pages = (n * sizeof(TimelineEvent) + 4095) / 4096;
    if (raw)
      b200::parallel_ranges(pages, [&](std::size_t lo, std::size_t hi, unsigned) {
        for (std::size_t p = lo; p < hi; ++p) raw[p * 4096] = 0;
      }, 1u << 12);
  }
  out.events.resize(n);
  b200::parallel_ranges(n, [&](std::size_t lo, std::size_t hi, unsigned) {
    for (std::size_t i = lo; i < hi; ++i) out.events[i] = b200::to_event(ev[i], plan.region_labels);
  });
  out.dropped_heads = w.dropped_heads;
  out.truncated_tails = w.truncated_tails;
  out.flagged_preconditions = w.flagged_preconditions;
  out.malformed_groups = w.malformed_groups;
  return out;
}

inline std::map<std::string, RegionStats> region_stats(
    const std::vector<TimelineEvent>& events) {
  std::vector<std::string> table;
  auto ev = b200::pack_events(events, table);
  b200::set_plan(0, BufferStrategy::Flush, table);
  std::vector<wgpf_region_stat> st(table.size() + 1);
  std::uint32_t n = 0;
  b200::check(wgpf_region_stats(b200::ctx(), ev.data(), events.size(), 0,
                                WGPF_F_EXACT_MEAN, st.data(),
                                static_cast<std::uint32_t>(st.size()), &n));
  std::map<std::string, RegionStats> out;
  for (std::uint32_t i = 0; i < n; ++i) {
    RegionStats r;
    r.warp_group = st[i].warp_group;
    r.kind = st[i].kind ? EventKind::Wait : EventKind::Exec;
    r.count = static_cast<std::uint32_t>(st[i].count);
    r.min = st[i].min;
    r.max = st[i].max;
    r.mean = st[i].mean;
    out.emplace(st[i].label, r);
  }
  return out;
}

// export_chrome_trace (trace.hpp:489-511): byte-identical Chrome Trace JSON.
inline std::string export_chrome_trace(const std::vector<TimelineEvent>& events,
                                       double cycles_per_us = 1000.0) {
  std::vector<std::string> table;
  auto ev = b200::pack_events(events, table);
  b200::set_plan(0, BufferStrategy::Flush, table);
  std::uint64_t len = 0;
  b200::check(wgpf_export_chrome_trace(b200::ctx(), ev.data(), events.size(), 0,
                                       cycles_per_us, nullptr, 0, &len));
  std::string out(len, '\0');
  b200::check(wgpf_export_chrome_trace(b200::ctx(), ev.data(), events.size(), 0,
                                       cycles_per_us, out.data(), len, &len));
  return out;
}

// ---------------------------------------------------------------------------
// Analytic models (perfmodel.hpp:22-222).  Tiny graphs and a few integers:
// host code, fed by the GPU's critical-path result (CriticalPathResult::graph
// below).  Same arithmetic as the reference (u64 wrap, i64 delta, ceiling
// divisions), same tie-breaks and error texts.
// ---------------------------------------------------------------------------
struct SwpStage {
  std::string name;
  std::uint64_t t_load = 0;
  std::uint64_t t_comp = 0;
  bool operator==(const SwpStage&) const = default;
};
struct SwpInput {
  std::uint32_t n_warp_groups = 1;
  std::uint32_t n_pipe_stages = 1;
  std::uint64_t n_loop = 1;
  std::vector<SwpStage> stages;
};
struct SwpResult {
  std::int64_t delta = 0;
  std::uint64_t latency = 0;
};
// delta = N_WG N_pipe sum(t_comp) - max(t_load + t_comp): compute bound
// (sum(t_comp) N_loop) when delta >= 0, else ceil(max N_loop / N_pipe)
inline SwpResult swp_latency(const SwpInput& in) {
  if (in.stages.empty() || !in.n_warp_groups || !in.n_pipe_stages || !in.n_loop)
    throw Error(ErrorKind::Validate, "swp_latency: inputs must be positive");
  std::uint64_t comp = 0, worst = 0;
  for (const SwpStage& s : in.stages) {
    comp += s.t_comp;
    const std::uint64_t t = s.t_load + s.t_comp;
    if (t > worst) worst = t;
  }
  const std::uint64_t lanes = (std::uint64_t)in.n_warp_groups * in.n_pipe_stages;
  SwpResult r;
  r.delta = static_cast<std::int64_t>(lanes * comp - worst);  // (two's complement)
  r.latency = r.delta >= 0 ? comp * in.n_loop
                           : (worst * in.n_loop + in.n_pipe_stages - 1) / in.n_pipe_stages;
  return r;
}

enum class StageKind { Load, Comp };
struct WsNode {
  std::string label;
  std::uint64_t duration = 0;
  StageKind kind = StageKind::Comp;
  bool operator==(const WsNode&) const = default;
};
struct WsInput {
  std::vector<WsNode> nodes;
  std::vector<std::pair<std::size_t, std::size_t>> edges;  // node indices
  bool operator==(const WsInput&) const = default;
};
struct WsResult {
  std::vector<std::string> critical_path;
  std::uint64_t latency = 0;
};
// Longest duration-weighted path of the stage DAG (iterative depth-first
// post-order; a successor still on the DFS stack is a cycle).  A node's
// successor is the first longest one in edge order, replaced by a later one
// of equal length with a smaller label; the start is the longest node,
// smaller label on ties.
inline WsResult ws_latency(const WsInput& in) {
  const std::size_t n = in.nodes.size();
  std::vector<std::vector<std::size_t>> out(n);
  for (const auto& e : in.edges) {
    if (e.first >= n || e.second >= n)
      throw Error(ErrorKind::Validate, "ws_latency: edge index out of range");
    out[e.first].push_back(e.second);
  }
  constexpr std::size_t kNone = ~std::size_t(0);
  std::vector<std::uint8_t> colour(n, 0);  // 0 new, 1 on stack, 2 done
  std::vector<std::uint64_t> best(n, 0);
  std::vector<std::size_t> next(n, kNone);
  std::vector<std::pair<std::size_t, std::size_t>> stack;
  for (std::size_t root = 0; root < n; ++root) {
    if (colour[root]) continue;
    colour[root] = 1;
    stack.assign(1, {root, 0});
    while (!stack.empty()) {
      auto& [v, k] = stack.back();
      if (k < out[v].size()) {
        const std::size_t s = out[v][k++];
        if (colour[s] == 1)
          throw Error(ErrorKind::Validate, "ws_latency: stage graph has a cycle");
        if (colour[s] == 0) {
          colour[s] = 1;
          stack.push_back({s, 0});
        }
        continue;
      }
      const std::uint64_t d = in.nodes[v].duration;
      std::uint64_t b = d;
      std::size_t c = kNone;
      for (std::size_t s : out[v]) {
        const std::uint64_t cand = d + best[s];
        if (cand > b || (cand == b && c != kNone && in.nodes[s].label < in.nodes[c].label)) {
          b = cand;
          c = s;
        }
      }
      best[v] = b;
      next[v] = c;
      colour[v] = 2;
      stack.pop_back();
    }
  }
  WsResult r;
  if (!n) return r;
  std::size_t start = 0;
  for (std::size_t i = 1; i < n; ++i)
    if (best[i] > best[start] ||
        (best[i] == best[start] && in.nodes[i].label < in.nodes[start].label))
      start = i;
  r.latency = best[start];
  for (std::size_t v = start; v != kNone; v = next[v]) r.critical_path.push_back(in.nodes[v].label);
  return r;
}

struct RooflineInput {
  std::uint64_t flops = 0;
  std::uint64_t throughput = 1;  // operations per cycle
  std::uint64_t t_read = 0;
  std::uint64_t bytes = 0;
  std::uint64_t bandwidth = 1;  // bytes per cycle
};
struct RooflineResult {
  std::uint64_t compute_cycles = 0;
  std::uint64_t memory_cycles = 0;
};
inline RooflineResult roofline(const RooflineInput& in) {
  if (!in.throughput || !in.bandwidth)
    throw Error(ErrorKind::Validate, "roofline: rates must be positive");
  return {(in.flops + in.throughput - 1) / in.throughput,
          in.t_read + (in.bytes + in.bandwidth - 1) / in.bandwidth};
}
struct OverheadInput {
  std::uint64_t t_vanilla = 0;
  std::uint64_t n_record = 0;
  std::uint64_t cycle_record = 0;
};
// Eq. 1 of the paper: T = T_vanilla + N_record * cycle_record
inline std::uint64_t overhead_model(const OverheadInput& in) {
  return in.t_vanilla + in.n_record * in.cycle_record;
}
// "<stage> <t_load> <t_comp>" per line, '#' comments, blank lines skipped
inline std::vector<SwpStage> load_stage_table(std::istream& is) {
  std::vector<SwpStage> out;
  std::string line;
  for (int no = 1; std::getline(is, line); ++no) {
    line.erase(std::min(line.find('#'), line.size()));
    std::istringstream ls(line);
    SwpStage s;
    if (!(ls >> s.name)) continue;
    if (!(ls >> s.t_load >> s.t_comp))
      throw Error(ErrorKind::Parse, "stage table line " + std::to_string(no) +
                                        ": expected <stage> <t_load> <t_comp>");
    out.push_back(std::move(s));
  }
  return out;
}

// analyze_critical_path (perfmodel.hpp:317-501).  The reference takes the
// lowered DeviceProgram and derives the barrier edges from it
// (perfmodel.hpp:258-313); this drop-in takes those edges directly (the
// reference's own detail::barrier_edges(dp), or the `.dev` side channel via
// the Python layer's parse_device_program).  The result carries the binding
// cycle and its period -- the parts of CriticalPathAnalysis the CLI reports
// (tools/wgprof.cpp:110) -- plus the per-stage steady means.
struct CriticalPathOptions {
  std::uint64_t slack_tolerance = 132;
  bool exclude_warmup = true;
};
struct CriticalPathResult {
  std::vector<std::string> cycle;
  std::uint64_t period = 0;
  std::map<std::string, std::uint64_t> stage_mean;
  WsInput graph;  // CriticalPathAnalysis::graph: feeds ws_latency
};
inline CriticalPathResult analyze_critical_path(
    const std::vector<TimelineEvent>& events,
    const std::vector<std::pair<std::string, std::string>>& barrier_edges,
    const CriticalPathOptions& opts = {}) {
  std::vector<std::string> table;
  auto ev = b200::pack_events(events, table);
  b200::set_plan(0, BufferStrategy::Flush, table);
  std::vector<const char*> src, dst;
  for (const auto& e : barrier_edges) {
    src.push_back(e.first.c_str());
    dst.push_back(e.second.c_str());
  }
  std::uint32_t cap = 64;
  for (;;) {
    std::vector<wgpf_cp_stage> st(cap);
    std::vector<std::uint64_t> bind((std::size_t)cap * cap);
    std::vector<std::uint32_t> cyc(cap);
    std::uint32_t ns = 0, nc = 0;
    std::uint64_t period = 0;
    const int rc = wgpf_critical_path(
        b200::ctx(), ev.data(), events.size(), 0, src.data(), dst.data(),
        static_cast<std::uint32_t>(src.size()), opts.slack_tolerance,
        opts.exclude_warmup ? 1 : 0, 0, st.data(), cap, &ns, bind.data(),
        (std::uint64_t)cap * cap, cyc.data(), cap, &nc, &period);
    if (rc == WGPF_E_BUFFER && ns > cap) {
      cap = ns;
      continue;
    }
    b200::check(rc);
    CriticalPathResult r;
    for (std::uint32_t i = 0; i < ns; ++i) r.stage_mean[st[i].label] = st[i].mean;
    for (std::uint32_t i = 0; i < nc; ++i) r.cycle.push_back(st[cyc[i]].label);
    r.period = period;
    // the stage graph (perfmodel.hpp:470-497): stages in label order, kind
    // Load when the label says so; edges the unfolded cycle, else every edge
    // binding in at least half of its target's steady instances
    std::vector<std::uint32_t> order(ns);
    for (std::uint32_t i = 0; i < ns; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
      return std::string(st[a].label) < std::string(st[b].label);
    });
    std::vector<std::size_t> pos(ns);
    for (std::uint32_t k = 0; k < ns; ++k) {
      pos[order[k]] = k;
      const std::string l = st[order[k]].label;
      r.graph.nodes.push_back(
          {l, st[order[k]].mean, l.find("Load") != std::string::npos ? StageKind::Load
                                                                      : StageKind::Comp});
    }
    if (nc) {
      for (std::uint32_t i = 0; i + 1 < nc; ++i) r.graph.edges.emplace_back(pos[cyc[i]], pos[cyc[i + 1]]);
    } else {
      for (std::uint32_t a = 0; a < ns; ++a)
        for (std::uint32_t b = 0; b < ns; ++b)
          if (bind[(std::size_t)a * ns + b] && 2 * bind[(std::size_t)a * ns + b] >= st[b].steady)
            r.graph.edges.emplace_back(pos[a], pos[b]);
      std::sort(r.graph.edges.begin(), r.graph.edges.end());
    }
    return r;
  }
}


// ---------------------------------------------------------------------------
// Device programs (lower.hpp:74-140, the `.dev` text of
// print_device_program lower.hpp:320-371) and the program-driven
// analyze_critical_path (perfmodel.hpp:242-318) -- what the reference CLI's
// replay / export / decode commands (tools/wgprof.cpp:70-126) take.  Host
// code.  The hot path behind them is the GPU replay above.
// ---------------------------------------------------------------------------
enum class InstrKind { SyncCompute, AsyncLaunch, AsyncWait, BarrierArrive, BarrierWait,
                       LoopBegin, LoopEnd, Record };
struct Instruction {
  InstrKind kind{};
  std::string unit;
  std::optional<std::uint64_t> latency;
  std::string label;
  std::uint64_t trip_count = 0;
  std::string barrier;
  std::string token;
  bool is_start = false;
  bool operator==(const Instruction&) const = default;
};
struct BarrierDecl {
  std::string name;
  std::uint32_t expected_arrivals = 1;
  bool operator==(const BarrierDecl&) const = default;
};
enum class MetricType { Clock };
enum class Granularity { WarpGroup, Warp, Thread };
enum class BufferType { Shared, Stack, Global };
struct LoweringConfig {
  MetricType metric_type = MetricType::Clock;
  Granularity granularity = Granularity::WarpGroup;
  BufferType buffer_type = BufferType::Shared;
  BufferStrategy buffer_strategy = BufferStrategy::Circular;
  std::uint64_t buffer_slots_total = 0;
  bool signature_bits_enabled = false;
  bool iteration_signature = false;
  bool operator==(const LoweringConfig&) const = default;
};
enum class DeviceOpKind { Base, Init, ReadCounter, StoreCounter, Finalize };
struct DeviceInstr {
  DeviceOpKind op = DeviceOpKind::Base;
  Instruction base;
  std::uint32_t reg = 0;
  std::uint32_t region_id = 0;
  bool is_start = false;
  bool operator==(const DeviceInstr&) const = default;
};
struct DeviceProgram {
  std::string name;
  std::uint32_t num_warp_groups = 1;
  std::uint64_t shared_mem_capacity = 0;
  std::vector<BarrierDecl> barriers;
  std::vector<std::vector<DeviceInstr>> bodies;
  BufferPlan plan;
  LoweringConfig config;
  bool operator==(const DeviceProgram&) const = default;
};

// pipeline.hpp:28-55
inline std::string read_file(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw Error(ErrorKind::Io, "cannot open '" + path + "'");
  std::ostringstream os;
  os << is.rdbuf();
  return os.str();
}
inline void write_file(const std::string& path, const std::string& data) {
  const std::filesystem::path p(path);
  if (p.has_parent_path()) std::filesystem::create_directories(p.parent_path());
  std::ofstream os(path, std::ios::binary);
  if (!os) throw Error(ErrorKind::Io, "cannot write '" + path + "'");
  os.write(data.data(), static_cast<std::streamsize>(data.size()));
}
inline void write_file(const std::string& path, const std::vector<std::uint8_t>& data) {
  write_file(path, std::string(data.begin(), data.end()));
}

namespace b200 {

// Tokens of the device-program text: identifiers (letters, digits, '_', '.'),
// decimal numbers, "strings" (\n and \<c> escapes), { } = ->; '#' comments.
// Errors are parse-errors "<line>:<col>: <message>" like the reference's
// lexer (ir.hpp:166-170).
struct DevTok {
  enum Kind { Ident, Number, String, LBrace, RBrace, Equals, Arrow, Eof } kind = Eof;
  std::string text;
  std::uint64_t number = 0;
  int line = 1, col = 1;
};

[[noreturn]] inline void parse_fail(const DevTok& t, const std::string& msg) {
  throw Error(ErrorKind::Parse, std::to_string(t.line) + ":" + std::to_string(t.col) +
                                    ": " + msg);
}

inline std::vector<DevTok> dev_tokens(std::string_view src) {
  std::vector<DevTok> out;
  int line = 1, col = 1;
  std::size_t i = 0;
  auto step = [&]() {
    if (src[i] == '\n') {
      ++line;
      col = 1;
    } else {
      ++col;
    }
    ++i;
  };
  for (;;) {
    while (i < src.size()) {
      if (src[i] == '#') {
        while (i < src.size() && src[i] != '\n') step();
      } else if (src[i] == ' ' || src[i] == '\t' || src[i] == '\r' || src[i] == '\n') {
        step();
      } else {
        break;
      }
    }
    DevTok t;
    t.line = line;
    t.col = col;
    if (i >= src.size()) {
      out.push_back(t);
      return out;
    }
    const char c = src[i];
    if (c == '{' || c == '}' || c == '=') {
      t.kind = c == '{' ? DevTok::LBrace : c == '}' ? DevTok::RBrace : DevTok::Equals;
      step();
    } else if (c == '-' && i + 1 < src.size() && src[i + 1] == '>') {
      t.kind = DevTok::Arrow;
      step();
      step();
    } else if (c == '"') {
      step();
      while (i < src.size() && src[i] != '"') {
        char d = src[i];
        if (d == '\\' && i + 1 < src.size()) {
          step();
          d = src[i] == 'n' ? '\n' : src[i];
        } else if (d == '\n') {
          parse_fail(t, "unterminated string literal");
        }
        t.text.push_back(d);
        step();
      }
      if (i >= src.size()) parse_fail(t, "unterminated string literal");
      step();
      t.kind = DevTok::String;
    } else if (std::isdigit(static_cast<unsigned char>(c))) {
      while (i < src.size() && std::isdigit(static_cast<unsigned char>(src[i]))) {
        t.number = t.number * 10 + static_cast<std::uint64_t>(src[i] - '0');
        t.text.push_back(src[i]);
        step();
      }
      t.kind = DevTok::Number;
    } else if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      while (i < src.size() && (std::isalnum(static_cast<unsigned char>(src[i])) ||
                                src[i] == '_' || src[i] == '.')) {
        t.text.push_back(src[i]);
        step();
      }
      t.kind = DevTok::Ident;
    } else {
      parse_fail(t, std::string("unexpected character '") + c + "'");
    }
    out.push_back(std::move(t));
  }
}

class DevParser {
 public:
  explicit DevParser(std::string_view text) : t_(dev_tokens(text)) {}
  const DevTok& peek(std::size_t k = 0) const {
    return t_[std::min(p_ + k, t_.size() - 1)];
  }
  DevTok take() {
    DevTok t = peek();
    if (p_ < t_.size() - 1) ++p_;
    return t;
  }
  DevTok want(DevTok::Kind k, const char* what) {
    if (peek().kind != k) parse_fail(peek(), std::string("expected ") + what);
    return take();
  }
  std::string keyword(const char* kw) {
    DevTok t = want(DevTok::Ident, (std::string("'") + kw + "'").c_str());
    if (t.text != kw) parse_fail(t, std::string("expected '") + kw + "'");
    return t.text;
  }
  std::uint64_t number_attr(const char* key) {
    DevTok k = want(DevTok::Ident, (std::string("'") + key + "'").c_str());
    if (k.text != key) parse_fail(k, std::string("expected '") + key + "'");
    want(DevTok::Equals, "'='");
    return want(DevTok::Number, (std::string("value of '") + key + "'").c_str()).number;
  }
  // key=value pairs up to the first token that does not start one
  std::vector<std::pair<std::string, DevTok>> attrs() {
    std::vector<std::pair<std::string, DevTok>> kv;
    while (peek().kind == DevTok::Ident && peek(1).kind == DevTok::Equals) {
      std::string key = take().text;
      take();
      DevTok v = take();
      if (v.kind != DevTok::Ident && v.kind != DevTok::Number && v.kind != DevTok::String)
        parse_fail(v, "expected attribute value");
      kv.emplace_back(std::move(key), std::move(v));
    }
    return kv;
  }
  static const DevTok* find(const std::vector<std::pair<std::string, DevTok>>& kv,
                            const char* key) {
    for (const auto& [k, v] : kv)
      if (k == key) return &v;
    return nullptr;
  }
  std::string ident_attr(const std::vector<std::pair<std::string, DevTok>>& kv,
                         const DevTok& at, const char* key, const char* ctx) {
    const DevTok* v = find(kv, key);
    if (!v) parse_fail(at, std::string(ctx) + " requires attribute '" + key + "'");
    if (v->kind != DevTok::Ident)
      parse_fail(*v, std::string("attribute '") + key + "' must be an identifier");
    return v->text;
  }
  std::optional<std::uint64_t> opt_number(
      const std::vector<std::pair<std::string, DevTok>>& kv, const char* key) {
    const DevTok* v = find(kv, key);
    if (!v) return std::nullopt;
    if (v->kind != DevTok::Number)
      parse_fail(*v, std::string("attribute '") + key + "' must be an integer");
    return v->number;
  }
  static std::string opt_string(const std::vector<std::pair<std::string, DevTok>>& kv,
                                const char* key) {
    const DevTok* v = find(kv, key);
    return v ? v->text : std::string();
  }
  std::uint32_t reg(const DevTok& r) {
    if (r.text.size() < 2 || r.text[0] != 'r') parse_fail(r, "expected register r<k>");
    return static_cast<std::uint32_t>(std::stoul(r.text.substr(1)));
  }

  void body(std::vector<DeviceInstr>& out) {
    for (;;) {
      const DevTok& t = peek();
      if (t.kind == DevTok::RBrace) {
        take();
        return;
      }
      if (t.kind == DevTok::Eof) parse_fail(t, "unexpected end of input inside a block");
      if (t.kind != DevTok::Ident) parse_fail(t, "expected an instruction");
      const DevTok kw = take();
      DeviceInstr d;
      if (kw.text == "init") {
        d.op = DeviceOpKind::Init;
      } else if (kw.text == "finalize") {
        d.op = DeviceOpKind::Finalize;
      } else if (kw.text == "read_counter") {
        want(DevTok::Arrow, "'->'");
        d.op = DeviceOpKind::ReadCounter;
        d.reg = reg(want(DevTok::Ident, "register"));
      } else if (kw.text == "store_counter") {
        d.op = DeviceOpKind::StoreCounter;
        d.reg = reg(want(DevTok::Ident, "register"));
        d.region_id = static_cast<std::uint32_t>(number_attr("region"));
        const DevTok se = want(DevTok::Ident, "'start' or 'end'");
        if (se.text != "start" && se.text != "end") parse_fail(se, "expected 'start' or 'end'");
        d.is_start = se.text == "start";
      } else if (kw.text == "for") {
        d.base.kind = InstrKind::LoopBegin;
        d.base.trip_count = want(DevTok::Number, "loop trip count").number;
        d.base.label = opt_string(attrs(), "label");
        want(DevTok::LBrace, "'{'");
        out.push_back(std::move(d));
        body(out);
        DeviceInstr e;
        e.base.kind = InstrKind::LoopEnd;
        out.push_back(std::move(e));
        continue;
      } else if (kw.text == "compute" || kw.text == "async_launch") {
        const auto kv = attrs();
        d.base.kind = kw.text == "compute" ? InstrKind::SyncCompute : InstrKind::AsyncLaunch;
        d.base.unit = ident_attr(kv, kw, "unit", kw.text.c_str());
        if (kw.text == "async_launch") d.base.token = ident_attr(kv, kw, "token", "async_launch");
        d.base.latency = opt_number(kv, "latency");
        d.base.label = opt_string(kv, "label");
      } else if (kw.text == "async_wait") {
        const auto kv = attrs();
        d.base.kind = InstrKind::AsyncWait;
        d.base.token = ident_attr(kv, kw, "token", "async_wait");
      } else if (kw.text == "arrive" || kw.text == "wait") {
        d.base.kind = kw.text == "arrive" ? InstrKind::BarrierArrive : InstrKind::BarrierWait;
        d.base.barrier = want(DevTok::Ident, "barrier name").text;
      } else if (kw.text == "record") {
        const DevTok se = want(DevTok::Ident, "'start' or 'end'");
        d.base.kind = InstrKind::Record;
        d.base.label = want(DevTok::String, "quoted region name").text;
        d.base.is_start = se.text == "start";
      } else {
        parse_fail(kw, "unknown instruction '" + kw.text + "'");
      }
      out.push_back(std::move(d));
    }
  }

  DeviceProgram program() {
    keyword("device");
    keyword("kernel");
    DeviceProgram dp;
    dp.name = want(DevTok::Ident, "kernel name").text;
    dp.num_warp_groups = static_cast<std::uint32_t>(number_attr("wgs"));
    dp.shared_mem_capacity = number_attr("smem");
    keyword("strategy");
    want(DevTok::Equals, "'='");
    const DevTok st = want(DevTok::Ident, "strategy value");
    if (st.text == "circular")
      dp.plan.strategy = BufferStrategy::Circular;
    else if (st.text == "flush")
      dp.plan.strategy = BufferStrategy::Flush;
    else
      parse_fail(st, "strategy must be circular or flush");
    dp.config.buffer_strategy = dp.plan.strategy;
    dp.plan.slots_per_warp_group = number_attr("slots_per_wg");
    dp.config.buffer_slots_total = dp.plan.slots_per_warp_group * dp.num_warp_groups;
    dp.config.signature_bits_enabled = number_attr("signature") != 0;
    dp.config.iteration_signature = number_attr("iter_sig") != 0;
    want(DevTok::LBrace, "'{'");
    dp.bodies.resize(dp.num_warp_groups);
    std::uint32_t next_wg = 0;
    for (;;) {
      const DevTok t = take();
      if (t.kind == DevTok::RBrace) break;
      if (t.kind == DevTok::Eof) parse_fail(t, "unexpected end of input inside device kernel");
      if (t.kind != DevTok::Ident) parse_fail(t, "expected 'region', 'barrier' or a wg block");
      if (t.text == "region") {
        const DevTok id = want(DevTok::Number, "region id");
        const DevTok label = want(DevTok::String, "region label");
        if (id.number != dp.plan.region_labels.size())
          parse_fail(id, "region ids must be dense and ascending");
        dp.plan.region_labels.push_back(label.text);
      } else if (t.text == "barrier") {
        BarrierDecl b;
        b.name = want(DevTok::Ident, "barrier name").text;
        b.expected_arrivals = static_cast<std::uint32_t>(number_attr("arrivals"));
        dp.barriers.push_back(std::move(b));
      } else if (t.text.size() > 2 && t.text.compare(0, 2, "wg") == 0) {
        const std::uint32_t idx = static_cast<std::uint32_t>(std::stoul(t.text.substr(2)));
        if (idx >= dp.num_warp_groups || idx != next_wg)
          parse_fail(t, "warp group blocks must appear as wg0..wgN-1 in order");
        ++next_wg;
        want(DevTok::LBrace, "'{'");
        body(dp.bodies[idx]);
      } else {
        parse_fail(t, "expected 'region', 'barrier' or a wg block");
      }
    }
    if (next_wg != dp.num_warp_groups)
      throw Error(ErrorKind::Parse, "device kernel is missing warp group bodies");
    return dp;
  }

 private:
  std::vector<DevTok> t_;
  std::size_t p_ = 0;
};

}  // namespace b200

// parse_device_program (lower.hpp:476-551): the `.dev` text back to a
// DeviceProgram (plan, barriers, bodies).
inline DeviceProgram parse_device_program(std::string_view text) {
  return b200::DevParser(text).program();
}

namespace detail {
// Barrier-derived candidate edges (perfmodel.hpp:258-313): for every barrier,
// the region whose end store is the last one before an arrive gates the
// region whose start store is the first one after a wait on it; sorted,
// unique, no self edges.
inline std::vector<std::pair<std::string, std::string>> barrier_edges(
    const DeviceProgram& dp) {
  std::vector<std::pair<std::string, std::string>> src, dst, out;  // (barrier, label)
  auto label = [&](std::uint32_t id) {
    return id < dp.plan.region_labels.size() ? dp.plan.region_labels[id] : std::string();
  };
  for (std::uint32_t wg = 0; wg < dp.num_warp_groups && wg < dp.bodies.size(); ++wg) {
    const auto& b = dp.bodies[wg];
    for (std::size_t i = 0; i < b.size(); ++i) {
      if (b[i].op != DeviceOpKind::Base) continue;
      const InstrKind k = b[i].base.kind;
      if (k == InstrKind::BarrierArrive) {
        for (std::size_t j = i; j-- > 0;)
          if (b[j].op == DeviceOpKind::StoreCounter && !b[j].is_start) {
            const std::string l = label(b[j].region_id);
            if (!l.empty()) src.emplace_back(b[i].base.barrier, l);
            break;
          }
      } else if (k == InstrKind::BarrierWait) {
        for (std::size_t j = i + 1; j < b.size(); ++j)
          if (b[j].op == DeviceOpKind::StoreCounter && b[j].is_start) {
            const std::string l = label(b[j].region_id);
            if (!l.empty()) dst.emplace_back(b[i].base.barrier, l);
            break;
          }
      }
    }
  }
  for (const auto& a : src)
    for (const auto& w : dst)
      if (a.first == w.first && a.second != w.second) out.emplace_back(a.second, w.second);
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}
}  // namespace detail

// CriticalPathAnalysis (perfmodel.hpp:242-246) and the reference's
// analyze_critical_path(events, dp, opts) (perfmodel.hpp:317-318): the GPU
// analysis with the program's barrier edges.
struct CriticalPathAnalysis {
  WsInput graph;
  std::vector<std::string> cycle;
  std::uint64_t period = 0;
};
inline CriticalPathAnalysis analyze_critical_path(const std::vector<TimelineEvent>& events,
                                                  const DeviceProgram& dp,
                                                  const CriticalPathOptions& opts = {}) {
  CriticalPathResult r = analyze_critical_path(events, detail::barrier_edges(dp), opts);
  CriticalPathAnalysis a;
  a.graph = std::move(r.graph);
  a.cycle = std::move(r.cycle);
  a.period = r.period;
  return a;
}

// The simulator totals the reports carry (vgpu.hpp:61-68); a replay of a
// trace file has none (tools/wgprof.cpp:111).
struct SimResult {
  GlobalTraceImage image;
  std::uint64_t total_cycles = 0;
  std::uint64_t vanilla_cycles = 0;
  std::uint64_t records_written = 0;
  std::vector<std::vector<ProfileRecord>> store_log;
};

#ifdef WGPROF_B200_HAVE_JSON
// make_replay_report (pipeline.hpp:146-178): the replay report from the GPU's
// statistics (region_stats above) and critical path.
inline nlohmann::ordered_json make_replay_report(const std::string& kernel,
                                                 const SimResult& sim,
                                                 const TraceReplay& tr,
                                                 const CriticalPathAnalysis& cp,
                                                 std::uint64_t record_cost) {
  using J = nlohmann::ordered_json;
  J rep;
  rep["kernel"] = kernel;
  rep["total_cycles"] = sim.total_cycles;
  rep["vanilla_cycles"] = sim.vanilla_cycles;
  rep["records_written"] = sim.records_written;
  rep["record_cost"] = record_cost;
  J regions = J::array();
  for (const auto& [label, st] : region_stats(tr.events)) {
    J r;
    r["region"] = label;
    r["warp_group"] = st.warp_group;
    r["kind"] = st.kind == EventKind::Wait ? "wait" : "exec";
    r["count"] = st.count;
    r["mean_duration"] = st.mean;
    r["min_duration"] = st.min;
    r["max_duration"] = st.max;
    regions.push_back(std::move(r));
  }
  rep["regions"] = std::move(regions);
  rep["critical_path"] = cp.cycle.empty() ? ws_latency(cp.graph).critical_path : cp.cycle;
  rep["iteration_period"] = cp.period;
  J w;
  w["dropped_heads"] = tr.dropped_heads;
  w["truncated_tails"] = tr.truncated_tails;
  w["flagged_preconditions"] = tr.flagged_preconditions;
  w["malformed_groups"] = tr.malformed_groups;
  rep["warnings"] = std::move(w);
  return rep;
}
#endif

}  // namespace wgprof
