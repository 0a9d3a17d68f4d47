// Compile check: the drop-in shim exposes the reference's wgprof signatures.
#include "wgprof_b200.hpp"

using namespace wgprof;

// Each line names a reference entry point with its reference signature.
[[maybe_unused]] static std::vector<DecodedStream> (*p_decode)(const GlobalTraceImage&, const BufferPlan&) = decode_image;
[[maybe_unused]] static std::vector<std::uint64_t> (*p_unwrap)(const std::vector<std::uint32_t>&) = unwrap_clock;
[[maybe_unused]] static PairResult (*p_pair)(const std::vector<ProfileRecord>&, const std::vector<std::string>&) = pair_records;
[[maybe_unused]] static ReplayResult (*p_replay)(const PairResult&, std::uint32_t, std::uint32_t, std::uint64_t) = replay;
[[maybe_unused]] static TraceReplay (*p_replay_image)(const GlobalTraceImage&, const BufferPlan&, std::uint64_t) = replay_image;
[[maybe_unused]] static std::map<std::string, RegionStats> (*p_stats)(const std::vector<TimelineEvent>&) = region_stats;
[[maybe_unused]] static GlobalTraceImage (*p_deser)(const std::vector<std::uint8_t>&) = deserialize_image;
[[maybe_unused]] static std::vector<std::uint8_t> (*p_ser)(const GlobalTraceImage&) = serialize_image;
