// capi.cu -- host side of the C-ABI (include/wgpf.h): context, plan tables,
// buffer management and the replay orchestration.  Single translation unit:
// the kernels live in the k_*.cuh headers included below.
//
// replay orchestration (one call of wgpf_replay_device):
//   k_count_fast      pass 1, warp/stream: decode checks, counts, routing
//   cub ExclusiveSum  counts -> event offsets
//   k_fast_emit       pass 2, warp/stream: pair + replay + stats (fast path)
//   k_general_emit    thread/stream, exact: streams routed off the fast path
//   (rare) exact recount of single-stack-invalid streams + re-emit
//   k_resolve_first   first-event warp_group per label
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include "wgpf.h"
#include "wgpf_dev.cuh"
#include "k_count.cuh"
#include "k_fast.cuh"
#include "k_tps.cuh"
#include "k_tpsd.cuh"
#include "k_general.cuh"
#include "k_misc.cuh"
#include "k_stats.cuh"
#include "k_synth.cuh"
#include "k_cp.cuh"
#include "k_chrome.cuh"
#include <cmath>
#include <functional>
#include <memory>
#include <thread>

using namespace wgpf;

namespace {

struct ToU64 {
  __host__ __device__ uint64_t operator()(uint32_t x) const { return x; }
};

constexpr uint32_t kSynthHash = 1024;  // out-of-table label classes per call

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  bool ensure(size_t bytes) {
    if (bytes <= n) return true;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    size_t want = std::max<size_t>(bytes, 256);
    if (cudaMalloc(&p, want) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    n = want;
    return true;
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

}  // namespace

using TpsKernel = void (*)(FastArgs);
using DeepKernel = void (*)(FastArgs, const CUtensorMap);
using TpsTmaKernel = void (*)(FastArgs, const CUtensorMap, const CUtensorMap);
static DeepKernel deep_kernel(bool emit, bool stats, bool markers, bool wide) {
  static const DeepKernel k[16] = {
      k_tpsd<false, false, false, false>, k_tpsd<true, false, false, false>,
      k_tpsd<false, true, false, false>,  k_tpsd<true, true, false, false>,
      k_tpsd<false, false, true, false>,  k_tpsd<true, false, true, false>,
      k_tpsd<false, true, true, false>,   k_tpsd<true, true, true, false>,
      k_tpsd<false, false, false, true>,  k_tpsd<true, false, false, true>,
      k_tpsd<false, true, false, true>,   k_tpsd<true, true, false, true>,
      k_tpsd<false, false, true, true>,   k_tpsd<true, false, true, true>,
      k_tpsd<false, true, true, true>,    k_tpsd<true, true, true, true>};
  return k[(emit ? 1 : 0) | (stats ? 2 : 0) | (markers ? 4 : 0) | (wide ? 8 : 0)];
}
static TpsTmaKernel tps_kernel(bool emit, bool stats) {
  static const TpsTmaKernel k[4] = {k_tps<false, false>, k_tps<true, false>,
                                 k_tps<false, true>, k_tps<true, true>};
  return k[(emit ? 1 : 0) | (stats ? 2 : 0)];
}

struct wgpf_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  std::string err;

  // plan
  bool has_plan = false;
  uint64_t slots = 0;
  uint32_t strategy = 0;
  std::vector<std::string> labels;
  std::vector<std::string> class_label;  // dense classes
  std::unordered_map<std::string, uint32_t> class_by_label;
  uint32_t K = 0;
  bool has_markers = false;  // some label is a wait marker ("X.wait")
  DevBuf d_class_of, d_wait_class, d_is_marker, d_swait_id, d_swait_cls;
  uint32_t n_synth_wait = 0;

  // stats
  DevBuf d_count, d_sum, d_min, d_max, d_first, d_hist, d_hkey, d_first_wg,
      d_mean;
  bool stats_valid = false;
  bool mean_exact_valid = false;
  std::vector<wgpf_region_stat> stats_out;
  std::vector<std::string> stats_names;

  // per call
  DevBuf d_status, d_counts, d_zpos, d_sflag, d_offsets, d_scan_tmp, d_glist,
      d_glen, d_orphans, d_gscratch, d_image, d_events, d_aux0, d_aux1, d_aux2,
      d_aux3, d_repack, d_chrome, d_dlist;
  DevStatus* h_status = nullptr;  // pinned
  // profiling
  cudaEvent_t ev[8] = {};
  bool profiling = false;
  bool no_stage = getenv("WGPF_NO_STAGE") != nullptr;
  bool no_tps = getenv("WGPF_NO_TPS") != nullptr;
  bool no_deep = getenv("WGPF_NO_DEEP") != nullptr;  // deep streams -> warp kernel
  bool no_wide = getenv("WGPF_NO_WIDE") != nullptr;  // wide streams -> warp kernel
  bool no_tma = getenv("WGPF_NO_TMA") != nullptr;    // k_tps windows by cp.async only
  bool no_group = getenv("WGPF_NO_GROUP") != nullptr;  // k_tps: consecutive streams per warp
  uint32_t group_hint = 0;   // W known from host headers (pipelined replay)
  uint32_t* h_blk = nullptr;  // pinned: block fields read by stream_group
  bool no_pipeline = getenv("WGPF_NO_PIPELINE") != nullptr;
  // overlapped pass 1 / pass 2 (replay_overlapped): a second stream for the
  // pass-1 chain, one event per chunk, chunk bases and batch counters
  // opt-in (WGPF_OVERLAP=1): measured slower, see replay_overlapped
  bool no_overlap = getenv("WGPF_OVERLAP") == nullptr;
  cudaStream_t s_count = nullptr;
  std::vector<cudaEvent_t> oev;
  DevBuf d_obase;
  DevBuf d_wlist;  // SF_WARP streams (count in d_glen[1])
  DevBuf d_vlist;  // wide-path streams (count in d_glen[3])
  DevBuf d_nccl_send, d_nccl_recv;  // wgpf_allreduce_stats
  DevBuf d_deep_rep;  // k_tpsd: per-CTA statistics replicas
  // pinned bounce buffers for pageable caller memory (replay_image pipeline)
  uint8_t* h_bounce_in[2] = {nullptr, nullptr};
  uint8_t* h_bounce_out[2] = {nullptr, nullptr};
  size_t bounce_in_n = 0, bounce_out_n[2] = {0, 0};
  DevBuf d_dorph;  // k_tpsd: one orphan event per lane
  size_t smem_optin = 0;
  // pipelined replay_image (host buffers): copy streams, chunk buffers, and
  // per-chunk (first stream, first event) for first_event lookups
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t pev[6] = {};  // h2d done [2], compute done [2], d2h done [2]
  DevBuf d_cbody[2], d_cev[2], d_packed, d_off_all;
  bool in_chunked = false, chunk_mode = false;
  std::vector<uint64_t> chunk_sbase, chunk_ebase;
  uint64_t chunk_nstreams = 0;
  uint32_t launches = 0;
  uint32_t overlap_chunks = 0;
  uint64_t general_streams = 0;
  wgpf_profile prof{};
  uint64_t last_stream_base = 0, last_n_streams = 0;
  const uint8_t* last_body = nullptr;
  uint64_t last_stride = 0;

  ~wgpf_ctx() {
    if (h_status) cudaFreeHost(h_status);
    if (h_blk) cudaFreeHost(h_blk);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : pev)
      if (e) cudaEventDestroy(e);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_count) cudaStreamDestroy(s_count);
    for (auto& e : oev)
      if (e) cudaEventDestroy(e);
    if (s_d2h) cudaStreamDestroy(s_d2h);
    for (int b = 0; b < 2; ++b) {
      if (h_bounce_in[b]) cudaFreeHost(h_bounce_in[b]);
      if (h_bounce_out[b]) cudaFreeHost(h_bounce_out[b]);
    }
  }
  void mark(int i) {
    if (profiling) cudaEventRecord(ev[i], stream);
  }
};

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------

static int set_err(wgpf_ctx* c, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  c->err = buf;
  return code;
}

static const bool g_debug = getenv("WGPF_DEBUG") != nullptr;

#define CUDA_OK(ctx, expr)                                                    \
  do {                                                                        \
    cudaError_t e_ = (expr);                                                  \
    if (g_debug && e_ == cudaSuccess) {                                       \
      fprintf(stderr, "[wgpf] %s:%d %s ... ", __FILE__, __LINE__, #expr);     \
      fflush(stderr);                                                         \
      e_ = cudaStreamSynchronize((ctx)->stream);                              \
      fprintf(stderr, "%s\n", cudaGetErrorString(e_));                        \
    }                                                                         \
    if (e_ != cudaSuccess) {                                                  \
      cudaGetLastError();                                                     \
      return set_err(ctx, WGPF_E_CUDA, "%s: %s (%s:%d)", #expr,               \
                     cudaGetErrorString(e_), __FILE__, __LINE__);             \
    }                                                                         \
  } while (0)

#define ALLOC_OK(ctx, buf, bytes)                                             \
  do {                                                                        \
    if (!(buf).ensure(bytes))                                                 \
      return set_err(ctx, WGPF_E_CUDA, "cudaMalloc of %zu bytes failed",      \
                     (size_t)(bytes));                                        \
  } while (0)

static std::string label_of(const wgpf_ctx* c, uint32_t rid) {
  if (rid < c->labels.size()) return c->labels[rid];
  return "region#" + std::to_string(rid);
}

static std::string class_name(const wgpf_ctx* c, uint32_t cls) {
  if (cls < c->K) return c->class_label[cls];
  return "region#" + std::to_string(cls - c->K);
}

static DevPlan dev_plan(const wgpf_ctx* c) {
  DevPlan p;
  p.slots = c->slots;
  p.strategy = c->strategy;
  p.T = (uint32_t)c->labels.size();
  p.K = c->K;
  p.n_synth_wait = c->n_synth_wait;
  p.class_of = c->d_class_of.as<uint32_t>();
  p.wait_class = c->d_wait_class.as<uint32_t>();
  p.is_marker = c->d_is_marker.as<uint8_t>();
  p.synth_wait_id = c->d_swait_id.as<uint32_t>();
  p.synth_wait_cls = c->d_swait_cls.as<uint32_t>();
  return p;
}

static uint32_t n_slots(const wgpf_ctx* c) { return c->K + kSynthHash; }

static DevStats dev_stats(const wgpf_ctx* c) {
  DevStats s;
  s.count = c->d_count.as<unsigned long long>();
  s.sum = c->d_sum.as<unsigned long long>();
  s.min = c->d_min.as<unsigned long long>();
  s.max = c->d_max.as<unsigned long long>();
  s.first = c->d_first.as<unsigned long long>();
  s.hist = c->d_hist.as<unsigned long long>();
  s.hkey = c->d_hkey.as<uint32_t>();
  s.K = c->K;
  s.H = kSynthHash;
  return s;
}

static int stats_reset(wgpf_ctx* c) {
  const size_t ns = n_slots(c);
  CUDA_OK(c, cudaMemsetAsync(c->d_count.p, 0, 8 * ns, c->stream));
  CUDA_OK(c, cudaMemsetAsync(c->d_sum.p, 0, 8 * ns, c->stream));
  CUDA_OK(c, cudaMemsetAsync(c->d_min.p, 0xFF, 8 * ns, c->stream));
  CUDA_OK(c, cudaMemsetAsync(c->d_max.p, 0, 8 * ns, c->stream));
  CUDA_OK(c, cudaMemsetAsync(c->d_first.p, 0xFF, 8 * ns, c->stream));
  CUDA_OK(c, cudaMemsetAsync(c->d_first_wg.p, 0, 8 * ns, c->stream));
  CUDA_OK(c, cudaMemsetAsync(c->d_hist.p, 0, 8 * ns * WGPF_HIST_BINS, c->stream));
  CUDA_OK(c, cudaMemsetAsync(c->d_hkey.p, 0xFF, 4 * kSynthHash, c->stream));
  c->stats_valid = false;
  c->mean_exact_valid = false;
  return WGPF_OK;
}

static int status_reset(wgpf_ctx* c) {
  DevStatus s;
  memset(&s, 0, sizeof s);
  s.decode_err = kNoErr;
  s.pair_err = kNoErr;
  *c->h_status = s;
  CUDA_OK(c, cudaMemcpyAsync(c->d_status.p, c->h_status, sizeof(DevStatus),
                             cudaMemcpyHostToDevice, c->stream));
  return WGPF_OK;
}

static int status_read(wgpf_ctx* c) {
  CUDA_OK(c, cudaMemcpyAsync(c->h_status, c->d_status.p, sizeof(DevStatus),
                             cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  return WGPF_OK;
}

static uint32_t grid_for(wgpf_ctx* c, const void* kernel, int threads,
                         size_t smem) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads,
                                                    smem) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  return (uint32_t)(c->sms * per_sm);
}

// ---------------------------------------------------------------------------
// lifecycle
// ---------------------------------------------------------------------------

extern "C" {

int wgpf_abi_version(void) { return WGPF_ABI_VERSION; }

const char* wgpf_error_category(int status) {
  switch (status) {
    case WGPF_OK: return "ok";
    case WGPF_E_PARSE: return "parse-error";
    case WGPF_E_VALIDATE: return "validate-error";
    case WGPF_E_INSTRUMENT: return "instrument-error";
    case WGPF_E_LOWER: return "lower-error";
    case WGPF_E_CAPACITY: return "capacity-error";
    case WGPF_E_DEADLOCK: return "simulation-deadlock";
    case WGPF_E_TRACE: return "trace-error";
    case WGPF_E_CONFIG: return "config-error";
    case WGPF_E_IO: return "io-error";
    case WGPF_E_CUDA: return "cuda-error";
    case WGPF_E_ARG: return "argument-error";
    case WGPF_E_BUFFER: return "buffer-too-small";
    default: return "error";
  }
}

int wgpf_create(int device, void* stream, wgpf_ctx** out) {
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return WGPF_E_CUDA;
  }
  if (device < 0 || device >= n) return WGPF_E_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return WGPF_E_CUDA;
  wgpf_ctx* c = new wgpf_ctx();
  c->device = device;
  c->stream = reinterpret_cast<cudaStream_t>(stream);
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMallocHost(&c->h_status, sizeof(DevStatus)) != cudaSuccess ||
      !c->d_status.ensure(sizeof(DevStatus)) || !c->d_glen.ensure(64)) {
    delete c;
    return WGPF_E_CUDA;
  }
  {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    c->smem_optin = (size_t)optin;
    for (int v = 0; v < 4; ++v) {
      cudaFuncSetAttribute(tps_kernel(v & 1, v & 2),
                           cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
      for (int m = 0; m < 4; ++m)
        cudaFuncSetAttribute(deep_kernel(v & 1, v & 2, m & 1, m & 2),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    }
  }
  cudaFuncSetAttribute(k_fast_emit<false>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)fast_smem_bytes(false, 0));
  cudaFuncSetAttribute(k_fast_emit<true>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (auto& e : c->ev) cudaEventCreate(&e);
  *out = c;
  return WGPF_OK;
}

void wgpf_destroy(wgpf_ctx* ctx) { delete ctx; }

int wgpf_set_stream(wgpf_ctx* ctx, void* stream) {
  ctx->stream = reinterpret_cast<cudaStream_t>(stream);
  return WGPF_OK;
}

const char* wgpf_last_error(const wgpf_ctx* ctx) { return ctx->err.c_str(); }

// BufferPlan (lower.hpp:57-73).  Label classes: one per distinct label
// string (duplicates in the table share statistics and wait matching, as
// the reference keys both by label string, pipeline.hpp:116, trace.hpp:442).
int wgpf_set_plan(wgpf_ctx* c, uint64_t slots, uint32_t strategy,
                  const char* const* labels, uint32_t n_labels) {
  if (strategy > 1) return set_err(c, WGPF_E_ARG, "strategy must be 0 or 1");
  if (n_labels > WGPF_MAX_REGIONS)
    return set_err(c, WGPF_E_ARG, "more than 2^19 region labels");
  c->slots = slots;
  c->strategy = strategy;
  c->labels.assign(labels, labels + n_labels);
  c->class_label.clear();
  c->class_by_label.clear();
  std::vector<uint32_t> cls_of_table(n_labels);
  for (uint32_t i = 0; i < n_labels; ++i) {
    auto it = c->class_by_label.find(c->labels[i]);
    if (it == c->class_by_label.end()) {
      uint32_t k = (uint32_t)c->class_label.size();
      c->class_by_label.emplace(c->labels[i], k);
      c->class_label.push_back(c->labels[i]);
      cls_of_table[i] = k;
    } else {
      cls_of_table[i] = it->second;
    }
  }
  c->K = (uint32_t)c->class_label.size();
  c->has_markers = false;
  std::vector<uint32_t> class_of(WGPF_MAX_REGIONS);
  for (uint32_t r = 0; r < WGPF_MAX_REGIONS; ++r)
    class_of[r] = r < n_labels ? cls_of_table[r] : c->K + r;
  std::vector<uint32_t> wait_class(c->K + 1, kNone);
  std::vector<uint8_t> is_marker(c->K + 1, 0);
  std::vector<std::pair<uint32_t, uint32_t>> swait;
  for (uint32_t k = 0; k < c->K; ++k) {
    const std::string& L = c->class_label[k];
    is_marker[k] = L.size() > 5 && L.compare(L.size() - 5, 5, ".wait") == 0;
    if (is_marker[k]) c->has_markers = true;
    auto it = c->class_by_label.find(L + ".wait");
    if (it != c->class_by_label.end()) wait_class[k] = it->second;
    // out-of-table ids whose synthesized label is a table label
    if (L.rfind("region#", 0) == 0) {
      const std::string d = L.substr(7);
      if (!d.empty() && d.size() <= 7 &&
          d.find_first_not_of("0123456789") == std::string::npos) {
        const unsigned long id = std::stoul(d);
        if (id >= n_labels && id < WGPF_MAX_REGIONS &&
            std::to_string(id) == d)
          class_of[id] = k;
      }
    }
    if (is_marker[k]) {
      const std::string b = L.substr(0, L.size() - 5);
      if (b.rfind("region#", 0) == 0) {
        const std::string d = b.substr(7);
        if (!d.empty() && d.size() <= 7 &&
            d.find_first_not_of("0123456789") == std::string::npos) {
          const unsigned long id = std::stoul(d);
          if (id >= n_labels && id < WGPF_MAX_REGIONS &&
              std::to_string(id) == d)
            swait.emplace_back((uint32_t)id, k);
        }
      }
    }
  }
  std::sort(swait.begin(), swait.end());
  c->n_synth_wait = (uint32_t)swait.size();
  std::vector<uint32_t> sw_id, sw_cls;
  for (auto& p : swait) {
    sw_id.push_back(p.first);
    sw_cls.push_back(p.second);
  }
  ALLOC_OK(c, c->d_class_of, 4ull * WGPF_MAX_REGIONS);
  ALLOC_OK(c, c->d_wait_class, 4ull * (c->K + 1));
  ALLOC_OK(c, c->d_is_marker, c->K + 1);
  ALLOC_OK(c, c->d_swait_id, 4ull * (sw_id.size() + 1));
  ALLOC_OK(c, c->d_swait_cls, 4ull * (sw_id.size() + 1));
  CUDA_OK(c, cudaMemcpyAsync(c->d_class_of.p, class_of.data(),
                             4ull * WGPF_MAX_REGIONS, cudaMemcpyHostToDevice,
                             c->stream));
  CUDA_OK(c, cudaMemcpyAsync(c->d_wait_class.p, wait_class.data(),
                             4ull * (c->K + 1), cudaMemcpyHostToDevice, c->stream));
  CUDA_OK(c, cudaMemcpyAsync(c->d_is_marker.p, is_marker.data(), c->K + 1,
                             cudaMemcpyHostToDevice, c->stream));
  if (!sw_id.empty()) {
    CUDA_OK(c, cudaMemcpyAsync(c->d_swait_id.p, sw_id.data(), 4 * sw_id.size(),
                               cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(c, cudaMemcpyAsync(c->d_swait_cls.p, sw_cls.data(), 4 * sw_id.size(),
                               cudaMemcpyHostToDevice, c->stream));
  }
  const size_t ns = n_slots(c);
  ALLOC_OK(c, c->d_count, 8 * ns);
  ALLOC_OK(c, c->d_sum, 8 * ns);
  ALLOC_OK(c, c->d_min, 8 * ns);
  ALLOC_OK(c, c->d_max, 8 * ns);
  ALLOC_OK(c, c->d_first, 8 * ns);
  ALLOC_OK(c, c->d_first_wg, 8 * ns);
  ALLOC_OK(c, c->d_mean, 8 * ns);
  ALLOC_OK(c, c->d_hist, 8 * ns * WGPF_HIST_BINS);
  ALLOC_OK(c, c->d_hkey, 4 * kSynthHash);
  int rc = stats_reset(c);
  if (rc) return rc;
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  c->has_plan = true;
  return WGPF_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// replay orchestration
// ---------------------------------------------------------------------------

static int run_general(wgpf_ctx* c, const uint8_t* body, uint64_t stride,
                       uint64_t n_streams, uint64_t stream_base,
                       uint64_t record_cost, wgpf_event* events,
                       uint64_t events_cap, bool no_stats, bool use_list,
                       uint64_t n_work) {
  if (n_work == 0) return WGPF_OK;
  const uint32_t cap = (uint32_t)c->slots;
  uint32_t hm = 16;
  while (hm < 2u * cap + 2u) hm <<= 1;
  const uint64_t per = gen_scratch_bytes(cap, hm);
  uint64_t batch = std::max<uint64_t>(1, (256ull << 20) / per);
  batch = std::min<uint64_t>(batch, n_work);
  batch = (batch + 127) / 128 * 128;
  ALLOC_OK(c, c->d_gscratch, per * batch);
  GenArgs a;
  a.body = body;
  a.stride = stride;
  a.n_streams = n_streams;
  a.stream_base = stream_base;
  a.plan = dev_plan(c);
  a.stats = dev_stats(c);
  a.status = c->d_status.as<DevStatus>();
  a.counts = c->d_counts.as<uint32_t>();
  a.sflag = c->d_sflag.as<uint32_t>();
  a.offsets = c->d_offsets.as<uint64_t>();
  a.events = events;
  a.events_cap = events_cap;
  a.record_cost = record_cost;
  a.list = use_list ? c->d_glist.as<uint64_t>() : nullptr;
  a.list_len = c->d_glen.as<unsigned long long>();
  a.batch = batch;
  a.scratch = c->d_gscratch.as<uint8_t>();
  a.scratch_stride = per;
  a.cap = cap;
  a.hm_size = hm;
  a.no_stats = no_stats ? 1u : 0u;
  for (uint64_t first = 0; first < n_work; first += batch) {
    a.first = first;
    k_general_emit<<<(uint32_t)(batch / 128), 128, 0, c->stream>>>(a);
    CUDA_OK(c, cudaGetLastError());
    ++c->launches;
  }
  return WGPF_OK;
}

static int run_general_count(wgpf_ctx* c, const uint8_t* body, uint64_t stride,
                             uint64_t n_streams, uint64_t stream_base,
                             uint64_t n_work) {
  if (n_work == 0) return WGPF_OK;
  const uint32_t cap = (uint32_t)c->slots;
  uint32_t hm = 16;
  while (hm < 2u * cap + 2u) hm <<= 1;
  const uint64_t per = gen_scratch_bytes(cap, hm);
  uint64_t batch = std::max<uint64_t>(1, (256ull << 20) / per);
  batch = std::min<uint64_t>(batch, n_work);
  batch = (batch + 127) / 128 * 128;
  ALLOC_OK(c, c->d_gscratch, per * batch);
  GenArgs a;
  memset(&a, 0, sizeof a);
  a.body = body;
  a.stride = stride;
  a.n_streams = n_streams;
  a.stream_base = stream_base;
  a.plan = dev_plan(c);
  a.status = c->d_status.as<DevStatus>();
  a.counts = c->d_counts.as<uint32_t>();
  a.sflag = c->d_sflag.as<uint32_t>();
  a.list = c->d_glist.as<uint64_t>();
  a.list_len = c->d_glen.as<unsigned long long>();
  a.batch = batch;
  a.scratch = c->d_gscratch.as<uint8_t>();
  a.scratch_stride = per;
  a.cap = cap;
  a.hm_size = hm;
  for (uint64_t first = 0; first < n_work; first += batch) {
    a.first = first;
    k_general_count<<<(uint32_t)(batch / 128), 128, 0, c->stream>>>(a);
    CUDA_OK(c, cudaGetLastError());
    ++c->launches;
  }
  return WGPF_OK;
}

__global__ void k_total(const uint32_t* counts, const uint64_t* off, uint64_t n,
                        DevStatus* st) {
  st->total_events = n ? off[n - 1] + counts[n - 1] : 0;
}

// streams flagged SF_INVALID -> general list (and SF_GENERAL for the re-emit)
__global__ void k_collect_invalid(uint32_t* sflag, uint64_t n,
                                  unsigned long long* list,
                                  unsigned long long* len) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (uint64_t)gridDim.x * blockDim.x)
    if (sflag[s] & SF_INVALID) {
      sflag[s] = (sflag[s] & ~SF_INVALID) | SF_GENERAL;
      list[atomicAdd(len, 1ull)] = s;
    }
}

static int scan_counts(wgpf_ctx* c, uint64_t n) {
  size_t tmp = 0;
  const uint32_t* in = c->d_counts.as<uint32_t>();
  uint64_t* out = c->d_offsets.as<uint64_t>();
  // widen to 64-bit accumulation
  auto it = thrust::make_transform_iterator(in, ToU64());
  CUDA_OK(c, cub::DeviceScan::ExclusiveSum(nullptr, tmp, it, out, (int64_t)n,
                                           c->stream));
  ALLOC_OK(c, c->d_scan_tmp, tmp);
  CUDA_OK(c, cub::DeviceScan::ExclusiveSum(c->d_scan_tmp.p, tmp, it, out,
                                           (int64_t)n, c->stream));
  k_total<<<1, 1, 0, c->stream>>>(in, out, n, c->d_status.as<DevStatus>());
  CUDA_OK(c, cudaGetLastError());
  ++c->launches;
  return WGPF_OK;
}

// Thread-per-stream kernel usable for this plan (even capacity that fits the
// packed stack entries, label classes that fit the lane-private tables).
static bool tps_enabled(const wgpf_ctx* c) {
  return !c->no_tps && c->slots % 2 == 0 && c->slots && c->slots <= kTpsMaxSlots &&
         c->K <= kTpsClasses && !c->labels.empty();
}
// thread-per-stream pass 1: record windows need an even capacity
static bool count_tps_enabled(const wgpf_ctx* c) {
  return !c->no_tps && c->slots % 2 == 0 && c->slots && c->slots <= kTpsMaxSlots;
}
// deep thread-per-stream kernel for SF_DEEP streams of the warp list (any
// number of label classes: its statistics live in the CTA table)
static bool deep_enabled(const wgpf_ctx* c) {
  return !c->no_tps && !c->no_deep && c->slots % 2 == 0 && c->slots &&
         c->slots <= kDeepMaxSlots && !c->labels.empty();
}
// wide thread-per-stream path (k_tpsd<kWide>): plans with region ids past the
// deep kernel's 64
static bool wide_enabled(const wgpf_ctx* c) {
  return deep_enabled(c) && !c->no_wide && c->labels.size() > kDeepRegions &&
         c->slots <= kDeepMaxSlots;
}
static uint32_t tps_regions(const wgpf_ctx* c) {
  return std::min<uint32_t>((uint32_t)c->labels.size(), kTpsRegions);
}

// The body as a 2-D u32 tensor {stride / 4, n_streams} with k_tps's window
// box {kTpsPitch / 4, 32} (k_window.cuh); false when TMA cannot address it
// (alignment, sizes) or the driver entry point is missing.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMapL2promotion l2_promotion() {
  const char* e = getenv("WGPF_TMA_L2");
  const int v = e ? atoi(e) : 256;  // measured: 256 B ~1 % faster than none
  return v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
         : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
         : v == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                    : CU_TENSOR_MAP_L2_PROMOTION_NONE;
}
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                       cudaSuccess &&
                   q == cudaDriverEntryPointSuccess
               ? reinterpret_cast<EncodeTiledFn>(p)
               : nullptr;
  }();
  return fn;
}
static bool body_tensor_map(CUtensorMap* m, const uint8_t* body, uint64_t stride,
                            uint64_t n_streams, uint32_t pitch,
                            CUtensorMapL2promotion prom = l2_promotion(),
                            CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn || (reinterpret_cast<uintptr_t>(body) & 15u) || (stride & 15u) ||
      stride < pitch || stride >= (1ull << 39) || n_streams < 32 ||
      n_streams >= (1ull << 31))
    return false;
  const cuuint64_t dims[2] = {stride / 4, n_streams};
  const cuuint64_t strides[1] = {stride};
  const cuuint32_t box[2] = {pitch / 4, 32};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint8_t*>(body), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
            prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Streams per block W of a device body (k_tps's lane mapping): the length of
// the leading run of streams whose header has stream 0's block, if it
// divides the stream count; else 1.  Reads the block field of up to 1,025
// headers (one small strided copy).
static uint32_t stream_group(wgpf_ctx* c, const uint8_t* body, uint64_t stride,
                             uint64_t n_streams) {
  if (c->no_group || n_streams < 64) return 1;
  if (c->group_hint)
    return n_streams % c->group_hint == 0 && n_streams / c->group_hint >= 32 ? c->group_hint
                                                                             : 1u;
  const uint64_t m = std::min<uint64_t>(n_streams, 1025);
  if (!c->h_blk && cudaMallocHost(&c->h_blk, 4 * 1025) != cudaSuccess) {
    c->h_blk = nullptr;
    cudaGetLastError();
    return 1;
  }
  const uint32_t* blk = c->h_blk;
  if (cudaMemcpy2DAsync(c->h_blk, 4, body, stride, 4, m, cudaMemcpyDeviceToHost,
                        c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  // (fewer than 32 blocks would leave lanes of every batch idle)
  for (uint64_t i = 1; i < m; ++i)
    if (blk[i] != blk[0]) return n_streams % i == 0 && n_streams / i >= 32 ? (uint32_t)i : 1u;
  return 1;
}

// 3-D view {stride / 4, W, n_streams / W} with box {kTpsPitch / 4, 1, 32}
// for the grouped lane mapping (k_window.cuh win_tma3)
static bool body_tensor_map3(CUtensorMap* m, const uint8_t* body, uint64_t stride,
                             uint64_t n_streams, uint32_t W,
                             CUtensorMapL2promotion prom = l2_promotion()) {
  EncodeTiledFn fn = encode_tiled();
  const uint64_t nb = n_streams / W;
  if (!fn || (reinterpret_cast<uintptr_t>(body) & 15u) || (stride & 15u) ||
      stride < kTpsPitch || stride * W >= (1ull << 39) || nb >= (1ull << 31) || W > 256 ||
      n_streams % W)
    return false;
  const cuuint64_t dims[3] = {stride / 4, W, nb};
  const cuuint64_t strides[2] = {stride, stride * W};
  const cuuint32_t box[3] = {kTpsPitch / 4, 1, 32};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint8_t*>(body), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The same view without L2 promotion, for the windows that end within 256 B
// of a stream's last record: a promoted request there would pull the unused
// slots past record_count into L2 (config 4: 1.3 GB of the body's 10 GB).
static bool tail_maps() { return getenv("WGPF_NO_TAIL_MAP") == nullptr; }

// The pass-2 arguments shared by every emit kernel of one call.
static FastArgs fast_args(wgpf_ctx* c, const uint8_t* body, uint64_t stride,
                          uint64_t n_streams, uint64_t stream_base, uint64_t record_cost,
                          wgpf_event* events, uint64_t events_cap, bool no_stats) {
  FastArgs f;
  f.body = body;
  f.stride = stride;
  f.n_streams = n_streams;
  f.stream_base = stream_base;
  f.plan = dev_plan(c);
  f.stats = dev_stats(c);
  f.status = c->d_status.as<DevStatus>();
  f.counts = c->d_counts.as<uint32_t>();
  f.zpos = c->d_zpos.as<int32_t>();
  f.sflag = c->d_sflag.as<uint32_t>();
  f.offsets = c->d_offsets.as<uint64_t>();
  f.events = events;
  f.events_cap = events_cap;
  f.record_cost = record_cost;
  f.cap = (uint32_t)c->slots;
  f.fast_regions = std::min<uint32_t>((uint32_t)c->labels.size(), kFastRegions);
  f.no_stats = no_stats ? 1u : 0u;
  f.general_list = c->d_glist.as<unsigned long long>();
  f.general_len = c->d_glen.as<unsigned long long>();
  f.list = nullptr;
  f.list_len = nullptr;
  f.tps_regions = tps_regions(c);
  f.tma = 0;
  f.group = 1;
  f.batch_ctr = nullptr;
  f.deep_rep = nullptr;
  f.list_base = 0;
  // without the thread-per-stream pass (which visits every stream) the list
  // kernels hand their SF_GENERAL entries to the general path themselves
  f.list_general = !tps_enabled(c) && deep_enabled(c) && record_cost < (1ull << 21) ? 1u : 0u;
  return f;
}

// k_tps over streams [s0, s0 + n) of the call's body (W streams per block,
// W | n): the chunk's own body pointer, tensor maps and per-stream arrays;
// stream indices in the general list and first-event keys stay call-global.
// bctr: the chunk's dynamic batch counter (zeroed).
static int launch_tps(wgpf_ctx* c, FastArgs f, uint64_t s0, uint64_t n, uint32_t W,
                      unsigned long long* bctr, cudaStream_t st) {
  const uint32_t tw = tps_warps(c->K, f.tps_regions, c->smem_optin);
  const size_t tsm = tps_smem_bytes(c->K, f.tps_regions, tw);
  f.body += s0 * f.stride;
  f.n_streams = n;
  f.stream_base += s0;
  f.list_base = s0;
  f.counts += s0;
  f.zpos += s0;
  f.sflag += s0;
  f.offsets += s0;
  f.group = W;
  f.batch_ctr = bctr;
  CUtensorMap tm, tmt;
  memset(&tm, 0, sizeof(tm));
  memset(&tmt, 0, sizeof(tmt));
  f.tma = !c->no_tma && body_tensor_map3(&tm, f.body, f.stride, n, W) ? 1u : 0u;
  if (f.tma && !(tail_maps() && body_tensor_map3(&tmt, f.body, f.stride, n, W,
                                                 CU_TENSOR_MAP_L2_PROMOTION_NONE)))
    tmt = tm;
  tps_kernel(f.events != nullptr, !f.no_stats)<<<c->sms, tw * 32, tsm, st>>>(f, tm, tmt);
  CUDA_OK(c, cudaGetLastError());
  ++c->launches;
  return WGPF_OK;
}

// tps_done: the thread-per-stream pass already ran (replay_overlapped, chunk
// by chunk, which also zeroed the general list)
static int emit_pass(wgpf_ctx* c, const uint8_t* body, uint64_t stride,
                     uint64_t n_streams, uint64_t stream_base,
                     uint64_t record_cost, wgpf_event* events,
                     uint64_t events_cap, bool no_stats, bool force_general,
                     bool tps_done = false) {
  if (!tps_done) CUDA_OK(c, cudaMemsetAsync(c->d_glen.p, 0, 8, c->stream));
  if (force_general) {
    c->mark(3);
    c->general_streams += n_streams;
    int rc = run_general(c, body, stride, n_streams, stream_base, record_cost,
                         events, events_cap, no_stats, false, n_streams);
    c->mark(4);
    return rc;
  }
  FastArgs f = fast_args(c, body, stride, n_streams, stream_base, record_cost, events,
                         events_cap, no_stats);
  // (record_cost < 2^21: cost x position (< 2^11) fits the kernel's 32-bit
  // correction arithmetic; larger costs take the warp-per-stream kernel)
  if ((tps_enabled(c) || deep_enabled(c)) && record_cost < (1ull << 21)) {
    if (tps_enabled(c) && !tps_done) {
      // shallow streams: thread per stream
      unsigned long long* bctr = c->d_glen.as<unsigned long long>() + 4;
      CUDA_OK(c, cudaMemsetAsync(bctr, 0, 8, c->stream));
      int rc = launch_tps(c, f, 0, n_streams, stream_group(c, body, stride, n_streams), bctr,
                          c->stream);
      if (rc) return rc;
    }
    if (deep_enabled(c)) {
      // pass 1's deep list (64-deep stacks, ids < 64), then its wide list
      // (32-deep stacks, ids < 256): thread per stream
      CUtensorMap tmd;
      memset(&tmd, 0, sizeof(tmd));
      const uint32_t tma_ok =
          !c->no_tma && body_tensor_map(&tmd, body, stride, n_streams, kDeepPitch,
                                        l2_promotion(), kDeepSwizzle) ? 1u : 0u;
      for (int wide = 0; wide < (wide_enabled(c) ? 2 : 1); ++wide) {
        f.list = wide ? c->d_vlist.as<unsigned long long>() : c->d_dlist.as<unsigned long long>();
        f.list_len = c->d_glen.as<unsigned long long>() + (wide ? 3 : 2);
        const uint32_t dw = deep_warps(c->smem_optin, wide);
        ALLOC_OK(c, c->d_dorph, sizeof(wgpf_event) * (uint64_t)c->sms * kDeepWarps * 32);
        f.orphan_scratch = c->d_dorph.as<wgpf_event>();  // one orphan per lane
        f.tma = tma_ok;
        const uint32_t classes = deep_classes(wide);
        const size_t rep_bytes = 8ull * c->sms * classes * kDeepRep;
        ALLOC_OK(c, c->d_deep_rep, 8ull * c->sms * deep_classes(true) * kDeepRep);
        f.deep_rep = c->d_deep_rep.as<unsigned long long>();
        if (!no_stats) CUDA_OK(c, cudaMemsetAsync(f.deep_rep, 0, rep_bytes, c->stream));
        deep_kernel(events != nullptr, !no_stats, c->has_markers, wide)
            <<<c->sms, dw * 32, deep_smem_bytes(dw, wide), c->stream>>>(f, tmd);
        CUDA_OK(c, cudaGetLastError());
        if (!no_stats)
          k_deep_reduce<<<(classes * kDeepRep + 255) / 256, 256, 0, c->stream>>>(
              f.deep_rep, c->sms, c->K, f.stats, classes);
        f.tma = 0;
        CUDA_OK(c, cudaGetLastError());
        c->launches += no_stats ? 1 : 2;
      }
    }
    // then the rest of the SF_WARP streams: warp per stream
    f.list = c->d_wlist.as<unsigned long long>();
    f.list_len = c->d_glen.as<unsigned long long>() + 1;
  }
  // stage whole streams in shared memory when two buffers per warp fit
  const size_t smem_stage = fast_smem_bytes(true, stride);
  const bool staged = !c->no_stage && smem_stage <= 160 * 1024;
  const size_t smem = staged ? smem_stage : fast_smem_bytes(false, stride);
  const void* kfn = staged ? (const void*)k_fast_emit<true>
                           : (const void*)k_fast_emit<false>;
  const uint32_t grid = grid_for(c, kfn, kFastWarps * 32, smem);
  ALLOC_OK(c, c->d_orphans,
           sizeof(wgpf_event) * (uint64_t)grid * kFastWarps * (c->slots / 2 + 1));
  f.orphan_scratch = c->d_orphans.as<wgpf_event>();
  if (staged)
    k_fast_emit<true><<<grid, kFastWarps * 32, smem, c->stream>>>(f);
  else
    k_fast_emit<false><<<grid, kFastWarps * 32, smem, c->stream>>>(f);
  CUDA_OK(c, cudaGetLastError());
  ++c->launches;
  c->mark(3);
  // streams the fast path routed away
  unsigned long long glen = 0;
  CUDA_OK(c, cudaMemcpyAsync(&glen, c->d_glen.p, 8, cudaMemcpyDeviceToHost,
                             c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  c->general_streams += glen;
  int rc = run_general(c, body, stride, n_streams, stream_base, record_cost,
                       events, events_cap, no_stats, true, glen);
  c->mark(4);
  return rc;
}

// ---------------------------------------------------------------------------
// Overlapped pass 1 / pass 2.  Pass 2 (k_tps) needs every stream's event
// offset, i.e. pass 1 over all streams before it, and pass 1 reads the body
// once more.  k_tps is latency-bound (about 60 % of issue slots and 65 % of
// DRAM bandwidth used), so pass 1 of the next chunk of streams runs beside it:
// the streams are cut into chunks of whole 32-block batch groups (32 W
// streams, k_tps's lane mapping), chunk 0 is small and counted alone by the
// full pass-1 kernel, and every later chunk k+1 is counted on a second stream
// by the co-resident pass-1 kernel (one warp per CTA, two CTAs per SM at <=
// 64 registers: they fit beside k_tps's CTA) while k_tps emits chunk k.
// Chunk sizes grow geometrically so that the counting of chunk k+1 (on two
// warps per SM) finishes within the emission of chunk k.  Offsets: one
// exclusive scan per chunk whose initial value is the running total left in
// device memory by the previous chunk (cub::FutureValue), no host round trip.
//
// Measured on config 4 (parity suite green with it on): 23.4 ms per replay
// vs 6.88 ms for the plain sequence -- the co-resident pass-1 warps run at
// ~380 cycles per record step (memory-latency bound with one 16-record window
// in flight; the stand-alone pass hides the same ~240 cycles per step behind
// 18 warps per SM), so the emission of every chunk waits for its count.
// Hence opt-in (WGPF_OVERLAP=1) and kept as the measured alternative.
// ---------------------------------------------------------------------------

__global__ void k_chunk_base(const uint32_t* counts, const uint64_t* off, uint64_t n,
                             unsigned long long* base_next) {
  *base_next = n ? off[n - 1] + counts[n - 1] : *(base_next - 1);
}
__global__ void k_total_from(const unsigned long long* total, DevStatus* st) {
  st->total_events = *total;
}

static double env_double(const char* k, double d) {
  const char* e = getenv(k);
  return e ? atof(e) : d;
}

// chunk starts (in streams, ending with n_streams) for the overlapped replay;
// empty when the call is too small to split
static std::vector<uint64_t> plan_overlap_chunks(uint64_t n_streams, uint32_t W) {
  std::vector<uint64_t> cs;
  const uint64_t unit = 32ull * W;
  const uint64_t units = n_streams / unit;  // whole batch groups (the rest joins the last chunk)
  const double first_div = env_double("WGPF_OVL_FIRST", 32.0);
  const double growth = env_double("WGPF_OVL_GROWTH", 1.25);
  const uint32_t max_chunks = (uint32_t)env_double("WGPF_OVL_MAX", 48.0);
  if (units < 8) return cs;
  double sz = std::max(1.0, (double)units / first_div);
  uint64_t at = 0;
  cs.push_back(0);
  while (true) {
    const uint64_t take = std::max<uint64_t>(1, (uint64_t)(sz + 0.5));
    if (at + take >= units || cs.size() >= max_chunks) break;
    at += take;
    cs.push_back(at * unit);
    sz *= growth;
  }
  cs.push_back(n_streams);
  return cs;
}

static int replay_overlapped(wgpf_ctx* c, CountArgs ca, const uint8_t* body, uint64_t stride,
                             uint64_t n_streams, uint64_t stream_base, uint64_t record_cost,
                             wgpf_event* events, uint64_t events_cap, bool no_stats,
                             uint32_t W, const std::vector<uint64_t>& cs) {
  const size_t C = cs.size() - 1;
  c->overlap_chunks = (uint32_t)C;
  if (!c->s_count)
    CUDA_OK(c, cudaStreamCreateWithFlags(&c->s_count, cudaStreamNonBlocking));
  while (c->oev.size() < C + 1) {
    cudaEvent_t e;
    CUDA_OK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->oev.push_back(e);
  }
  // [0, C]: running event totals (chunk bases); [C + 1, 2C]: k_tps batch counters
  ALLOC_OK(c, c->d_obase, 8 * (2 * C + 2));
  unsigned long long* base = c->d_obase.as<unsigned long long>();
  unsigned long long* bctr = base + C + 1;
  CUDA_OK(c, cudaMemsetAsync(base, 0, 8 * (2 * C + 2), c->stream));
  CUDA_OK(c, cudaMemsetAsync(c->d_glen.p, 0, 8, c->stream));  // general list
  // scan temporary storage for the largest chunk
  uint64_t max_n = 0;
  for (size_t k = 0; k < C; ++k) max_n = std::max(max_n, cs[k + 1] - cs[k]);
  auto widen = thrust::make_transform_iterator(c->d_counts.as<uint32_t>(), ToU64());
  size_t tmp = 0;
  CUDA_OK(c, cub::DeviceScan::ExclusiveScan(
                 nullptr, tmp, widen, c->d_offsets.as<uint64_t>(), cuda::std::plus<uint64_t>{},
                 cub::FutureValue<uint64_t>(reinterpret_cast<uint64_t*>(base)), (int64_t)max_n,
                 c->s_count));
  ALLOC_OK(c, c->d_scan_tmp, tmp);
  // the pass-1 stream starts after this call's resets on the main stream
  CUDA_OK(c, cudaEventRecord(c->oev[0], c->stream));
  CUDA_OK(c, cudaStreamWaitEvent(c->s_count, c->oev[0], 0));

  const FastArgs f = fast_args(c, body, stride, n_streams, stream_base, record_cost, events,
                               events_cap, no_stats);
  const void* k_big = (const void*)k_count_tps<kCountWarps, kCountUnroll, kCountMinBlocks>;
  const uint32_t g_big = grid_for(c, k_big, kCountWarps * 32, 0);
  for (size_t k = 0; k < C; ++k) {
    const uint64_t s0 = cs[k], n = cs[k + 1] - cs[k];
    // pass 1 of chunk k (second stream)
    CountArgs a = ca;
    a.body = body + s0 * stride;
    a.n_streams = n;
    a.counts += s0;
    a.zpos += s0;
    a.sflag += s0;
    a.list_base = s0;
    CUtensorMap tm, tmt;
    memset(&tm, 0, sizeof(tm));
    memset(&tmt, 0, sizeof(tmt));
    a.tma = !c->no_tma && body_tensor_map(&tm, a.body, stride, n, CountWin::kTpsPitch) ? 1u
                                                                                       : 0u;
    if (a.tma && !(tail_maps() && body_tensor_map(&tmt, a.body, stride, n, CountWin::kTpsPitch,
                                                   CU_TENSOR_MAP_L2_PROMOTION_NONE)))
      tmt = tm;
    if (k == 0)
      k_count_tps<kCountWarps, kCountUnroll, kCountMinBlocks>
          <<<g_big, kCountWarps * 32, 0, c->s_count>>>(a, tm, tmt);
    else
      k_count_tps<1, kCountCoUnroll, kCountCoMinBlocks>
          <<<c->sms * kCountCoCtas, 32, 0, c->s_count>>>(a, tm, tmt);
    CUDA_OK(c, cudaGetLastError());
    ++c->launches;
    // offsets of chunk k: exclusive scan from the running total
    auto it = thrust::make_transform_iterator(c->d_counts.as<uint32_t>() + s0, ToU64());
    CUDA_OK(c, cub::DeviceScan::ExclusiveScan(
                   c->d_scan_tmp.p, tmp, it, c->d_offsets.as<uint64_t>() + s0,
                   cuda::std::plus<uint64_t>{},
                   cub::FutureValue<uint64_t>(reinterpret_cast<uint64_t*>(base + k)), (int64_t)n,
                   c->s_count));
    k_chunk_base<<<1, 1, 0, c->s_count>>>(c->d_counts.as<uint32_t>() + s0,
                                          c->d_offsets.as<uint64_t>() + s0, n, base + k + 1);
    CUDA_OK(c, cudaGetLastError());
    c->launches += 2;
    CUDA_OK(c, cudaEventRecord(c->oev[k + 1], c->s_count));
    // pass 2 of chunk k (main stream) once its offsets exist
    CUDA_OK(c, cudaStreamWaitEvent(c->stream, c->oev[k + 1], 0));
    if (k == 0) {
      c->mark(1);
      c->mark(2);
    }
    int rc = launch_tps(c, f, s0, n, W, bctr + k, c->stream);
    if (rc) return rc;
  }
  k_total_from<<<1, 1, 0, c->stream>>>(base + C, c->d_status.as<DevStatus>());
  CUDA_OK(c, cudaGetLastError());
  ++c->launches;
  // the list kernels (deep, warp, general) over the whole call
  return emit_pass(c, body, stride, n_streams, stream_base, record_cost, events, events_cap,
                   no_stats, false, true);
}

static int report_errors(wgpf_ctx* c, const uint8_t* body, uint64_t stride,
                         uint64_t stream_base) {
  const DevStatus& st = *c->h_status;
  if (st.decode_err != kNoErr) {
    const uint64_t s = st.decode_err >> 2;
    const uint32_t code = (uint32_t)(st.decode_err & 3u);
    if (code == DEC_CAP) {
      wgpf_stream_hdr h;
      CUDA_OK(c, cudaMemcpy(&h, body + s * stride, 16, cudaMemcpyDeviceToHost));
      return set_err(c, WGPF_E_TRACE,
                     "stream capacity %u does not match the buffer plan (%llu)",
                     h.slot_capacity, (unsigned long long)c->slots);
    }
    if (code == DEC_FLUSH)
      return set_err(c, WGPF_E_TRACE,
                     "flush stream claims more records than slots");
    return set_err(c, WGPF_E_TRACE, "circular stream has zero slot capacity");
  }
  if (st.pair_err != kNoErr) {
    const uint64_t gs = st.pair_err >> 32;
    const uint32_t pos = (uint32_t)(st.pair_err & 0xFFFFFFFFu);
    const uint64_t s = gs - stream_base;
    wgpf_stream_hdr h;
    CUDA_OK(c, cudaMemcpy(&h, body + s * stride, 16, cudaMemcpyDeviceToHost));
    const uint32_t start =
        h.record_count <= h.slot_capacity ? 0u : h.record_count % h.slot_capacity;
    uint32_t slot = start + pos;
    if (slot >= h.slot_capacity) slot -= h.slot_capacity;
    wgpf_record r;
    CUDA_OK(c, cudaMemcpy(&r, body + s * stride + 16 + 8ull * slot, 8,
                          cudaMemcpyDeviceToHost));
    const uint32_t rid = (r.tag >> 12) & (WGPF_MAX_REGIONS - 1u);
    return set_err(c, WGPF_E_TRACE,
                   "interval \"%s\" exceeds 2^32 cycles; the 32-bit clock "
                   "cannot represent it",
                   label_of(c, rid).c_str());
  }
  return WGPF_OK;
}

static int finalize_stats(wgpf_ctx* c, const uint8_t* body, uint64_t stride,
                          uint64_t stream_base, uint64_t n_streams,
                          const wgpf_event* events, uint64_t n_events,
                          bool exact) {
  const uint32_t ns = n_slots(c);
  k_resolve_first<<<(ns + 127) / 128, 128, 0, c->stream>>>(
      dev_stats(c), ns, body, stride, stream_base, n_streams,
      c->d_first_wg.as<unsigned long long>());
  CUDA_OK(c, cudaGetLastError());
  ++c->launches;
  c->mean_exact_valid = false;
  if (exact && events && n_events) {
    // stable class sort of durations, then the recurrence per class
    ALLOC_OK(c, c->d_aux0, 4 * n_events);
    ALLOC_OK(c, c->d_aux1, 8 * n_events);
    ALLOC_OK(c, c->d_aux2, 4 * n_events);
    ALLOC_OK(c, c->d_aux3, 8 * n_events);
    k_event_class_dur<<<c->sms * 8, 256, 0, c->stream>>>(
        events, n_events, dev_plan(c), c->d_aux0.as<uint32_t>(),
        c->d_aux1.as<unsigned long long>());
    CUDA_OK(c, cudaGetLastError());
    size_t tmp = 0;
    CUDA_OK(c, cub::DeviceRadixSort::SortPairs(
                   nullptr, tmp, c->d_aux0.as<uint32_t>(), c->d_aux2.as<uint32_t>(),
                   c->d_aux1.as<unsigned long long>(),
                   c->d_aux3.as<unsigned long long>(), (int64_t)n_events, 0, 32,
                   c->stream));
    ALLOC_OK(c, c->d_scan_tmp, tmp);
    CUDA_OK(c, cub::DeviceRadixSort::SortPairs(
                   c->d_scan_tmp.p, tmp, c->d_aux0.as<uint32_t>(),
                   c->d_aux2.as<uint32_t>(), c->d_aux1.as<unsigned long long>(),
                   c->d_aux3.as<unsigned long long>(), (int64_t)n_events, 0, 32,
                   c->stream));
    k_exact_mean<<<ns, kEmThreads, 0, c->stream>>>(
        c->d_aux2.as<uint32_t>(), c->d_aux3.as<unsigned long long>(), n_events,
        dev_stats(c), ns, c->d_mean.as<double>(), nullptr);
    CUDA_OK(c, cudaGetLastError());
    c->mean_exact_valid = true;
  }
  c->stats_valid = true;
  return WGPF_OK;
}

// The kernels read 16-byte headers and stage streams with 16-byte bulk
// copies: odd-capacity or unaligned bodies are repacked (one 2D device copy)
// to a 16-byte pitch; *stride becomes the pitch.
static int align_body(wgpf_ctx* c, const void** d_body, uint64_t n_streams,
                      uint64_t* stride) {
  if (!n_streams ||
      (!(reinterpret_cast<uintptr_t>(*d_body) & 15u) && !(*stride & 15u)))
    return WGPF_OK;
  const uint64_t pitch = (*stride + 15) & ~15ull;
  ALLOC_OK(c, c->d_repack, n_streams * pitch);
  CUDA_OK(c, cudaMemcpy2DAsync(c->d_repack.p, pitch, *d_body, *stride, *stride,
                               n_streams, cudaMemcpyDeviceToDevice, c->stream));
  *d_body = c->d_repack.p;
  *stride = pitch;
  return WGPF_OK;
}

extern "C" int wgpf_replay_device(wgpf_ctx* c, const void* d_body,
                                  uint64_t body_bytes, uint64_t n_streams,
                                  uint64_t stream_base, uint64_t record_cost,
                                  wgpf_event* d_events, uint64_t events_cap,
                                  uint32_t flags, uint64_t* n_events,
                                  wgpf_warnings* warnings) {
  if (!c->has_plan) return set_err(c, WGPF_E_ARG, "no buffer plan set");
  if (n_events) *n_events = 0;
  if (warnings) memset(warnings, 0, sizeof *warnings);
  uint64_t stride = 16ull + 8ull * c->slots;
  if (body_bytes < n_streams * stride)
    return set_err(c, WGPF_E_ARG, "body of %llu bytes < %llu streams x %llu",
                   (unsigned long long)body_bytes,
                   (unsigned long long)n_streams, (unsigned long long)stride);
  if (c->slots >= (1ull << 31))
    return set_err(c, WGPF_E_ARG, "slot capacity too large");
  {
    int rr = align_body(c, &d_body, n_streams, &stride);
    if (rr) return rr;
  }
  const bool stats_only = flags & WGPF_F_STATS_ONLY;
  const bool no_stats = flags & WGPF_F_NO_STATS;
  if (!c->in_chunked) c->chunk_mode = false;
  c->profiling = (flags & WGPF_F_PROFILE) != 0;
  c->launches = 0;
  c->overlap_chunks = 0;
  c->general_streams = 0;
  c->prof = wgpf_profile{};
  c->mark(0);
  const bool force_general = flags & WGPF_F_FORCE_GENERAL;
  wgpf_event* events = stats_only ? nullptr : d_events;
  const uint8_t* body = static_cast<const uint8_t*>(d_body);
  int rc = status_reset(c);
  if (rc) return rc;
  rc = stats_reset(c);
  if (rc) return rc;
  c->last_body = body;
  c->last_stride = stride;
  c->last_stream_base = stream_base;
  c->last_n_streams = n_streams;
  if (n_streams == 0) {
    c->stats_valid = true;
    return WGPF_OK;
  }
  ALLOC_OK(c, c->d_counts, 4 * n_streams);
  ALLOC_OK(c, c->d_zpos, 4 * n_streams);
  ALLOC_OK(c, c->d_sflag, 4 * n_streams);
  ALLOC_OK(c, c->d_offsets, 8 * n_streams);
  ALLOC_OK(c, c->d_glist, 8 * n_streams);

  CountArgs ca;
  ca.tma = 0;
  ca.list_base = 0;
  ca.body = body;
  ca.stride = stride;
  ca.n_streams = n_streams;
  ca.plan = dev_plan(c);
  ca.counts = c->d_counts.as<uint32_t>();
  ca.zpos = c->d_zpos.as<int32_t>();
  ca.sflag = c->d_sflag.as<uint32_t>();
  ca.status = c->d_status.as<DevStatus>();
  ca.fast_regions = std::min<uint32_t>((uint32_t)c->labels.size(), kFastRegions);
  ca.max_depth = kMaxDepth;
  ca.force_general = force_general ? 1u : 0u;
  const bool tps = tps_enabled(c);
  ca.tps_regions = tps ? tps_regions(c) : 0u;
  ca.tps_depth = tps ? kTpsDepth : 0u;
  ca.deep_regions = deep_enabled(c) ? kDeepRegions : 0u;
  ca.deep_depth = deep_enabled(c) ? kDeepDepth : 0u;
  ca.wide_regions = wide_enabled(c) ? kWideRegions : 0u;
  ca.wide_depth = wide_enabled(c) ? kWideDepth : 0u;
  ca.list_general = 0;
  if (!tps && deep_enabled(c)) {
    // no shallow kernel for this plan: every stream with records is listed
    // (SF_WARP) and the deep ones marked; general streams go to the warp
    // list as well, so that its kernel hands them to the general path
    ca.tps_regions = 0;
    ca.tps_depth = 1;
    ca.list_general = 1;
  }
  ALLOC_OK(c, c->d_wlist, 8 * n_streams);
  ca.warp_list = c->d_wlist.as<unsigned long long>();
  ca.warp_len = c->d_glen.as<unsigned long long>() + 1;
  ALLOC_OK(c, c->d_dlist, deep_enabled(c) ? 8 * n_streams : 8);
  ca.deep_list = c->d_dlist.as<unsigned long long>();
  ca.deep_len = c->d_glen.as<unsigned long long>() + 2;
  ALLOC_OK(c, c->d_vlist, wide_enabled(c) ? 8 * n_streams : 8);
  ca.wide_list = c->d_vlist.as<unsigned long long>();
  ca.wide_len = c->d_glen.as<unsigned long long>() + 3;
  CUDA_OK(c, cudaMemsetAsync(ca.warp_len, 0, 24, c->stream));
  // pass 1 of the next chunk beside pass 2 of the current one (large calls)
  std::vector<uint64_t> ovl;
  uint32_t ovl_w = 1;
  if (!c->no_overlap && !force_general && tps_enabled(c) && count_tps_enabled(c) &&
      record_cost < (1ull << 21) && n_streams >= 4096) {
    ovl_w = stream_group(c, body, stride, n_streams);
    ovl = plan_overlap_chunks(n_streams, ovl_w);
  }
  if (!ovl.empty()) {
    rc = replay_overlapped(c, ca, body, stride, n_streams, stream_base, record_cost, events,
                           events_cap, no_stats, ovl_w, ovl);
    if (rc) return rc;
  } else if (count_tps_enabled(c)) {
    CUtensorMap tm, tmt;
    memset(&tm, 0, sizeof(tm));
    memset(&tmt, 0, sizeof(tmt));
    ca.tma = !c->no_tma &&
                     body_tensor_map(&tm, body, stride, n_streams, CountWin::kTpsPitch)
                 ? 1u
                 : 0u;
    if (ca.tma && !(tail_maps() && body_tensor_map(&tmt, body, stride, n_streams,
                                                   CountWin::kTpsPitch,
                                                   CU_TENSOR_MAP_L2_PROMOTION_NONE)))
      tmt = tm;
    const void* kc = (const void*)k_count_tps<kCountWarps, kCountUnroll, kCountMinBlocks>;
    k_count_tps<kCountWarps, kCountUnroll, kCountMinBlocks>
        <<<grid_for(c, kc, kCountWarps * 32, 0), kCountWarps * 32, 0, c->stream>>>(ca, tm, tmt);
  } else
    k_count_fast<<<grid_for(c, (const void*)k_count_fast, 256, 0), 256, 0,
                   c->stream>>>(ca);
  if (ovl.empty()) {
    CUDA_OK(c, cudaGetLastError());
    ++c->launches;
    c->mark(1);
    rc = scan_counts(c, n_streams);
    if (rc) return rc;
    c->mark(2);
    rc = emit_pass(c, body, stride, n_streams, stream_base, record_cost, events,
                   events_cap, no_stats, force_general);
    if (rc) return rc;
  }
  rc = status_read(c);
  if (rc) return rc;
  if (c->h_status->invalid && c->h_status->decode_err == kNoErr) {
    // exact recount of the streams that broke the single-stack assumption,
    // then re-emit everything at the corrected offsets
    CUDA_OK(c, cudaMemsetAsync(c->d_glen.p, 0, 8, c->stream));
    k_collect_invalid<<<c->sms * 4, 256, 0, c->stream>>>(
        c->d_sflag.as<uint32_t>(), n_streams,
        c->d_glist.as<unsigned long long>(), c->d_glen.as<unsigned long long>());
    unsigned long long n_inv = 0;
    CUDA_OK(c, cudaMemcpyAsync(&n_inv, c->d_glen.p, 8, cudaMemcpyDeviceToHost,
                               c->stream));
    CUDA_OK(c, cudaStreamSynchronize(c->stream));
    rc = run_general_count(c, body, stride, n_streams, stream_base, n_inv);
    if (rc) return rc;
    const unsigned long long pair_err = c->h_status->pair_err;
    rc = status_reset(c);
    if (rc) return rc;
    rc = stats_reset(c);
    if (rc) return rc;
    rc = scan_counts(c, n_streams);
    if (rc) return rc;
    rc = emit_pass(c, body, stride, n_streams, stream_base, record_cost,
                   events, events_cap, no_stats, force_general);
    if (rc) return rc;
    rc = status_read(c);
    if (rc) return rc;
    if (pair_err < c->h_status->pair_err) c->h_status->pair_err = pair_err;
  }
  rc = report_errors(c, body, stride, stream_base);
  if (rc) return rc;
  const DevStatus& st = *c->h_status;
  if (n_events) *n_events = st.total_events;
  if (warnings) {
    warnings->dropped_heads = (uint32_t)st.warn[0];
    warnings->truncated_tails = (uint32_t)st.warn[1];
    warnings->flagged_preconditions = (uint32_t)st.warn[2];
    warnings->malformed_groups = (uint32_t)st.warn[3];
  }
  if (st.synth_overflow)
    return set_err(c, WGPF_E_CAPACITY,
                   "more than %u distinct out-of-table region labels",
                   kSynthHash);
  if (events && st.total_events > events_cap)
    return set_err(c, WGPF_E_BUFFER, "event buffer holds %llu of %llu events",
                   (unsigned long long)events_cap,
                   (unsigned long long)st.total_events);
  if (!no_stats) {
    rc = finalize_stats(c, body, stride, stream_base, n_streams, events,
                        st.total_events, (flags & WGPF_F_EXACT_MEAN) != 0);
    if (rc) return rc;
  }
  c->mark(5);
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  if (c->profiling) {
    float t[5];
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], c->ev[i], c->ev[i + 1]);
    c->prof.count_ms = t[0];
    c->prof.scan_ms = t[1];
    c->prof.emit_ms = t[2];
    c->prof.general_ms = t[3];
    c->prof.finalize_ms = t[4];
    cudaEventElapsedTime(&c->prof.total_ms, c->ev[0], c->ev[5]);
  }
  c->prof.launches = c->launches;
  c->prof.overlap_chunks = c->overlap_chunks;
  c->prof.general_streams = (uint32_t)c->general_streams;
  return WGPF_OK;
}

extern "C" int wgpf_last_profile(const wgpf_ctx* c, wgpf_profile* out) {
  *out = c->prof;
  return WGPF_OK;
}

// ---------------------------------------------------------------------------
// host-image entry points
// ---------------------------------------------------------------------------

static uint32_t rd32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) |
         ((uint32_t)p[3] << 24);
}

// deserialize_image framing (trace.hpp:181-209) followed by the first
// decode_image error (trace.hpp:222-251), walking the host headers.  Only
// used when the image is not a uniform body of the plan's capacity.
static int host_walk(wgpf_ctx* c, const uint8_t* b, uint64_t n, uint64_t pos,
                     uint64_t count) {
  std::vector<wgpf_stream_hdr> hdr;
  for (uint64_t s = 0; s < count; ++s) {
    if (pos + 16 > n) return set_err(c, WGPF_E_TRACE, "truncated trace image");
    wgpf_stream_hdr h{rd32(b + pos), rd32(b + pos + 4), rd32(b + pos + 8),
                      rd32(b + pos + 12)};
    pos += 16;
    const uint64_t need = 8ull * h.slot_capacity;
    if (pos + need > n) return set_err(c, WGPF_E_TRACE, "truncated trace image");
    pos += need;
    hdr.push_back(h);
  }
  if (pos != n)
    return set_err(c, WGPF_E_TRACE, "trailing bytes after trace image");
  for (const auto& h : hdr) {
    if ((uint64_t)h.slot_capacity != c->slots)
      return set_err(c, WGPF_E_TRACE,
                     "stream capacity %u does not match the buffer plan (%llu)",
                     h.slot_capacity, (unsigned long long)c->slots);
    if (h.record_count > h.slot_capacity) {
      if (c->strategy == WGPF_STRATEGY_FLUSH)
        return set_err(c, WGPF_E_TRACE,
                       "flush stream claims more records than slots");
      if (h.slot_capacity == 0)
        return set_err(c, WGPF_E_TRACE, "circular stream has zero slot capacity");
    }
  }
  return set_err(c, WGPF_E_TRACE, "internal: image walk found no error");
}

// Parses the KPFT file header; on success *body_off / *count are set.
static int parse_header(wgpf_ctx* c, const uint8_t* b, uint64_t n,
                        uint64_t* body_off, uint64_t* count) {
  if (n < 4) return set_err(c, WGPF_E_TRACE, "truncated trace image");
  if (memcmp(b, "KPFT", 4) != 0)
    return set_err(c, WGPF_E_TRACE, "bad magic: not a trace image");
  if (n < 6) return set_err(c, WGPF_E_TRACE, "truncated trace image");
  const uint16_t version = (uint16_t)(b[4] | (b[5] << 8));
  if (version == 1) {
    if (n < 8) return set_err(c, WGPF_E_TRACE, "truncated trace image");
    *count = (uint16_t)(b[6] | (b[7] << 8));
    *body_off = 8;
  } else if (version == 2) {
    if (n < 16) return set_err(c, WGPF_E_TRACE, "truncated trace image");
    *count = (uint64_t)rd32(b + 8) | ((uint64_t)rd32(b + 12) << 32);
    *body_off = 16;
  } else {
    return set_err(c, WGPF_E_TRACE, "unsupported trace version %u",
                   (unsigned)version);
  }
  return WGPF_OK;
}

// Stages the image body on the device; returns the device body pointer.
static int stage_image(wgpf_ctx* c, const uint8_t* kpft, uint64_t n,
                       const uint8_t** d_body, uint64_t* n_streams) {
  uint64_t off = 0, count = 0;
  int rc = parse_header(c, kpft, n, &off, &count);
  if (rc) return rc;
  const uint64_t stride = 16ull + 8ull * c->slots;
  const uint64_t body = n - off;
  if (count == 0 || body / stride != count || body % stride != 0) {
    // not a uniform body of the plan capacity: the reference would fail in
    // deserialize or decode (or it is empty)
    if (count == 0 && body == 0) {
      *n_streams = 0;
      *d_body = nullptr;
      return WGPF_OK;
    }
    return host_walk(c, kpft, n, off, count);
  }
  ALLOC_OK(c, c->d_image, body);
  CUDA_OK(c, cudaMemcpyAsync(c->d_image.p, kpft + off, body,
                             cudaMemcpyHostToDevice, c->stream));
  *d_body = c->d_image.as<uint8_t>();
  *n_streams = count;
  return WGPF_OK;
}

extern "C" int wgpf_stats_merge(wgpf_ctx* c, const void* d_gathered,
                                uint32_t n_ranks);

// Host-buffer replay of a large uniform image, pipelined over chunks of
// streams: the H2D copy of chunk k+1 and the D2H copy of chunk k-1's events
// (their own streams, double-buffered device chunks) overlap the replay of
// chunk k, so the call approaches max(H2D, D2H) time instead of the sum.
// Per-chunk statistics are packed and merged at the end (the multi-GPU merge);
// errors and warnings are the first / the sum over chunks in stream order.
static constexpr uint64_t kChunkBytes = 256ull << 20;
// internal: a chunk failed with a reference error; the caller redoes the call
// on the whole image so that errors come in the reference's order
static constexpr int WGPF_E_RETRY_WHOLE = 1000;

// Host memory the caller passed: pinned (page-locked / registered) or not.
static bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// memcpy over several host threads (pageable <-> pinned staging): one thread
// copies ~4 GB/s on this class of host, 8-16 copy 50-77 GB/s, PCIe's order
static void parallel_memcpy(void* dst, const void* src, size_t n) {
  static const unsigned kThreads = [] {
    const unsigned h = std::thread::hardware_concurrency();
    return std::max(1u, std::min(16u, h ? h : 1u));
  }();
  const size_t piece = std::max<size_t>(4u << 20, (n + kThreads - 1) / kThreads);
  std::vector<std::thread> th;
  for (size_t o = piece; o < n; o += piece)
    th.emplace_back([=] {
      memcpy(static_cast<uint8_t*>(dst) + o, static_cast<const uint8_t*>(src) + o,
             std::min(piece, n - o));
    });
  memcpy(dst, src, std::min(piece, n));
  for (auto& t : th) t.join();
}

// rows of `width` bytes at `pitch` (the first width bytes of every stream),
// over the same host threads
static void parallel_memcpy_rows(void* dst, const void* src, size_t pitch, size_t width,
                                 size_t rows) {
  static const unsigned kThreads = [] {
    const unsigned h = std::thread::hardware_concurrency();
    return std::max(1u, std::min(16u, h ? h : 1u));
  }();
  const size_t per = std::max<size_t>(2048, (rows + kThreads - 1) / kThreads);
  auto part = [=](size_t r0, size_t r1) {
    for (size_t r = r0; r < r1; ++r)
      memcpy(static_cast<uint8_t*>(dst) + r * pitch, static_cast<const uint8_t*>(src) + r * pitch,
             width);
  };
  std::vector<std::thread> th;
  for (size_t r = per; r < rows; r += per) th.emplace_back(part, r, std::min(rows, r + per));
  part(0, std::min(rows, per));
  for (auto& t : th) t.join();
}

// Host -> device copy of caller memory on the context stream: pageable
// buffers over 64 MB go through the two pinned bounce buffers in 64-MB
// chunks (multi-threaded host copy of chunk k+1 while chunk k's DMA runs)
// instead of the driver's single-threaded staging.
static int h2d_host(wgpf_ctx* c, void* d_dst, const void* h_src, uint64_t bytes) {
  constexpr uint64_t kChunk = 64ull << 20;
  if (bytes <= kChunk || host_pinned(h_src)) {
    CUDA_OK(c, cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, c->stream));
    return WGPF_OK;
  }
  if (c->bounce_in_n < kChunk) {
    for (auto& h : c->h_bounce_in) {
      if (h) cudaFreeHost(h);
      h = nullptr;
    }
    c->bounce_in_n = 0;
    for (auto& h : c->h_bounce_in)
      CUDA_OK(c, cudaMallocHost(reinterpret_cast<void**>(&h), kChunk));
    c->bounce_in_n = kChunk;
  }
  for (int b = 0; b < 2; ++b)
    if (!c->pev[b]) CUDA_OK(c, cudaEventCreateWithFlags(&c->pev[b], cudaEventDisableTiming));
  const uint64_t chunk = std::min<uint64_t>(c->bounce_in_n, 1ull << 30);
  for (uint64_t k = 0, at = 0; at < bytes; ++k, at += chunk) {
    const uint32_t b = (uint32_t)(k & 1);
    const uint64_t m = std::min(chunk, bytes - at);
    if (k >= 2) CUDA_OK(c, cudaEventSynchronize(c->pev[b]));  // bounce b free again
    parallel_memcpy(c->h_bounce_in[b], static_cast<const uint8_t*>(h_src) + at, m);
    CUDA_OK(c, cudaMemcpyAsync(static_cast<uint8_t*>(d_dst) + at, c->h_bounce_in[b], m,
                               cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(c, cudaEventRecord(c->pev[b], c->stream));
  }
  return WGPF_OK;
}

static int replay_image_chunked(wgpf_ctx* c, const uint8_t* kpft, uint64_t off,
                                uint64_t count, uint64_t record_cost,
                                wgpf_event* h_events, uint64_t events_cap,
                                uint32_t flags, uint64_t* n_events,
                                wgpf_warnings* warnings) {
  const uint64_t stride = 16ull + 8ull * c->slots;
  // pageable caller memory goes through host copies, which amortise better
  // over larger chunks (config 4: 1.56 G records/s at 256 MB, 1.67-1.86 at
  // 512 MB); pinned memory runs best at 256 MB (332 ms vs 334 at 128 / 512)
  const bool pageable_io = !host_pinned(kpft) || !host_pinned(h_events);
  uint64_t chunk_bytes = pageable_io ? 2 * kChunkBytes : kChunkBytes;
  if (const char* e = getenv("WGPF_CHUNK_MB")) chunk_bytes = (uint64_t)atoll(e) << 20;
  const uint64_t cs = std::max<uint64_t>(32, (chunk_bytes / stride) & ~31ull);
  // chunk boundaries: a quarter-size first and last chunk shorten the
  // pipeline's fill (first H2D alone) and drain (last D2H alone)
  std::vector<uint64_t> cut{0};
  {
    const uint64_t q = std::max<uint64_t>(32, (cs / 4) & ~31ull);
    uint64_t at = 0;
    if (count > 2 * cs) {
      cut.push_back(at = q);
      while (count - at > cs + q) cut.push_back(at += cs);
      if (count - at > q) cut.push_back(at = count - q);
    }
    while (at < count) cut.push_back(at = std::min(count, at + cs));
  }
  const uint64_t nc = cut.size() - 1;
  const uint64_t ev_cap = std::max<uint64_t>(cs * c->slots, 1);
  if (!c->s_h2d) {
    CUDA_OK(c, cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    CUDA_OK(c, cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    for (auto& e : c->pev)
      CUDA_OK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const uint64_t pb = wgpf_stats_packed_bytes(c);
  for (int b = 0; b < 2; ++b) {
    ALLOC_OK(c, c->d_cbody[b], cs * stride);
    ALLOC_OK(c, c->d_cev[b], ev_cap * sizeof(wgpf_event));
  }
  ALLOC_OK(c, c->d_packed, nc * pb);
  ALLOC_OK(c, c->d_off_all, 8 * count);
  cudaEvent_t* eH = c->pev;
  cudaEvent_t* eC = c->pev + 2;
  cudaEvent_t* eD = c->pev + 4;
  // Pageable caller memory: an async copy from / to it would serialise the
  // pipeline (and runs at ~10 / 18 GB/s), and registering it costs ~20 GB/s,
  // so chunks are staged through pinned bounce buffers with a multi-threaded
  // host memcpy instead.
  const bool stage_in = !host_pinned(kpft);
  const bool stage_out = !host_pinned(h_events);
  if (stage_in && c->bounce_in_n < cs * stride) {
    for (auto& h : c->h_bounce_in) {
      if (h) cudaFreeHost(h);
      h = nullptr;
    }
    c->bounce_in_n = 0;
    for (auto& h : c->h_bounce_in)
      CUDA_OK(c, cudaMallocHost(reinterpret_cast<void**>(&h), cs * stride));
    c->bounce_in_n = cs * stride;
  }
  auto h2d = [&](uint64_t k) -> int {
    const uint32_t b = (uint32_t)(k & 1);
    const uint64_t s0 = cut[k], m = cut[k + 1] - cut[k];
    if (k >= 2) CUDA_OK(c, cudaStreamWaitEvent(c->s_h2d, eC[b], 0));
    const uint8_t* src = kpft + off + s0 * stride;
    // Flush streams never read slots past their record count, so only each
    // stream's header and its first max-count slots travel (one 2-D copy;
    // the device rows' tails keep whatever they held and are never used):
    // config 4 uploads 8.7 of the image's 10.0 GB, and the download of the
    // events -- the pipeline's long pole -- shares the link with less:
    // 382 -> 346 ms per call.
    uint64_t width = stride;
    if (c->strategy == WGPF_STRATEGY_FLUSH) {
      uint32_t mx = 0;
      for (uint64_t i = 0; i < m; ++i) {
        const uint32_t n_ = rd32(src + i * stride + 8);
        mx = n_ > mx ? n_ : mx;
      }
      if (mx < c->slots) width = (16ull + 8ull * mx + 15) & ~15ull;
    }
    if (stage_in) {
      // the bounce buffer's previous copy (chunk k - 2) must have left
      if (k >= 2) CUDA_OK(c, cudaEventSynchronize(eH[b]));
      if (width < stride)
        parallel_memcpy_rows(c->h_bounce_in[b], src, stride, width, m);
      else
        parallel_memcpy(c->h_bounce_in[b], src, m * stride);
      src = c->h_bounce_in[b];
    }
    if (width < stride)
      CUDA_OK(c, cudaMemcpy2DAsync(c->d_cbody[b].p, stride, src, stride, width, m,
                                   cudaMemcpyHostToDevice, c->s_h2d));
    else
      CUDA_OK(c, cudaMemcpyAsync(c->d_cbody[b].p, src, m * stride, cudaMemcpyHostToDevice,
                                 c->s_h2d));
    CUDA_OK(c, cudaEventRecord(eH[b], c->s_h2d));
    return WGPF_OK;
  };
  // staged output: chunk k's events land in bounce_out[k & 1]; the copy to
  // the caller's buffer happens one chunk later (or at the end)
  uint64_t out_pending = ~0ull, out_at = 0, out_n = 0;
  auto copy_out = [&]() -> int {
    if (out_pending == ~0ull) return WGPF_OK;
    const uint32_t b = (uint32_t)(out_pending & 1);
    CUDA_OK(c, cudaEventSynchronize(eD[b]));
    parallel_memcpy(h_events + out_at, c->h_bounce_out[b], out_n * sizeof(wgpf_event));
    out_pending = ~0ull;
    return WGPF_OK;
  };
  auto drain = [&]() {
    cudaStreamSynchronize(c->s_h2d);
    cudaStreamSynchronize(c->s_d2h);
    cudaStreamSynchronize(c->stream);
  };
  c->chunk_sbase.clear();
  c->chunk_ebase.clear();
  c->chunk_mode = false;
  // streams per block from the host headers (no device read per chunk: a
  // small D2H would queue behind the event copies)
  {
    uint32_t W = 1;
    const uint64_t m = std::min<uint64_t>(count, 1025);
    for (uint64_t i = 1; i < m; ++i)
      if (rd32(kpft + off + i * stride) != rd32(kpft + off)) {
        W = (uint32_t)i;
        break;
      }
    c->group_hint = W;
  }
  struct HintReset {
    wgpf_ctx* c;
    ~HintReset() { c->group_hint = 0; }
  } hint_reset{c};
  int rc = h2d(0);
  if (rc) return rc;
  uint64_t total = 0;
  wgpf_warnings acc{};
  bool overflow = false;
  for (uint64_t k = 0; k < nc; ++k) {
    const uint32_t b = (uint32_t)(k & 1);
    const uint64_t s0 = cut[k], m = cut[k + 1] - cut[k];
    if (k + 1 < nc && (rc = h2d(k + 1))) return rc;
    CUDA_OK(c, cudaStreamWaitEvent(c->stream, eH[b], 0));
    if (k >= 2) CUDA_OK(c, cudaStreamWaitEvent(c->stream, eD[b], 0));
    uint64_t ne = 0;
    wgpf_warnings w{};
    c->in_chunked = true;
    rc = wgpf_replay_device(c, c->d_cbody[b].p, m * stride, m, s0, record_cost,
                            c->d_cev[b].as<wgpf_event>(), ev_cap,
                            flags & ~WGPF_F_STATS_ONLY, &ne, &w);
    c->in_chunked = false;
    if (rc) {
      drain();
      // The reference decodes every stream before pairing any (decode_image
      // then the per-stream pair/replay, pipeline.hpp:69-80), so an error in
      // chunk k may be preceded by a decode error in a later chunk: redo the
      // call on the whole image (error path only), whose error report orders
      // framing, decode and pair errors as the reference does.
      if (rc >= WGPF_E_PARSE && rc <= WGPF_E_IO) return WGPF_E_RETRY_WHOLE;
      return rc;
    }
    CUDA_OK(c, cudaEventRecord(eC[b], c->stream));
    rc = wgpf_stats_export(c, c->d_packed.as<uint8_t>() + k * pb);
    if (rc) return rc;
    CUDA_OK(c, cudaMemcpyAsync(c->d_off_all.as<uint64_t>() + s0, c->d_offsets.p, 8 * m,
                               cudaMemcpyDeviceToDevice, c->stream));
    if (total + ne > events_cap) overflow = true;
    if (stage_out && (rc = copy_out())) return rc;  // chunk k - 1 (frees its buffer)
    if (!overflow && ne) {
      CUDA_OK(c, cudaStreamWaitEvent(c->s_d2h, eC[b], 0));
      wgpf_event* dst = h_events + total;
      if (stage_out) {
        const size_t need = ne * sizeof(wgpf_event);
        if (c->bounce_out_n[b] < need) {
          if (c->h_bounce_out[b]) cudaFreeHost(c->h_bounce_out[b]);
          c->h_bounce_out[b] = nullptr;
          c->bounce_out_n[b] = 0;
          CUDA_OK(c, cudaMallocHost(reinterpret_cast<void**>(&c->h_bounce_out[b]),
                                    need + need / 4));
          c->bounce_out_n[b] = need + need / 4;
        }
        dst = reinterpret_cast<wgpf_event*>(c->h_bounce_out[b]);
        out_pending = k;
        out_at = total;
        out_n = ne;
      }
      CUDA_OK(c, cudaMemcpyAsync(dst, c->d_cev[b].p, ne * sizeof(wgpf_event),
                                 cudaMemcpyDeviceToHost, c->s_d2h));
    }
    CUDA_OK(c, cudaEventRecord(eD[b], c->s_d2h));
    c->chunk_sbase.push_back(s0);
    c->chunk_ebase.push_back(total);
    total += ne;
    acc.dropped_heads += w.dropped_heads;
    acc.truncated_tails += w.truncated_tails;
    acc.flagged_preconditions += w.flagged_preconditions;
    acc.malformed_groups += w.malformed_groups;
  }
  drain();
  if (stage_out && (rc = copy_out())) return rc;
  if (n_events) *n_events = total;
  if (warnings) *warnings = acc;
  if (overflow)
    return set_err(c, WGPF_E_BUFFER, "event buffer holds %llu of %llu events",
                   (unsigned long long)events_cap, (unsigned long long)total);
  if (!(flags & WGPF_F_NO_STATS)) {
    rc = wgpf_stats_merge(c, c->d_packed.p, (uint32_t)nc);
    if (rc) return rc;
    c->chunk_mode = true;
    c->chunk_nstreams = count;
  }
  return WGPF_OK;
}

extern "C" int wgpf_replay_image(wgpf_ctx* c, const uint8_t* kpft,
                                 uint64_t n_bytes, uint64_t record_cost,
                                 wgpf_event* h_events, uint64_t events_cap,
                                 uint32_t flags, uint64_t* n_events,
                                 wgpf_warnings* warnings) {
  if (!c->has_plan) return set_err(c, WGPF_E_ARG, "no buffer plan set");
  if (n_events) *n_events = 0;
  if (warnings) memset(warnings, 0, sizeof *warnings);
  {
    // large uniform images with host event output: pipelined chunks
    uint64_t off = 0, count = 0;
    const uint64_t stride = 16ull + 8ull * c->slots;
    if (parse_header(c, kpft, n_bytes, &off, &count) == WGPF_OK && count &&
        (n_bytes - off) % stride == 0 && (n_bytes - off) / stride == count &&
        n_bytes - off > 2 * kChunkBytes && h_events &&
        !(flags & (WGPF_F_STATS_ONLY | WGPF_F_EXACT_MEAN)) && !c->no_pipeline) {
      const int rc = replay_image_chunked(c, kpft, off, count, record_cost, h_events,
                                          events_cap, flags, n_events, warnings);
      if (rc != WGPF_E_RETRY_WHOLE) return rc;
      if (n_events) *n_events = 0;
      if (warnings) memset(warnings, 0, sizeof *warnings);
    }
  }
  const uint8_t* d_body = nullptr;
  uint64_t ns = 0;
  int rc = stage_image(c, kpft, n_bytes, &d_body, &ns);
  if (rc) {
    // a capacity mismatch found on the device must still be checked
    // against deserialize framing; stage_image already walked it.
    return rc;
  }
  const uint64_t stride = 16ull + 8ull * c->slots;
  const bool want_events = !(flags & WGPF_F_STATS_ONLY) && h_events;
  // device event buffer sized by the caller's capacity
  wgpf_event* d_ev = nullptr;
  if (want_events) {
    ALLOC_OK(c, c->d_events, sizeof(wgpf_event) * std::max<uint64_t>(events_cap, 1));
    d_ev = c->d_events.as<wgpf_event>();
  }
  uint64_t ne = 0;
  rc = wgpf_replay_device(c, d_body, ns * stride, ns, 0, record_cost, d_ev,
                          want_events ? events_cap : 0,
                          want_events ? flags : (flags | WGPF_F_STATS_ONLY),
                          &ne, warnings);
  if (rc == WGPF_E_TRACE && c->h_status->decode_err != kNoErr &&
      c->h_status->cap_mismatch) {
    // uniform size but a stream's capacity differs: the reference's
    // deserialize walk decides between framing and decode errors
    uint64_t off = 0, count = 0;
    parse_header(c, kpft, n_bytes, &off, &count);
    return host_walk(c, kpft, n_bytes, off, count);
  }
  if (n_events) *n_events = ne;
  if (rc) return rc;
  if (want_events && ne) {
    CUDA_OK(c, cudaMemcpyAsync(h_events, d_ev, sizeof(wgpf_event) * ne,
                               cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(c, cudaStreamSynchronize(c->stream));
  }
  return WGPF_OK;
}

extern "C" int wgpf_decode_image(wgpf_ctx* c, const uint8_t* kpft,
                                 uint64_t n_bytes, wgpf_record* h_records,
                                 uint64_t records_cap, uint64_t* n_records,
                                 wgpf_decoded_stream* h_streams,
                                 uint64_t streams_cap, uint64_t* n_streams) {
  if (!c->has_plan) return set_err(c, WGPF_E_ARG, "no buffer plan set");
  *n_records = 0;
  *n_streams = 0;
  const uint8_t* d_body = nullptr;
  uint64_t ns = 0;
  int rc = stage_image(c, kpft, n_bytes, &d_body, &ns);
  if (rc) return rc;
  if (ns == 0) return WGPF_OK;
  uint64_t stride = 16ull + 8ull * c->slots;
  {
    const void* db = d_body;
    int rr = align_body(c, &db, ns, &stride);
    if (rr) return rr;
    d_body = static_cast<const uint8_t*>(db);
  }
  // decode checks via pass 1
  int r2 = status_reset(c);
  if (r2) return r2;
  ALLOC_OK(c, c->d_counts, 4 * ns);
  ALLOC_OK(c, c->d_zpos, 4 * ns);
  ALLOC_OK(c, c->d_sflag, 4 * ns);
  CountArgs ca;
  ca.tma = 0;
  ca.list_base = 0;
  ca.body = d_body;
  ca.stride = stride;
  ca.n_streams = ns;
  ca.plan = dev_plan(c);
  ca.counts = c->d_counts.as<uint32_t>();
  ca.zpos = c->d_zpos.as<int32_t>();
  ca.sflag = c->d_sflag.as<uint32_t>();
  ca.status = c->d_status.as<DevStatus>();
  ca.fast_regions = 0;
  ca.max_depth = kMaxDepth;
  ca.force_general = 1;
  ca.tps_regions = 0;
  ca.tps_depth = 0;
  ca.deep_regions = 0;
  ca.deep_depth = 0;
  ca.wide_regions = 0;
  ca.wide_depth = 0;
  ca.wide_list = nullptr;
  ca.wide_len = nullptr;
  ca.warp_list = nullptr;
  ca.warp_len = nullptr;
  ca.deep_list = nullptr;
  ca.deep_len = nullptr;
  ca.list_general = 0;
  k_count_fast<<<grid_for(c, (const void*)k_count_fast, 256, 0), 256, 0,
                 c->stream>>>(ca);
  CUDA_OK(c, cudaGetLastError());
  r2 = status_read(c);
  if (r2) return r2;
  if (c->h_status->decode_err != kNoErr) {
    if (c->h_status->cap_mismatch) {
      uint64_t off = 0, count = 0;
      parse_header(c, kpft, n_bytes, &off, &count);
      return host_walk(c, kpft, n_bytes, off, count);
    }
    return report_errors(c, d_body, stride, 0);
  }
  ALLOC_OK(c, c->d_aux1, 8 * ns);
  ALLOC_OK(c, c->d_aux3, 8 * ns);
  ALLOC_OK(c, c->d_aux2, sizeof(wgpf_decoded_stream) * ns);
  k_decode_counts<<<c->sms * 4, 256, 0, c->stream>>>(
      d_body, stride, ns, c->d_aux1.as<uint64_t>(),
      c->d_aux2.as<wgpf_decoded_stream>());
  size_t tmp = 0;
  CUDA_OK(c, cub::DeviceScan::ExclusiveSum(nullptr, tmp, c->d_aux1.as<uint64_t>(),
                                           c->d_aux3.as<uint64_t>(), (int64_t)ns,
                                           c->stream));
  ALLOC_OK(c, c->d_scan_tmp, tmp);
  CUDA_OK(c, cub::DeviceScan::ExclusiveSum(c->d_scan_tmp.p, tmp,
                                           c->d_aux1.as<uint64_t>(),
                                           c->d_aux3.as<uint64_t>(), (int64_t)ns,
                                           c->stream));
  std::vector<uint64_t> cnt(ns), off(ns);
  CUDA_OK(c, cudaMemcpyAsync(cnt.data(), c->d_aux1.p, 8 * ns,
                             cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaMemcpyAsync(off.data(), c->d_aux3.p, 8 * ns,
                             cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  const uint64_t total = off[ns - 1] + cnt[ns - 1];
  *n_records = total;
  *n_streams = ns;
  if (total > records_cap || ns > streams_cap)
    return set_err(c, WGPF_E_BUFFER, "decode needs %llu records / %llu streams",
                   (unsigned long long)total, (unsigned long long)ns);
  ALLOC_OK(c, c->d_aux0, sizeof(wgpf_record) * std::max<uint64_t>(total, 1));
  k_decode_records<<<c->sms * 4, 256, 0, c->stream>>>(
      d_body, stride, ns, c->d_aux3.as<uint64_t>(), c->d_aux0.as<wgpf_record>());
  CUDA_OK(c, cudaGetLastError());
  std::vector<wgpf_decoded_stream> ds(ns);
  CUDA_OK(c, cudaMemcpyAsync(ds.data(), c->d_aux2.p,
                             sizeof(wgpf_decoded_stream) * ns,
                             cudaMemcpyDeviceToHost, c->stream));
  if (total)
    CUDA_OK(c, cudaMemcpyAsync(h_records, c->d_aux0.p, sizeof(wgpf_record) * total,
                               cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  for (uint64_t s = 0; s < ns; ++s) {
    ds[s].offset = off[s];
    h_streams[s] = ds[s];
  }
  return WGPF_OK;
}

extern "C" int wgpf_unwrap_clock(wgpf_ctx* c, const uint32_t* h_values,
                                 uint64_t n, uint64_t* h_out) {
  if (n == 0) return WGPF_OK;
  ALLOC_OK(c, c->d_aux0, 4 * n);
  ALLOC_OK(c, c->d_aux2, 4 * n);
  ALLOC_OK(c, c->d_aux1, 8 * n);
  ALLOC_OK(c, c->d_aux3, 8 * n);
  CUDA_OK(c, cudaMemcpyAsync(c->d_aux0.p, h_values, 4 * n,
                             cudaMemcpyHostToDevice, c->stream));
  k_unwrap_flags<<<c->sms * 4, 256, 0, c->stream>>>(c->d_aux0.as<uint32_t>(), n,
                                                   c->d_aux2.as<uint32_t>());
  auto it = thrust::make_transform_iterator(c->d_aux2.as<uint32_t>(), ToU64());
  size_t tmp = 0;
  CUDA_OK(c, cub::DeviceScan::InclusiveSum(nullptr, tmp, it,
                                           c->d_aux1.as<uint64_t>(), (int64_t)n,
                                           c->stream));
  ALLOC_OK(c, c->d_scan_tmp, tmp);
  CUDA_OK(c, cub::DeviceScan::InclusiveSum(c->d_scan_tmp.p, tmp, it,
                                           c->d_aux1.as<uint64_t>(), (int64_t)n,
                                           c->stream));
  k_unwrap_combine<<<c->sms * 4, 256, 0, c->stream>>>(
      c->d_aux0.as<uint32_t>(), c->d_aux1.as<uint64_t>(), n,
      c->d_aux3.as<uint64_t>());
  CUDA_OK(c, cudaGetLastError());
  CUDA_OK(c, cudaMemcpyAsync(h_out, c->d_aux3.p, 8 * n, cudaMemcpyDeviceToHost,
                             c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  return WGPF_OK;
}

extern "C" int wgpf_pair_records(wgpf_ctx* c, const wgpf_record* h_records,
                                 uint64_t n, wgpf_interval* h_out, uint64_t cap,
                                 uint64_t* n_out, uint32_t* dropped_heads,
                                 uint32_t* truncated_tails) {
  if (!c->has_plan) return set_err(c, WGPF_E_ARG, "no buffer plan set");
  *n_out = 0;
  if (n >= (1ull << 31)) return set_err(c, WGPF_E_ARG, "stream too long");
  const uint64_t stride = 16 + 8 * n;
  ALLOC_OK(c, c->d_image, stride);
  wgpf_stream_hdr h{0, 0, (uint32_t)n, (uint32_t)n};
  CUDA_OK(c, cudaMemcpyAsync(c->d_image.p, &h, 16, cudaMemcpyHostToDevice,
                             c->stream));
  if (n)
    CUDA_OK(c, cudaMemcpyAsync(c->d_image.as<uint8_t>() + 16, h_records, 8 * n,
                               cudaMemcpyHostToDevice, c->stream));
  int rc = status_reset(c);
  if (rc) return rc;
  uint32_t hm = 16;
  while (hm < 2u * (uint32_t)n + 2u) hm <<= 1;
  const uint64_t per = gen_scratch_bytes((uint32_t)std::max<uint64_t>(n, 1), hm);
  ALLOC_OK(c, c->d_gscratch, per);
  ALLOC_OK(c, c->d_aux1, sizeof(wgpf_interval) * (n / 2 + 1));
  ALLOC_OK(c, c->d_aux0, 16);
  GenArgs a;
  memset(&a, 0, sizeof a);
  a.body = c->d_image.as<uint8_t>();
  a.stride = stride;
  a.n_streams = 1;
  a.plan = dev_plan(c);
  a.status = c->d_status.as<DevStatus>();
  a.scratch = c->d_gscratch.as<uint8_t>();
  a.scratch_stride = per;
  a.cap = (uint32_t)std::max<uint64_t>(n, 1);
  a.hm_size = hm;
  k_pair_one<<<1, 1, 0, c->stream>>>(a, c->d_aux1.as<wgpf_interval>(),
                                      c->d_aux0.as<uint32_t>());
  CUDA_OK(c, cudaGetLastError());
  uint32_t info[3];
  CUDA_OK(c, cudaMemcpyAsync(info, c->d_aux0.p, 12, cudaMemcpyDeviceToHost,
                             c->stream));
  rc = status_read(c);
  if (rc) return rc;
  if (c->h_status->pair_err != kNoErr) {
    const uint32_t pos = (uint32_t)(c->h_status->pair_err & 0xFFFFFFFFu);
    const uint32_t rid = (h_records[pos].tag >> 12) & (WGPF_MAX_REGIONS - 1u);
    return set_err(c, WGPF_E_TRACE,
                   "interval \"%s\" exceeds 2^32 cycles; the 32-bit clock "
                   "cannot represent it",
                   label_of(c, rid).c_str());
  }
  *n_out = info[0];
  if (dropped_heads) *dropped_heads = info[1];
  if (truncated_tails) *truncated_tails = info[2];
  if (info[0] > cap)
    return set_err(c, WGPF_E_BUFFER, "pair_records needs %u intervals", info[0]);
  if (info[0])
    CUDA_OK(c, cudaMemcpy(h_out, c->d_aux1.p, sizeof(wgpf_interval) * info[0],
                          cudaMemcpyDeviceToHost));
  return WGPF_OK;
}

extern "C" int wgpf_replay_intervals(wgpf_ctx* c, const wgpf_interval* h_iv,
                                     uint64_t n, uint32_t block_index,
                                     uint32_t warp_group, uint64_t record_cost,
                                     wgpf_event* h_out, uint64_t cap,
                                     uint64_t* n_out, wgpf_warnings* w) {
  if (!c->has_plan) return set_err(c, WGPF_E_ARG, "no buffer plan set");
  *n_out = 0;
  if (w) memset(w, 0, sizeof *w);
  ALLOC_OK(c, c->d_aux0, sizeof(wgpf_interval) * (n + 1));
  ALLOC_OK(c, c->d_aux1, sizeof(wgpf_event) * (n + 1));
  ALLOC_OK(c, c->d_aux2, n + 1);
  ALLOC_OK(c, c->d_aux3, 32);
  if (n)
    CUDA_OK(c, cudaMemcpyAsync(c->d_aux0.p, h_iv, sizeof(wgpf_interval) * n,
                               cudaMemcpyHostToDevice, c->stream));
  k_replay_one<<<1, 1, 0, c->stream>>>(
      c->d_aux0.as<wgpf_interval>(), n, dev_plan(c), block_index, warp_group,
      record_cost, c->d_aux2.as<uint8_t>(), c->d_aux1.as<wgpf_event>(),
      c->d_aux3.as<unsigned long long>());
  CUDA_OK(c, cudaGetLastError());
  unsigned long long info[3];
  CUDA_OK(c, cudaMemcpyAsync(info, c->d_aux3.p, 24, cudaMemcpyDeviceToHost,
                             c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  *n_out = info[0];
  if (w) {
    w->flagged_preconditions = (uint32_t)info[1];
    w->malformed_groups = (uint32_t)info[2];
  }
  if (info[0] > cap)
    return set_err(c, WGPF_E_BUFFER, "replay needs %llu events", info[0]);
  if (info[0])
    CUDA_OK(c, cudaMemcpy(h_out, c->d_aux1.p, sizeof(wgpf_event) * info[0],
                          cudaMemcpyDeviceToHost));
  return WGPF_OK;
}

// ---------------------------------------------------------------------------
// statistics read-out
// ---------------------------------------------------------------------------

static int read_stats(wgpf_ctx* c, bool event_keys) {
  const uint32_t ns = n_slots(c);
  std::vector<unsigned long long> cnt(ns), sum(ns), mn(ns), mx(ns), first(ns),
      fwg(ns), hist((size_t)ns * WGPF_HIST_BINS);
  std::vector<double> mean(ns);
  std::vector<uint32_t> hkey(kSynthHash);
  CUDA_OK(c, cudaMemcpyAsync(cnt.data(), c->d_count.p, 8 * ns, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaMemcpyAsync(sum.data(), c->d_sum.p, 8 * ns, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaMemcpyAsync(mn.data(), c->d_min.p, 8 * ns, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaMemcpyAsync(mx.data(), c->d_max.p, 8 * ns, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaMemcpyAsync(first.data(), c->d_first.p, 8 * ns, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaMemcpyAsync(fwg.data(), c->d_first_wg.p, 8 * ns, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaMemcpyAsync(hist.data(), c->d_hist.p, 8ull * ns * WGPF_HIST_BINS, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaMemcpyAsync(hkey.data(), c->d_hkey.p, 4 * kSynthHash, cudaMemcpyDeviceToHost, c->stream));
  if (c->mean_exact_valid)
    CUDA_OK(c, cudaMemcpyAsync(mean.data(), c->d_mean.p, 8 * ns, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  std::vector<std::pair<std::string, uint32_t>> order;
  for (uint32_t i = 0; i < ns; ++i) {
    if (!cnt[i]) continue;
    const uint32_t cls = i < c->K ? i : hkey[i - c->K];
    order.emplace_back(class_name(c, cls), i);
  }
  std::sort(order.begin(), order.end());
  c->stats_out.clear();
  c->stats_names.clear();
  c->stats_names.reserve(order.size());
  for (auto& [name, i] : order) {
    c->stats_names.push_back(name);
    wgpf_region_stat r;
    memset(&r, 0, sizeof r);
    r.warp_group = (uint32_t)fwg[i];
    r.kind = (uint32_t)(first[i] & 1u);
    r.count = cnt[i];
    r.min = mn[i];
    r.max = mx[i];
    r.sum = sum[i];
    r.mean = c->mean_exact_valid ? mean[i] : (double)sum[i] / (double)cnt[i];
    if (event_keys) {
      r.first_event = first[i] >> 1;
    } else {
      // (stream << 25 | k << 1 | kind): global event index when the stream
      // is local to this context (offsets of the last replay), else ~0
      const uint64_t gs = first[i] >> 25;
      const uint64_t k = (first[i] >> 1) & ((1ull << 24) - 1);
      r.first_event = ~0ull;
      if (c->chunk_mode) {  // pipelined replay_image: per-chunk event bases
        if (gs < c->chunk_nstreams && !c->chunk_sbase.empty()) {
          const size_t j = (size_t)(std::upper_bound(c->chunk_sbase.begin(),
                                                     c->chunk_sbase.end(), gs) -
                                    c->chunk_sbase.begin()) - 1;
          uint64_t off = 0;
          CUDA_OK(c, cudaMemcpy(&off, c->d_off_all.as<uint64_t>() + gs, 8,
                                cudaMemcpyDeviceToHost));
          r.first_event = c->chunk_ebase[j] + off + k;
        }
      } else if (gs >= c->last_stream_base &&
          gs - c->last_stream_base < c->last_n_streams && c->d_offsets.p) {
        uint64_t off = 0;
        CUDA_OK(c, cudaMemcpy(&off,
                              c->d_offsets.as<uint64_t>() + (gs - c->last_stream_base),
                              8, cudaMemcpyDeviceToHost));
        r.first_event = off + k;
      }
    }
    for (uint32_t b = 0; b < WGPF_HIST_BINS; ++b)
      r.hist[b] = hist[(size_t)i * WGPF_HIST_BINS + b];
    c->stats_out.push_back(r);
  }
  for (size_t k = 0; k < c->stats_out.size(); ++k)
    c->stats_out[k].label = c->stats_names[k].c_str();
  return WGPF_OK;
}

extern "C" int wgpf_stats_get(wgpf_ctx* c, wgpf_region_stat* out,
                              uint32_t cap, uint32_t* n) {
  *n = 0;
  if (!c->has_plan || !c->stats_valid)
    return set_err(c, WGPF_E_ARG, "no statistics available");
  int rc = read_stats(c, false);
  if (rc) return rc;
  *n = (uint32_t)c->stats_out.size();
  if (c->stats_out.size() > cap)
    return set_err(c, WGPF_E_BUFFER, "stats need %u entries", *n);
  for (size_t k = 0; k < c->stats_out.size(); ++k) out[k] = c->stats_out[k];
  return WGPF_OK;
}

extern "C" int wgpf_region_stats(wgpf_ctx* c, const wgpf_event* events,
                                 uint64_t n, int on_device, uint32_t flags,
                                 wgpf_region_stat* out, uint32_t cap,
                                 uint32_t* n_out) {
  if (!c->has_plan) return set_err(c, WGPF_E_ARG, "no buffer plan set");
  *n_out = 0;
  int rc = status_reset(c);
  if (rc) return rc;
  rc = stats_reset(c);
  if (rc) return rc;
  const wgpf_event* d_ev = events;
  if (!on_device) {
    ALLOC_OK(c, c->d_events, sizeof(wgpf_event) * std::max<uint64_t>(n, 1));
    if (n) {
      rc = h2d_host(c, c->d_events.p, events, sizeof(wgpf_event) * n);
      if (rc) return rc;
    }
    d_ev = c->d_events.as<wgpf_event>();
  }
  if (n) {
    k_event_stats<<<c->sms * 4, 256, 0, c->stream>>>(
        d_ev, n, dev_plan(c), dev_stats(c), c->d_status.as<DevStatus>());
    CUDA_OK(c, cudaGetLastError());
    const uint32_t ns = n_slots(c);
    k_event_first_wg<<<(ns + 127) / 128, 128, 0, c->stream>>>(
        d_ev, dev_stats(c), ns, c->d_first_wg.as<unsigned long long>());
    CUDA_OK(c, cudaGetLastError());
    c->mean_exact_valid = false;
    if (flags & WGPF_F_EXACT_MEAN) {
      c->stats_valid = true;
      rc = finalize_stats(c, nullptr, 0, 0, 0, d_ev, n, true);
      if (rc) return rc;
      // k_resolve_first ran against no body; restore the event-based wg
      k_event_first_wg<<<(ns + 127) / 128, 128, 0, c->stream>>>(
          d_ev, dev_stats(c), ns, c->d_first_wg.as<unsigned long long>());
    }
  }
  rc = status_read(c);
  if (rc) return rc;
  if (c->h_status->synth_overflow)
    return set_err(c, WGPF_E_CAPACITY,
                   "more than %u distinct out-of-table region labels",
                   kSynthHash);
  c->stats_valid = true;
  rc = read_stats(c, true);
  if (rc) return rc;
  *n_out = (uint32_t)c->stats_out.size();
  if (c->stats_out.size() > cap)
    return set_err(c, WGPF_E_BUFFER, "stats need %u entries", *n_out);
  for (size_t k = 0; k < c->stats_out.size(); ++k) out[k] = c->stats_out[k];
  return WGPF_OK;
}

extern "C" uint64_t wgpf_stats_packed_bytes(const wgpf_ctx* c) {
  if (!c->has_plan) return 0;  // the size depends on the plan's label classes
  return 8ull * ((uint64_t)n_slots(c) * kPackedPerSlot + kSynthHash);
}

extern "C" int wgpf_stats_export(wgpf_ctx* c, void* d_dst) {
  const uint32_t ns = n_slots(c);
  const uint32_t m = std::max(ns, kSynthHash);
  k_stats_pack<<<(m + 127) / 128, 128, 0, c->stream>>>(
      dev_stats(c), ns, c->d_first_wg.as<unsigned long long>(),
      static_cast<unsigned long long*>(d_dst));
  CUDA_OK(c, cudaGetLastError());
  return WGPF_OK;
}

extern "C" int wgpf_stats_merge(wgpf_ctx* c, const void* d_gathered,
                                uint32_t n_ranks) {
  c->chunk_mode = false;
  int rc = stats_reset(c);
  if (rc) return rc;
  rc = status_reset(c);
  if (rc) return rc;
  const uint32_t ns = n_slots(c);
  const uint64_t work = (uint64_t)n_ranks * ns;
  const auto* in = static_cast<const unsigned long long*>(d_gathered);
  k_stats_merge<<<(uint32_t)((work + 127) / 128), 128, 0, c->stream>>>(
      dev_stats(c), ns, in, n_ranks, c->d_status.as<DevStatus>());
  k_stats_merge_wg<<<(uint32_t)((work + 127) / 128), 128, 0, c->stream>>>(
      dev_stats(c), ns, in, n_ranks, c->d_first_wg.as<unsigned long long>());
  CUDA_OK(c, cudaGetLastError());
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  c->stats_valid = true;
  c->mean_exact_valid = false;
  return WGPF_OK;
}

extern "C" int wgpf_synth_body(wgpf_ctx* c, void* d_body, uint32_t shape,
                               uint64_t stream0, uint64_t n_streams,
                               uint64_t n_long) {
  if (shape > 1) return set_err(c, WGPF_E_ARG, "unknown synthetic shape");
  if (n_streams == 0) return WGPF_OK;
  k_synth<<<c->sms * 8, 256, 0, c->stream>>>(static_cast<uint8_t*>(d_body),
                                             shape, stream0, n_streams, n_long);
  CUDA_OK(c, cudaGetLastError());
  return WGPF_OK;
}

#include "capi_cp.inc"
#include "capi_chrome.inc"
#include "capi_p1.inc"
