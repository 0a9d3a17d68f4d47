/*
 * wgpf.h -- C-ABI of the B200-native KPerfIR trace post-processor (P2) and the
 * host helpers of the device instrumentation runtime (P1).
 *
 * This is the drop-in boundary.  The reference (arXiv 2505.21661,
 * /root/reference/proj) exposes its hot path as inline C++ functions in
 * namespace wgprof; each entry point below states the reference function it
 * replaces (file:line, relative to proj/include/).  include/wgprof_b200.hpp
 * wraps this ABI back into those exact C++ signatures (value semantics,
 * wgprof::Error exceptions), and paper_2505_21661_b200/trace.py mirrors them in
 * Python.  INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - No exceptions cross the ABI; every call returns a wgpf_status.  Status
 *    1..9 are the reference's ErrorKind values + 1 (wgprof/error.hpp:8-18), so
 *    a shim rethrows wgprof::Error((ErrorKind)(status - 1), wgpf_last_error()).
 *  - Caller-allocated outputs with capacity / count out-parameters.  When a
 *    capacity is too small the call returns WGPF_E_BUFFER and writes the
 *    needed count.
 *  - All device work is stream-ordered on the context's CUDA stream.  Calls
 *    that return host values synchronise that stream.
 *  - One context per host thread; contexts are independent (the reference
 *    functions are pure).
 *  - There is no CPU fallback: without a usable CUDA device wgpf_create fails
 *    with WGPF_E_CUDA.
 */
#ifndef WGPF_H
#define WGPF_H

#include <stddef.h>
#include <stdint.h>

#include "wgpf_format.h"

#ifdef __cplusplus
extern "C" {
#endif

#define WGPF_ABI_VERSION 1

typedef enum wgpf_status {
  WGPF_OK = 0,
  WGPF_E_PARSE = 1,      /* ErrorKind::Parse      "parse-error"         */
  WGPF_E_VALIDATE = 2,   /* ErrorKind::Validate   "validate-error"      */
  WGPF_E_INSTRUMENT = 3, /* ErrorKind::Instrument "instrument-error"    */
  WGPF_E_LOWER = 4,      /* ErrorKind::Lower      "lower-error"         */
  WGPF_E_CAPACITY = 5,   /* ErrorKind::Capacity   "capacity-error"      */
  WGPF_E_DEADLOCK = 6,   /* ErrorKind::Deadlock   "simulation-deadlock" */
  WGPF_E_TRACE = 7,      /* ErrorKind::Trace      "trace-error"         */
  WGPF_E_CONFIG = 8,     /* ErrorKind::Config     "config-error"        */
  WGPF_E_IO = 9,         /* ErrorKind::Io         "io-error"            */
  WGPF_E_CUDA = 10,      /* CUDA runtime failure / no device           */
  WGPF_E_ARG = 11,       /* invalid argument                            */
  WGPF_E_BUFFER = 12     /* caller buffer too small (count written)     */
} wgpf_status;

typedef struct wgpf_ctx wgpf_ctx;

typedef struct wgpf_warnings { /* TraceReplay counters, pipeline.hpp:58-64 */
  uint32_t dropped_heads;
  uint32_t truncated_tails;
  uint32_t flagged_preconditions;
  uint32_t malformed_groups;
} wgpf_warnings;

typedef struct wgpf_decoded_stream { /* DecodedStream, trace.hpp:215-220 */
  uint32_t block_index;
  uint32_t warp_group;
  uint32_t dropped_records;
  uint32_t pad;
  uint64_t offset; /* first record in the flat record output */
  uint64_t count;
} wgpf_decoded_stream;

typedef struct wgpf_interval { /* RawInterval, trace.hpp:278-286 (label -> id) */
  uint32_t region_id;
  uint32_t iteration;
  uint64_t start;
  uint64_t end;
  uint64_t start_pos;
  uint64_t end_pos;
} wgpf_interval;

typedef struct wgpf_region_stat { /* RegionStats, pipeline.hpp:105-112 + ext */
  const char* label;    /* owned by the context, valid until the next call */
  uint32_t warp_group;  /* of the first event with this label */
  uint32_t kind;        /* 0 exec, 1 wait (first event)        */
  uint64_t count;
  uint64_t min;
  uint64_t max;
  uint64_t sum;         /* exact integer sum of durations      */
  double mean;          /* see WGPF_F_EXACT_MEAN               */
  uint64_t first_event; /* global event index of the first event */
  uint64_t hist[WGPF_HIST_BINS]; /* wgpf_hist_bin() bins          */
} wgpf_region_stat;

/* replay flags */
#define WGPF_F_STATS_ONLY 0x1u  /* do not materialise events (stats only) */
#define WGPF_F_EXACT_MEAN 0x2u  /* mean by the reference's order-dependent
                                   double recurrence (pipeline.hpp:129),
                                   bit-exact; needs materialised events.
                                   Default: mean = (double)sum / count.   */
#define WGPF_F_FORCE_GENERAL 0x4u /* route every stream through the general
                                     (thread-per-stream) kernels            */
#define WGPF_F_NO_STATS 0x8u    /* skip region statistics                  */
#define WGPF_F_PROFILE 0x10u    /* record per-phase CUDA-event timings     */

/* Per-phase device time of the last wgpf_replay_device (WGPF_F_PROFILE) and
 * the number of this library's kernels it launched. */
typedef struct wgpf_profile {
  float count_ms;    /* pass 1 (k_count_tps / k_count_fast); overlapped
                        replay: pass 1 + scan of the first chunk only   */
  float scan_ms;     /* event-offset scan (0 when overlapped)          */
  float emit_ms;     /* pass 2 fast paths (k_tps, k_tpsd, k_fast_emit);
                        overlapped replay: with pass 1 of every later
                        chunk running beside it                        */
  float general_ms;  /* general path (k_general_emit), if any      */
  float finalize_ms; /* statistics finalisation                    */
  float total_ms;
  uint32_t launches;        /* kernels of this library launched     */
  uint32_t general_streams; /* streams taken by the general path   */
  uint32_t overlap_chunks;  /* chunks of the overlapped pass 1 / pass 2
                               (0: not overlapped)                     */
  uint32_t reserved;
} wgpf_profile;
int wgpf_last_profile(const wgpf_ctx* ctx, wgpf_profile* out);

/* ----------------------------------------------------------------------- */
/* Lifecycle                                                                 */
/* ----------------------------------------------------------------------- */

int wgpf_abi_version(void);
/* device: CUDA ordinal; stream: cudaStream_t (NULL = legacy default). */
int wgpf_create(int device, void* stream, wgpf_ctx** out);
void wgpf_destroy(wgpf_ctx* ctx);
int wgpf_set_stream(wgpf_ctx* ctx, void* stream);
const char* wgpf_last_error(const wgpf_ctx* ctx);
/* Error::category() for a status (error.hpp:29-51). */
const char* wgpf_error_category(int status);

/* BufferPlan (lower.hpp:57-73): slots per stream, strategy, region table. */
int wgpf_set_plan(wgpf_ctx* ctx, uint64_t slots_per_warp_group,
                  uint32_t strategy, const char* const* region_labels,
                  uint32_t n_labels);

/* ----------------------------------------------------------------------- */
/* P2: the trace post-processor                                              */
/* ----------------------------------------------------------------------- */

/*
 * replay_image (pipeline.hpp:66-81) = decode_image (trace.hpp:222) +
 * pair_records (trace.hpp:294) + replay (trace.hpp:398) per stream, events
 * concatenated in image order, warnings summed; plus region_stats
 * (pipeline.hpp:114) and duration histograms over the produced events.
 *
 * Device variant: d_body is a KPFT body (per stream: 16-byte header + slots)
 * already resident in HBM, n_streams streams of uniform stride
 * 16 + 8 * plan.slots.  stream_base is the global index of the first stream
 * (multi-GPU shards; 0 otherwise).  d_events (device) may be NULL with
 * WGPF_F_STATS_ONLY.  Synchronises the context stream before returning.
 */
int wgpf_replay_device(wgpf_ctx* ctx, const void* d_body, uint64_t body_bytes,
                       uint64_t n_streams, uint64_t stream_base,
                       uint64_t record_cost, wgpf_event* d_events,
                       uint64_t events_cap, uint32_t flags,
                       uint64_t* n_events, wgpf_warnings* warnings);

/*
 * Host variant (the reference-facing call): a complete KPFT v1 or v2 image in
 * host memory -> events in host memory.  Includes the host->device copy of
 * the image and the device->host copy of the events.  deserialize_image
 * errors (trace.hpp:181-209) are reproduced exactly.
 */
int wgpf_replay_image(wgpf_ctx* ctx, const uint8_t* kpft, uint64_t n_bytes,
                      uint64_t record_cost, wgpf_event* h_events,
                      uint64_t events_cap, uint32_t flags, uint64_t* n_events,
                      wgpf_warnings* warnings);

/* decode_image (trace.hpp:222-251) on a host KPFT image. */
int wgpf_decode_image(wgpf_ctx* ctx, const uint8_t* kpft, uint64_t n_bytes,
                      wgpf_record* h_records, uint64_t records_cap,
                      uint64_t* n_records, wgpf_decoded_stream* h_streams,
                      uint64_t streams_cap, uint64_t* n_streams);

/* unwrap_clock (trace.hpp:257-272). */
int wgpf_unwrap_clock(wgpf_ctx* ctx, const uint32_t* h_values, uint64_t n,
                      uint64_t* h_out);

/* pair_records (trace.hpp:294-346) on one chronological stream. */
int wgpf_pair_records(wgpf_ctx* ctx, const wgpf_record* h_records, uint64_t n,
                      wgpf_interval* h_out, uint64_t cap, uint64_t* n_out,
                      uint32_t* dropped_heads, uint32_t* truncated_tails);

/* replay (trace.hpp:398-487) on one stream's intervals. */
int wgpf_replay_intervals(wgpf_ctx* ctx, const wgpf_interval* h_iv, uint64_t n,
                          uint32_t block_index, uint32_t warp_group,
                          uint64_t record_cost, wgpf_event* h_out,
                          uint64_t cap, uint64_t* n_out,
                          wgpf_warnings* warnings);

/* Region statistics of the last replay (sorted by label bytes, as the
 * reference's std::map).  *n receives the number of labels. */
int wgpf_stats_get(wgpf_ctx* ctx, wgpf_region_stat* out, uint32_t cap,
                   uint32_t* n);

/* region_stats (pipeline.hpp:114-133) over an arbitrary event array
 * (device pointer when on_device != 0, else host). */
int wgpf_region_stats(wgpf_ctx* ctx, const wgpf_event* events, uint64_t n,
                      int on_device, uint32_t flags, wgpf_region_stat* out,
                      uint32_t cap, uint32_t* n_out);

/* Multi-GPU: export this rank's packed statistics (device buffer of
 * wgpf_stats_packed_bytes() bytes), and merge n_ranks gathered exports (one
 * after the other in d_gathered) into this context's statistics.  The caller
 * moves the bytes (e.g. one NCCL all-gather over NVLink).  The packed size
 * depends on the plan's label classes: 0 before wgpf_set_plan. */
uint64_t wgpf_stats_packed_bytes(const wgpf_ctx* ctx);
int wgpf_stats_export(wgpf_ctx* ctx, void* d_dst);
int wgpf_stats_merge(wgpf_ctx* ctx, const void* d_gathered, uint32_t n_ranks);

/* The same combination in one call over NCCL: export, one ncclAllGather of
 * the packed tables on the context stream (NVLink / NVSwitch), merge -- the
 * path's single collective.  nccl_comm is an ncclComm_t of
 * the participating ranks (ncclCommInitRank, or a framework's communicator);
 * afterwards every rank holds the whole trace's statistics.  libnccl.so.2 is
 * resolved at run time, so C / C++ hosts need no torch. */
int wgpf_allreduce_stats(wgpf_ctx* ctx, void* nccl_comm);

/* ----------------------------------------------------------------------- */
/* Interval-overlap analysis (K6)                                            */
/* ----------------------------------------------------------------------- */

typedef struct wgpf_cp_stage {
  const char* label;   /* owned by the context; stages sorted by label */
  uint64_t mean;       /* llround(sum / n) over the steady window */
  uint64_t steady;     /* steady-window instances */
  uint32_t warp_group; /* of the stage's lowest-iteration event */
  uint32_t pad;
} wgpf_cp_stage;

/*
 * analyze_critical_path (perfmodel.hpp:317-501) over an event array (device
 * pointer when on_device != 0).  barrier_src/dst: barrier-derived candidate
 * edges as label pairs (perfmodel.hpp:258-313 derives them from the lowered
 * program).  Outputs: stages (sorted by label), binding counts as an
 * n_stages x n_stages row-major matrix (row = gating stage, column = gated
 * stage), and the binding cycle (stage indices, rotated to the smallest
 * label) with its period.  gate_by_block selects per-(block, warp_group)
 * gating instead of the reference's per-warp_group gating (:373).
 */
int wgpf_critical_path(wgpf_ctx* ctx, const wgpf_event* events, uint64_t n,
                       int on_device, const char* const* barrier_src,
                       const char* const* barrier_dst, uint32_t n_barrier,
                       uint64_t slack, int exclude_warmup, int gate_by_block,
                       wgpf_cp_stage* stages, uint32_t stages_cap,
                       uint32_t* n_stages, uint64_t* binding,
                       uint64_t binding_cap, uint32_t* cycle,
                       uint32_t cycle_cap, uint32_t* n_cycle, uint64_t* period);

/* Role overlap counters (framework definition, oracle/wgpf_oracle.h
 * wgpo_overlap): per block, producer (role 0) / consumer (role 1) busy time
 * as the union of their Exec intervals, their intersection, the block span
 * and bubbles, summed over blocks. */
typedef struct wgpf_overlap {
  uint64_t blocks, span;
  uint64_t busy[2];
  uint64_t both;
  uint64_t bubble[2];
} wgpf_overlap;
int wgpf_overlap_counters(wgpf_ctx* ctx, const wgpf_event* events, uint64_t n,
                          int on_device, const uint8_t* role_of_wg,
                          uint32_t n_roles, wgpf_overlap* out);

/* export_chrome_trace (trace.hpp:493-511): the reference's Chrome Trace JSON
 * (nlohmann dump(2) layout, "\n"-terminated) for an event array (device
 * pointer when on_device != 0).  out == NULL queries *len. */
int wgpf_export_chrome_trace(wgpf_ctx* ctx, const wgpf_event* events, uint64_t n,
                             int on_device, double cycles_per_us, char* out,
                             uint64_t cap, uint64_t* len);

/* A double as nlohmann 3.11.3 serialises it (Grisu2 shortest digits, the
 * library's fixed / exponent layout, "null" when not finite) -- the number
 * format of the reference's JSON reports (pipeline.hpp:146-240).  Host code,
 * no device needed.  Returns the length written (<= 32), or -1 if cap < 33. */
int wgpf_format_json_double(double x, char* out, uint64_t cap);

/* ----------------------------------------------------------------------- */
/* P1 host helpers (the device runtime is include/wgpf_device.cuh)          */
/* ----------------------------------------------------------------------- */

/* HBM bytes the flushed profile of a grid needs: ctas x streams_per_cta x
 * (16-byte stream header + 8 x slots) -- the KPFT body Engine::image
 * (vgpu.hpp:136-148) copies out.  Host arithmetic, no device needed. */
uint64_t wgpf_profile_bytes(uint64_t ctas, uint32_t streams_per_cta,
                            uint64_t slots);

/*
 * Engine::image (vgpu.hpp:136-148) for a device profile: the n_streams-stream
 * body the kernels flushed to d_profile, checked and copied out as a KPFT
 * image (v1 when n_streams <= 65,535 -- readable by the reference's
 * deserialize_image -- else v2).  Checks, in the reference's order:
 *  - d_validate (optional, the error word of debug-mode recorders,
 *    wgpf_dev::Recorder<..., kValidate>): the first pairing violation of the
 *    lowest stream -> WGPF_E_INSTRUMENT with validate_record_pairing's text
 *    (instrument.hpp:60-105);
 *  - plan strategy Flush and record_count > slot_capacity (the recorder kept
 *    the first capacity records and counted the rest) -> WGPF_E_CAPACITY
 *    "wg<k>: flush buffer overflow after <cap> records" (vgpu.hpp:261-265).
 * out == NULL only checks and reports *n_bytes.
 */
int wgpf_collect(wgpf_ctx* ctx, const void* d_profile, uint64_t n_streams,
                 const uint64_t* d_validate, uint8_t* out, uint64_t cap,
                 uint64_t* n_bytes);

/* A scope program: per stream role (warp / warp group) a body of record and
 * loop ops, the device counterpart of the KernelProgram bodies lower() reads
 * (ir.hpp Instruction kinds Record / LoopBegin / LoopEnd). */
#define WGPF_OP_START 0u   /* record start "label"              */
#define WGPF_OP_END 1u     /* record end "label"                */
#define WGPF_OP_LOOP 2u    /* for <trips> {                     */
#define WGPF_OP_ENDLOOP 3u /* }                                 */
typedef struct wgpf_scope_op {
  uint32_t op;
  uint32_t pad;
  uint64_t trips;    /* WGPF_OP_LOOP */
  const char* label; /* WGPF_OP_START / WGPF_OP_END */
} wgpf_scope_op;

typedef struct wgpf_lower_cfg { /* LoweringConfig, lower.hpp:44-55 */
  const char* name;             /* kernel name (validate messages) */
  uint32_t strategy;            /* WGPF_STRATEGY_CIRCULAR / _FLUSH */
  int signature_bits;           /* signature_bits_enabled */
  int iteration_signature;      /* iteration_signature */
  int global_buffer;            /* BufferType::Global: no smem check */
  uint64_t slots_total;         /* buffer_slots_total, 0 = from the program */
  uint64_t smem_capacity;       /* KernelProgram::shared_mem_capacity */
} wgpf_lower_cfg;

typedef struct wgpf_lowered {
  uint64_t slots_per_stream;   /* BufferPlan::slots_per_warp_group */
  uint64_t smem_bytes_per_cta; /* device layout: streams x (16 + 8 x slots) */
  uint32_t n_regions;          /* region table size (ids 0 .. n-1) */
  uint32_t pad;
} wgpf_lowered;

/*
 * lower() (lower.hpp:220-301) of a scope program: the loop / record checks of
 * validate (ir.hpp:347-390, WGPF_E_VALIDATE), validate_record_pairing
 * (instrument.hpp:60-105, WGPF_E_INSTRUMENT), the signature-mode conflict
 * (WGPF_E_LOWER), dense region ids in first-appearance order
 * (region_of_op[i] for every op, ~0 for loop ops; the region table is the
 * labels in id order), the buffer plan (flush: the largest dynamic record
 * count; circular: plan_slots; explicit slots_total must divide by the
 * stream count) and the shared-memory budget (WGPF_E_CAPACITY), with the
 * reference's messages in err.  ops holds the bodies back to back.  Host
 * code, no device needed.
 */
int wgpf_lower_scopes(const wgpf_scope_op* ops, const uint32_t* body_len,
                      uint32_t n_bodies, const wgpf_lower_cfg* cfg,
                      uint32_t* region_of_op, wgpf_lowered* out, char* err,
                      uint64_t err_cap);

/*
 * Cross-SM time alignment: rewrites events (device pointer when on_device)
 * from their CTA's SM-local clock into one global cycle domain -- cycles at
 * cycles_per_ns since the earliest CTA start -- using the runtime's per-CTA
 * timing records (h_timing[block_index], host memory).  Durations are
 * unchanged; start times of all CTAs become comparable (Chrome export with
 * cycles_per_us = 1000 x cycles_per_ns puts them on one timeline).
 * cycles_per_ns <= 0 measures the SM clock rate from the records (total
 * cycles / total ns); the rate used is returned in *used_cycles_per_ns.
 * The reference has a single cycle domain (its vGPU clock); this is the B200
 * counterpart.
 */
int wgpf_align_events(wgpf_ctx* ctx, wgpf_event* events, uint64_t n, int on_device,
                      const wgpf_cta_timing* h_timing, uint64_t n_ctas,
                      double cycles_per_ns, double* used_cycles_per_ns);

/* ----------------------------------------------------------------------- */
/* Synthetic trace generator (bench / tests)    */
/* ----------------------------------------------------------------------- */

#define WGPF_SYNTH_MIXED 0u  /* config 4: producers/consumers, flush, cap 256 */
#define WGPF_SYNTH_NESTED 1u /* config 5: 64 nested scopes, circular 1000 w */

int wgpf_synth_body(wgpf_ctx* ctx, void* d_body, uint32_t shape,
                    uint64_t stream0, uint64_t n_streams, uint64_t n_long);

#ifdef __cplusplus
}
#endif

#endif /* WGPF_H */
