/*
 * wgpf_format.h -- on-wire / in-HBM layouts shared by the device runtime (P1),
 * the decode kernels (P2), the C-ABI, the C++ shim and the CPU oracle.
 *
 * Plain C, usable from C, C++ and CUDA device code.
 *
 * Record (8 bytes, little endian), reference wgprof/trace.hpp:15-35,58-99:
 *   u32 tag     = start<<31 | region<<12 | signature&0xFFF  (region: 19 bits)
 *   u32 payload = 32-bit clock capture
 *
 * KPFT image, reference wgprof/trace.hpp:25-28,158-209:
 *   "KPFT", u16 version=1, u16 stream_count, then per stream
 *   { u32 block_index, u32 warp_group, u32 record_count, u32 slot_capacity }
 *   followed by slot_capacity raw records (buffer order).
 *
 * The per-stream block { 16-byte header, slot_capacity records } is the
 * "KPFT body".  The device runtime's finalize (P1) writes exactly this body to
 * HBM, so a device profile buffer prefixed with the 8-byte v1 header is a
 * valid reference image (<= 65535 streams).
 *
 * KPFT v2 (this framework's container for > 65535 streams; not readable by the
 * reference, which rejects version != 1, trace.hpp:187-190):
 *   "KPFT", u16 version=2, u16 reserved=0, u64 stream_count, then the same
 *   body.  Any contiguous run of <= 65535 streams of a v2 body prefixed with a
 *   v1 header is a valid v1 image (tests/test_format.py round-trips chunks
 *   through the reference deserialize_image).
 */
#ifndef WGPF_FORMAT_H
#define WGPF_FORMAT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WGPF_START_FLAG 0x80000000u     /* trace.hpp:32 kStartFlag       */
#define WGPF_SIGNATURE_MASK 0xFFFu      /* trace.hpp:33 kSignatureMask   */
#define WGPF_REGION_BITS 19u            /* lower.hpp:35 kRegionIdBits    */
#define WGPF_MAX_REGIONS (1u << 19)     /* lower.hpp:36 kMaxRegions      */
#define WGPF_RECORD_BYTES 8u            /* lower.hpp:37 kRecordBytes     */
#define WGPF_STREAM_HDR_BYTES 16u       /* trace.hpp:169-172             */
#define WGPF_KPFT_V1_HDR_BYTES 8u       /* "KPFT" u16 ver u16 count      */
#define WGPF_KPFT_V2_HDR_BYTES 16u      /* "KPFT" u16 ver u16 0 u64 count */
#define WGPF_KPFT_V1_MAX_STREAMS 0xFFFFu /* trace.hpp:162-163            */

/* BufferStrategy, reference lower.hpp:42 (enum order Circular, Flush). */
#define WGPF_STRATEGY_CIRCULAR 0u
#define WGPF_STRATEGY_FLUSH 1u

/* One raw record. */
typedef struct wgpf_record {
  uint32_t tag;
  uint32_t payload;
} wgpf_record;

/* KPFT per-stream header, byte-identical to trace.hpp:169-172. */
typedef struct wgpf_stream_hdr {
  uint32_t block_index;
  uint32_t warp_group;
  uint32_t record_count;  /* total writes (may exceed capacity: circular) */
  uint32_t slot_capacity;
} wgpf_stream_hdr;

/*
 * Decoded timeline event, 32 bytes (reference TimelineEvent, trace.hpp:354-367,
 * with the label string replaced by the region id; the label is
 * plan.region_labels[id] or "region#<id>", trace.hpp:302-306).
 */
typedef struct wgpf_event {
  uint64_t start;
  uint64_t end;
  uint32_t region;       /* region id | WGPF_EV_WAIT | WGPF_EV_CORRECTED */
  uint32_t iteration;
  uint32_t block_index;
  uint32_t warp_group;
} wgpf_event;

/*
 * Per-CTA timing side record of the device runtime (wgpf_dev::CtaTiming,
 * include/wgpf_device.cuh), 32 bytes: the SM, and %globaltimer (ns, one
 * clock for the whole GPU) with %clock (cycles, per SM) at the CTA's start
 * and end -- what wgpf_align_events uses to put the SM-local record clocks
 * of all CTAs on one timeline.
 */
typedef struct wgpf_cta_timing {
  uint32_t smid;
  uint32_t streams;
  uint64_t gt_start;  /* %globaltimer at init (ns) */
  uint64_t gt_end;    /* %globaltimer at finalize (ns) */
  uint32_t clk_start; /* %clock at init */
  uint32_t clk_end;   /* %clock at finalize */
} wgpf_cta_timing;

#define WGPF_EV_WAIT 0x80000000u      /* EventKind::Wait (else Exec)      */
#define WGPF_EV_CORRECTED 0x40000000u /* TimelineEvent::corrected         */
#define WGPF_EV_REGION_MASK 0x0007FFFFu

/* Duration histogram: 64 half-octave bins (this framework's definition; the
 * reference has no histograms).  bin(d) = d for d < 4; otherwise with
 * k = floor(log2 d): 2k + ((d >> (k-1)) & 1).  bin(2^32-1) = 63. */
#define WGPF_HIST_BINS 64u

static inline uint32_t wgpf_hist_bin(uint64_t d) {
  if (d < 4u) return (uint32_t)d;
  uint32_t k = 63u - (uint32_t)__builtin_clzll(d);
  uint32_t b = 2u * k + (uint32_t)((d >> (k - 1u)) & 1u);
  return b < WGPF_HIST_BINS ? b : WGPF_HIST_BINS - 1u;
}

#ifdef __cplusplus
}
#endif

#endif /* WGPF_FORMAT_H */
