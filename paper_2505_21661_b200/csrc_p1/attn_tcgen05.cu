// attn_tcgen05.cu -- config-3 workload: a warp-specialised attention forward
// O = softmax(Q K^T / sqrt(d)) V for bf16 Q, K, V, O laid out [B*H, S, d],
// d = 128, on sm_100a, optionally instrumented with the P1 runtime.
//
// Structure: the B200 form of the reference's fa3 case-study kernel
// (fixtures/fa3_vanilla.kir: K / V producers, two consumers that each run
// GEMM0 -> softmax -> GEMM1 and ping-pong on the tensor core), with the
// same scope names, so the P2 overlap analyser reads the device trace the way
// the reference reads its vGPU trace.
//
//   warp 0      K producer: Q tiles once, then K_j via TMA into a KV_STAGES ring
//   warp 1      V producer: V_j via TMA into its ring
//   warps 2-5   consumer c0 (query rows q0 .. q0+127)
//   warps 6-9   consumer c1 (query rows q0+128 .. q0+255)
//
// A consumer's warp 0 lane 0 issues its own tcgen05.mma (any thread may);
// the four warps of the group own TMEM lane quadrants (warp % 4), i.e. one
// query row per thread.  TMEM (512 columns): S_c / P_c at 128 c, O_c at
// 256 + 128 c.  Per KV tile j (128 keys):
//   GEMM0  S_c = Q_c K_j^T          (SS, K-major, 8 x 128x128x16)
//   softmax  row max, lazy rescale of O_c (only when the running max grows
//          by more than 2^8; FA4's trick, exact after the final 1/l), P = 2^(s
//          - m) to bf16, written back into S_c's columns (tcgen05.st)
//   GEMM1  O_c += P_c V_j          (TS: A = P from TMEM, B = V MN-major)
// and GEMM0 of tile j+1 is issued right behind GEMM1 of tile j by the same
// thread (in-order tcgen05 pipe: it overwrites P only after GEMM1 read it;
// its completion implies GEMM1's, which is what the O rescale needs).
//
// Scopes (region ids) follow the reference's async pattern
// (instrument.hpp:14-25: S(X) before the launch, E(X) before the wait,
// S(X.wait) E(X.wait) after it): producers "Load K"/"Load V" (+ ".wait":
// the TMA completion), consumers "GEMM0.cN" (+ ".wait": S ready, which also
// retires the GEMM1 issued just before), "Softmax.cN", "GEMM1.cN".  One profile stream per warp, circular,
// PROF_CAP slots.
//
// The consumers alternate softmax turns every tile (named-barrier tokens),
// so one consumer's softmax runs beside the other's GEMMs.
//
// KV_STAGES = 1 mirrors fa3_vanilla (single-buffered K / V slots: the next
// load waits for both consumers' GEMMs); 2 double-buffers them.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "tc_sm100.cuh"
#include "wgpf_device.cuh"

namespace {

constexpr uint32_t HD = 128;                  // head dim
constexpr uint32_t BQ = 128, BKV = 128;       // rows per consumer / keys per tile
constexpr uint32_t TILE = 128 * HD * 2;       // 32 KB bf16 tile
constexpr uint32_t HALF = TILE / 2;           // one 64-column TMA box
constexpr uint32_t NWARPS = 10, THREADS = NWARPS * 32;
constexpr uint32_t PROF_CAP = 64;
constexpr uint32_t PROF_BYTES = wgpf_dev::smem_bytes(NWARPS, PROF_CAP);
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t IDESC_S = tc::idesc_bf16(128, 128, false);
constexpr uint32_t IDESC_PV = tc::idesc_bf16(128, HD, true);
constexpr float RESCALE_LOG2 = 8.0f;
#ifndef WGPF_ATTN_MUFU_PAIRS
#define WGPF_ATTN_MUFU_PAIRS 16
#endif
constexpr int kMufuPairs = WGPF_ATTN_MUFU_PAIRS;
// Per-tile softmax tokens between the consumers (FA3's warp-scheduler
// barriers).  Measured (B=16 H=16 S=8192, plain TFLOP/s / overhead): kv 1
// 1,042 / 4.0 % vs 1,033 / 4.1 % with only the initial stagger; kv 2 980 /
// 1.4 % vs 920 / 0.1 %.  Issuing the MMAs from a converged warp with
// elect.sync (the GEMM's fix) was faster still without the tokens (1,110 /
// 1,063) but its instrumented double-buffered variant fell into lockstep
// (24 % overhead); with the tokens it measured 1,017 / 978 -- not kept.
#ifndef WGPF_ATTN_PINGPONG
#define WGPF_ATTN_PINGPONG 1
#endif  // of 16 pairs per chunk: ex2 on MUFU

enum : uint32_t {
  R_LOAD_K, R_LOAD_K_WAIT, R_LOAD_V, R_LOAD_V_WAIT,
  R_C0,  // + 4 * c: GEMM0, GEMM0.wait, Softmax, GEMM1
};

template <uint32_t kStages>
constexpr uint32_t smem_bytes(bool instrument) {
  return 1024 + 2 * TILE + 2 * kStages * TILE + 256 + (instrument ? PROF_BYTES : 0);
}

// K-major tile (Q or K): k-step kk (16 columns of d) inside box kk / 4.
__device__ __forceinline__ uint64_t kmaj(uint32_t base, uint32_t kk) {
  return tc::desc_k_sw128(base + (kk >> 2) * HALF + (kk & 3u) * 32u);
}

template <bool kInstr, uint32_t kStages>
__global__ void __launch_bounds__(THREADS, 1)
    k_attn(const __grid_constant__ CUtensorMap tq,
           const __grid_constant__ CUtensorMap tk,
           const __grid_constant__ CUtensorMap tv, __nv_bfloat16* O,
           uint32_t S, float scale_log2, uint8_t* profile,
           wgpf_dev::CtaTiming* timing) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* qs = smem;                         // 2 tiles
  uint8_t* ks = qs + 2 * TILE;                // kStages tiles
  uint8_t* vs = ks + kStages * TILE;          // kStages tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(vs + kStages * TILE);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + kStages;
  uint64_t* v_full = k_empty + kStages;
  uint64_t* v_empty = v_full + kStages;
  uint64_t* s_full = v_empty + kStages;  // [2]
  uint64_t* o_done = s_full + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
  uint8_t* prof = reinterpret_cast<uint8_t*>(bars) + 256;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t bh = blockIdx.y;
  const uint32_t q0 = blockIdx.x * (2 * BQ);
  const uint32_t nkv = S / BKV;
  const uint64_t cta = (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const int row0 = (int)(bh * S);  // first row of this head in [B*H*S, d]

  // the uninstrumented twin uses the null recorder (strip_profiling)
  std::conditional_t<kInstr, wgpf_dev::Recorder<true>, wgpf_dev::NullRecorder> rec;
  if constexpr (kInstr) {
    rec.init(prof, warp, PROF_CAP, lane == 0);
    if (threadIdx.x == 0 && timing) {
      timing[cta].smid = wgpf_dev::smid();
      timing[cta].streams = NWARPS;
      timing[cta].gt_start = wgpf_dev::globaltimer();
      timing[cta].clk_start = wgpf_dev::clock32();
    }
  }

  if (warp == 0 && lane == 0) {
    tc::prefetch_map(&tq);
    tc::prefetch_map(&tk);
    tc::prefetch_map(&tv);
    tc::mbar_init(q_full, 1);
    for (uint32_t s = 0; s < kStages; ++s) {
      tc::mbar_init(&k_full[s], 1);
      tc::mbar_init(&k_empty[s], 2);  // one commit per consumer
      tc::mbar_init(&v_full[s], 1);
      tc::mbar_init(&v_empty[s], 2);
    }
    for (uint32_t c = 0; c < 2; ++c) {
      tc::mbar_init(&s_full[c], 1);
      tc::mbar_init(&o_done[c], 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<TMEM_COLS>(tmem_slot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 2) {
    // ---------------- producers: warp 0 = K (and Q), warp 1 = V -------------
    const bool is_k = warp == 0;
    const CUtensorMap* map = is_k ? &tk : &tv;
    uint64_t* full = is_k ? k_full : v_full;
    uint64_t* empty = is_k ? k_empty : v_empty;
    uint8_t* ring = is_k ? ks : vs;
    const uint32_t R = is_k ? R_LOAD_K : R_LOAD_V;
    if (is_k && lane == 0) {
      tc::mbar_expect_tx(q_full, 2 * TILE);
      for (uint32_t c = 0; c < 2; ++c) {
        tc::tma_load_2d(&tq, q_full, qs + c * TILE, 0, row0 + (int)(q0 + c * BQ));
        tc::tma_load_2d(&tq, q_full, qs + c * TILE + HALF, 64,
                        row0 + (int)(q0 + c * BQ));
      }
    }
    for (uint32_t j = 0; j < nkv; ++j) {
      const uint32_t s = j % kStages, ph = (j / kStages) & 1u;
      if (lane == 0) tc::mbar_wait(&empty[s], ph ^ 1u);
      __syncwarp();
      // the async pattern around the TMA launch and its completion wait
      // (insert_async_pattern, instrument.hpp:145-153)
      wgpf_dev::async_region(
          rec, R, R + 1,
          [&] {
            if (lane == 0) {
              uint8_t* dst = ring + s * TILE;
              tc::mbar_expect_tx(&full[s], TILE);
              tc::tma_load_2d(map, &full[s], dst, 0, row0 + (int)(j * BKV));
              tc::tma_load_2d(map, &full[s], dst + HALF, 64, row0 + (int)(j * BKV));
            }
            __syncwarp();
          },
          [&] {
            if (lane == 0) tc::mbar_wait(&full[s], ph);
            __syncwarp();
          });
    }
  } else {
    // ---------------- consumers ----------------
    const uint32_t c = (warp - 2) >> 2;
    const bool issuer = ((warp - 2) & 3u) == 0 && lane == 0;
    const uint32_t quad = warp & 3u;  // TMEM lane quadrant
    const uint32_t lane_base = (quad * 32u) << 16;
    const uint32_t tS = tmem + c * 128u;          // S, then P (bf16 pairs)
    const uint32_t tO = tmem + 256u + c * 128u;
    const uint32_t R = R_C0 + 4u * c;
    const uint32_t qbase = tc::smem_u32(qs + c * TILE);
    const uint32_t kbase = tc::smem_u32(ks), vbase = tc::smem_u32(vs);

    tc::mbar_wait(q_full, 0);
#if !WGPF_ATTN_PINGPONG
    if (c == 1) tc::bar_sync(3, 256);  // start one softmax behind c0 (ping-pong)
#endif
    // GEMM0: S = Q K_j^T into tS (issued one iteration ahead, right behind
    // GEMM1 of the previous tile; tcgen05.mma from one thread executes in
    // order, so it overwrites P only after GEMM1 has consumed it, and its
    // commit implies that GEMM1 -- and with it O -- is complete)
    auto gemm0 = [&](uint32_t jj) {
      const uint32_t s1 = jj % kStages, ph1 = (jj / kStages) & 1u;
      tc::mbar_wait(&k_full[s1], ph1);
      if constexpr (kInstr) rec.start(R + 0);
      if (issuer) {
        tc::fence_after();
        const uint32_t kt = kbase + s1 * TILE;
#pragma unroll
        for (uint32_t kk = 0; kk < HD / 16; ++kk)
          tc::mma_ss(tS, kmaj(qbase, kk), kmaj(kt, kk), IDESC_S, kk);
        tc::mma_commit(&s_full[c]);
        tc::mma_commit(&k_empty[s1]);
      }
      __syncwarp();
      if constexpr (kInstr) rec.end(R + 0);
    };
    gemm0(0);
    float m = -INFINITY, l = 0.f;
    for (uint32_t j = 0; j < nkv; ++j) {
      const uint32_t s = j % kStages, ph = (j / kStages) & 1u;
      tc::mbar_wait(&s_full[c], j & 1u);
      tc::fence_after();
      if constexpr (kInstr) {
        rec.start(R + 1);
        rec.end(R + 1);
      }
#if WGPF_ATTN_PINGPONG
      // softmax turns alternate between the consumers every tile (named
      // barrier tokens: c0 waits on 3 for c1's previous softmax, c1 on 4 for
      // c0's current one), so one consumer's softmax always runs beside the
      // other's GEMMs -- FA3's warp-scheduler barriers
      if (c == 1) tc::bar_sync(4, 256);
      else if (j > 0) tc::bar_sync(3, 256);
#endif
      if constexpr (kInstr) rec.start(R + 2);
      // ---- softmax ----
      // pass 1: row max (S stays in TMEM; pass 2 reloads it)
      // (four independent max chains: the 3-input max has a few cycles of
      // latency and a single chain would serialise the pass)
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll 1
      for (uint32_t ch = 0; ch < 4; ++ch) {
        uint32_t v[32];
        tc::tmem_ld32(tS + lane_base + ch * 32u, v);
        tc::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; i += 2)
          mx4[(i >> 1) & 3] = tc::max3(mx4[(i >> 1) & 3], __uint_as_float(v[i]),
                                       __uint_as_float(v[i + 1]));
      }
      const float mx = fmaxf(tc::max3(mx4[0], mx4[1], mx4[2]), mx4[3]);
      const float m_new = fmaxf(m, mx * scale_log2);
      const bool grow = m_new > m + RESCALE_LOG2;
      if (j > 0 && __any_sync(0xFFFFFFFFu, grow)) {
        const float f = grow ? tc::ex2(m - m_new) : 1.f;
#pragma unroll
        for (uint32_t ch = 0; ch < 4; ++ch) {
          uint32_t v[32];
          tc::tmem_ld32(tO + lane_base + ch * 32u, v);
          tc::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i)
            v[i] = __float_as_uint(__uint_as_float(v[i]) * f);
          tc::tmem_st32(tO + lane_base + ch * 32u, v);
        }
      }
      if (grow) {
        l *= tc::ex2(m - m_new);
        m = m_new;
      }
      // pass 2: P = 2^(s scale - m) in bf16 pairs over S's first 64 columns.
      // Chunk ch reads S columns 32ch .. 32ch+31, then P chunk ch overwrites
      // columns 16ch .. 16ch+15 -- all of them already read.  Packed f32x2
      // arithmetic; pairs [0, kMufuPairs) take ex2.approx (MUFU), the rest
      // the polynomial on the FMA pipe.
      const uint64_t sc2 = tc::pack2(scale_log2, scale_log2);
      const uint64_t nm2 = tc::pack2(-m, -m);
      uint64_t l2a = tc::pack2(0.f, 0.f), l2b = l2a;  // two sum chains
      auto chunk = [&](uint32_t ch, const uint32_t (&v)[32]) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t x = tc::fma2(tc::pack2(__uint_as_float(v[2 * i]),
                                                __uint_as_float(v[2 * i + 1])),
                                      sc2, nm2);
          uint64_t e;
          float x0, x1;
          tc::unpack2(x, x0, x1);
          if (i < kMufuPairs)
            e = tc::pack2(tc::ex2(x0), tc::ex2(x1));
          else
            e = tc::exp2_poly2(tc::pack2(fmaxf(x0, -125.f), fmaxf(x1, -125.f)));
          if (i & 1)
            l2b = tc::add2(l2b, e);
          else
            l2a = tc::add2(l2a, e);
          float a, b;
          tc::unpack2(e, a, b);
          __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
          pk[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        tc::tmem_st16(tS + lane_base + ch * 16u, pk);
      };
#pragma unroll 1
      for (uint32_t ch = 0; ch < 4; ++ch) {
        uint32_t v[32];
        tc::tmem_ld32(tS + lane_base + ch * 32u, v);
        tc::tmem_wait_ld();
        chunk(ch, v);
      }
      {
        float la, lb;
        tc::unpack2(tc::add2(l2a, l2b), la, lb);
        l += la + lb;
      }
      tc::tmem_wait_st();
      tc::fence_before();
      tc::bar_sync(1 + c, 128);  // P (and a rescaled O) of all 128 rows stored
#if WGPF_ATTN_PINGPONG
      if (c == 0) tc::bar_arrive(4, 256);
      else if (j + 1 < nkv) tc::bar_arrive(3, 256);
#else
      if (c == 0 && j == 0) tc::bar_arrive(3, 256);
#endif
      if constexpr (kInstr) rec.end(R + 2);
      // ---- GEMM1: O += P V_j ----
      tc::mbar_wait(&v_full[s], ph);
      if constexpr (kInstr) rec.start(R + 3);
      if (issuer) {
        tc::fence_after();
        const uint32_t vt = vbase + s * TILE;
#pragma unroll
        for (uint32_t kk = 0; kk < BKV / 16; ++kk)
          tc::mma_ts(tO, tS + kk * 8u, tc::desc_mn_sw128(vt + kk * 2048u, HALF),
                     IDESC_PV, (j | kk) != 0u);
        tc::mma_commit(&v_empty[s]);
        if (j + 1 == nkv) tc::mma_commit(o_done + c);
      }
      __syncwarp();
      if constexpr (kInstr) rec.end(R + 3);
      if (j + 1 < nkv) gemm0(j + 1);
    }
    tc::mbar_wait(o_done + c, 0);
    tc::fence_after();
    // ---- epilogue: O / l -> bf16 -> HBM (one row per thread) ----
    const float inv = 1.f / l;
    const uint64_t orow = (uint64_t)row0 + q0 + c * BQ + quad * 32u + lane;
    uint4* dst = reinterpret_cast<uint4*>(O + orow * HD);
#pragma unroll
    for (uint32_t ch = 0; ch < 4; ++ch) {
      uint32_t v[32];
      tc::tmem_ld32(tO + lane_base + ch * 32u, v);
      tc::tmem_wait_ld();
      uint32_t o[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * i]) * inv,
                                                 __uint_as_float(v[2 * i + 1]) * inv);
        o[i] = *reinterpret_cast<uint32_t*>(&h);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dst[ch * 4 + i] = make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
    }
  }

  if constexpr (kInstr) rec.close((uint32_t)cta, warp, PROF_CAP);
  tc::fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc<TMEM_COLS>(tmem);
  if constexpr (kInstr) {
    wgpf_dev::flush(prof, profile, cta, PROF_BYTES, threadIdx.x, THREADS);
    if (threadIdx.x == 0 && timing) {
      timing[cta].gt_end = wgpf_dev::globaltimer();
      timing[cta].clk_end = wgpf_dev::clock32();
    }
  }
}

template <bool kInstr, uint32_t kStages>
int launch(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
           void* O, uint32_t BH, uint32_t S, float scale_log2, void* prof,
           void* timing, cudaStream_t st) {
  auto* kfn = k_attn<kInstr, kStages>;
  constexpr uint32_t smem = smem_bytes<kStages>(kInstr);
  if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
      cudaSuccess)
    return 10;
  dim3 grid(S / (2 * BQ), BH);
  kfn<<<grid, THREADS, smem, st>>>(tq, tk, tv, static_cast<__nv_bfloat16*>(O), S,
                                   scale_log2, static_cast<uint8_t*>(prof),
                                   static_cast<wgpf_dev::CtaTiming*>(timing));
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}

}  // namespace

// Labels of the attention kernel's region ids (the plan's region table).
extern "C" const char* wgpf_attn_label(uint32_t id) {
  static const char* L[] = {"Load K",   "Load K.wait",   "Load V",
                            "Load V.wait", "GEMM0.c0", "GEMM0.c0.wait",
                            "Softmax.c0",  "GEMM1.c0", "GEMM0.c1",
                            "GEMM0.c1.wait", "Softmax.c1", "GEMM1.c1"};
  return id < sizeof(L) / sizeof(L[0]) ? L[id] : nullptr;
}

extern "C" uint64_t wgpf_attn_profile_bytes(uint32_t BH, uint32_t S) {
  return wgpf_dev::profile_bytes((uint64_t)BH * (S / (2 * BQ)), NWARPS, PROF_CAP);
}

extern "C" uint32_t wgpf_attn_smem_bytes(int instrument, int kv_stages) {
  return kv_stages == 1 ? smem_bytes<1>(instrument != 0)
                        : smem_bytes<2>(instrument != 0);
}

// O = softmax(Q K^T * scale) V; Q, K, V, O bf16 [BH, S, 128] contiguous;
// S % 256 == 0.  scale <= 0 selects 1/sqrt(128).  kv_stages 1 or 2.
// instrument != 0 writes the KPFT body (wgpf_attn_profile_bytes) to d_profile
// and 32-B CTA side records to d_timing (may be null).
extern "C" int wgpf_attn_bf16(const void* Q, const void* K, const void* V, void* O,
                              uint32_t BH, uint32_t S, float scale, int kv_stages,
                              int instrument, void* d_profile, void* d_timing,
                              void* stream) {
  if (S == 0 || S % (2 * BQ) || BH == 0 || BH > 65535 ||
      (kv_stages != 1 && kv_stages != 2))
    return 11;
  if (instrument && !d_profile) return 11;
  CUtensorMap tq, tk, tv;
  const uint64_t rows = (uint64_t)BH * S;
  if (!tc::make_map_bf16(&tq, Q, rows, HD, 128) ||
      !tc::make_map_bf16(&tk, K, rows, HD, 128) ||
      !tc::make_map_bf16(&tv, V, rows, HD, 128))
    return 10;
  if (scale <= 0.f) scale = 0.08838834764831845f;  // 1/sqrt(128)
  const float sl2 = scale * 1.4426950408889634f;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (instrument)
    return kv_stages == 1
               ? launch<true, 1>(tq, tk, tv, O, BH, S, sl2, d_profile, d_timing, st)
               : launch<true, 2>(tq, tk, tv, O, BH, S, sl2, d_profile, d_timing, st);
  return kv_stages == 1
             ? launch<false, 1>(tq, tk, tv, O, BH, S, sl2, nullptr, nullptr, st)
             : launch<false, 2>(tq, tk, tv, O, BH, S, sl2, nullptr, nullptr, st);
}
