// gemm_tcgen05.cu -- config-2 workload: bf16 GEMM C[M,N] = A[M,K] . B[N,K]^T
// (fp32 accumulate in TMEM) on sm_100a with TMA loads, tcgen05.mma issued by
// one thread, and a warp-specialised pipeline; optionally instrumented with
// the P1 runtime (include/wgpf_device.cuh) -- one profile stream per warp,
// 64 slots each in a shared-memory circular buffer (3 KB + headers per CTA).
//
// Roles (6 warps): warp 0 TMA producer, warp 1 MMA issuer (+ TMEM owner),
// warps 2-5 epilogue (TMEM lanes 32*(w%4) .. +32).  Two shapes:
//   CTA pair (M % 256 == 0, the default): a cluster of 2 CTAs on one TPC
//     computes a 256x256 tile with UMMA 256x256x16 (cta_group::2) issued by
//     the leader CTA; each CTA stages its 128 rows of A and its 128-row half
//     of B (6 smem stages of 32 KB): per 128x256 of output an SM stages and
//     feeds the tensor core 2/3 of the single-CTA bytes (A 128 + B 128 rows
//     instead of A 128 + B 256).  Each CTA's TMEM holds its 128 rows of the
//     accumulator.  8192^3: ~1,560 TFLOP/s (~93 % of cuBLAS on the same box;
//     single-CTA ~1,300), profiles/r02_gemm_pair.json.
//   single CTA (M % 128 == 0): tile 128x256x64, UMMA 128x256x16
//     (cta_group::1), 4 smem stages of 48 KB.
// Both: 2 x 256 TMEM columns (double-buffered accumulator).
//
// Scopes (region ids): 0 tile, 1 tma.stall, 2 tma.issue, 3 mma.stall,
// 4 mma.issue, 5 epi.stall, 6 epi.ld, 7 epi.st (the stalls are sync scopes
// around mbarrier waits: no ".wait" suffix, which replay reserves for the
// async pattern's wait markers, trace.hpp:377-382).  Placed by the
// instrumentation-pass helpers of wgpf_device.cuh, not by hand: the tile is
// a wgpf_dev::Scope, each role's pipeline phases a wgpf_dev::Chain
// (stall -> issue -> stall ...); the plain twin is the same source on
// wgpf_dev::NullRecorder.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "wgpf_device.cuh"

namespace {

constexpr uint32_t BM = 128, BN = 256, BK = 64;
constexpr uint32_t NWARPS = 6, THREADS = NWARPS * 32;
constexpr uint32_t PROF_CAP = 64;
constexpr uint32_t PROF_BYTES = wgpf_dev::smem_bytes(NWARPS, PROF_CAP);
constexpr uint32_t TMEM_COLS = 512;  // two 128 x 256 fp32 accumulators

// per-shape constants (kPair: the CTA-pair kernel)
template <bool kPair>
struct Geo {
  static constexpr uint32_t TM = kPair ? 256 : BM;       // tile rows (both CTAs)
  static constexpr uint32_t STAGES = kPair ? 6 : 4;
  static constexpr uint32_t A_BYTES = BM * BK * 2;        // this CTA's A rows
  static constexpr uint32_t B_BYTES = (kPair ? BN / 2 : BN) * BK * 2;  // its B rows
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  // bytes the MMA's full barrier waits for (both CTAs' loads when paired)
  static constexpr uint32_t TX_BYTES = (kPair ? 2 : 1) * STAGE_BYTES;
  static constexpr uint32_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256 + PROF_BYTES;
  // kind::f16, A/B bf16, D f32, K-major both, M = TM, N = 256
  static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) |
                                    ((BN >> 3) << 17) | ((TM >> 4) << 24);
};

enum : uint32_t { R_TILE, R_TMA_WAIT, R_TMA, R_MMA_WAIT, R_MMA, R_EPI_WAIT,
                  R_EPI_LD, R_EPI_ST };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// cluster-scope wait (the barrier's arrivals come from the peer CTA too)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_idx() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

// K-major, 128-byte swizzle UMMA shared-memory descriptor (SBO = 1024 B).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);  // start address
  d |= (uint64_t)1 << 16;                  // LBO (16 B, unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO
  d |= (uint64_t)1 << 46;                  // version (sm100)
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}

// One stage's loads issued by an elected lane of a converged warp: the
// expected bytes on this CTA's full barrier bar (tx != 0: the leader) and the
// A and B boxes completing on fb (the leader's full barrier, a cluster
// address when paired).
template <bool kPair>
__device__ __forceinline__ void tma_kblock(const CUtensorMap* ma, const CUtensorMap* mb,
                                           uint32_t fb, uint32_t sa, uint32_t sb, int k,
                                           int m0, int n0, uint32_t tx, uint32_t bar) {
  if constexpr (kPair)
    asm volatile(
        "{\n.reg .pred e, x;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.and.b32 x, %8, 0, e;\n"
        "@x mbarrier.arrive.expect_tx.shared::cta.b64 _, [%9], %8;\n"
        "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%3], [%0, {%5, %6}], [%2];\n"
        "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%4], [%1, {%5, %7}], [%2];\n"
        "}\n" ::"l"(reinterpret_cast<uint64_t>(ma)),
        "l"(reinterpret_cast<uint64_t>(mb)), "r"(fb), "r"(sa), "r"(sb), "r"(k), "r"(m0),
        "r"(n0), "r"(tx), "r"(bar)
        : "memory");
  else
    asm volatile(
        "{\n.reg .pred e, x;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.and.b32 x, %8, 0, e;\n"
        "@x mbarrier.arrive.expect_tx.shared::cta.b64 _, [%9], %8;\n"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%3], [%0, {%5, %6}], [%2];\n"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%4], [%1, {%5, %7}], [%2];\n"
        "}\n" ::"l"(reinterpret_cast<uint64_t>(ma)),
        "l"(reinterpret_cast<uint64_t>(mb)), "r"(fb), "r"(sa), "r"(sb), "r"(k), "r"(m0),
        "r"(n0), "r"(tx), "r"(bar)
        : "memory");
}

// One k-block (BK = 64: four K = 16 MMAs) and its stage's commit, issued by
// one elected lane of a converged warp: the descriptors advance by 32 B
// (2 in the 16-B address field) inside the asm, so the warp spends a handful
// of instructions per k-block instead of a per-MMA uniform-register
// waterfall (the MMA issuer is a single warp feeding two SMs' tensor cores).
template <bool kPair>
__device__ __forceinline__ void umma_kblock(uint32_t tmem, uint64_t da, uint64_t db,
                                            uint32_t accumulate, uint32_t bar) {
  if constexpr (kPair)
    asm volatile(
        "{\n"
        ".reg .pred e, p, t;\n"
        ".reg .b64 a1, a2, a3, b1, b2, b3;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 t, 0, 0;\n"
        "add.s64 a1, %1, 2;\n add.s64 a2, %1, 4;\n add.s64 a3, %1, 6;\n"
        "add.s64 b1, %2, 2;\n add.s64 b2, %2, 4;\n add.s64 b3, %2, 6;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, t;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%5], %6;\n"
        "}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(Geo<true>::IDESC), "r"(accumulate), "r"(bar), "h"((uint16_t)3)
        : "memory");
  else
    asm volatile(
        "{\n"
        ".reg .pred e, p, t;\n"
        ".reg .b64 a1, a2, a3, b1, b2, b3;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 t, 0, 0;\n"
        "add.s64 a1, %1, 2;\n add.s64 a2, %1, 4;\n add.s64 a3, %1, 6;\n"
        "add.s64 b1, %2, 2;\n add.s64 b2, %2, 4;\n add.s64 b3, %2, 6;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, t;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n"
        "}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(Geo<false>::IDESC), "r"(accumulate), "r"(bar)
        : "memory");
}

// MMA completion -> an mbarrier arrive, by an elected lane of a converged
// warp (kPair: on the barrier at the same offset in both CTAs of the pair)
template <bool kPair>
__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
  if constexpr (kPair)
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;\n}\n" ::"r"(bar), "h"((uint16_t)3)
        : "memory");
  else
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
            bar)
        : "memory");
}

// Persistent: one CTA per SM walks tiles t = blockIdx.x, += gridDim.x in a
// grouped raster (kGroupM m-blocks x all n-blocks, m fastest) so a wave's A
// and B tiles stay in L2.  Two TMEM accumulators (2 x 256 columns): the MMA
// warp fills one while the epilogue drains the other (tmem_full / tmem_empty
// barriers), so the epilogue overlaps the next tile's main loop.
// measured (8192^3, CTA pairs): groups of 2 / 4 / 8 / 16 / 32 pair m-blocks
// give 1,466 / 1,535 / 1,588 / 1,574 / 1,484 TFLOP/s with DRAM reads
// following (1.07 GB at 8, 1.52 at 4); L2 evict_last / evict_first hints on
// the A / B loads did not help (1,545-1,597)
#ifndef WGPF_GEMM_GROUP_M
#define WGPF_GEMM_GROUP_M 8
#endif
constexpr uint32_t kGroupM = WGPF_GEMM_GROUP_M;

__device__ __forceinline__ void tile_coords(uint32_t t, uint32_t nM, uint32_t nN,
                                            uint32_t& mb, uint32_t& nb) {
  const uint32_t per_group = kGroupM * nN;
  const uint32_t g = t / per_group, r = t % per_group;
  const uint32_t gm = min(kGroupM, nM - g * kGroupM);  // m-blocks in this group
  mb = g * kGroupM + r % gm;
  nb = r / gm;
}

// kMode: 0 plain, 1 one clock capture per RecordOp, 2 adjacent END/START
// RecordOps at scope boundaries share a capture (Recorder::mark).
// kPair: clusters of 2 CTAs (cluster rank 0 issues the pair's MMAs); tiles
// go to clusters, t = cluster index, += cluster count.
template <int kMode, bool kPair>
__global__ void __launch_bounds__(THREADS, 1)
    k_gemm(const __grid_constant__ CUtensorMap ta,
           const __grid_constant__ CUtensorMap tb, __nv_bfloat16* C, uint32_t M,
           uint32_t N, uint32_t K, uint8_t* profile,
           wgpf_dev::CtaTiming* timing) {
  using G = Geo<kPair>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::STAGES * G::STAGE_BYTES);
  uint64_t* empty = full + G::STAGES;
  uint64_t* tmem_full = empty + G::STAGES;   // [2]
  uint64_t* tmem_empty = tmem_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  uint8_t* prof = smem + G::STAGES * G::STAGE_BYTES + 256;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t nM = M / G::TM, nN = N / BN, n_tiles = nM * nN;
  const uint32_t nk = K / BK;
  const uint64_t cta = blockIdx.x;
  const uint32_t rank = kPair ? cluster_rank() : 0u;  // 0: MMA leader
  const uint32_t t0 = kPair ? cluster_idx() : blockIdx.x;
  const uint32_t tstep = kPair ? cluster_count() : gridDim.x;

  // the uninstrumented twin records nothing (strip_profiling)
  using Rec = std::conditional_t<kMode == 0, wgpf_dev::NullRecorder, wgpf_dev::Recorder<true>>;
  using Tile = wgpf_dev::Scope<Rec>;
  using Phases = wgpf_dev::Chain<Rec, kMode == 2>;
  Rec rec;
  if constexpr (kMode != 0) {
    rec.init(prof, warp, PROF_CAP, lane == 0);
    if (threadIdx.x == 0 && timing) {
      timing[cta].smid = wgpf_dev::smid();
      timing[cta].streams = NWARPS;
      timing[cta].gt_start = wgpf_dev::globaltimer();
      timing[cta].clk_start = wgpf_dev::clock32();
    }
  }

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)));
    for (uint32_t s = 0; s < G::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (uint32_t a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      // one arrive per epilogue warp (of both CTAs when paired)
      mbar_init(&tmem_empty[a], kPair ? 8 : 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    // (paired: warp 1 of both CTAs allocates the same columns)
    if constexpr (kPair) {
      asm volatile(
          "tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
              smem_u32(tmem_slot)),
          "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile(
          "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
              smem_u32(tmem_slot)),
          "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  // paired: the peer's loads and arrivals target the leader's barriers
  if constexpr (kPair) cluster_sync(); else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    uint32_t it = 0;  // k-block counter across tiles
    for (uint32_t t = t0; t < n_tiles; t += tstep) {
      uint32_t mb, nb;
      tile_coords(t, nM, nN, mb, nb);
      // this CTA's A rows and B rows (paired: its halves of the 256-row tile
      // and of the 256 columns)
      const uint32_t m0 = mb * G::TM + rank * BM;
      const uint32_t n0 = nb * BN + rank * (BN / 2);
      Tile tile(rec, R_TILE);
      Phases ph_(rec);  // tma.stall -> tma.issue per k-block
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % G::STAGES, ph = (it / G::STAGES) & 1u;
        ph_.to(R_TMA_WAIT, R_TMA);
        mbar_wait(&empty[s], ph ^ 1u);
        __syncwarp();
        ph_.to(R_TMA, R_TMA_WAIT);
        {
          const uint32_t a = smem_u32(stage_base + s * G::STAGE_BYTES);
          const uint32_t fb = kPair ? peer_addr(&full[s], 0) : smem_u32(&full[s]);
          tma_kblock<kPair>(&ta, &tb, fb, a, a + G::A_BYTES, (int)(kb * BK), (int)m0, (int)n0,
                            rank == 0 ? G::TX_BYTES : 0u, smem_u32(&full[s]));
        }
        ph_.iteration_end();
      }
    }
    if constexpr (kPair) {
      // the leader's last MMA commits arrive on this CTA's empty barriers:
      // wait for them before the CTA can exit
      if (lane == 0)
        for (uint32_t i = 0; i < G::STAGES; ++i, ++it)
          mbar_wait(&empty[it % G::STAGES], ((it / G::STAGES) & 1u) ^ 1u);
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (paired: the leader CTA only) ----------------
    uint32_t it = 0, tl = 0;
    for (uint32_t t = t0; rank == 0 && t < n_tiles; t += tstep, ++tl) {
      const uint32_t acc = tl & 1u, aph = (tl >> 1) & 1u;
      const uint32_t dt = tmem + acc * BN;
      Tile tile(rec, R_TILE);
      // the epilogue has drained this accumulator (two tiles ago)
      if (lane == 0) {
        if constexpr (kPair) mbar_wait_cluster(&tmem_empty[acc], aph ^ 1u);
        else mbar_wait(&tmem_empty[acc], aph ^ 1u);
      }
      __syncwarp();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      Phases ph_(rec);  // mma.stall -> mma.issue per k-block
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % G::STAGES, ph = (it / G::STAGES) & 1u;
        ph_.to(R_MMA_WAIT, R_MMA);
        mbar_wait(&full[s], ph);
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        ph_.to(R_MMA, R_MMA_WAIT);
        const uint32_t a = smem_u32(stage_base + s * G::STAGE_BYTES);
        umma_kblock<kPair>(dt, umma_desc(a), umma_desc(a + G::A_BYTES), kb, smem_u32(&empty[s]));
        if (kb == nk - 1) umma_commit_elect<kPair>(smem_u32(&tmem_full[acc]));
        ph_.iteration_end();
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> registers -> bf16 -> HBM -----------
    const uint32_t quad = warp & 3u;  // TMEM lane quadrant of this warp
    // the accumulator's empty barrier lives in the leader CTA when paired
    const uint32_t te0 = kPair ? peer_addr(&tmem_empty[0], 0) : smem_u32(&tmem_empty[0]);
    uint32_t tl = 0;
    for (uint32_t t = t0; t < n_tiles; t += tstep, ++tl) {
      uint32_t mb, nb;
      tile_coords(t, nM, nN, mb, nb);
      const uint32_t m0 = mb * G::TM + rank * BM, n0 = nb * BN;
      const uint32_t acc = tl & 1u, aph = (tl >> 1) & 1u;
      const uint32_t row = m0 + quad * 32u + lane;
      Tile tile(rec, R_TILE);
      Phases ph_(rec);  // epi.stall, then epi.ld -> epi.st per 32 columns
      ph_.to(R_EPI_WAIT);
      mbar_wait(&tmem_full[acc], aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      ph_.iteration_end();
      const uint32_t taddr = tmem + acc * BN + ((quad * 32u) << 16);
      for (uint32_t c = 0; c < BN; c += 32) {
        ph_.to(R_EPI_LD, c ? R_EPI_ST : R_EPI_WAIT);
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,"
            "%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,"
            "%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]),
              "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]),
              "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
              "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c + 32 == BN) {
          // the accumulator is in registers: hand it back to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if constexpr (kPair)
              asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                               te0 + 8u * acc)
                           : "memory");
            else
              asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(te0 + 8u * acc)
                           : "memory");
          }
        }
        ph_.to(R_EPI_ST, R_EPI_LD);
        uint4 out[4];
        uint32_t* o = reinterpret_cast<uint32_t*>(out);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * j]),
                                                   __uint_as_float(v[2 * j + 1]));
          o[j] = *reinterpret_cast<uint32_t*>(&h);
        }
        if (row < M) {
          uint4* dst = reinterpret_cast<uint4*>(C + (uint64_t)row * N + n0 + c);
#pragma unroll
          for (int j = 0; j < 4; ++j) dst[j] = out[j];
        }
        ph_.iteration_end();
      }
    }
  }

  if constexpr (kMode != 0) rec.close((uint32_t)cta, warp, PROF_CAP);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  // paired: both CTAs are done with the pair's TMEM and barriers
  if constexpr (kPair) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(TMEM_COLS));
  }
  if constexpr (kMode != 0) {
    wgpf_dev::flush_bulk(prof, profile, cta, PROF_BYTES, threadIdx.x, THREADS);
    if (threadIdx.x == 0 && timing) {
      timing[cta].gt_end = wgpf_dev::globaltimer();
      timing[cta].clk_end = wgpf_dev::clock32();
    }
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// the CTA-pair kernel for M % 256 == 0 (WGPF_GEMM_SINGLE=1 forces the
// single-CTA kernel, for A/B runs)
bool use_pair(uint32_t M) {
  static int single = -1;
  if (single < 0) {
    const char* e = getenv("WGPF_GEMM_SINGLE");
    single = e && atoi(e) ? 1 : 0;
  }
  return !single && M % 256 == 0;
}

// CTA pairs that can be resident at once (a pair needs both SMs of a TPC)
uint32_t max_pairs() {
  static int n = 0;
  if (!n) {
    auto* kfn = k_gemm<1, true>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Geo<true>::SMEM_BYTES);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (sm_count() / 2));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = Geo<true>::SMEM_BYTES;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, kfn, &cfg) != cudaSuccess || c <= 0) {
      cudaGetLastError();
      c = sm_count() / 2;
    }
    n = c;
  }
  return (uint32_t)n;
}

uint32_t grid_ctas(uint32_t M, uint32_t N) {
  if (use_pair(M)) {
    const uint32_t tiles = (M / 256) * (N / BN), p = max_pairs();
    return 2u * (tiles < p ? tiles : p);
  }
  const uint32_t tiles = (M / BM) * (N / BN);
  return tiles < (uint32_t)sm_count() ? tiles : (uint32_t)sm_count();
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t,
                                void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*,
                                CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault,
                                &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols,
              uint32_t box_rows) {
  EncodeTiled fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// C[M,N] = A[M,K] . B[N,K]^T (bf16 in/out, fp32 accumulate).  M % 128 (the
// CTA-pair kernel when M % 256 == 0),
// N % 256, K % 64 must be 0.  instrument != 0 runs the P1-instrumented kernel
// and writes the KPFT body to d_profile (wgpf_gemm_profile_bytes) and the CTA
// side records to d_timing (32 B per CTA, may be null).
// one profile segment per CTA of the persistent grid (min(tiles, SMs))
extern "C" uint64_t wgpf_gemm_profile_bytes(uint32_t M, uint32_t N) {
  return wgpf_dev::profile_bytes(grid_ctas(M, N), NWARPS, PROF_CAP);
}
extern "C" uint32_t wgpf_gemm_ctas(uint32_t M, uint32_t N) { return grid_ctas(M, N); }

// (per CTA, of the kernel an M % 256 == 0 GEMM runs)
extern "C" uint32_t wgpf_gemm_smem_bytes(int instrument) {
  const uint32_t b = use_pair(256) ? Geo<true>::SMEM_BYTES : Geo<false>::SMEM_BYTES;
  return instrument ? b : b - PROF_BYTES;
}

namespace {
template <bool kPair>
cudaError_t launch_gemm(int mode, const CUtensorMap& ta, const CUtensorMap& tb, void* C,
                        uint32_t M, uint32_t N, uint32_t K, void* d_profile,
                        void* d_timing, cudaStream_t st) {
  using G = Geo<kPair>;
  auto* kfn = mode == 0 ? k_gemm<0, kPair> : mode == 2 ? k_gemm<2, kPair> : k_gemm<1, kPair>;
  const uint32_t smem = mode ? G::SMEM_BYTES : G::SMEM_BYTES - PROF_BYTES;
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid_ctas(M, N));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kPair ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kfn, ta, tb, static_cast<__nv_bfloat16*>(C), M, N, K,
                            static_cast<uint8_t*>(mode ? d_profile : nullptr),
                            static_cast<wgpf_dev::CtaTiming*>(mode ? d_timing : nullptr));
}
}  // namespace

extern "C" int wgpf_gemm_bf16(const void* A, const void* B, void* C, uint32_t M,
                              uint32_t N, uint32_t K, int instrument,
                              void* d_profile, void* d_timing, void* stream) {
  if (M % BM || N % BN || K % BK || K == 0) return 11;
  const bool pair = use_pair(M);
  CUtensorMap ta, tb;
  // box rows: this CTA's 128 rows of A; its B rows (half of 256 when paired)
  if (!make_map(&ta, A, M, K, BM) || !make_map(&tb, B, N, K, pair ? BN / 2 : BN)) return 10;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // instrument = 1: one capture per RecordOp; 2: shared boundary captures
  // (WGPF_P1_MODE overrides, for A/B runs)
  int mode = 0;
  if (instrument) {
    mode = instrument;
    if (const char* e = getenv("WGPF_P1_MODE")) mode = atoi(e);
    if (mode != 2) mode = 1;
  }
  const cudaError_t e = pair ? launch_gemm<true>(mode, ta, tb, C, M, N, K, d_profile, d_timing, st)
                             : launch_gemm<false>(mode, ta, tb, C, M, N, K, d_profile, d_timing, st);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? 0 : 10;
}
