// gemm_tcgen05.cu -- config-2 workload: bf16 GEMM C[M,N] = A[M,K] . B[N,K]^T
// (fp32 accumulate in TMEM) on sm_100a with TMA loads, tcgen05.mma issued by
// one thread, and a warp-specialised pipeline; optionally instrumented with
// the P1 runtime (include/wgpf_device.cuh) -- one profile stream per warp,
// 64 slots each in a shared-memory circular buffer (3 KB + headers per CTA).
//
// Roles (6 warps): warp 0 TMA producer, warp 1 MMA issuer (+ TMEM owner),
// warps 2-5 epilogue (TMEM lanes 32*(w%4) .. +32).  Tile 128x256x64, UMMA
// 128x256x16 (cta_group::1), 4 smem stages of 48 KB, 2 x 256 TMEM columns
// (double-buffered accumulator).
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

constexpr uint32_t BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr uint32_t NWARPS = 6, THREADS = NWARPS * 32;
constexpr uint32_t PROF_CAP = 64;
constexpr uint32_t PROF_BYTES = wgpf_dev::smem_bytes(NWARPS, PROF_CAP);
constexpr uint32_t TMEM_COLS = 512;  // two 128 x 256 fp32 accumulators
constexpr uint32_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256 + PROF_BYTES;

enum : uint32_t { R_TILE, R_TMA_WAIT, R_TMA, R_MMA_WAIT, R_MMA, R_EPI_WAIT,
                  R_EPI_LD, R_EPI_ST };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
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

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar,
                                            void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
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

// kind::f16, A/B bf16, D f32, K-major both, M = 128, N = 256.
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) |
                           ((BN >> 3) << 17) | ((BM >> 4) << 24);

__device__ __forceinline__ void umma(uint32_t tmem, uint64_t a, uint64_t b,
                                     uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// Persistent: one CTA per SM walks tiles t = blockIdx.x, += gridDim.x in a
// grouped raster (kGroupM m-blocks x all n-blocks, m fastest) so a wave's A
// and B tiles stay in L2.  Two TMEM accumulators (2 x 256 columns): the MMA
// warp fills one while the epilogue drains the other (tmem_full / tmem_empty
// barriers), so the epilogue overlaps the next tile's main loop.
constexpr uint32_t kGroupM = 8;

__device__ __forceinline__ void tile_coords(uint32_t t, uint32_t nM, uint32_t nN,
                                            uint32_t& mb, uint32_t& nb) {
  const uint32_t per_group = kGroupM * nN;
  const uint32_t g = t / per_group, r = t % per_group;
  const uint32_t gm = min(kGroupM, nM - g * kGroupM);  // m-blocks in this group
  mb = g * kGroupM + r % gm;
  nb = r / gm;
}

// kMode: 0 plain, 1 one clock capture per RecordOp, 2 adjacent END/START
// RecordOps at scope boundaries share a capture (Recorder::mark)
template <int kMode>
__global__ void __launch_bounds__(THREADS, 1)
    k_gemm(const __grid_constant__ CUtensorMap ta,
           const __grid_constant__ CUtensorMap tb, __nv_bfloat16* C, uint32_t M,
           uint32_t N, uint32_t K, uint8_t* profile,
           wgpf_dev::CtaTiming* timing) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;   // [2]
  uint64_t* tmem_empty = tmem_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  uint8_t* prof = smem + STAGES * STAGE_BYTES + 256;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t nM = M / BM, nN = N / BN, n_tiles = nM * nN;
  const uint32_t nk = K / BK;
  const uint64_t cta = blockIdx.x;

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
    for (uint32_t s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (uint32_t a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
            smem_u32(tmem_slot)),
        "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    uint32_t it = 0;  // k-block counter across tiles
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      uint32_t mb, nb;
      tile_coords(t, nM, nN, mb, nb);
      const uint32_t m0 = mb * BM, n0 = nb * BN;
      Tile tile(rec, R_TILE);
      Phases ph_(rec);  // tma.stall -> tma.issue per k-block
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % STAGES, ph = (it / STAGES) & 1u;
        ph_.to(R_TMA_WAIT, R_TMA);
        if (lane == 0) mbar_wait(&empty[s], ph ^ 1u);
        __syncwarp();
        ph_.to(R_TMA, R_TMA_WAIT);
        if (lane == 0) {
          uint8_t* a = stage_base + s * STAGE_BYTES;
          mbar_expect_tx(&full[s], STAGE_BYTES);
          tma_load_2d(&ta, &full[s], a, (int)(kb * BK), (int)m0);
          tma_load_2d(&tb, &full[s], a + A_BYTES, (int)(kb * BK), (int)n0);
        }
        __syncwarp();
        ph_.iteration_end();
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    uint32_t it = 0, tl = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
      const uint32_t acc = tl & 1u, aph = (tl >> 1) & 1u;
      const uint32_t dt = tmem + acc * BN;
      Tile tile(rec, R_TILE);
      // the epilogue has drained this accumulator (two tiles ago)
      if (lane == 0) mbar_wait(&tmem_empty[acc], aph ^ 1u);
      __syncwarp();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      Phases ph_(rec);  // mma.stall -> mma.issue per k-block
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % STAGES, ph = (it / STAGES) & 1u;
        ph_.to(R_MMA_WAIT, R_MMA);
        if (lane == 0) mbar_wait(&full[s], ph);
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        ph_.to(R_MMA, R_MMA_WAIT);
        if (lane == 0) {
          const uint32_t a = smem_u32(stage_base + s * STAGE_BYTES);
          const uint32_t b = a + A_BYTES;
#pragma unroll
          for (uint32_t k = 0; k < BK / 16; ++k)
            umma(dt, umma_desc(a + 32u * k), umma_desc(b + 32u * k), (kb | k) != 0u);
          umma_commit(&empty[s]);
          if (kb == nk - 1) umma_commit(&tmem_full[acc]);
        }
        __syncwarp();
        ph_.iteration_end();
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> registers -> bf16 -> HBM -----------
    const uint32_t quad = warp & 3u;  // TMEM lane quadrant of this warp
    uint32_t tl = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
      uint32_t mb, nb;
      tile_coords(t, nM, nN, mb, nb);
      const uint32_t m0 = mb * BM, n0 = nb * BN;
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
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                             smem_u32(&tmem_empty[acc]))
                         : "memory");
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
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
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

uint32_t grid_ctas(uint32_t M, uint32_t N) {
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

// C[M,N] = A[M,K] . B[N,K]^T (bf16 in/out, fp32 accumulate).  M % 128,
// N % 256, K % 64 must be 0.  instrument != 0 runs the P1-instrumented kernel
// and writes the KPFT body to d_profile (wgpf_gemm_profile_bytes) and the CTA
// side records to d_timing (32 B per CTA, may be null).
// one profile segment per CTA of the persistent grid (min(tiles, SMs))
extern "C" uint64_t wgpf_gemm_profile_bytes(uint32_t M, uint32_t N) {
  return wgpf_dev::profile_bytes(grid_ctas(M, N), NWARPS, PROF_CAP);
}
extern "C" uint32_t wgpf_gemm_ctas(uint32_t M, uint32_t N) { return grid_ctas(M, N); }

extern "C" uint32_t wgpf_gemm_smem_bytes(int instrument) {
  return instrument ? SMEM_BYTES : SMEM_BYTES - PROF_BYTES;
}

extern "C" int wgpf_gemm_bf16(const void* A, const void* B, void* C, uint32_t M,
                              uint32_t N, uint32_t K, int instrument,
                              void* d_profile, void* d_timing, void* stream) {
  if (M % BM || N % BN || K % BK || K == 0) return 11;
  CUtensorMap ta, tb;
  if (!make_map(&ta, A, M, K, BM) || !make_map(&tb, B, N, K, BN)) return 10;
  dim3 grid(grid_ctas(M, N));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (instrument) {
    // instrument = 1: one capture per RecordOp; 2: shared boundary captures
    // (WGPF_P1_MODE overrides, for A/B runs)
    int mode = instrument;
    if (const char* e = getenv("WGPF_P1_MODE")) mode = atoi(e);
    auto* kfn = mode == 2 ? k_gemm<2> : k_gemm<1>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    kfn<<<grid, THREADS, SMEM_BYTES, st>>>(
        ta, tb, static_cast<__nv_bfloat16*>(C), M, N, K,
        static_cast<uint8_t*>(d_profile),
        static_cast<wgpf_dev::CtaTiming*>(d_timing));
  } else {
    cudaFuncSetAttribute(k_gemm<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SMEM_BYTES - PROF_BYTES);
    k_gemm<0><<<grid, THREADS, SMEM_BYTES - PROF_BYTES, st>>>(
        ta, tb, static_cast<__nv_bfloat16*>(C), M, N, K, nullptr, nullptr);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 10;
}
