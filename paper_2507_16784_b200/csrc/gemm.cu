// Skinny weight-streaming GEMM for decode steps on the 5th-gen tensor cores:
// Y[M,N] (+)= X[M,K] . W[K,N] with M <= 64 rows (one decode row per request),
// bf16 in, fp32 accumulate in TMEM.
//
// At decode batch sizes the four per-layer GEMMs read ~284 MB of weights for
// 64 rows: pure weight streaming, so the kernel is built around keeping HBM
// busy.  Weights are stored transposed (Wt [N,K], K contiguous) and play the
// MMA's A operand (UMMA M = 128 weight rows), the activations are B (UMMA
// N = 64 rows), so D^T = Wt . X^T lands in TMEM as 128 lanes (output columns)
// x 64 TMEM columns (rows of Y).
//
// The (n-block 128 x k-block 128) chunk space is split evenly over persistent
// CTAs (stream-K).  Warp roles per CTA (one CTA per SM):
//   warp 0     TMA producer: cp.async.bulk.tensor 2D loads (128B swizzle) of the
//              W (128x128) and X (64x128) tiles into a 4-stage ring (48 KiB/stage)
//   warp 1     TMEM owner + MMA issuer: one thread issues tcgen05.mma
//              (kind::f16, 128x64x16) and tcgen05.commit's the stage back
//   warps 2-5  epilogue: tcgen05.ld the 128x64 accumulator (double-buffered in
//              TMEM, so the next n-block's MMAs overlap the epilogue), then
//              write Y (+ residual) directly when one CTA covered the whole
//              n-block, else park an fp32 partial in a workspace; the last CTA
//              to arrive on the n-block's counter merges the partials.
// Programmatic dependent launch: the weight tiles of the first stages stream
// before the preceding kernel has finished; activation tiles, the residual and
// the workspace wait for it (griddepcontrol.wait).
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"

namespace tim {

struct GCfg {
  static constexpr int BM = 64;                 // activation rows (UMMA N)
  static constexpr int BN = 128;                // weight rows per tile (UMMA M)
  static constexpr int BK = 128;                // k per stage
  static constexpr int KB = 64;                 // k extent of one TMA box (128 bytes)
  static constexpr int NKB = BK / KB;
  static constexpr int W_BOX = BN * KB * 2;     // 16 KiB
  static constexpr int X_BOX = BM * KB * 2;     // 8 KiB
  static constexpr int W_BYTES = NKB * W_BOX;
  static constexpr int STAGE_BYTES = NKB * (W_BOX + X_BOX);
  static constexpr int STAGES = 4;
  static constexpr int THREADS = 6 * 32;
  static constexpr int TMEM_COLS = 2 * BM;      // two accumulator buffers
  static constexpr int OUT_BYTES = BM * BN * 2;  // bf16 residual-in / Y-out staging tile
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + OUT_BYTES + 256;
};

TIM_DEV void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor: K-major operand, 128B swizzle, 8-row groups
// 1024 bytes apart (the layout TMA writes for a 128-byte-wide box).
TIM_DEV uint64_t umma_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major, M=128, N=64
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(GCfg::BM >> 3) << 17) |
                            ((uint32_t)(GCfg::BN >> 4) << 24);

TIM_DEV void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
      : "memory");
}

TIM_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

TIM_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
TIM_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

TIM_DEV void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(taddr));
}

__device__ unsigned long long g_gtrace[160 * 16];   // per-CTA phase timestamps (diagnostics)
TIM_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GT(i) do { if (trace) g_gtrace[blockIdx.x * 16 + (i)] = gtime(); } while (0)

struct Piece {   // the chunks [lo, hi) of one n-block owned by this CTA
  int nb;
  int64_t lo, hi;
};

__global__ void __launch_bounds__(GCfg::THREADS, 1)
    gemm_skinny_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tw,
                       __nv_bfloat16* y, const __nv_bfloat16* res,   // may alias (in-place residual)
                       int M, int N, int K, float* __restrict__ ws, int32_t* __restrict__ counters, int trace) {
  using C = GCfg;
  griddep_launch();
  if (threadIdx.x == 0) GT(0);   // the next kernel may launch as soon as our CTAs retire
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* otile = reinterpret_cast<__nv_bfloat16*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + C::OUT_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;       // [2] accumulator ready
  uint64_t* tempty = tfull + 2;              // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* sflag = reinterpret_cast<int*>(tmem_slot + 1);

  const int nblk = N / C::BN, kblk = K / C::BK;
  const int64_t total = (int64_t)nblk * kblk;
  const int64_t G = gridDim.x < total ? gridDim.x : total;
  const int c = blockIdx.x;
  if (c >= G) return;
  const int64_t start = (int64_t)c * total / G, end = (int64_t)(c + 1) * total / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tw)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tx)) : "memory");
      const int64_t n = end - start;
      const int pre = n < C::STAGES ? (int)n : C::STAGES;
      // weights never depend on the preceding kernel: fill the ring's W halves first
      for (int it = 0; it < pre; ++it) {
        const int64_t ch = start + it;
        const int nb = (int)(ch / kblk), kb = (int)(ch - (int64_t)nb * kblk);
        uint8_t* base = smem + it * C::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[it], C::STAGE_BYTES);
#pragma unroll
        for (int j = 0; j < C::NKB; ++j)
          tma_load_2d(base + j * C::W_BOX, &tw, kb * C::BK + j * C::KB, nb * C::BN, &full[it]);
      }
      GT(1);
      griddep_wait();   // activations come from the preceding kernel
      GT(2);
      for (int it = 0; it < pre; ++it) {
        const int64_t ch = start + it;
        const int nb = (int)(ch / kblk), kb = (int)(ch - (int64_t)nb * kblk);
        uint8_t* base = smem + it * C::STAGE_BYTES + C::W_BYTES;
#pragma unroll
        for (int j = 0; j < C::NKB; ++j)
          tma_load_2d(base + j * C::X_BOX, &tx, kb * C::BK + j * C::KB, 0, &full[it]);
      }
      for (int it = pre; it < n; ++it) {
        const int64_t ch = start + it;
        const int nb = (int)(ch / kblk), kb = (int)(ch - (int64_t)nb * kblk);
        const int stg = it % C::STAGES;
        mbar_wait(&empty[stg], ((it / C::STAGES) & 1) ^ 1);
        uint8_t* base = smem + stg * C::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[stg], C::STAGE_BYTES);
#pragma unroll
        for (int j = 0; j < C::NKB; ++j)
          tma_load_2d(base + j * C::W_BOX, &tw, kb * C::BK + j * C::KB, nb * C::BN, &full[stg]);
#pragma unroll
        for (int j = 0; j < C::NKB; ++j)
          tma_load_2d(base + C::W_BYTES + j * C::X_BOX, &tx, kb * C::BK + j * C::KB, 0, &full[stg]);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t sbase = smem_u32(smem);
      int it = 0, pi = 0;
      for (int64_t ch = start; ch < end; ++pi) {
        const int nb = (int)(ch / kblk);
        const int64_t pend = end < (int64_t)(nb + 1) * kblk ? end : (int64_t)(nb + 1) * kblk;
        const int a = pi & 1;
        if (pi >= 2) mbar_wait(&tempty[a], ((pi >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + a * C::BM;
        for (bool first = true; ch < pend; ++ch, ++it, first = false) {
          const int stg = it % C::STAGES;
          mbar_wait(&full[stg], (it / C::STAGES) & 1);
          if (it == 0) GT(3);
          tc_fence_after();
          const uint32_t wb = sbase + stg * C::STAGE_BYTES, xb = wb + C::W_BYTES;
#pragma unroll
          for (int kk = 0; kk < C::BK / 16; ++kk) {
            const uint32_t off = (kk & 3) * 32;
            umma_f16(d, umma_desc(wb + (kk >> 2) * C::W_BOX + off), umma_desc(xb + (kk >> 2) * C::X_BOX + off),
                     (first && kk == 0) ? 0u : 1u);
          }
          umma_commit(&empty[stg]);   // stage reusable once these MMAs have read it
        }
        umma_commit(&tfull[a]);       // accumulator complete
      }
      GT(4);
    }
  } else {
    // ---------------------------------------------------------- epilogue
    griddep_wait();   // residual / workspace / counters are shared with the preceding kernel
    const int q = warp & 3;                    // TMEM lane quadrant this warp may access
    const int r = q * 32 + lane;               // output column within the n-block
    int pi = 0;
    for (int64_t ch = start; ch < end; ++pi) {
      const int nb = (int)(ch / kblk);
      const int64_t nb_lo = (int64_t)nb * kblk, nb_hi = nb_lo + kblk;
      ch = end < nb_hi ? end : nb_hi;
      const int a = pi & 1;
      const int n0 = nb * C::BN;
      // residual tile [64 rows][128 cols] of this block: cp.async'ed into the
      // staging tile while the MMAs are still running (res may alias y; only
      // the last piece of the block writes y, after every piece passed here)
      if (res) {
#pragma unroll
        for (int i = 0; i < C::OUT_BYTES / 16 / 128; ++i) {
          const int ck = (threadIdx.x - 64) + 128 * i, row = ck >> 4, c16 = ck & 15;
          if (row < M) cp_async16(otile + row * C::BN + c16 * 8, res + (int64_t)row * N + n0 + c16 * 8);
        }
        cp_async_commit();
      }
      mbar_wait(&tfull[a], (pi >> 1) & 1);
      if (threadIdx.x == 64) GT(5);
      tc_fence_after();
      float v[C::BM];
      {
        uint32_t t0[32], t1[32];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + a * C::BM;
        tmem_ld32(ta, t0);
        tmem_ld32(ta + 32, t1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          v[j] = __uint_as_float(t0[j]);
          v[32 + j] = __uint_as_float(t1[j]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);

      const int64_t c_first = (nb_lo * G + G - 1) / total;   // first CTA whose range meets the n-block
      int64_t c_last = (nb_hi * G - 1) / total;               // CTA holding chunk nb_hi-1
      if (c_last >= G) c_last = G - 1;
      bool write_out = c_first == c_last;
      if (!write_out) {
        // split n-block: every piece adds into the block's fp32 tile in L2
        // ([16][128][4]: a warp's v4 reductions are 512 contiguous bytes);
        // the last piece to arrive reads the sum back and re-zeroes the tile.
        float* tile = ws + (int64_t)nb * (C::BM * C::BN) + r * 4;
#pragma unroll
        for (int jq = 0; jq < C::BM / 4; ++jq)
          asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(tile + jq * C::BN * 4),
                       "f"(v[4 * jq]), "f"(v[4 * jq + 1]), "f"(v[4 * jq + 2]), "f"(v[4 * jq + 3])
                       : "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          int old;
          asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                       : "=r"(old) : "l"(counters + nb) : "memory");
          const int last = old == (int)(c_last - c_first);
          if (last) counters[nb] = 0;
          *sflag = last;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) GT(7);
        write_out = *sflag != 0;
        if (write_out) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
#pragma unroll
          for (int jq = 0; jq < C::BM / 4; ++jq) {
            const float4 t4 = __ldcg(reinterpret_cast<const float4*>(tile + jq * C::BN * 4));
            v[4 * jq] = t4.x; v[4 * jq + 1] = t4.y; v[4 * jq + 2] = t4.z; v[4 * jq + 3] = t4.w;
          }
#pragma unroll
          for (int jq = 0; jq < C::BM / 4; ++jq)
            __stcg(reinterpret_cast<float4*>(tile + jq * C::BN * 4), make_float4(0.f, 0.f, 0.f, 0.f));
          if (trace && threadIdx.x == 64) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : "f"(v[63]));
            g_gtrace[blockIdx.x * 16 + 8] = t;
          }
        }
      }
      if (write_out) {
        // this thread's column (+ residual) -> staging tile; then 16-byte rows out
        if (res) cp_async_wait<0>();
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
        for (int j = 0; j < C::BM; ++j) {
          if (j < M) {
            __nv_bfloat16* o = otile + j * C::BN + r;
            float val = v[j];
            if (res) val += __bfloat162float(*o);
            *o = __float2bfloat16_rn(val);
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
        for (int i = 0; i < C::OUT_BYTES / 16 / 128; ++i) {
          const int ck = (threadIdx.x - 64) + 128 * i, row = ck >> 4, c16 = ck & 15;
          if (row < M)
            *reinterpret_cast<uint4*>(y + (int64_t)row * N + n0 + c16 * 8) =
                *reinterpret_cast<const uint4*>(otile + row * C::BN + c16 * 8);
        }
      } else if (res) {
        cp_async_wait<0>();   // drain the unused prefetch before the tile is refilled
      }
    }
  }
  if (threadIdx.x == 64) GT(6);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS)
                 : "memory");
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

}  // namespace tim

using namespace tim;

extern "C" int32_t tim_tmap_2d_bf16(void* tmap_out, const void* base, int64_t rows, int64_t cols,
                                    int32_t box_rows, int32_t box_cols) {
  if (g_encode == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    const cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || fn == nullptr) {
      set_last_error("cuTensorMapEncodeTiled unavailable");
      return TIM_CUDA_ERROR;
    }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (box_cols * 2 != 128 || box_rows > 256 || (cols * 2) % 16) {
    set_last_error("tmap: box must be 128 bytes wide, row pitch a multiple of 16 bytes");
    return TIM_BAD_ARGUMENT;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = g_encode(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                              2, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return TIM_CUDA_ERROR;
  }
  return TIM_OK;
}

static int g_gemm_trace = 0;
extern "C" int32_t tim_gemm_trace(int32_t on, uint64_t* out, int32_t n) {
  g_gemm_trace = on;
  if (out) {
    if (cudaMemcpyFromSymbol(out, g_gtrace, sizeof(uint64_t) * n) != cudaSuccess) return TIM_CUDA_ERROR;
  }
  return TIM_OK;
}

extern "C" int64_t tim_gemm_ws_floats(int32_t n_ctas, int32_t n) {
  (void)n_ctas;
  return (int64_t)(n / GCfg::BN) * GCfg::BM * GCfg::BN;
}

extern "C" int32_t tim_gemm_skinny(const void* tmap_x, const void* tmap_w, void* y, const void* res,
                                   int32_t M, int32_t N, int32_t K, float* ws, int32_t* counters,
                                   int32_t n_ctas, void* stream) {
  if (M > GCfg::BM || M <= 0 || N % GCfg::BN || K % GCfg::BK) {
    set_last_error("gemm_skinny: M <= 64, N %% 128 == 0, K %% 128 == 0 required (M=%d N=%d K=%d)", M, N, K);
    return TIM_BAD_ARGUMENT;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_skinny_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GCfg::SMEM);
    attr = true;
  }
  CUtensorMap mx, mw;
  memcpy(&mx, tmap_x, sizeof(mx));
  memcpy(&mw, tmap_w, sizeof(mw));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(GCfg::THREADS);
  cfg.dynamicSmemBytes = GCfg::SMEM;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_skinny_kernel, mx, mw, (__nv_bfloat16*)y,
                                           (const __nv_bfloat16*)res, M, N, K, ws, counters, g_gemm_trace);
  if (e != cudaSuccess) {
    set_last_error("gemm_skinny launch: %s", cudaGetErrorString(e));
    return TIM_CUDA_ERROR;
  }
  return check_launch("gemm_skinny");
}
