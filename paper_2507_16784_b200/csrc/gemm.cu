// Skinny weight-streaming GEMM for decode steps: Y[M,N] (+)= X[M,K] . W[K,N]
// with M <= 64 rows (one decode row per request), bf16 in, fp32 accumulate.
//
// At decode batch sizes the four per-layer GEMMs read ~284 MB of weights for
// 64 rows: pure weight streaming.  Weights are stored transposed (Wt [N,K],
// K contiguous) so an output-column block is one contiguous slab.  The
// (n-block x k-block) chunk space is split evenly over persistent CTAs
// (stream-K): one producer warp issues TMA 2D tile loads (cp.async.bulk.tensor,
// 128B swizzle, SASS UTMALDG) of 64x64 W and X boxes into a 3-stage ring;
// 8 consumer warps run mma.sync m16n8k16 (2 n-halves x 4 k-slices of a
// 64-k box).  The k-slice partials meet in a shared fp32 tile; an n-block
// covered by one CTA is written directly (+ residual R for the o_proj / down
// projections), otherwise partials go to a workspace and the last CTA merges
// them.  The launch uses programmatic dependent launch: the weight tiles of
// the first stages stream before the preceding kernel has finished; only the
// activation tiles wait for it.
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"

namespace tim {

struct GCfg {
  static constexpr int BM = 64, BN = 64, BK = 256, KB = 64;     // KB: k extent of one TMA box
  static constexpr int NKB = BK / KB;                            // boxes per stage per operand
  static constexpr int BOX_BYTES = 64 * KB * 2;                  // 8 KiB
  static constexpr int W_BYTES = NKB * BOX_BYTES;                // 32 KiB
  static constexpr int X_BYTES = NKB * BOX_BYTES;                // 32 KiB
  static constexpr int STAGE_BYTES = W_BYTES + X_BYTES;
  static constexpr int STAGES = 3;
  static constexpr int THREADS = 9 * 32;
  static constexpr int RED_BYTES = BM * BN * 4;                  // fp32 k-slice reduction tile
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + RED_BYTES + 2 * STAGES * 8 + 64;
};

TIM_DEV void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// byte offset of (row, 16-byte chunk) inside a 128B-swizzled box of 128-byte rows
TIM_DEV uint32_t swz(int row, int chunk) { return row * 128 + ((chunk ^ (row & 7)) << 4); }

__global__ void __launch_bounds__(GCfg::THREADS, 1)
    gemm_skinny_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tw,
                       __nv_bfloat16* y, const __nv_bfloat16* res,   // may alias (in-place residual)
                       int M, int N, int K, float* __restrict__ ws, int32_t* __restrict__ counters,
                       int max_slots) {
  using C = GCfg;
  griddep_launch();   // the next kernel may launch as soon as our CTAs retire
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* red = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + C::RED_BYTES);
  uint64_t* empty = full + C::STAGES;
  int* sflag = reinterpret_cast<int*>(empty + C::STAGES);

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
      mbar_init(&empty[s], 8);
    }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < C::BM * C::BN; i += blockDim.x) red[i] = 0.f;
  __syncthreads();

  if (warp == 8) {
    // ---------------------------------------------------------- producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tw)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tx)) : "memory");
      bool waited = false;
      int it = 0;
      for (int64_t ch = start; ch < end; ++ch, ++it) {
        const int nb = (int)(ch / kblk), kb = (int)(ch - (int64_t)nb * kblk);
        const int stg = it % C::STAGES;
        if (it >= C::STAGES) mbar_wait(&empty[stg], ((it / C::STAGES) & 1) ^ 1);
        uint8_t* base = smem + stg * C::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[stg], C::STAGE_BYTES);
        // weights never depend on the preceding kernel: stream them first
#pragma unroll
        for (int j = 0; j < C::NKB; ++j)
          tma_load_2d(base + j * C::BOX_BYTES, &tw, kb * C::BK + j * C::KB, nb * C::BN, &full[stg]);
        if (!waited) {
          griddep_wait();   // activations come from the preceding kernel
          waited = true;
        }
#pragma unroll
        for (int j = 0; j < C::NKB; ++j)
          tma_load_2d(base + C::W_BYTES + j * C::BOX_BYTES, &tx, kb * C::BK + j * C::KB, 0, &full[stg]);
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  // warp = (kh, nq): k half of the stage (boxes 2kh, 2kh+1) x 16-column quarter.
  griddep_wait();                      // residual input may come from the preceding kernel
  const int kh = warp >> 2, nq = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const uint32_t sbase = smem_u32(smem);
  int it = 0;
  int64_t ch = start;
  while (ch < end) {
    const int nb = (int)(ch / kblk);
    const int64_t nb_lo = (int64_t)nb * kblk, nb_hi = nb_lo + kblk;
    const int64_t pend = end < nb_hi ? end : nb_hi;
    float acc[4][2][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = acc[a][b][2] = acc[a][b][3] = 0.f;

    for (; ch < pend; ++ch, ++it) {
      const int stg = it % C::STAGES;
      mbar_wait(&full[stg], (it / C::STAGES) & 1);
#pragma unroll
      for (int bx = 0; bx < 2; ++bx) {
        const uint32_t wbox = sbase + stg * C::STAGE_BYTES + (kh * 2 + bx) * C::BOX_BYTES;
        const uint32_t xbox = wbox + C::W_BYTES;
#pragma unroll
        for (int ks = 0; ks < C::KB / 16; ++ks) {
          uint32_t b0, b1, b2, b3;
          {
            const int mi = lane >> 3;
            const int n = nq * 16 + (mi >> 1) * 8 + (lane & 7);
            ldsm_x4(b0, b1, b2, b3, wbox + swz(n, ks * 2 + (mi & 1)));
          }
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            uint32_t a0, a1, a2, a3;
            const int mi = lane >> 3;
            const int row = mt * 16 + (lane & 7) + (mi & 1) * 8;
            ldsm_x4(a0, a1, a2, a3, xbox + swz(row, ks * 2 + (mi >> 1)));
            mma_bf16(acc[mt][0], a0, a1, a2, a3, b0, b1);
            mma_bf16(acc[mt][1], a0, a1, a2, a3, b2, b3);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stg]);
    }

    // ---- k-half reduction: kh=1 warps park their tile in smem, kh=0 warps add it
    if (kh == 1) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = mt * 16 + g + 8 * h, col = nq * 16 + nt * 8 + 2 * t;
            *reinterpret_cast<float2*>(&red[row * C::BN + col]) =
                make_float2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]);
          }
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (kh == 0) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = mt * 16 + g + 8 * h, col = nq * 16 + nt * 8 + 2 * t;
            float2* p = reinterpret_cast<float2*>(&red[row * C::BN + col]);
            const float2 o = *p;
            *p = make_float2(o.x + acc[mt][nt][2 * h], o.y + acc[mt][nt][2 * h + 1]);
          }
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");

    const int64_t c_first = (nb_lo * G + G - 1) / total;   // first CTA whose range meets the n-block
    int64_t c_last = ((nb_hi) * G - 1) / total;            // CTA holding chunk nb_hi-1
    if (c_last >= G) c_last = G - 1;
    const int npieces = (int)(c_last - c_first + 1);
    const int n0 = nb * C::BN;
    bool write_out = npieces == 1;
    if (!write_out) {
      const int64_t slot = c + nb;
      float* dst = ws + slot * (C::BM * C::BN);
      for (int i = threadIdx.x; i < C::BM * C::BN / 4; i += 256)
        __stcg(reinterpret_cast<float4*>(dst) + i, reinterpret_cast<const float4*>(red)[i]);
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (threadIdx.x == 0) {
        int old;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                     : "=r"(old) : "l"(counters + nb) : "memory");
        const int last = old == npieces - 1;
        if (last) counters[nb] = 0;
        *sflag = last;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      write_out = *sflag != 0;
      if (write_out) {
        for (int i = threadIdx.x; i < C::BM * C::BN / 4; i += 256) {
          float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int64_t cc = c_first; cc <= c_last; ++cc) {
            const float4 v = __ldcg(reinterpret_cast<const float4*>(ws + (cc + nb) * (C::BM * C::BN)) + i);
            s4.x += v.x; s4.y += v.y; s4.z += v.z; s4.w += v.w;
          }
          reinterpret_cast<float4*>(red)[i] = s4;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
    }
    if (write_out) {
      // epilogue: y = (res +) acc for the valid rows, 4 columns per thread
      for (int i = threadIdx.x; i < C::BM * C::BN / 4; i += 256) {
        const int row = i / (C::BN / 4), col = (i - row * (C::BN / 4)) * 4;
        if (row >= M) continue;
        const float4 v = reinterpret_cast<const float4*>(red)[i];
        float o0 = v.x, o1 = v.y, o2 = v.z, o3 = v.w;
        const int64_t off = (int64_t)row * N + n0 + col;
        if (res) {
          uint2 rr;
          asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(rr.x), "=r"(rr.y) : "l"(res + off));
          const __nv_bfloat162 r01 = *reinterpret_cast<const __nv_bfloat162*>(&rr.x);
          const __nv_bfloat162 r23 = *reinterpret_cast<const __nv_bfloat162*>(&rr.y);
          o0 += __low2float(r01); o1 += __high2float(r01);
          o2 += __low2float(r23); o3 += __high2float(r23);
        }
        uint2 pk;
        pk.x = pack_bf16(o0, o1);
        pk.y = pack_bf16(o2, o3);
        *reinterpret_cast<uint2*>(y + off) = pk;
      }
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
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

extern "C" int64_t tim_gemm_ws_floats(int32_t n_ctas, int32_t n) {
  return (int64_t)(n_ctas + n / GCfg::BN) * GCfg::BM * GCfg::BN;
}

extern "C" int32_t tim_gemm_skinny(const void* tmap_x, const void* tmap_w, void* y, const void* res,
                                   int32_t M, int32_t N, int32_t K, float* ws, int32_t* counters,
                                   int32_t n_ctas, void* stream) {
  if (M > GCfg::BM || M <= 0 || N % GCfg::BN || K % GCfg::BK) {
    set_last_error("gemm_skinny: M <= 64, N %% 64 == 0, K %% 256 == 0 required (M=%d N=%d K=%d)", M, N, K);
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
                                           (const __nv_bfloat16*)res, M, N, K, ws, counters,
                                           n_ctas + N / GCfg::BN);
  if (e != cudaSuccess) {
    set_last_error("gemm_skinny launch: %s", cudaGetErrorString(e));
    return TIM_CUDA_ERROR;
  }
  return check_launch("gemm_skinny");
}
