// Paged GQA attention over the retained working memory (page size 1).
//
// Reference semantics (model.py:139-159): per layer, queries of the new block
// attend every page of the request's table (the retained prefix, fully
// visible) plus the new block causally; scores = q.k / sqrt(D), softmax with
// max subtraction, ctx = softmax @ V.  The reference has Hq == Hkv; GQA maps
// q head h to kv head h / (Hq/Hkv) (HF repeat_kv convention).
//
// K1 (decode, bf16 KV): persistent stream-K kernel.  The concatenated kv
//   tokens of all decode queries are split evenly over the CTAs, so load is
//   balanced whatever the retained lengths are.  One CTA = 1 producer warp
//   that streams whole page rows (all kv heads of a token: Hkv*D*2 bytes,
//   contiguous in the [layer][page][Hkv][D] pool) into a multi-stage shared
//   ring with TMA bulk copies (cp.async.bulk, SASS UBLKCP) + mbarriers, and
//   Hkv consumer warps (one per kv head) that run QK^T and PV on the tensor
//   cores (mma.sync m16n8k16 bf16, fp32 accumulate) with an online softmax.
//   Queries split across CTAs are merged in-kernel (K6) by the last CTA to
//   finish (threadfence + counter), with a log-sum-exp combine.
// K2 (extend / re-encode, bf16 KV): FA2-style q-tiles of 64 rows
//   (queries x group heads) per (item, kv head), cp.async 3-stage ring.
// Generic (fp32 / any): warp per (row, q head), exact two-pass softmax; used
//   for the fp32 parity configuration.
#include "common.cuh"

namespace tim {

constexpr float kLog2e = 1.4426950408889634f;
constexpr int kMaxHeads = 128;      // hq bound for the in-kernel combine
constexpr int kCombineChunk = 8;    // partials merged per smem pass
constexpr int kIdChunk = 1024;      // page ids staged per producer refill (multiple of TK)

// ===================================================================== K1
template <int D, int HKV>
struct DecCfg {
  static constexpr int TK = 16;                       // tokens per stage
  static constexpr int ROW_BYTES = HKV * D * 2;       // one page, all kv heads, one layer
  static constexpr int ROW_STRIDE = ROW_BYTES + 16;   // +16B: conflict-free ldmatrix rows
  static constexpr int STAGE_BYTES = 2 * TK * ROW_STRIDE;
  static constexpr int STAGES_RAW = 204800 / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr int THREADS = (HKV + 1) * 32;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 2 * STAGES * 8 + 16 + kIdChunk * 4;
  static constexpr int KC = D / 16;
  static constexpr int NT = D / 8;
};

__device__ __forceinline__ int64_t cta_of(int64_t x, int64_t G, int64_t N) {
  return ((x + 1) * G - 1) / N;
}

template <int D, int HKV>
__global__ void __launch_bounds__(DecCfg<D, HKV>::THREADS, 1)
    attn_decode_kernel(const int32_t* __restrict__ step, const __nv_bfloat16* __restrict__ q,
                       __nv_bfloat16* __restrict__ out, const __nv_bfloat16* __restrict__ kl,
                       const __nv_bfloat16* __restrict__ vl, const int32_t* __restrict__ tables,
                       int64_t tstride, int hq, float scale, float* __restrict__ ws,
                       int32_t* __restrict__ counters, int max_dec) {
  using C = DecCfg<D, HKV>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  int* sflag = reinterpret_cast<int*>(empty + C::STAGES);
  __shared__ float s_m[kMaxHeads], s_inv[kMaxHeads];
  __shared__ float s_w[kCombineChunk][kMaxHeads];

  const tim_step_header& hd = *reinterpret_cast<const tim_step_header*>(step);
  const int n_dec = hd.n_dec;
  const int64_t N = hd.dec_total;
  if (n_dec == 0 || N == 0) return;
  const int64_t G = gridDim.x < N ? gridDim.x : N;
  const int c = blockIdx.x;
  if (c >= G) return;
  const int32_t* dec = step + hd.off_dec;
  const int32_t* prefix = step + hd.off_dec_prefix;
  const int64_t start = (int64_t)c * N / G, end = (int64_t)(c + 1) * N / G;

  // first segment of this CTA: largest r with prefix[r] <= start
  int r0 = 0;
  {
    int lo = 0, hi = n_dec - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= start) lo = mid; else hi = mid - 1;
    }
    r0 = lo;
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], HKV);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == HKV) {
    // ------------------------------------------------------------ producer
    // Page ids of the piece are staged into shared memory a chunk at a time
    // (one coalesced read per kIdChunk tokens), so the id latency is off the
    // per-stage critical path; each stage is then 2*TK bulk copies.
    int32_t* s_ids = reinterpret_cast<int32_t*>(sflag + 4);
    int it = 0;
    for (int r = r0; r < n_dec && prefix[r] < end; ++r) {
      const int64_t lo = prefix[r], hi = prefix[r + 1];
      const int p0 = (int)((start > lo ? start : lo) - lo);
      const int p1 = (int)((end < hi ? end : hi) - lo);
      const int32_t* trow = tables + (int64_t)dec[r * TIM_DEC_FIELDS + 1] * tstride;
      for (int c0 = p0; c0 < p1; c0 += kIdChunk) {
        const int c1 = (p1 - c0) < kIdChunk ? p1 : c0 + kIdChunk;
        __syncwarp();
#pragma unroll 8
        for (int i = lane; i < c1 - c0; i += 32) s_ids[i] = __ldg(trow + c0 + i);
        __syncwarp();
        for (int k0 = c0; k0 < c1; k0 += C::TK, ++it) {
          const int ntok = (c1 - k0) < C::TK ? (c1 - k0) : C::TK;
          const int stg = it % C::STAGES;
          if (it >= C::STAGES) mbar_wait(&empty[stg], ((it / C::STAGES) & 1) ^ 1);
          if (lane == 0) mbar_arrive_expect_tx(&full[stg], 2 * C::TK * C::ROW_BYTES);
          __syncwarp();
          const int row = lane & (C::TK - 1);
          const int32_t page = s_ids[k0 - c0 + (row < ntok ? row : ntok - 1)];  // pad rows repeat a valid row
          uint8_t* base = smem + stg * C::STAGE_BYTES + (lane >= C::TK ? C::TK * C::ROW_STRIDE : 0);
          const __nv_bfloat16* src = (lane >= C::TK ? vl : kl) + (int64_t)page * (HKV * D);
          bulk_g2s(base + row * C::ROW_STRIDE, src, C::ROW_BYTES, &full[stg]);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int grp = hq / HKV;             // q heads per kv head (rows used of the m16 tile)
  const int g = lane >> 2, t = lane & 3;
  const float sl = scale * kLog2e;
  const uint32_t smem_base = smem_u32(smem);
  float* ws_o = ws;
  float* ws_ml = ws + (int64_t)(gridDim.x + max_dec) * hq * D;
  int it = 0;

  for (int r = r0; r < n_dec && prefix[r] < end; ++r) {
    const int64_t lo = prefix[r], hi = prefix[r + 1];
    const int p0 = (int)((start > lo ? start : lo) - lo);
    const int p1 = (int)((end < hi ? end : hi) - lo);
    const int qrow = dec[r * TIM_DEC_FIELDS + 0];

    // Q fragments (A operand, rows = heads of this kv group, k = d)
    uint32_t qa[C::KC][4];
    {
      const __nv_bfloat16* qb = q + ((int64_t)qrow * hq + warp * grp) * D;
#pragma unroll
      for (int kc = 0; kc < C::KC; ++kc) {
        const int d0 = kc * 16 + 2 * t;
        qa[kc][0] = g < grp ? *reinterpret_cast<const uint32_t*>(qb + g * D + d0) : 0u;
        qa[kc][1] = g + 8 < grp ? *reinterpret_cast<const uint32_t*>(qb + (g + 8) * D + d0) : 0u;
        qa[kc][2] = g < grp ? *reinterpret_cast<const uint32_t*>(qb + g * D + d0 + 8) : 0u;
        qa[kc][3] = g + 8 < grp ? *reinterpret_cast<const uint32_t*>(qb + (g + 8) * D + d0 + 8) : 0u;
      }
    }
    float o[C::NT][4];
#pragma unroll
    for (int i = 0; i < C::NT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

    for (int k0 = p0; k0 < p1; k0 += C::TK, ++it) {
      const int ntok = (p1 - k0) < C::TK ? (p1 - k0) : C::TK;
      const int stg = it % C::STAGES;
      mbar_wait(&full[stg], (it / C::STAGES) & 1);
      const uint32_t kbase = smem_base + stg * C::STAGE_BYTES + warp * D * 2;
      const uint32_t vbase = kbase + C::TK * C::ROW_STRIDE;

      float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
      {
        const int mi = lane >> 3;
        const int tok = (lane & 7) + (mi >> 1) * 8;
        const uint32_t a = kbase + tok * C::ROW_STRIDE + (mi & 1) * 16;
#pragma unroll
        for (int kc = 0; kc < C::KC; ++kc) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(b0, b1, b2, b3, a + kc * 32);
          mma_bf16(s0, qa[kc][0], qa[kc][1], qa[kc][2], qa[kc][3], b0, b1);
          mma_bf16(s1, qa[kc][0], qa[kc][1], qa[kc][2], qa[kc][3], b2, b3);
        }
      }
      // online softmax (log2 domain); row g -> v[0], row g+8 -> v[1]
      float v[2][4] = {{s0[0], s0[1], s1[0], s1[1]}, {s0[2], s0[3], s1[2], s1[3]}};
      const int tk[4] = {2 * t, 2 * t + 1, 8 + 2 * t, 9 + 2 * t};
      float corr[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[h][j] = tk[j] < ntok ? v[h][j] * sl : -INFINITY;
          mx = fmaxf(mx, v[h][j]);
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float mnew = fmaxf(m_r[h], mx);
        const float muse = mnew == -INFINITY ? 0.f : mnew;
        corr[h] = fast_exp2(m_r[h] - muse);
        float sum = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[h][j] = fast_exp2(v[h][j] - muse);
          sum += v[h][j];
        }
        l_r[h] = l_r[h] * corr[h] + sum;
        m_r[h] = mnew;
      }
#pragma unroll
      for (int i = 0; i < C::NT; ++i) {
        o[i][0] *= corr[0];
        o[i][1] *= corr[0];
        o[i][2] *= corr[1];
        o[i][3] *= corr[1];
      }
      const uint32_t pa0 = pack_bf16(v[0][0], v[0][1]);
      const uint32_t pa1 = pack_bf16(v[1][0], v[1][1]);
      const uint32_t pa2 = pack_bf16(v[0][2], v[0][3]);
      const uint32_t pa3 = pack_bf16(v[1][2], v[1][3]);
      {
        const int mi = lane >> 3;
        const int tok = (lane & 7) + (mi & 1) * 8;
        const uint32_t a = vbase + tok * C::ROW_STRIDE + (mi >> 1) * 16;
#pragma unroll
        for (int j = 0; j < C::NT / 2; ++j) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(b0, b1, b2, b3, a + j * 32);
          mma_bf16(o[2 * j], pa0, pa1, pa2, pa3, b0, b1);
          mma_bf16(o[2 * j + 1], pa0, pa1, pa2, pa3, b2, b3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stg]);
    }

    // ------------------------------------------------------------ epilogue
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 1);
      l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 2);
    }
    const int64_t c_first = cta_of(lo, G, N), c_last = cta_of(hi - 1, G, N);
    const int npieces = (int)(c_last - c_first + 1);
    if (npieces == 1) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = g + 8 * h;
        if (rr < grp) {
          const float inv = 1.f / l_r[h];
          __nv_bfloat16* ob = out + ((int64_t)qrow * hq + warp * grp + rr) * D;
#pragma unroll
          for (int i = 0; i < C::NT; ++i)
            *reinterpret_cast<uint32_t*>(ob + i * 8 + 2 * t) =
                pack_bf16(o[i][2 * h] * inv, o[i][2 * h + 1] * inv);
        }
      }
      continue;
    }
    const int64_t slot = c + r;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rr = g + 8 * h;
      if (rr < grp) {
        const int head = warp * grp + rr;
        float* ob = ws_o + (slot * hq + head) * D;
#pragma unroll
        for (int i = 0; i < C::NT; ++i)
          __stcg(reinterpret_cast<float2*>(ob + i * 8 + 2 * t), make_float2(o[i][2 * h], o[i][2 * h + 1]));
        if (t == 0) __stcg(reinterpret_cast<float2*>(ws_ml + (slot * hq + head) * 2), make_float2(m_r[h], l_r[h]));
      }
    }
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"n"(HKV * 32));
    if (threadIdx.x == 0) {
      const int old = atomicAdd(&counters[r], 1);
      const int last = old == npieces - 1;
      if (last) counters[r] = 0;
      *sflag = last;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(HKV * 32));
    if (*sflag) {
      __threadfence();
      // K6: log-sum-exp merge of this query's partials (slots c' + r).  Per
      // head: M = max m_p, weight_p = exp2(m_p - M) / sum_q exp2(m_q - M) l_q;
      // then every thread merges float4 slices of the hq*D outputs.
      const int nthr = HKV * 32;
      for (int h = threadIdx.x; h < hq; h += nthr) {
        float M = -INFINITY;
        for (int64_t cc = c_first; cc <= c_last; ++cc)
          M = fmaxf(M, __ldcg(ws_ml + ((cc + r) * hq + h) * 2));
        float den = 0.f;
        for (int64_t cc = c_first; cc <= c_last; ++cc) {
          const float2 ml = __ldcg(reinterpret_cast<const float2*>(ws_ml + ((cc + r) * hq + h) * 2));
          den += (ml.x == -INFINITY ? 0.f : fast_exp2(ml.x - M)) * ml.y;
        }
        s_m[h] = M;
        s_inv[h] = 1.f / den;
      }
      constexpr int V4 = 4;  // float4 slices per thread per pass
      const int n4 = hq * D / 4;
      for (int base = 0; base < n4; base += nthr * V4) {
        float4 acc[V4];
#pragma unroll
        for (int k = 0; k < V4; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t c0 = c_first; c0 <= c_last; c0 += kCombineChunk) {
          const int np = (int)((c_last - c0 + 1) < kCombineChunk ? (c_last - c0 + 1) : kCombineChunk);
          asm volatile("bar.sync 1, %0;" ::"n"(HKV * 32));
          for (int i = threadIdx.x; i < np * hq; i += nthr) {
            const int pp = i / hq, h = i - pp * hq;
            const float mm = __ldcg(ws_ml + ((c0 + pp + r) * hq + h) * 2);
            s_w[pp][h] = mm == -INFINITY ? 0.f : fast_exp2(mm - s_m[h]) * s_inv[h];
          }
          asm volatile("bar.sync 1, %0;" ::"n"(HKV * 32));
          for (int pp = 0; pp < np; ++pp) {
            const float4* src = reinterpret_cast<const float4*>(ws_o + (c0 + pp + r) * hq * D);
#pragma unroll
            for (int k = 0; k < V4; ++k) {
              const int e4 = base + threadIdx.x + k * nthr;
              if (e4 < n4) {
                const float w = s_w[pp][(e4 * 4) / D];
                const float4 v = __ldcg(src + e4);
                acc[k].x += w * v.x; acc[k].y += w * v.y; acc[k].z += w * v.z; acc[k].w += w * v.w;
              }
            }
          }
        }
#pragma unroll
        for (int k = 0; k < V4; ++k) {
          const int e4 = base + threadIdx.x + k * nthr;
          if (e4 < n4) {
            uint2 pk;
            pk.x = pack_bf16(acc[k].x, acc[k].y);
            pk.y = pack_bf16(acc[k].z, acc[k].w);
            *reinterpret_cast<uint2*>(out + (int64_t)qrow * hq * D + e4 * 4) = pk;
          }
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(HKV * 32));
  }
}

// ===================================================================== K2
template <int D>
struct ExtCfg {
  static constexpr int TK = 32;
  static constexpr int ROW_BYTES = D * 2;
  static constexpr int ROW_STRIDE = ROW_BYTES + 16;
  static constexpr int STAGES = 3;
  static constexpr int STAGE_BYTES = 2 * TK * ROW_STRIDE;
  static constexpr int THREADS = 128;  // 4 warps x 16 rows
  static constexpr int SMEM = STAGES * STAGE_BYTES;
  static constexpr int KC = D / 16;
  static constexpr int NT = D / 8;
  static constexpr int CHUNKS = ROW_BYTES / 16;
};

template <int D>
__global__ void __launch_bounds__(ExtCfg<D>::THREADS)
    attn_extend_kernel(const int32_t* __restrict__ step, const __nv_bfloat16* __restrict__ q,
                       __nv_bfloat16* __restrict__ out, const __nv_bfloat16* __restrict__ kl,
                       const __nv_bfloat16* __restrict__ vl, const int32_t* __restrict__ tables,
                       int64_t tstride, int hq, int hkv, float scale) {
  using C = ExtCfg<D>;
  extern __shared__ __align__(128) uint8_t smem[];
  const tim_step_header& hd = *reinterpret_cast<const tim_step_header*>(step);
  if ((int)blockIdx.x >= hd.n_ext) return;
  const int32_t* item = step + hd.off_ext + blockIdx.x * TIM_EXT_FIELDS;
  const int row_off = item[0], slot = item[1], m = item[2], n = item[3], q0 = item[4];
  const int kvh = blockIdx.y;
  const int grp = hq / hkv;
  const int qpw = 16 / grp;                   // queries per warp
  const int q_end = (q0 + 4 * qpw) < n ? (q0 + 4 * qpw) : n;
  const int kend = m + q_end;                 // keys [0, kend)
  const int32_t* trow = tables + (int64_t)slot * tstride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const float sl = scale * kLog2e;

  // rows of this warp: rr -> (query qi, head)
  int qi_r[2], valid_r[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int rr = g + 8 * h;
    qi_r[h] = q0 + warp * qpw + rr / grp;
    valid_r[h] = qi_r[h] < n;
  }
  uint32_t qa[C::KC][4];
#pragma unroll
  for (int kc = 0; kc < C::KC; ++kc) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rr = g + 8 * h;
      const __nv_bfloat16* qb = q + ((int64_t)(row_off + qi_r[h]) * hq + kvh * grp + rr % grp) * D + kc * 16 + 2 * t;
      qa[kc][h] = valid_r[h] ? *reinterpret_cast<const uint32_t*>(qb) : 0u;
      qa[kc][h + 2] = valid_r[h] ? *reinterpret_cast<const uint32_t*>(qb + 8) : 0u;
    }
  }

  auto load_tile = [&](int tile, int stg) {
    const int k0 = tile * C::TK;
    uint8_t* kb = smem + stg * C::STAGE_BYTES;
    uint8_t* vb = kb + C::TK * C::ROW_STRIDE;
    for (int e = threadIdx.x; e < C::TK * C::CHUNKS; e += C::THREADS) {
      const int row = e / C::CHUNKS, ch = e - row * C::CHUNKS;
      int tok = k0 + row;
      tok = tok < kend ? tok : kend - 1;
      const int64_t page = trow[tok];
      const int64_t off = (page * hkv + kvh) * D + ch * 8;
      cp_async16(kb + row * C::ROW_STRIDE + ch * 16, kl + off);
      cp_async16(vb + row * C::ROW_STRIDE + ch * 16, vl + off);
    }
  };

  float o[C::NT][4];
#pragma unroll
  for (int i = 0; i < C::NT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  const int ntiles = (kend + C::TK - 1) / C::TK;
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < ntiles) load_tile(s, s);
    cp_async_commit();
  }
  const uint32_t smem_base = smem_u32(smem);
  for (int tile = 0; tile < ntiles; ++tile) {
    const int nxt = tile + C::STAGES - 1;
    if (nxt < ntiles) load_tile(nxt, nxt % C::STAGES);
    cp_async_commit();
    cp_async_wait<C::STAGES - 1>();
    __syncthreads();
    const int stg = tile % C::STAGES;
    const uint32_t kbase = smem_base + stg * C::STAGE_BYTES;
    const uint32_t vbase = kbase + C::TK * C::ROW_STRIDE;
    const int k0 = tile * C::TK;

    float s[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {  // token blocks of 16
      const int mi = lane >> 3;
      const int tok = nb * 16 + (lane & 7) + (mi >> 1) * 8;
      const uint32_t a = kbase + tok * C::ROW_STRIDE + (mi & 1) * 16;
#pragma unroll
      for (int kc = 0; kc < C::KC; ++kc) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(b0, b1, b2, b3, a + kc * 32);
        mma_bf16(s[2 * nb], qa[kc][0], qa[kc][1], qa[kc][2], qa[kc][3], b0, b1);
        mma_bf16(s[2 * nb + 1], qa[kc][0], qa[kc][1], qa[kc][2], qa[kc][3], b2, b3);
      }
    }
    float corr[2];
    float p[2][8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int lim = m + qi_r[h];  // causal: key j visible iff j <= m + qi
      float mx = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int key = k0 + nt * 8 + 2 * t + j;
          const float x = (key <= lim && key < kend) ? s[nt][2 * h + j] * sl : -INFINITY;
          p[h][nt * 2 + j] = x;
          mx = fmaxf(mx, x);
        }
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float mnew = fmaxf(m_r[h], mx);
      const float muse = mnew == -INFINITY ? 0.f : mnew;
      corr[h] = fast_exp2(m_r[h] - muse);
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        p[h][j] = fast_exp2(p[h][j] - muse);
        sum += p[h][j];
      }
      l_r[h] = l_r[h] * corr[h] + sum;
      m_r[h] = mnew;
    }
#pragma unroll
    for (int i = 0; i < C::NT; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
#pragma unroll
    for (int kb = 0; kb < 2; ++kb) {  // k16 blocks of tokens
      const uint32_t pa0 = pack_bf16(p[0][kb * 4 + 0], p[0][kb * 4 + 1]);
      const uint32_t pa1 = pack_bf16(p[1][kb * 4 + 0], p[1][kb * 4 + 1]);
      const uint32_t pa2 = pack_bf16(p[0][kb * 4 + 2], p[0][kb * 4 + 3]);
      const uint32_t pa3 = pack_bf16(p[1][kb * 4 + 2], p[1][kb * 4 + 3]);
      const int mi = lane >> 3;
      const int tok = kb * 16 + (lane & 7) + (mi & 1) * 8;
      const uint32_t a = vbase + tok * C::ROW_STRIDE + (mi >> 1) * 16;
#pragma unroll
      for (int j = 0; j < C::NT / 2; ++j) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(b0, b1, b2, b3, a + j * 32);
        mma_bf16(o[2 * j], pa0, pa1, pa2, pa3, b0, b1);
        mma_bf16(o[2 * j + 1], pa0, pa1, pa2, pa3, b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 1);
    l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 2);
    if (!valid_r[h]) continue;
    const int rr = g + 8 * h;
    const float inv = 1.f / l_r[h];
    __nv_bfloat16* ob = out + ((int64_t)(row_off + qi_r[h]) * hq + kvh * grp + rr % grp) * D;
#pragma unroll
    for (int i = 0; i < C::NT; ++i)
      *reinterpret_cast<uint32_t*>(ob + i * 8 + 2 * t) = pack_bf16(o[i][2 * h] * inv, o[i][2 * h + 1] * inv);
  }
}

// ================================================================ generic
// Warp per (row, q head); exact two-pass softmax in fp32 (model.py:154-159).
template <typename T>
__global__ void attn_generic_kernel(const int32_t* __restrict__ step, const T* __restrict__ q,
                                    T* __restrict__ out, const T* __restrict__ kl,
                                    const T* __restrict__ vl, const int32_t* __restrict__ tables,
                                    int64_t tstride, int hq, int hkv, int D, float scale) {
  const tim_step_header& hd = *reinterpret_cast<const tim_step_header*>(step);
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int row = wid / hq, head = wid - row * hq;
  if (row >= hd.n_rows) return;
  const int32_t* segs = step + hd.off_segs;
  int lo = 0, hi = hd.n_segs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid * TIM_SEG_FIELDS + 3] <= row) lo = mid; else hi = mid - 1;
  }
  const int slot = segs[lo * TIM_SEG_FIELDS], m = segs[lo * TIM_SEG_FIELDS + 1];
  const int i = row - segs[lo * TIM_SEG_FIELDS + 3];
  const int kv_len = m + i + 1;  // prefix fully visible + causal within the new block
  const int kvh = head / (hq / hkv);
  const int32_t* trow = tables + (int64_t)slot * tstride;
  constexpr int MAXE = 8;  // D <= 256
  float qv[MAXE], ov[MAXE];
  const T* qp = q + ((int64_t)row * hq + head) * D;
#pragma unroll
  for (int k = 0; k < MAXE; ++k) {
    const int e = lane + 32 * k;
    qv[k] = e < D ? to_f32(qp[e]) : 0.f;
    ov[k] = 0.f;
  }
  float mx = -INFINITY;
  for (int j = 0; j < kv_len; ++j) {
    const T* kp = kl + ((int64_t)trow[j] * hkv + kvh) * D;
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < MAXE; ++k) {
      const int e = lane + 32 * k;
      if (e < D) acc += qv[k] * to_f32(kp[e]);
    }
    mx = fmaxf(mx, warp_sum(acc) * scale);
  }
  float den = 0.f;
  for (int j = 0; j < kv_len; ++j) {
    const int64_t pg = trow[j];
    const T* kp = kl + (pg * hkv + kvh) * D;
    const T* vp = vl + (pg * hkv + kvh) * D;
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < MAXE; ++k) {
      const int e = lane + 32 * k;
      if (e < D) acc += qv[k] * to_f32(kp[e]);
    }
    const float w = expf(warp_sum(acc) * scale - mx);
    den += w;
#pragma unroll
    for (int k = 0; k < MAXE; ++k) {
      const int e = lane + 32 * k;
      if (e < D) ov[k] += w * to_f32(vp[e]);
    }
  }
  T* op = out + ((int64_t)row * hq + head) * D;
#pragma unroll
  for (int k = 0; k < MAXE; ++k) {
    const int e = lane + 32 * k;
    if (e < D) op[e] = from_f32<T>(ov[k] / den);
  }
}

template <int D, int HKV>
int32_t launch_decode(const int32_t* step, const void* q, void* out, const void* kl, const void* vl,
                      const int32_t* tables, int64_t tstride, int hq, float scale, float* ws,
                      int32_t* counters, int n_ctas, int max_dec, cudaStream_t st) {
  using C = DecCfg<D, HKV>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_kernel<D, HKV>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  attn_decode_kernel<D, HKV><<<n_ctas, C::THREADS, C::SMEM, st>>>(
      step, (const __nv_bfloat16*)q, (__nv_bfloat16*)out, (const __nv_bfloat16*)kl,
      (const __nv_bfloat16*)vl, tables, tstride, hq, scale, ws, counters, max_dec);
  return check_launch("attn_decode");
}

template <int D>
int32_t launch_extend(const int32_t* step, int max_items, const void* q, void* out, const void* kl,
                      const void* vl, const int32_t* tables, int64_t tstride, int hq, int hkv,
                      float scale, cudaStream_t st) {
  using C = ExtCfg<D>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_extend_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  dim3 grid(max_items, hkv);
  attn_extend_kernel<D><<<grid, C::THREADS, C::SMEM, st>>>(
      step, (const __nv_bfloat16*)q, (__nv_bfloat16*)out, (const __nv_bfloat16*)kl,
      (const __nv_bfloat16*)vl, tables, tstride, hq, hkv, scale);
  return check_launch("attn_extend");
}

}  // namespace tim

using namespace tim;

static bool tensor_core_shape(int32_t hq, int32_t hkv, int32_t head_dim) {
  if (hkv <= 0 || hq % hkv) return false;
  const int grp = hq / hkv;
  const bool grp_ok = grp == 1 || grp == 2 || grp == 4 || grp == 8 || grp == 16;
  const bool hkv_ok = hkv == 1 || hkv == 2 || hkv == 4 || hkv == 8;
  return grp_ok && hkv_ok && (head_dim == 64 || head_dim == 128);
}

extern "C" int64_t tim_decode_ws_floats(int32_t n_ctas, int32_t max_dec, int32_t hq, int32_t head_dim) {
  return (int64_t)(n_ctas + max_dec) * hq * (head_dim + 2);
}

extern "C" int32_t tim_extend_queries_per_item(int32_t hq, int32_t hkv, int32_t head_dim, int32_t dtype) {
  if (dtype == TIM_DTYPE_BF16 && tensor_core_shape(hq, hkv, head_dim)) return 64 / (hq / hkv);
  return 1 << 30;  // generic path: whole segments
}

static int32_t launch_generic(const int32_t* step, int32_t n_rows, const void* q, void* out,
                              const void* kl, const void* vl, const int32_t* tables,
                              int64_t tstride, int32_t hq, int32_t hkv, int32_t D, float scale,
                              int32_t dtype, cudaStream_t st) {
  if (D > 256) { set_last_error("head_dim > 256 unsupported"); return TIM_UNSUPPORTED; }
  const int64_t warps = (int64_t)n_rows * hq;
  const int blocks = (int)((warps * 32 + 255) / 256);
  if (blocks <= 0) return TIM_OK;
  if (dtype == TIM_DTYPE_F32) {
    attn_generic_kernel<float><<<blocks, 256, 0, st>>>(step, (const float*)q, (float*)out,
                                                       (const float*)kl, (const float*)vl, tables,
                                                       tstride, hq, hkv, D, scale);
  } else {
    attn_generic_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
        step, (const __nv_bfloat16*)q, (__nv_bfloat16*)out, (const __nv_bfloat16*)kl,
        (const __nv_bfloat16*)vl, tables, tstride, hq, hkv, D, scale);
  }
  return check_launch("attn_generic");
}

// Rows handled: decode queries listed in the step (n_dec).  For the fp32 /
// generic configuration every row is handled by tim_attn_extend instead.
extern "C" int32_t tim_attn_decode(const int32_t* step, const void* q, void* out, const void* k_layer,
                                   const void* v_layer, const int32_t* block_tables,
                                   int64_t table_stride, int32_t hq, int32_t hkv, int32_t head_dim,
                                   float scale, float* ws, int32_t* counters, int32_t n_ctas,
                                   int32_t max_dec, int32_t dtype, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype != TIM_DTYPE_BF16 || !tensor_core_shape(hq, hkv, head_dim)) {
    set_last_error("tim_attn_decode: tensor-core path needs bf16, hkv in {1,2,4,8}, "
                   "group in {1,2,4,8,16}, D in {64,128}");
    return TIM_UNSUPPORTED;
  }
  if (n_ctas <= 0) return TIM_OK;
#define TIM_DEC(DD, HH)                                                                        \
  if (head_dim == DD && hkv == HH)                                                             \
    return launch_decode<DD, HH>(step, q, out, k_layer, v_layer, block_tables, table_stride, hq, \
                                 scale, ws, counters, n_ctas, max_dec, st);
  TIM_DEC(128, 8) TIM_DEC(128, 4) TIM_DEC(128, 2) TIM_DEC(128, 1)
  TIM_DEC(64, 8) TIM_DEC(64, 4) TIM_DEC(64, 2) TIM_DEC(64, 1)
#undef TIM_DEC
  return TIM_UNSUPPORTED;
}

extern "C" int32_t tim_attn_extend(const int32_t* step, int32_t max_items, const void* q, void* out,
                                   const void* k_layer, const void* v_layer,
                                   const int32_t* block_tables, int64_t table_stride, int32_t hq,
                                   int32_t hkv, int32_t head_dim, float scale, int32_t dtype,
                                   void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (max_items <= 0) return TIM_OK;
  if (dtype == TIM_DTYPE_BF16 && tensor_core_shape(hq, hkv, head_dim)) {
    if (head_dim == 128)
      return launch_extend<128>(step, max_items, q, out, k_layer, v_layer, block_tables, table_stride, hq, hkv, scale, st);
    return launch_extend<64>(step, max_items, q, out, k_layer, v_layer, block_tables, table_stride, hq, hkv, scale, st);
  }
  // generic path: max_items is the number of rows to cover
  return launch_generic(step, max_items, q, out, k_layer, v_layer, block_tables, table_stride, hq,
                        hkv, head_dim, scale, dtype, st);
}
