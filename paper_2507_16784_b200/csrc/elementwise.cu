// K3 (fused RoPE + page store) and the small per-row kernels of the forward:
// embedding gather, weightless RMSNorm, SiLU, greedy argmax.
#include "common.cuh"

namespace tim {

// Vector of V elements of T moved as one 16-byte access.
template <typename T>
struct alignas(16) Vec {
  static constexpr int V = 16 / sizeof(T);
  T v[V];
};

template <typename T>
TIM_DEV Vec<T> ldv(const T* p) { return *reinterpret_cast<const Vec<T>*>(p); }
template <typename T>
TIM_DEV void stv(T* p, const Vec<T>& x) { *reinterpret_cast<Vec<T>*>(p) = x; }

// Weightless RMSNorm commutes with the following GEMM (rms(h) @ W ==
// (h @ W) / rms_scale), so the forward runs its GEMMs on the raw residual
// stream and applies the per-row scale in the consumer kernel (model.py:69-70).

// silu(x) = x * sigmoid(x) with the SFU exponential (ex2.approx): relative
// error ~1e-7, far inside the 1e-5 fp32 parity bound, and ~8x fewer
// instructions than expf on a 12288-wide MLP row.
TIM_DEV float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

// Block-wide sum of one float per thread (every thread gets the total).
template <int NT>
TIM_DEV float block_sum(float v) {
  __shared__ float red[NT / 32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) tot += red[w];
  return tot;
}

// K3: RoPE + page store, fused with the preceding RMSNorm scale.  One CTA per
// row; every global load of the row (the residual h for the RMS scale, the
// q/k halves and v vectors, cos/sin) is issued before the block reduction, so
// the kernel costs one memory round trip.  qkv row layout: [q heads | k heads
// | v heads] x D, the column order of the fused [wq | wk | wv] GEMM.
// Rotate-half convention (model.py:118-125): out[i] = x1*cos - x2*sin,
// out[i+half] = x1*sin + x2*cos.  Items beyond NT*MAXI per row (larger
// models) take a second, unbuffered pass.
template <typename T, int NT, int MAXI>
__global__ void __launch_bounds__(NT, 3)
    rope_kv_kernel(const T* __restrict__ qkv, const T* __restrict__ h, int dm, float eps,
                   const int32_t* __restrict__ row_pos, const int32_t* __restrict__ row_pages,
                   const float* __restrict__ cos_tab, const float* __restrict__ sin_tab, int hq,
                   int hkv, int D, T* __restrict__ q_out, T* __restrict__ k_layer,
                   T* __restrict__ v_layer) {
  constexpr int V = Vec<T>::V;
  constexpr int MAXH = 16 / V;   // dm <= 4096 in registers; wider rows take the loop below
  griddep_launch();   // the attention kernel may start streaming old pages now
  griddep_wait();     // qkv / h come from the preceding GEMM (programmatic launch)
  const int r = blockIdx.x;
  const int half = D >> 1;
  const int gph = half / V;                       // rope vector groups per head
  const int n_rope = (hq + hkv) * gph;
  const int total = n_rope + hkv * D / V;
  const int pos = row_pos[r];
  const int page = row_pages[r];
  const T* x = qkv + (int64_t)r * (hq + 2 * hkv) * D;
  const float* ct = cos_tab + (int64_t)pos * half;
  const float* st = sin_tab + (int64_t)pos * half;
  const T* hr = h ? h + (int64_t)r * dm : nullptr;

  Vec<T> hv[MAXH], av[MAXI], bv[MAXI];
  float cs[MAXI][V], sn[MAXI][V];
#pragma unroll
  for (int k = 0; k < MAXH; ++k) {
    const int e = (threadIdx.x + k * NT) * V;
    if (hr && e < dm) hv[k] = ldv(hr + e);
  }
#pragma unroll
  for (int k = 0; k < MAXI; ++k) {
    const int it = threadIdx.x + k * NT;
    if (it < n_rope) {
      const int head = it / gph, c = (it - head * gph) * V;
      av[k] = ldv(x + head * D + c);
      bv[k] = ldv(x + head * D + half + c);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        cs[k][j] = ct[c + j];
        sn[k][j] = st[c + j];
      }
    } else if (it < total) {
      av[k] = ldv(x + (hq + hkv) * D + (it - n_rope) * V);
    }
  }
  float inv = 1.f;
  if (hr) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < MAXH; ++k) {
      const int e = (threadIdx.x + k * NT) * V;
      if (e < dm) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const float f = to_f32(hv[k].v[j]);
          acc += f * f;
        }
      }
    }
    for (int e = (threadIdx.x + MAXH * NT) * V; e < dm; e += NT * V) {   // dm > NT*V*MAXH
      const Vec<T> y = ldv(hr + e);
#pragma unroll
      for (int j = 0; j < V; ++j) acc += to_f32(y.v[j]) * to_f32(y.v[j]);
    }
    inv = 1.f / sqrtf(block_sum<NT>(acc) / (float)dm + eps);
  }
  auto emit = [&](int it, const Vec<T>& a, const Vec<T>& b, const float* c_, const float* s_) {
    if (it < n_rope) {
      const int head = it / gph, c = (it - head * gph) * V;
      Vec<T> o1, o2;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const float x1 = to_f32(a.v[j]) * inv, x2 = to_f32(b.v[j]) * inv;
        o1.v[j] = from_f32<T>(x1 * c_[j] - x2 * s_[j]);
        o2.v[j] = from_f32<T>(x1 * s_[j] + x2 * c_[j]);
      }
      T* dst;
      if (head < hq) {
        dst = q_out + ((int64_t)r * hq + head) * D;
      } else {
        if (page < 0) return;
        dst = k_layer + ((int64_t)page * hkv + (head - hq)) * D;
      }
      stv(dst + c, o1);
      stv(dst + half + c, o2);
    } else if (page >= 0) {
      Vec<T> o;
#pragma unroll
      for (int j = 0; j < V; ++j) o.v[j] = from_f32<T>(to_f32(a.v[j]) * inv);
      stv(v_layer + (int64_t)page * hkv * D + (it - n_rope) * V, o);
    }
  };
#pragma unroll
  for (int k = 0; k < MAXI; ++k) {
    const int it = threadIdx.x + k * NT;
    if (it < total) emit(it, av[k], bv[k], cs[k], sn[k]);
  }
  for (int it = threadIdx.x + MAXI * NT; it < total; it += NT) {   // rows wider than NT*MAXI items
    Vec<T> a, b;
    float c_[V], s_[V];
    if (it < n_rope) {
      const int head = it / gph, c = (it - head * gph) * V;
      a = ldv(x + head * D + c);
      b = ldv(x + head * D + half + c);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        c_[j] = ct[c + j];
        s_[j] = st[c + j];
      }
    } else {
      a = ldv(x + (hq + hkv) * D + (it - n_rope) * V);
    }
    emit(it, a, b, c_, s_);
  }
}

// u = silu(u * inv_rms(h_row)) in place: the MLP input RMSNorm folded behind
// the W1 GEMM (model.py:161).  One CTA per row, all loads issued before the
// reduction (one round trip); widths beyond NT*V*MAXU take a second pass.
template <typename T, int NT, int MAXU>
__global__ void __launch_bounds__(NT, 3)
    silu_rms_kernel(T* __restrict__ u, int width, const T* __restrict__ h, int dm, float eps) {
  constexpr int V = Vec<T>::V;
  constexpr int MAXH = 16 / V;   // dm <= 4096 in registers; wider rows take the loop below
  griddep_launch();   // the down-projection GEMM may start streaming its weights
  griddep_wait();     // u / h come from the preceding GEMM (programmatic launch)
  const int r = blockIdx.x;
  T* row = u + (int64_t)r * width;
  const T* hr = h ? h + (int64_t)r * dm : nullptr;
  Vec<T> hv[MAXH], uv[MAXU];
#pragma unroll
  for (int k = 0; k < MAXH; ++k) {
    const int e = (threadIdx.x + k * NT) * V;
    if (hr && e < dm) hv[k] = ldv(hr + e);
  }
#pragma unroll
  for (int k = 0; k < MAXU; ++k) {
    const int e = (threadIdx.x + k * NT) * V;
    if (e < width) uv[k] = ldv(row + e);
  }
  float inv = 1.f;
  if (hr) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < MAXH; ++k) {
      const int e = (threadIdx.x + k * NT) * V;
      if (e < dm) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const float f = to_f32(hv[k].v[j]);
          acc += f * f;
        }
      }
    }
    for (int e = (threadIdx.x + MAXH * NT) * V; e < dm; e += NT * V) {
      const Vec<T> y = ldv(hr + e);
#pragma unroll
      for (int j = 0; j < V; ++j) acc += to_f32(y.v[j]) * to_f32(y.v[j]);
    }
    inv = 1.f / sqrtf(block_sum<NT>(acc) / (float)dm + eps);
  }
#pragma unroll
  for (int k = 0; k < MAXU; ++k) {
    const int e = (threadIdx.x + k * NT) * V;
    if (e < width) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const float f = to_f32(uv[k].v[j]) * inv;
        uv[k].v[j] = from_f32<T>(silu(f));
      }
      stv(row + e, uv[k]);
    }
  }
  for (int e = (threadIdx.x + MAXU * NT) * V; e < width; e += NT * V) {
    Vec<T> a = ldv(row + e);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const float f = to_f32(a.v[j]) * inv;
      a.v[j] = from_f32<T>(silu(f));
    }
    stv(row + e, a);
  }
}

template <typename T>
__global__ void embed_kernel(const int32_t* __restrict__ toks, const T* __restrict__ emb, int dm,
                             T* __restrict__ h) {
  const int r = blockIdx.x;
  const T* src = emb + (int64_t)toks[r] * dm;
  T* dst = h + (int64_t)r * dm;
  for (int e = threadIdx.x; e < dm; e += blockDim.x) dst[e] = src[e];
}

// Weightless RMSNorm (model.py:69-70): x / sqrt(mean(x^2) + eps), fp32 math.
template <typename T>
__global__ void rmsnorm_kernel(const T* __restrict__ x, int64_t xs, T* __restrict__ y, int64_t ys,
                               int dm, float eps) {
  const int r = blockIdx.x;
  const T* xr = x + (int64_t)r * xs;
  T* yr = y + (int64_t)r * ys;
  float acc = 0.f;
  for (int e = threadIdx.x; e < dm; e += blockDim.x) {
    const float v = to_f32(xr[e]);
    acc += v * v;
  }
  __shared__ float red[32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float denom = sqrtf(red[0] / (float)dm + eps);
  for (int e = threadIdx.x; e < dm; e += blockDim.x) yr[e] = from_f32<T>(to_f32(xr[e]) / denom);
}

template <typename T>
__global__ void silu_kernel(T* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = to_f32(x[i]);
    x[i] = from_f32<T>(v / (1.0f + expf(-v)));
  }
}

// One warp per row; ties resolve to the lowest id (np.argmax semantics).
// With a mask table, only ids admitted by the row's mask compete
// (np.where(allowed, logits, -inf), model.py:186-192); a row whose mask admits
// nothing below `vocab` writes -1 (EmptyMask).
template <typename T>
__global__ void argmax_kernel(const T* __restrict__ logits, int n_rows, int vocab, int32_t* out,
                              const int32_t* __restrict__ mask_ids, const uint32_t* __restrict__ masks,
                              int words) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n_rows) return;
  const T* row = logits + (int64_t)warp * vocab;
  const int mid = mask_ids ? mask_ids[warp] : -1;
  const uint32_t* mrow = mid >= 0 ? masks + (int64_t)mid * words : nullptr;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = lane; i < vocab; i += 32) {
    if (mrow && (i >= 32 * words || !((mrow[i >> 5] >> (i & 31)) & 1u))) continue;
    const float v = to_f32(row[i]);
    if (bi == 0x7fffffff || v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (oi != 0x7fffffff && (bi == 0x7fffffff || ov > best || (ov == best && oi < bi))) { best = ov; bi = oi; }
  }
  if (lane == 0) out[warp] = bi == 0x7fffffff ? (mrow ? -1 : 0) : bi;
}

}  // namespace tim

using namespace tim;

// Launch with programmatic stream serialization: the grid may be scheduled
// while the preceding kernel drains; the kernels above wait (griddepcontrol)
// before touching its outputs.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int block, cudaStream_t st, Args... args) {
  prefer_shared(kern);
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = st;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

#define TIM_DISPATCH(dtype, ...)                                   \
  do {                                                             \
    if ((dtype) == TIM_DTYPE_F32) {                                \
      using T = float;                                             \
      __VA_ARGS__;                                                 \
    } else if ((dtype) == TIM_DTYPE_BF16) {                        \
      using T = __nv_bfloat16;                                     \
      __VA_ARGS__;                                                 \
    } else {                                                       \
      set_last_error("unsupported dtype %d", (int)(dtype));        \
      return TIM_UNSUPPORTED;                                      \
    }                                                              \
  } while (0)

extern "C" int32_t tim_rope_kv_store(const void* qkv, const void* h, int32_t dm, float eps,
                                     int32_t n_rows, const int32_t* row_pos,
                                     const int32_t* row_pages, const float* cos_tab,
                                     const float* sin_tab, int32_t hq, int32_t hkv,
                                     int32_t head_dim, void* q_out, void* k_layer, void* v_layer,
                                     int32_t dtype, void* stream) {
  if (n_rows <= 0) return TIM_OK;
  const int V = dtype == TIM_DTYPE_BF16 ? 8 : 4;
  if (head_dim % (2 * V) || dm % V) {
    set_last_error("rope_kv_store: head_dim must be a multiple of %d and dm of %d", 2 * V, V);
    return TIM_BAD_ARGUMENT;
  }
  TIM_DISPATCH(dtype, launch_pdl(rope_kv_kernel<T, 256, 2>, n_rows, 256, (cudaStream_t)stream,
                                 (const T*)qkv, (const T*)h, dm, eps, row_pos, row_pages, cos_tab,
                                 sin_tab, hq, hkv, head_dim, (T*)q_out, (T*)k_layer, (T*)v_layer));
  return check_launch("rope_kv_store");
}

extern "C" int32_t tim_silu_rms(void* u, int32_t n_rows, int32_t width, const void* h, int32_t dm,
                                float eps, int32_t dtype, void* stream) {
  if (n_rows <= 0) return TIM_OK;
  const int V = dtype == TIM_DTYPE_BF16 ? 8 : 4;
  if (width % V || dm % V) {
    set_last_error("silu_rms: width and dm must be multiples of %d", V);
    return TIM_BAD_ARGUMENT;
  }
  TIM_DISPATCH(dtype, launch_pdl(silu_rms_kernel<T, 256, 6>, n_rows, 256, (cudaStream_t)stream, (T*)u,
                                 width, (const T*)h, dm, eps));
  return check_launch("silu_rms");
}

extern "C" int32_t tim_embed(const int32_t* row_tokens, int32_t n_rows, const void* emb, int32_t dm,
                             void* h, int32_t dtype, void* stream) {
  if (n_rows <= 0) return TIM_OK;
  TIM_DISPATCH(dtype, prefer_shared(embed_kernel<T>); embed_kernel<T><<<n_rows, 256, 0, (cudaStream_t)stream>>>(
                          row_tokens, (const T*)emb, dm, (T*)h));
  return check_launch("embed");
}

extern "C" int32_t tim_rmsnorm(const void* x, int64_t x_stride, void* y, int64_t y_stride,
                               int32_t n_rows, int32_t dm, float eps, int32_t dtype, void* stream) {
  if (n_rows <= 0) return TIM_OK;
  TIM_DISPATCH(dtype, prefer_shared(rmsnorm_kernel<T>); rmsnorm_kernel<T><<<n_rows, 512, 0, (cudaStream_t)stream>>>(
                          (const T*)x, x_stride, (T*)y, y_stride, dm, eps));
  return check_launch("rmsnorm");
}

extern "C" int32_t tim_silu(void* x, int64_t n, int32_t dtype, void* stream) {
  if (n <= 0) return TIM_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  TIM_DISPATCH(dtype, prefer_shared(silu_kernel<T>); silu_kernel<T><<<(int)blocks, 256, 0, (cudaStream_t)stream>>>((T*)x, n));
  return check_launch("silu");
}

extern "C" int32_t tim_argmax(const void* logits, int32_t n_rows, int32_t vocab, int32_t* out,
                              int32_t dtype, void* stream) {
  if (n_rows <= 0) return TIM_OK;
  const int blocks = (n_rows * 32 + 255) / 256;
  TIM_DISPATCH(dtype, prefer_shared(argmax_kernel<T>); argmax_kernel<T><<<blocks, 256, 0, (cudaStream_t)stream>>>(
                          (const T*)logits, n_rows, vocab, out, nullptr, nullptr, 0));
  return check_launch("argmax");
}

extern "C" int32_t tim_masked_argmax(const void* logits, int32_t n_rows, int32_t vocab, const int32_t* mask_ids,
                                     const uint32_t* masks, int32_t words, int32_t* out, int32_t dtype,
                                     void* stream) {
  if (n_rows <= 0) return TIM_OK;
  if (!mask_ids || !masks || words <= 0) return TIM_BAD_ARGUMENT;
  const int blocks = (n_rows * 32 + 255) / 256;
  TIM_DISPATCH(dtype, prefer_shared(argmax_kernel<T>); argmax_kernel<T><<<blocks, 256, 0, (cudaStream_t)stream>>>(
                          (const T*)logits, n_rows, vocab, out, mask_ids, masks, words));
  return check_launch("masked_argmax");
}
