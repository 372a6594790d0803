// K3 (fused RoPE + page store) and the small per-row kernels of the forward:
// embedding gather, weightless RMSNorm, SiLU, greedy argmax.
#include "common.cuh"

namespace tim {

// Vector of V elements of T moved as one 16-byte access.
template <typename T>
struct Vec {
  static constexpr int V = 16 / sizeof(T);
  T v[V];
};

template <typename T>
TIM_DEV Vec<T> ldv(const T* p) { return *reinterpret_cast<const Vec<T>*>(p); }
template <typename T>
TIM_DEV void stv(T* p, const Vec<T>& x) { *reinterpret_cast<Vec<T>*>(p) = x; }

// 1 / sqrt(mean(h_row^2) + eps) of one row, all threads of the CTA get it.
// Weightless RMSNorm commutes with the following GEMM (rms(h) @ W ==
// (h @ W) / rms_scale), so the forward runs its GEMMs on the raw residual
// stream and applies this per-row scale in the consumer kernel (model.py:69-70).
template <typename T>
TIM_DEV float row_inv_rms(const T* __restrict__ h, int dm, float eps) {
  constexpr int V = Vec<T>::V;
  __shared__ float red[32];
  float acc = 0.f;
  for (int e = threadIdx.x * V; e < dm; e += blockDim.x * V) {
    const Vec<T> x = ldv(h + e);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const float f = to_f32(x.v[k]);
      acc += f * f;
    }
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
  __syncthreads();
  return 1.f / sqrtf(tot / (float)dm + eps);
}

// K3: RoPE + page store, fused with the preceding RMSNorm scale.  Grid
// (rows, splits); the row's work items (rotated q/k vectors, v vectors) are
// divided over the splits.  qkv row layout: [q heads | k heads | v heads] x D,
// the column order of the fused [wq | wk | wv] GEMM.  Rotate-half convention
// (model.py:118-125): out[i] = x1*cos - x2*sin, out[i+half] = x1*sin + x2*cos.
template <typename T>
__global__ void __launch_bounds__(128)
    rope_kv_kernel(const T* __restrict__ qkv, const T* __restrict__ h, int dm, float eps,
                   const int32_t* __restrict__ row_pos, const int32_t* __restrict__ row_pages,
                   const float* __restrict__ cos_tab, const float* __restrict__ sin_tab, int hq,
                   int hkv, int D, T* __restrict__ q_out, T* __restrict__ k_layer,
                   T* __restrict__ v_layer) {
  constexpr int V = Vec<T>::V;
  griddep_launch();   // the attention kernel may start staging its page ids now
  const int r = blockIdx.x;
  const float inv = h ? row_inv_rms(h + (int64_t)r * dm, dm, eps) : 1.f;
  const int half = D >> 1;
  const int gph = half / V;                       // rope vector groups per head
  const int n_rope = (hq + hkv) * gph;
  const int n_v = hkv * D / V;
  const int total = n_rope + n_v;
  const int per = (total + gridDim.y - 1) / gridDim.y;
  const int i0 = blockIdx.y * per, i1 = min(total, i0 + per);
  const int pos = row_pos[r];
  const int page = row_pages[r];
  const T* x = qkv + (int64_t)r * (hq + 2 * hkv) * D;
  const float* ct = cos_tab + (int64_t)pos * half;
  const float* st = sin_tab + (int64_t)pos * half;
  for (int it = i0 + threadIdx.x; it < i1; it += blockDim.x) {
    if (it < n_rope) {
      const int head = it / gph, c = (it - head * gph) * V;
      const T* src = x + head * D;
      const Vec<T> a = ldv(src + c), b = ldv(src + half + c);
      Vec<T> o1, o2;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float x1 = to_f32(a.v[k]) * inv, x2 = to_f32(b.v[k]) * inv;
        const float cs = ct[c + k], sn = st[c + k];
        o1.v[k] = from_f32<T>(x1 * cs - x2 * sn);
        o2.v[k] = from_f32<T>(x1 * sn + x2 * cs);
      }
      T* dst;
      if (head < hq) {
        dst = q_out + ((int64_t)r * hq + head) * D;
      } else {
        if (page < 0) continue;
        dst = k_layer + ((int64_t)page * hkv + (head - hq)) * D;
      }
      stv(dst + c, o1);
      stv(dst + half + c, o2);
    } else if (page >= 0) {
      const int e = (it - n_rope) * V;
      const Vec<T> a = ldv(x + (hq + hkv) * D + e);
      Vec<T> o;
#pragma unroll
      for (int k = 0; k < V; ++k) o.v[k] = from_f32<T>(to_f32(a.v[k]) * inv);
      stv(v_layer + (int64_t)page * hkv * D + e, o);
    }
  }
}

// u = silu(u * inv_rms(h_row)) in place: the MLP input RMSNorm folded behind
// the W1 GEMM (model.py:161), grid (rows, splits).
template <typename T>
__global__ void __launch_bounds__(128)
    silu_rms_kernel(T* __restrict__ u, int width, const T* __restrict__ h, int dm, float eps) {
  constexpr int V = Vec<T>::V;
  griddep_launch();   // the down-projection GEMM may start streaming its weights
  const int r = blockIdx.x;
  const float inv = h ? row_inv_rms(h + (int64_t)r * dm, dm, eps) : 1.f;
  const int nv = width / V;
  const int per = (nv + gridDim.y - 1) / gridDim.y;
  const int i0 = blockIdx.y * per, i1 = min(nv, i0 + per);
  T* row = u + (int64_t)r * width;
  for (int it = i0 + threadIdx.x; it < i1; it += blockDim.x) {
    Vec<T> a = ldv(row + it * V);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const float f = to_f32(a.v[k]) * inv;
      a.v[k] = from_f32<T>(f / (1.0f + expf(-f)));
    }
    stv(row + it * V, a);
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
template <typename T>
__global__ void argmax_kernel(const T* __restrict__ logits, int n_rows, int vocab, int32_t* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n_rows) return;
  const T* row = logits + (int64_t)warp * vocab;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = lane; i < vocab; i += 32) {
    const float v = to_f32(row[i]);
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if (lane == 0) out[warp] = bi == 0x7fffffff ? 0 : bi;
}

}  // namespace tim

using namespace tim;

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
  const int items = (hq + hkv) * (head_dim / 2 / V) + hkv * head_dim / V;
  const int splits = items > 512 ? 4 : (items > 256 ? 2 : 1);
  dim3 grid(n_rows, splits);
  TIM_DISPATCH(dtype, rope_kv_kernel<T><<<grid, 128, 0, (cudaStream_t)stream>>>(
                          (const T*)qkv, (const T*)h, dm, eps, row_pos, row_pages, cos_tab, sin_tab,
                          hq, hkv, head_dim, (T*)q_out, (T*)k_layer, (T*)v_layer));
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
  const int splits = width / V >= 1024 ? 8 : (width / V >= 256 ? 2 : 1);
  dim3 grid(n_rows, splits);
  TIM_DISPATCH(dtype, silu_rms_kernel<T><<<grid, 128, 0, (cudaStream_t)stream>>>(
                          (T*)u, width, (const T*)h, dm, eps));
  return check_launch("silu_rms");
}

extern "C" int32_t tim_embed(const int32_t* row_tokens, int32_t n_rows, const void* emb, int32_t dm,
                             void* h, int32_t dtype, void* stream) {
  if (n_rows <= 0) return TIM_OK;
  TIM_DISPATCH(dtype, embed_kernel<T><<<n_rows, 256, 0, (cudaStream_t)stream>>>(
                          row_tokens, (const T*)emb, dm, (T*)h));
  return check_launch("embed");
}

extern "C" int32_t tim_rmsnorm(const void* x, int64_t x_stride, void* y, int64_t y_stride,
                               int32_t n_rows, int32_t dm, float eps, int32_t dtype, void* stream) {
  if (n_rows <= 0) return TIM_OK;
  TIM_DISPATCH(dtype, rmsnorm_kernel<T><<<n_rows, 512, 0, (cudaStream_t)stream>>>(
                          (const T*)x, x_stride, (T*)y, y_stride, dm, eps));
  return check_launch("rmsnorm");
}

extern "C" int32_t tim_silu(void* x, int64_t n, int32_t dtype, void* stream) {
  if (n <= 0) return TIM_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  TIM_DISPATCH(dtype, silu_kernel<T><<<(int)blocks, 256, 0, (cudaStream_t)stream>>>((T*)x, n));
  return check_launch("silu");
}

extern "C" int32_t tim_argmax(const void* logits, int32_t n_rows, int32_t vocab, int32_t* out,
                              int32_t dtype, void* stream) {
  if (n_rows <= 0) return TIM_OK;
  const int blocks = (n_rows * 32 + 255) / 256;
  TIM_DISPATCH(dtype, argmax_kernel<T><<<blocks, 256, 0, (cudaStream_t)stream>>>(
                          (const T*)logits, n_rows, vocab, out));
  return check_launch("argmax");
}
