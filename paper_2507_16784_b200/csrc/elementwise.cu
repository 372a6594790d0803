// K3 (fused RoPE + page store) and the small per-row kernels of the forward:
// embedding gather, weightless RMSNorm, SiLU, greedy argmax.
#include "common.cuh"

namespace tim {

// K3: one CTA per row.  qkv row layout: [q heads | k heads | v heads] x D, the
// column order of the fused [wq | wk | wv] GEMM.  Rotate-half convention
// (model.py:118-125): out[i] = x1*cos - x2*sin, out[i+half] = x1*sin + x2*cos.
template <typename T>
__global__ void rope_kv_kernel(const T* __restrict__ qkv, const int32_t* __restrict__ row_pos,
                               const int32_t* __restrict__ row_pages, const float* __restrict__ cos_tab,
                               const float* __restrict__ sin_tab, int hq, int hkv, int D,
                               T* __restrict__ q_out, T* __restrict__ k_layer, T* __restrict__ v_layer) {
  const int r = blockIdx.x;
  const int half = D >> 1;
  const int pos = row_pos[r];
  const int page = row_pages[r];
  const int width = (hq + 2 * hkv) * D;
  const T* x = qkv + (int64_t)r * width;
  const float* ct = cos_tab + (int64_t)pos * half;
  const float* st = sin_tab + (int64_t)pos * half;
  const int nq = hq * half, nk = hkv * half;
  // rotated pairs of q and k
  for (int e = threadIdx.x; e < nq + nk; e += blockDim.x) {
    const bool isq = e < nq;
    const int ee = isq ? e : e - nq;
    const int head = ee / half, i = ee - head * half;
    const T* src = x + (isq ? 0 : hq * D) + head * D;
    const float x1 = to_f32(src[i]), x2 = to_f32(src[i + half]);
    const float c = ct[i], s = st[i];
    const float o1 = x1 * c - x2 * s;
    const float o2 = x1 * s + x2 * c;
    if (isq) {
      T* dst = q_out + (int64_t)r * hq * D + head * D;
      dst[i] = from_f32<T>(o1);
      dst[i + half] = from_f32<T>(o2);
    } else if (page >= 0) {
      T* dst = k_layer + ((int64_t)page * hkv + head) * D;
      dst[i] = from_f32<T>(o1);
      dst[i + half] = from_f32<T>(o2);
    }
  }
  if (page >= 0) {
    const T* vsrc = x + (hq + hkv) * D;
    T* vdst = v_layer + (int64_t)page * hkv * D;
    for (int e = threadIdx.x; e < hkv * D; e += blockDim.x) vdst[e] = vsrc[e];
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

extern "C" int32_t tim_rope_kv_store(const void* qkv, int32_t n_rows, const int32_t* row_pos,
                                     const int32_t* row_pages, const float* cos_tab,
                                     const float* sin_tab, int32_t hq, int32_t hkv,
                                     int32_t head_dim, void* q_out, void* k_layer, void* v_layer,
                                     int32_t dtype, void* stream) {
  if (n_rows <= 0) return TIM_OK;
  if (head_dim % 2) { set_last_error("head_dim must be even"); return TIM_BAD_ARGUMENT; }
  TIM_DISPATCH(dtype, rope_kv_kernel<T><<<n_rows, 256, 0, (cudaStream_t)stream>>>(
                          (const T*)qkv, row_pos, row_pages, cos_tab, sin_tab, hq, hkv, head_dim,
                          (T*)q_out, (T*)k_layer, (T*)v_layer));
  return check_launch("rope_kv_store");
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
