// Why does a 64-row SiLU*RMS row kernel take ~9 us?  Variants of the same
// body: plain launch vs programmatic launch (+griddepcontrol), with and
// without the RMS block reduction, timed over 200 back-to-back launches.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2507_16784_b200/csrc -o /tmp/rp tools/rowkernel_probe.cu
#include <cstdio>
#include "common.cuh"
using namespace tim;

template <int MODE>   // bit0: griddep calls, bit1: block reduction
__global__ void __launch_bounds__(256) k(__nv_bfloat16* u, int width, const __nv_bfloat16* h, int dm) {
  if (MODE & 1) { griddep_launch(); griddep_wait(); }
  const int r = blockIdx.x;
  __nv_bfloat16* row = u + (int64_t)r * width;
  uint4 uv[6], hv[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) hv[i] = *reinterpret_cast<const uint4*>(h + (int64_t)r * dm + (threadIdx.x + i * 256) * 8);
#pragma unroll
  for (int i = 0; i < 6; ++i) uv[i] = *reinterpret_cast<const uint4*>(row + (threadIdx.x + i * 256) * 8);
  float inv = 1.f;
  if (MODE & 2) {
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(&hv[i]);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += __bfloat162float(p[j]) * __bfloat162float(p[j]);
    }
    __shared__ float red[8];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    float tot = 0.f;
    for (int w = 0; w < 8; ++w) tot += red[w];
    inv = rsqrtf(tot / dm + 1e-6f);
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(&uv[i]);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float f = __bfloat162float(p[j]) * inv;
      p[j] = __float2bfloat16_rn(__fdividef(f, 1.f + __expf(-f)));
    }
    *reinterpret_cast<uint4*>(row + (threadIdx.x + i * 256) * 8) = uv[i];
  }
}

template <int MODE>
float run(int T, __nv_bfloat16* u, __nv_bfloat16* h, bool pdl, cudaStream_t st) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(T);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  for (int i = 0; i < 10; ++i) cudaLaunchKernelEx(&cfg, k<MODE>, u, 12288, (const __nv_bfloat16*)h, 4096);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  for (int i = 0; i < 200; ++i) cudaLaunchKernelEx(&cfg, k<MODE>, u, 12288, (const __nv_bfloat16*)h, 4096);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000 / 200;
}

int main() {
  cudaStream_t st;
  cudaStreamCreate(&st);
  __nv_bfloat16 *u, *h;
  cudaMalloc(&u, 2048 * 12288 * 2);
  cudaMalloc(&h, 2048 * 4096 * 2);
  cudaMemset(u, 0, 2048 * 12288 * 2);
  cudaMemset(h, 0, 2048 * 4096 * 2);
  for (int T : {1, 64, 680}) {
    printf("{\"rows\": %d, \"plain\": %.2f, \"plain_rms\": %.2f, \"pdl_griddep\": %.2f, \"pdl_griddep_rms\": %.2f}\n", T,
           run<0>(T, u, h, false, st), run<2>(T, u, h, false, st), run<1>(T, u, h, true, st), run<3>(T, u, h, true, st));
  }
  return 0;
}
