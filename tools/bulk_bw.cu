// Floor for the decode kernel's access pattern: stream N random 2 KiB page rows
// (K and V) into a 3-stage x 64 KiB shared ring per SM with cp.async.bulk and
// mbarriers, no math.  Prints us and GB/s for several N.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2507_16784_b200/csrc tools/bulk_bw.cu -o /tmp/bulk_bw
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include "common.cuh"

using namespace tim;
constexpr int TK = 16, STAGES = 3;

template <int ROW>
__global__ void __launch_bounds__(64) stream_rows(const int32_t* pages, int64_t n_tok,
                                                    const uint8_t* kpool, const uint8_t* vpool,
                                                    int consumers_work) {
  constexpr int STRIDE = ROW + 16, STAGE_BYTES = 2 * TK * STRIDE;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const int64_t G = gridDim.x;
  const int64_t start = blockIdx.x * n_tok / G, end = (blockIdx.x + 1) * n_tok / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  int it = 0;
  if (warp == 0) {
    for (int64_t k0 = start; k0 < end; k0 += TK, ++it) {
      const int stg = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty[stg], ((it / STAGES) & 1) ^ 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[stg], 2 * TK * ROW);
      __syncwarp();
      const int row = lane & (TK - 1);
      int64_t tok = k0 + row;
      if (tok >= end) tok = end - 1;
      const int page = pages[tok];
      uint8_t* base = smem + stg * STAGE_BYTES + (lane >= TK ? TK * STRIDE : 0);
      bulk_g2s(base + row * STRIDE, (lane >= TK ? vpool : kpool) + (int64_t)page * ROW, ROW, &full[stg]);
    }
  } else {
    float acc = 0.f;
    for (int64_t k0 = start; k0 < end; k0 += TK, ++it) {
      const int stg = it % STAGES;
      mbar_wait(&full[stg], (it / STAGES) & 1);
      if (consumers_work) acc += reinterpret_cast<const float*>(smem + stg * STAGE_BYTES)[lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stg]);
    }
    if (acc == 12345.f) printf("x");
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t cap = 1 << 21;  // 1 KiB rows addressable up to 2M (2 GiB per pool)
  uint8_t *K, *V;
  cudaMalloc(&K, cap * 2048);
  cudaMalloc(&V, cap * 2048);
  cudaMemset(K, 1, cap * 2048);
  cudaMemset(V, 1, cap * 2048);
  std::vector<int32_t> perm(cap);
  for (int i = 0; i < cap; ++i) perm[i] = i;
  std::shuffle(perm.begin(), perm.end(), std::mt19937(1));
  int32_t* pages;
  cudaMalloc(&pages, cap * 4);
  cudaMemcpy(pages, perm.data(), cap * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto kern, int row, int ctas, const char* tag) {
    const int smem = STAGES * 2 * TK * (row + 16) + 64;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int64_t n : {20000L, 46000L, 127000L, 382000L, 1000000L}) {
      const int64_t nrows = n * 2048 / row;   // same bytes for both row sizes
      for (int rep = 0; rep < 3; ++rep) kern<<<ctas, 64, smem>>>(pages, nrows, K, V, 1);
      cudaEventRecord(a);
      const int iters = 20;
      for (int rep = 0; rep < iters; ++rep)
        kern<<<ctas, 64, smem>>>(pages + (rep * nrows) % (cap - nrows), nrows, K, V, 1);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double us = ms * 1000.0 / iters;
      const double bytes = (double)nrows * row * 2;
      printf("{\"cfg\": \"%s\", \"MB\": %.1f, \"us\": %.2f, \"GBs\": %.0f}\n", tag, bytes / 1e6, us,
             bytes / us / 1e3);
    }
  };
  run(stream_rows<2048>, 2048, sms, "2KiB rows, 1 CTA/SM");
  run(stream_rows<1024>, 1024, 2 * sms, "1KiB rows, 2 CTA/SM");
  run(stream_rows<2048>, 2048, 2 * sms, "2KiB rows, 2 CTA/SM (2 waves?)");
  return 0;
}
