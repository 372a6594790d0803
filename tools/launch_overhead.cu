// Event-timed cost of launching an (almost) empty persistent grid, as bench.py
// times the layer-0 attention: 148 CTAs x 288 threads, with/without ~200 KB of
// dynamic shared memory and with/without the programmatic-launch attribute.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lo tools/launch_overhead.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel(int* flag) {
  extern __shared__ int s[];
  if (flag && threadIdx.x == 0 && blockIdx.x == 100000) s[0] = *flag;
}
__global__ void spin_kernel(long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > ns) break;
  }
}

int main() {
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 210000);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int smem : {0, 100000, 203000}) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      for (int prev = 0; prev < 2; ++prev) {
        float tot = 0;
        const int iters = 50;
        for (int i = 0; i < iters + 5; ++i) {
          if (prev) spin_kernel<<<148, 32, 0, st>>>(20000);   // a busy predecessor (20 us)
          cudaEventRecord(a, st);
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(148);
          cfg.blockDim = dim3(288);
          cfg.dynamicSmemBytes = smem;
          cfg.stream = st;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = pdl;
          cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
          cudaEventRecord(b, st);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (i >= 5) tot += ms;
        }
        printf("{\"smem\": %d, \"pdl\": %d, \"busy_predecessor\": %d, \"us\": %.2f}\n", smem, pdl, prev,
               tot * 1000 / iters);
      }
    }
  }
  return 0;
}
