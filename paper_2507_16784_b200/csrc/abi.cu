// ABI utilities: error strings, launch checks, device queries.
#include <cstdarg>
#include <cstdio>
#include "common.cuh"

namespace tim {

static thread_local char g_last_error[512] = {0};

void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

void prefer_shared_carveout(const void* kern) {
  static const void* done[64];
  static int n = 0;
  for (int i = 0; i < n; ++i)
    if (done[i] == kern) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (n < 64) done[n++] = kern;
}

int32_t check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error("%s: %s", what, cudaGetErrorString(e));
    return TIM_CUDA_ERROR;
  }
  return TIM_OK;
}

}  // namespace tim

extern "C" int32_t tim_abi_version(void) { return 1; }

extern "C" const char* tim_last_error(void) { return tim::g_last_error; }

extern "C" int32_t tim_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

extern "C" int32_t tim_read_error(int32_t* err_dev, int32_t* code_out, int32_t* detail_out,
                                  void* stream) {
  int32_t host[2] = {0, 0};
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(host, err_dev, sizeof(host), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && host[0] != 0) e = cudaMemsetAsync(err_dev, 0, sizeof(host), st);
  if (e != cudaSuccess) {
    tim::set_last_error("read_error: %s", cudaGetErrorString(e));
    return TIM_CUDA_ERROR;
  }
  *code_out = host[0];
  *detail_out = host[1];
  return TIM_OK;
}

namespace {
__global__ void noop_kernel() { tim::griddep_launch(); }
}  // namespace

// Diagnostics: an empty grid launched exactly like the attention kernel
// (n_ctas x threads, `smem` dynamic shared bytes, programmatic launch), so
// bench.py can measure the fixed cost CUDA-event bracketing adds to a launch.
extern "C" int32_t tim_noop(int32_t n_ctas, int32_t threads, int32_t smem, void* stream) {
  static int attr_smem = -1;
  if (smem > attr_smem) {
    cudaFuncSetAttribute(noop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_smem = smem;
  }
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, noop_kernel) != cudaSuccess) return tim::check_launch("noop");
  return tim::check_launch("noop");
}
