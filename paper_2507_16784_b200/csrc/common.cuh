// Shared device helpers for libtimrun (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include "timrun.h"

#define TIM_DEV __device__ __forceinline__

namespace tim {

// ---------------------------------------------------------------- step access
struct Step {
  const int32_t* base;
  TIM_DEV const tim_step_header& h() const { return *reinterpret_cast<const tim_step_header*>(base); }
  TIM_DEV const int32_t* at(int32_t off) const { return base + off; }
};

TIM_DEV void raise_error(int32_t* err, int32_t code, int32_t detail) {
  if (err == nullptr) return;
  if (atomicCAS(err, 0, code) == 0) err[1] = detail;
}

// ------------------------------------------------------------------ smem/PTX
TIM_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

TIM_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
TIM_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
TIM_DEV void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
TIM_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
TIM_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
TIM_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "TIM_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TIM_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared (SASS UBLKCP), completion counted on `bar`.
TIM_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// The same with an L2 cache policy (createpolicy): streamed page rows are
// marked evict-first so the stream does not flush the small hot working set
// (plan, block tables, parked split partials, instructions) out of L2.
TIM_DEV uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
TIM_DEV void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Ampere-style 16B async copy (LDGSTS).
TIM_DEV void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
TIM_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
TIM_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ldmatrix / mma.sync (bf16, fp32 accumulate)
TIM_DEV void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
TIM_DEV void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
TIM_DEV void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                      uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

TIM_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Programmatic dependent launch (sm_90+): a dependent grid may start early;
// griddep_wait() blocks until the preceding grid finished and its memory is
// visible, griddep_launch() lets the next grid start.
TIM_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
TIM_DEV void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

TIM_DEV float fast_exp2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <typename T>
TIM_DEV float to_f32(T v);
template <>
TIM_DEV float to_f32<float>(float v) { return v; }
template <>
TIM_DEV float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
TIM_DEV T from_f32(float v);
template <>
TIM_DEV float from_f32<float>(float v) { return v; }
template <>
TIM_DEV __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

TIM_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
TIM_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace tim

// host-side error plumbing shared by the ABI translation units
namespace tim {
void set_last_error(const char* fmt, ...);
int32_t check_launch(const char* what);

// Every small kernel of a step asks for the max-shared carveout.  A kernel
// with little or no shared memory otherwise lets the SMs switch to a large-L1
// configuration, and the ~200 KB-per-CTA attention launch that follows it has
// to switch them back: measured on B200 (tools/carveout_probe.py), an empty
// 148 x 320 grid with 203 KB of dynamic smem bracketed by CUDA events takes
// 10.2 us after a 0-smem kernel and 6.1 us after any kernel that kept the
// shared carveout.  Idempotent, once per kernel.
void prefer_shared_carveout(const void* kern);
template <typename K>
inline void prefer_shared(K kern) { prefer_shared_carveout(reinterpret_cast<const void*>(kern)); }
}  // namespace tim
