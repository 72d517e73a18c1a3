// common.cuh — device/host helpers shared by the CUDA kernels of libreadme_b200 (product code).
// Nothing here is shared with oracle/ (the test oracle); see DESIGN.md "Oracle independence".
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/readme.h"

namespace readme {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------------------------------
// Host-side error plumbing (thread-local message, status codes).
void set_error(const char* fmt, ...);
readme_status cuda_fail(cudaError_t e, const char* where);

#define README_CHECK_ARG(cond, ...)              \
  do {                                           \
    if (!(cond)) {                               \
      ::readme::set_error(__VA_ARGS__);          \
      return README_ERR_INVALID_ARG;             \
    }                                            \
  } while (0)

#define README_CUDA(call)                                              \
  do {                                                                 \
    cudaError_t e_ = (call);                                           \
    if (e_ != cudaSuccess) return ::readme::cuda_fail(e_, #call);      \
  } while (0)

#define README_TRY(expr)            \
  do {                              \
    readme_status s_ = (expr);      \
    if (s_ != README_OK) return s_; \
  } while (0)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
inline size_t dt_size(readme_dtype dt) { return dt == README_BF16 ? 2 : 4; }

int num_sms();  // cached per device

// ---------------------------------------------------------------------------------------------------
// Device helpers.
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint64_t ld_relaxed_gpu_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint4 ld_nc_v4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
// round-to-nearest-even pack of two floats into bf16x2 (lo in the low half)
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ---------------------------------------------------------------------------------------------------
// Timeline trace for measurement only (readme_debug_trace): when a device buffer is registered, the
// dispatch / route / expert FFN kernels record %globaltimer extremes into it (slot meanings in capi.cu).
// Null by default: the kernels then skip it entirely.
extern uint64_t* g_trace_buf;
extern uint64_t* g_tile_trace;  // per-tile records of the single-launch FFN (readme_debug_tile_trace)
extern int32_t g_tile_trace_max;
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_min(uint64_t* tr, int i) {
  if (tr) atomicMin(reinterpret_cast<unsigned long long*>(tr + i), static_cast<unsigned long long>(globaltimer_ns()));
}
__device__ __forceinline__ void trace_max(uint64_t* tr, int i) {
  if (tr) atomicMax(reinterpret_cast<unsigned long long*>(tr + i), static_cast<unsigned long long>(globaltimer_ns()));
}

}  // namespace readme
