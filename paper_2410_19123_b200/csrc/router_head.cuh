// router_head.cuh — the pre-gating router's gating head for ONE token, computed by one warp (NEXT-1 of
// SURVEY §8(f); §2.3, reading Q15): logits = (RMSNorm(h2) * g_f) . W_head^T in fp32, h2 the
// 512-wide output of the router block. Shared by the separate head kernel (router.cu) and the route launch
// that consumes the hidden state directly (route.cu), so both produce bit-identical logits.
#pragma once

#include "common.cuh"

namespace readme {

constexpr int kRouterDim = 512;

__device__ __forceinline__ float head_warp_sum(float v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// w(n, c) returns W_head[n][c] as fp32 (from shared memory, fp32 or bf16: the value is the same). Lane 0
// stores the N logits through out(n, value).
template <class W, class Out>
__device__ __forceinline__ void head_logits_warp(const __nv_bfloat16* __restrict__ h2row,
                                                 const __nv_bfloat16* __restrict__ gf, W w, int N, float eps,
                                                 int lane, Out out) {
  float v[16];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = __bfloat162float(h2row[lane + 32 * i]);
    ss = fmaf(v[i], v[i], ss);
  }
  ss = head_warp_sum(ss);
  const float r = rsqrtf(ss / kRouterDim + eps);
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] *= r * __bfloat162float(gf[lane + 32 * i]);
  for (int n = 0; n < N; ++n) {
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) acc = fmaf(v[i], w(n, lane + 32 * i), acc);
    acc = head_warp_sum(acc);
    if (lane == 0) out(n, acc);
  }
}

}  // namespace readme
