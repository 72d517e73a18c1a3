// ffn_f32.cu — a6/a7 in fp32 on CUDA cores (FFMA, no TF32), for the tiny fp32 config (H=64, d=128,
// T=256) whose tolerance (1e-4) TF32 would break. Same math as the bf16 tensor-core path
// (SwiGLU reading Q4):
//     h_r = silu(x_r W_gate[e]^T) * (x_r W_up[e]^T),   y_r = h_r W_down[e]^T,   e = segment % E.
// Grid = (segment m-tiles of 32 rows) x (n-tiles of 32 columns); the tile list is derived on the device
// from `offsets`, so the call needs no host synchronisation. Accumulation is fp32, k ascending.
#include <math.h>

#include "kernels.h"

namespace readme {

namespace {

constexpr int kTm = 32, kTn = 32;
constexpr int kMaxSeg = 512;

// K per staged block: the whole K of the tiny config in as few serial load rounds as shared memory allows
// (64 with three operand tiles, 128 with two)
template <bool kSwiGLU>
__global__ void __launch_bounds__(256)
ffn_f32_kernel(const float* __restrict__ A, int64_t rows, int K, int N, int E, int nseg,
               const int32_t* __restrict__ offsets, const float* __restrict__ B0, const float* __restrict__ B1,
               float* __restrict__ C, const int32_t* __restrict__ src, const float* __restrict__ residual) {
  constexpr int kTk = kSwiGLU ? 64 : 128;
  __shared__ int s_off[kMaxSeg + 1];
  __shared__ int s_tstart[kMaxSeg + 1];
  __shared__ float sA[kTm][kTk + 1];
  __shared__ float sB0[kTn][kTk + 1];
  __shared__ float sB1[kSwiGLU ? kTn : 1][kTk + 1];
  const int tid = threadIdx.x;
  for (int i = tid; i <= nseg; i += blockDim.x) s_off[i] = offsets[i];
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int g = 0; g < nseg; ++g) {
      s_tstart[g] = acc;
      acc += (s_off[g + 1] - s_off[g] + kTm - 1) / kTm;
    }
    s_tstart[nseg] = acc;
  }
  __syncthreads();
  const int mtile = blockIdx.x;
  if (mtile >= s_tstart[nseg]) return;
  int g = 0;
  while (s_tstart[g + 1] <= mtile) ++g;
  const int e = g % E;
  const int64_t r0 = s_off[g] + static_cast<int64_t>(mtile - s_tstart[g]) * kTm;
  const int64_t rend = s_off[g + 1];
  const int n0 = blockIdx.y * kTn;
  const int tx = tid % kTn, ty = tid / kTn;  // 32 x 8

  const float* Be0 = B0 + static_cast<int64_t>(e) * N * K;
  const float* Be1 = kSwiGLU ? B1 + static_cast<int64_t>(e) * N * K : nullptr;
  float acc0[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k0 = 0; k0 < K; k0 += kTk) {
    for (int i = ty; i < kTm; i += 8) {
#pragma unroll
      for (int cc = tx; cc < kTk; cc += kTn) {
        const int64_t r = r0 + i;
        sA[i][cc] = (r < rend && k0 + cc < K) ? A[r * K + k0 + cc] : 0.f;
        const int n = n0 + i;
        sB0[i][cc] = (n < N && k0 + cc < K) ? Be0[static_cast<int64_t>(n) * K + k0 + cc] : 0.f;
        if constexpr (kSwiGLU)
          sB1[i][cc] = (n < N && k0 + cc < K) ? Be1[static_cast<int64_t>(n) * K + k0 + cc] : 0.f;
      }
    }
    __syncthreads();
    const int kk = min(kTk, K - k0);
    for (int q = 0; q < kk; ++q) {
      const float b0 = sB0[tx][q];
      float b1 = 0.f;
      if constexpr (kSwiGLU) b1 = sB1[tx][q];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = sA[ty + 8 * i][q];
        acc0[i] = fmaf(a, b0, acc0[i]);
        if constexpr (kSwiGLU) acc1[i] = fmaf(a, b1, acc1[i]);
      }
    }
    __syncthreads();
  }
  const int n = n0 + tx;
  if (n >= N) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + ty + 8 * i;
    if (r >= rend) continue;
    float v = acc0[i];
    if constexpr (kSwiGLU) v = v / (1.0f + expf(-v)) * acc1[i];
    int64_t orow = r;
    if (src) {  // fused combine (k == 1): row r holds token src[r]
      orow = src[r];
      if (orow < 0 || orow >= rows) continue;
    }
    if (residual) v += residual[orow * N + n];
    C[orow * N + n] = v;
  }
}

}  // namespace

readme_status launch_gate_up_f32(const float* xs, int64_t rows, int32_t H, int32_t E, int32_t d, int32_t nseg,
                                 const int32_t* offsets, const float* wg, const float* wu, float* h, cudaStream_t st) {
  if (rows == 0) return README_OK;
  if (nseg > kMaxSeg) {
    set_error("fp32 expert FFN supports at most %d segments (got %d)", kMaxSeg, nseg);
    return README_ERR_UNSUPPORTED;
  }
  const int64_t mtiles_ub = nseg + (rows + kTm - 1) / kTm;
  dim3 g(static_cast<unsigned>(mtiles_ub), (d + kTn - 1) / kTn);
  ffn_f32_kernel<true><<<g, 256, 0, st>>>(xs, rows, H, d, E, nseg, offsets, wg, wu, h, nullptr, nullptr);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_down_f32(const float* h, int64_t rows, int32_t H, int32_t E, int32_t d, int32_t nseg,
                              const int32_t* offsets, const float* wd, float* out, const int32_t* src,
                              const float* residual, cudaStream_t st) {
  if (rows == 0) return README_OK;
  if (nseg > kMaxSeg) {
    set_error("fp32 expert FFN supports at most %d segments (got %d)", kMaxSeg, nseg);
    return README_ERR_UNSUPPORTED;
  }
  const int64_t mtiles_ub = nseg + (rows + kTm - 1) / kTm;
  dim3 g(static_cast<unsigned>(mtiles_ub), (H + kTn - 1) / kTn);
  ffn_f32_kernel<false><<<g, 256, 0, st>>>(h, rows, d, H, E, nseg, offsets, wd, nullptr, out, src, residual);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

}  // namespace readme
