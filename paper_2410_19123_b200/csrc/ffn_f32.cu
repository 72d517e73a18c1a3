// ffn_f32.cu — a6/a7 in fp32 on CUDA cores (FFMA, no TF32), for the tiny fp32 config (H=64, d=128,
// T=256) whose tolerance (1e-4) TF32 would break. Same math as the bf16 tensor-core path
// (SwiGLU reading Q4):
//     h_r = silu(x_r W_gate[e]^T) * (x_r W_up[e]^T),   y_r = h_r W_down[e]^T,   e = segment % E.
// Two forms: the two-pass ffn_f32_kernel (grid = segment m-tiles of 32 rows x n-tiles of 32 columns) and, for
// H, d <= 128, ffn_f32_fused_kernel (a6 + a7 in one launch, below). Tile lists are derived on the device from
// `offsets`, so no call needs a host synchronisation. Accumulation is fp32, k ascending, in both.
#include <math.h>

#include <mutex>

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

// a6 + a7 (+ fused combine, + a5 as a row gather) in ONE launch for small layers (H, d <= 128: the tiny fp32
// config). The layer is latency-bound there (12.6 MFLOP, every operand cold in DRAM), so a CTA owns an 8-row
// m-tile of one segment (one row per thread row: many CTAs, little serial work each) and pulls everything it
// needs in one round of loads — its rows of x (gathered straight
// from the token-order input, x[gsrc[r] / k], when `gx` is set) and the expert's whole W_gate, W_up and W_down
// slices — into shared memory, then computes h (kept in shared memory) and y with no further global loads:
// no x_sorted, no h in global memory, no second launch. Every output element is the same fmaf chain (k
// ascending from 0) with the same SiLU expression and residual add as ffn_f32_kernel's two passes: bitwise
// equal to them (tested).
constexpr int kFusedMax = 128, kRt = 8;  // rows per CTA: one per thread row, so 8x the CTAs of a 32-row tile
__host__ __device__ constexpr size_t fused_smem_floats(int H, int d) {
  return static_cast<size_t>(kRt) * (H + 1) + 2ull * d * (H + 1) + static_cast<size_t>(H) * (d + 1) +
         static_cast<size_t>(kRt) * (d + 1);
}
// global -> shared copies with no register round trip (LDGSTS): every one of a CTA's loads is in flight at
// once, which is what a cold, latency-bound layer needs; 4-byte granules keep the +1-float row padding that
// makes the compute loops' column reads conflict-free
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void load_rows_to_smem(float* dst, int ld, const float* __restrict__ srcp, int nrows,
                                                  int ncols, int warp, int lane) {
  // row-major [nrows][ncols] -> rows of ld floats; a warp per row, coalesced
  for (int r = warp; r < nrows; r += 32) {
    const float* s = srcp + static_cast<int64_t>(r) * ncols;
    float* o = dst + r * ld;
    for (int c = lane; c < ncols; c += 32) cp_async4(o + c, s + c);
  }
}
__global__ void __launch_bounds__(1024)
ffn_f32_fused_kernel(const float* __restrict__ A, const float* __restrict__ gx, int gk, int64_t rows, int H, int d,
                     int E, int nseg, const int32_t* __restrict__ offsets, const float* __restrict__ Wg,
                     const float* __restrict__ Wu, const float* __restrict__ Wd, float* __restrict__ C,
                     const int32_t* __restrict__ gsrc, const int32_t* __restrict__ osrc,
                     const float* __restrict__ residual) {
  extern __shared__ float smf[];
  __shared__ int s_off[kMaxSeg + 1];
  __shared__ int s_tstart[kMaxSeg + 1];
  const int tid = threadIdx.x;
  for (int i = tid; i <= nseg; i += blockDim.x) s_off[i] = offsets[i];
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int g = 0; g < nseg; ++g) {
      s_tstart[g] = acc;
      acc += (s_off[g + 1] - s_off[g] + kRt - 1) / kRt;
    }
    s_tstart[nseg] = acc;
  }
  __syncthreads();
  const int mtile = blockIdx.x;
  if (mtile >= s_tstart[nseg]) return;
  int g = 0;
  while (s_tstart[g + 1] <= mtile) ++g;
  const int e = g % E;
  const int64_t r0 = s_off[g] + static_cast<int64_t>(mtile - s_tstart[g]) * kRt;
  const int64_t rend = s_off[g + 1];
  const int ldA = H + 1, ldH = d + 1;
  float* sA = smf;                                   // [8][H]   the m-tile's input rows
  float* sG = sA + kRt * ldA;                        // [d][H]   W_gate[e]
  float* sU = sG + d * ldA;                          // [d][H]   W_up[e]
  float* sD = sU + d * ldA;                          // [H][d]   W_down[e]
  float* sH = sD + H * ldH;                          // [8][d]   h rows
  // one round of loads: the rows (x_sorted rows, or x[gsrc[r] / k] gathered; rows past the segment are zero)
  // and the expert's three weight slices
  const int warp = tid / 32, lane = tid % 32;
  if (warp < kRt) {  // the rows: warp w stages row w of the tile
    const int64_t r = r0 + warp;
    const float* arow = nullptr;
    if (r < rend) {
      if (gx) {
        const int64_t sl = gsrc[r];
        arow = (sl >= 0 && sl < rows) ? gx + (sl / gk) * H : nullptr;
      } else {
        arow = A + r * H;
      }
    }
    for (int c = lane; c < H; c += 32) {
      if (arow) cp_async4(sA + warp * ldA + c, arow + c);
      else sA[warp * ldA + c] = 0.f;
    }
  }
  load_rows_to_smem(sG, ldA, Wg + static_cast<int64_t>(e) * d * H, d, H, warp, lane);
  load_rows_to_smem(sU, ldA, Wu + static_cast<int64_t>(e) * d * H, d, H, warp, lane);
  load_rows_to_smem(sD, ldH, Wd + static_cast<int64_t>(e) * H * d, H, d, warp, lane);
  cp_async_wait_all();
  __syncthreads();
  // 1024 threads = 32 columns x 8 rows x 4 column groups: thread (tx, ty, tg) owns row ty and column
  // tg * 32 + tx of h, then of y (H, d <= 128), so each output element is one thread's single fmaf chain
  const int tx = tid % kTn, ty = (tid / kTn) % kRt, tg = tid / (kTn * kRt);
  const float* arow = sA + ty * ldA;
  // a6: h = silu(x Wg^T) * (x Wu^T)
  if (tg * kTn + tx < d) {
    const int n = tg * kTn + tx;
    float acc0 = 0.f, acc1 = 0.f;
    const float* bg = sG + n * ldA;
    const float* bu = sU + n * ldA;
#pragma unroll 8
    for (int q = 0; q < H; ++q) {
      const float a = arow[q];
      acc0 = fmaf(a, bg[q], acc0);
      acc1 = fmaf(a, bu[q], acc1);
    }
    sH[ty * ldH + n] = acc0 / (1.0f + expf(-acc0)) * acc1;
  }
  __syncthreads();
  // a7 (+ a8): y = h Wd^T, stored to y_sorted or, fused, to y[osrc[r]] (+ residual)
  const int64_t r = r0 + ty;
  const float* hrow = sH + ty * ldH;
  {
    const int n = tg * kTn + tx;
    if (n >= H || r >= rend) return;
    float acc = 0.f;
    const float* bd = sD + n * ldH;
#pragma unroll 8
    for (int q = 0; q < d; ++q) acc = fmaf(hrow[q], bd[q], acc);
    int64_t orow = r;
    if (osrc) {
      orow = osrc[r];
      if (orow < 0 || orow >= rows) return;
    }
    float v = acc;
    if (residual) v += residual[orow * H + n];
    C[orow * H + n] = v;
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

bool ffn_f32_fusable(int32_t H, int32_t d) {
  return H <= kFusedMax && d <= kFusedMax && H % 4 == 0 && d % 4 == 0 &&
         fused_smem_floats(H, d) * sizeof(float) <= 200u * 1024u;
}

readme_status launch_ffn_f32_fused(const float* xs, const float* x, const int32_t* gsrc, int32_t k, int64_t rows,
                                   int32_t H, int32_t E, int32_t d, int32_t nseg, const int32_t* offsets, const float* wg,
                                   const float* wu, const float* wd, float* out, const int32_t* src,
                                   const float* residual, cudaStream_t st) {
  if (rows == 0) return README_OK;
  if (nseg > kMaxSeg || !ffn_f32_fusable(H, d)) {
    set_error("fused fp32 FFN: needs <= %d segments and H, d <= %d", kMaxSeg, kFusedMax);
    return README_ERR_UNSUPPORTED;
  }
  const int64_t mtiles_ub = nseg + (rows + kRt - 1) / kRt;
  const size_t smem = fused_smem_floats(H, d) * sizeof(float);
  static std::once_flag once[64];  // the opt-in shared-memory size, once per device
  static cudaError_t attr_err[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  std::call_once(once[dev], [dev] {
    attr_err[dev] = cudaFuncSetAttribute(ffn_f32_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  README_CUDA(attr_err[dev]);
  ffn_f32_fused_kernel<<<static_cast<unsigned>(mtiles_ub), 1024, smem, st>>>(xs, x, k, rows, H, d, E, nseg, offsets,
                                                                          wg, wu, wd, out, gsrc, src, residual);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

}  // namespace readme
