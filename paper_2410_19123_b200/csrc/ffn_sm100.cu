// ffn_sm100.cu — a6/a7: the grouped SwiGLU expert GEMMs on the 5th-generation tensor cores (bf16).
//
// Paper: each expert is a neuron subset of the dense FFN, F_i(x) = W_2 M_i^T sigma(M_i W_1 x)
// (§3), SwiGLU form (Q4): for the rows r of expert e (segment g, e = g % E)
//     GEMM1 (kMode 0):  h_r = silu(x_r . W_gate[e]^T) * (x_r . W_up[e]^T)     [rows, d], bf16 (Q11)
//     GEMM2 (kMode 1):  y_r = h_r . W_down[e]^T                                 [rows, H], bf16
// The expert layers are where the paper says the time goes.
//
// B200 design (one persistent CTA per SM, warp-specialised, 192 threads):
//   warp 0    TMA producer: A tile [128 x 64] of the expert-contiguous rows and the B tile(s) of the
//             expert's weights (3-D tensor maps [E][N][K], so a partial N tile is zero-filled per expert)
//             land in a kStages-deep shared-memory ring (128-byte swizzle), completion via mbarrier tx.
//   warp 1    allocates 512 TMEM columns (two 128 x 256 fp32 accumulators) and one elected lane issues
//             tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256, K=16) x 4 per stage; tcgen05.commit
//             frees the smem stage and, after the last K block, hands the accumulator to the epilogue.
//   warps 2-5 epilogue: tcgen05.ld (32 lanes x 32 columns per instruction) -> fp32 SiLU(gate)*up (GEMM1)
//             or plain convert (GEMM2) -> bf16 -> 16-byte global stores, predicated to the expert's rows,
//             so a tile that overhangs into the next expert's rows never clobbers them.
//   GEMM1 interleaves gate and up inside ONE MMA: the B tile is 128 rows of W_gate followed by the same
//   128 rows of W_up, so accumulator columns [0,128) are gate and [128,256) are up for the same neurons.
// Tile order: segment-major, then N tile, then M tile fastest, statically strided over the persistent
// grid, so co-resident CTAs share the expert's weight tile in L2. The tile list is derived on the device
// from `offsets` (no host synchronisation; CUDA-graph capturable). No split-K: every output element has a
// fixed K order, so results are bitwise batch-invariant and permutation-equivariant (P4, P13).
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "kernels.h"
#include "tc_common.cuh"

namespace readme {

using namespace tc;

namespace {

constexpr int kBM = 128;     // rows per tile (TMEM lanes)
constexpr int kBN = 256;     // MMA N (accumulator columns)
constexpr int kBK = 64;      // K per stage: one 128-byte swizzle row of bf16
constexpr int kUK = 16;      // K per tcgen05.mma (kind::f16)
constexpr int kStages = 4;
constexpr int kThreads = 192;
constexpr int kMaxSeg = 512;
constexpr int kABytes = kBM * kBK * 2;  // 16 KB
constexpr int kBBytes = kBN * kBK * 2;  // 32 KB
constexpr int kTmemCols = 512;

struct __align__(8) Smem {
  uint8_t a[kStages][kABytes];
  uint8_t b[kStages][kBBytes];
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  int seg_off[kMaxSeg + 1];
  int tile_start[kMaxSeg + 1];
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;  // + alignment slack (swizzle-128B needs 1024 B)

struct Tile {
  int g;       // segment
  int m0;      // first row (global row index into the expert-contiguous buffer)
  int mrows;   // rows of this tile that belong to the segment
  int n0;      // first output column
};

__device__ __forceinline__ Tile decode_tile(const Smem& s, int t, int nseg, int NT, int bn_out, int& gcur) {
  while (gcur + 1 < nseg && s.tile_start[gcur + 1] <= t) ++gcur;
  const int g = gcur;
  const int cnt = s.seg_off[g + 1] - s.seg_off[g];
  const int mt_g = (cnt + kBM - 1) / kBM;
  const int local = t - s.tile_start[g];
  const int nt = local / mt_g, mt = local % mt_g;
  Tile tl;
  tl.g = g;
  tl.m0 = s.seg_off[g] + mt * kBM;
  tl.mrows = min(kBM, cnt - mt * kBM);
  tl.n0 = nt * bn_out;
  return tl;
}


template <int kMode>
__global__ void __launch_bounds__(kThreads, 1)
ffn_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                const __grid_constant__ CUtensorMap tmB1, int K, int N, int E, int nseg,
                const int32_t* __restrict__ offsets, __nv_bfloat16* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
  constexpr int kBnOut = kMode == 0 ? kBN / 2 : kBN;  // output columns per tile
  const int NT = (N + kBnOut - 1) / kBnOut;
  const int KB = (K + kBK - 1) / kBK;

  // ---- setup: segment table, tile prefix, barriers, TMEM ----
  for (int i = tid; i <= nseg; i += kThreads) s.seg_off[i] = offsets[i];
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB0);
    if (kMode == 0) prefetch_tmap(&tmB1);
  }
  if (warp == 1) {
    tmem_alloc<1>(&s.tmem_base, kTmemCols);
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int g = 0; g < nseg; ++g) {
      s.tile_start[g] = acc;
      acc += (s.seg_off[g + 1] - s.seg_off[g] + kBM - 1) / kBM * NT;
    }
    s.tile_start[nseg] = acc;
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s.tfull[i], 1);
      mbar_init(&s.tempty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const int ntiles = s.tile_start[nseg];
  const uint32_t tmem_base = s.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      int gcur = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const Tile tl = decode_tile(s, t, nseg, NT, kBnOut, gcur);
        const int e = tl.g % E;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&s.empty[stage], phase ^ 1);
          mbar_expect_tx(&s.full[stage], kABytes + kBBytes);
          tma_load_2d(&tmA, s.a[stage], &s.full[stage], kb * kBK, tl.m0);
          if (kMode == 0) {
            tma_load_3d(&tmB0, s.b[stage], &s.full[stage], kb * kBK, tl.n0, e);
            tma_load_3d(&tmB1, s.b[stage] + kBBytes / 2, &s.full[stage], kb * kBK, tl.n0, e);
          } else {
            tma_load_3d(&tmB0, s.b[stage], &s.full[stage], kb * kBK, tl.n0, e);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idesc = idesc_bf16(kBM, kBN);
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int acc = i & 1;
        const uint32_t use = static_cast<uint32_t>(i >> 1);
        mbar_wait(&s.tempty[acc], (use & 1u) ^ 1u);
        fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * kBN);
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&s.full[stage], phase);
          fence_after();
          const uint32_t a0 = smem_u32(s.a[stage]), b0 = smem_u32(s.b[stage]);
#pragma unroll
          for (int kk = 0; kk < kBK / kUK; ++kk) {
            mma_f16<1>(d_tmem, sdesc_sw128(a0 + kk * kUK * 2), sdesc_sw128(b0 + kk * kUK * 2), idesc,
                   (kb | kk) != 0 ? 1u : 0u);
          }
          commit(&s.empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        commit(&s.tfull[acc]);
      }
    }
  } else {
    // ===== epilogue: warps 2..5 -> TMEM lane quarter (warp % 4) =====
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int gcur = 0, i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const Tile tl = decode_tile(s, t, nseg, NT, kBnOut, gcur);
      const int acc = i & 1;
      const uint32_t use = static_cast<uint32_t>(i >> 1);
      mbar_wait(&s.tfull[acc], use & 1u);
      fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * kBN);
      const bool valid = row < tl.mrows;
      __nv_bfloat16* orow = out + static_cast<int64_t>(tl.m0 + row) * N;
      if (kMode == 0) {
#pragma unroll 1
        for (int c = 0; c < kBN / 2; c += 32) {
          uint32_t gr[32], ur[32];
          tmem_ld32(taddr + c, gr);
          tmem_ld32(taddr + kBN / 2 + c, ur);
          tmem_wait_ld();
          const int col0 = tl.n0 + c;
          if (valid) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              if (col0 + j < N) {
                uint4 v;
                v.x = pack_bf16x2(silu(__uint_as_float(gr[j + 0])) * __uint_as_float(ur[j + 0]),
                                  silu(__uint_as_float(gr[j + 1])) * __uint_as_float(ur[j + 1]));
                v.y = pack_bf16x2(silu(__uint_as_float(gr[j + 2])) * __uint_as_float(ur[j + 2]),
                                  silu(__uint_as_float(gr[j + 3])) * __uint_as_float(ur[j + 3]));
                v.z = pack_bf16x2(silu(__uint_as_float(gr[j + 4])) * __uint_as_float(ur[j + 4]),
                                  silu(__uint_as_float(gr[j + 5])) * __uint_as_float(ur[j + 5]));
                v.w = pack_bf16x2(silu(__uint_as_float(gr[j + 6])) * __uint_as_float(ur[j + 6]),
                                  silu(__uint_as_float(gr[j + 7])) * __uint_as_float(ur[j + 7]));
                st_v4(reinterpret_cast<uint4*>(orow + col0 + j), v);
              }
            }
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < kBN; c += 32) {
          uint32_t vr[32];
          tmem_ld32(taddr + c, vr);
          tmem_wait_ld();
          const int col0 = tl.n0 + c;
          if (valid) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              if (col0 + j < N) {
                uint4 v;
                v.x = pack_bf16x2(__uint_as_float(vr[j + 0]), __uint_as_float(vr[j + 1]));
                v.y = pack_bf16x2(__uint_as_float(vr[j + 2]), __uint_as_float(vr[j + 3]));
                v.z = pack_bf16x2(__uint_as_float(vr[j + 4]), __uint_as_float(vr[j + 5]));
                v.w = pack_bf16x2(__uint_as_float(vr[j + 6]), __uint_as_float(vr[j + 7]));
                st_v4(reinterpret_cast<uint4*>(orow + col0 + j), v);
              }
            }
          }
        }
      }
      fence_before();
      mbar_arrive(&s.tempty[acc]);
    }
  }

  // ---- teardown ----
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 1) {
    tmem_dealloc<1>(tmem_base, kTmemCols);
  }
}

// ---- host: tensor maps ------------------------------------------------------------------------------
}  // namespace
namespace tc {
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}
}  // namespace

bool make_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_in,
                 uint32_t box_out) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_in, box_out};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map_3d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t mid, uint64_t outer, uint32_t box_in,
                 uint32_t box_mid) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {inner, mid, outer};
  cuuint64_t strides[2] = {inner * 2, inner * mid * 2};
  cuuint32_t box[3] = {box_in, box_mid, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace tc

namespace {
readme_status set_smem_attr() {
  static std::once_flag once[64];
  static cudaError_t err[64];
  int dev = 0;
  README_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) dev = 0;
  std::call_once(once[dev], [&] {
    err[dev] = cudaFuncSetAttribute(ffn_gemm_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmemBytes));
    if (err[dev] == cudaSuccess)
      err[dev] = cudaFuncSetAttribute(ffn_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kSmemBytes));
  });
  if (err[dev] != cudaSuccess) return cuda_fail(err[dev], "cudaFuncSetAttribute(ffn_gemm_kernel)");
  return README_OK;
}

}  // namespace

readme_status launch_gemm_1cta(int mode, const __nv_bfloat16* A, int64_t rows, int32_t K, int32_t N, int32_t E,
                               int32_t nseg, const int32_t* offsets, const __nv_bfloat16* B0,
                               const __nv_bfloat16* B1, __nv_bfloat16* out, cudaStream_t st) {
  if (rows == 0) return README_OK;
  if (nseg > kMaxSeg) {
    set_error("bf16 expert FFN supports at most %d segments (got %d)", kMaxSeg, nseg);
    return README_ERR_UNSUPPORTED;
  }
  readme_status rs = set_smem_attr();
  if (rs != README_OK) return rs;
  CUtensorMap mA, mB0, mB1;
  const uint32_t bn_box = mode == 0 ? kBN / 2 : kBN;
  bool ok = tc::make_map_2d(&mA, A, K, rows, kBK, kBM) && tc::make_map_3d(&mB0, B0, K, N, E, kBK, bn_box) &&
            (mode == 1 || tc::make_map_3d(&mB1, B1, K, N, E, kBK, bn_box));
  if (!ok) {
    set_error("cuTensorMapEncodeTiled failed (driver entry point missing or bad shape/alignment)");
    return README_ERR_CUDA;
  }
  if (mode == 1) mB1 = mB0;
  const int64_t mt_ub = nseg + (rows + kBM - 1) / kBM;
  const int nsm = num_sms();
  const int64_t tiles = mt_ub * ((N + bn_box - 1) / bn_box);
  const int grid = static_cast<int>(tiles < nsm ? tiles : nsm);
  if (mode == 0)
    ffn_gemm_kernel<0><<<grid, kThreads, kSmemBytes, st>>>(mA, mB0, mB1, K, N, E, nseg, offsets, out);
  else
    ffn_gemm_kernel<1><<<grid, kThreads, kSmemBytes, st>>>(mA, mB0, mB1, K, N, E, nseg, offsets, out);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

// Kernel choice: the CTA-pair kernel by default; README_FFN_KERNEL=1cta selects the single-CTA one (kept
// for A/B measurement). The scattered (fused-combine) epilogue exists only in the CTA-pair kernel.
bool force_1cta() {
  const char* v = getenv("README_FFN_KERNEL");
  return v && strcmp(v, "1cta") == 0;
}  // (=split / =unfused keep the CTA-pair kernels; see capi.cu ffn_path())

readme_status launch_gate_up_bf16(const __nv_bfloat16* xs, int64_t rows, int32_t H, int32_t E, int32_t d,
                                  int32_t nseg, const int32_t* offsets, const __nv_bfloat16* wg,
                                  const __nv_bfloat16* wu, __nv_bfloat16* h, cudaStream_t st) {
  if (force_1cta()) return launch_gemm_1cta(0, xs, rows, H, d, E, nseg, offsets, wg, wu, h, st);
  return launch_gemm_2cta(0, xs, rows, H, d, E, nseg, offsets, wg, wu, h, nullptr, nullptr, st);
}

readme_status launch_down_bf16(const __nv_bfloat16* h, int64_t rows, int32_t H, int32_t E, int32_t d, int32_t nseg,
                               const int32_t* offsets, const __nv_bfloat16* wd, __nv_bfloat16* out,
                               const int32_t* src, const __nv_bfloat16* residual, cudaStream_t st) {
  if (force_1cta() && src == nullptr && residual == nullptr)
    return launch_gemm_1cta(1, h, rows, d, H, E, nseg, offsets, wd, wd, out, st);
  return launch_gemm_2cta(1, h, rows, d, H, E, nseg, offsets, wd, nullptr, out, src, residual, st);
}

}  // namespace readme
