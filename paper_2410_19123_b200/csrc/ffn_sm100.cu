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
#include <cudaTypedefs.h>

#include <mutex>

#include "kernels.h"

namespace readme {

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

// ---- PTX wrappers ----------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, void* dst, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, void* dst, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T, both K-major.
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor for a K-major operand tile stored by TMA with 128-byte swizzle:
// rows of 128 B, 8-row core groups 1024 B apart (SBO), LBO unused for swizzled K-major (=1),
// version 1 (sm_100), layout type 2 = SWIZZLE_128B. Advancing K by 16 bf16 = +32 B on the start address.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;           // LBO (16 B units)
  d |= static_cast<uint64_t>(1024u >> 4) << 32;   // SBO (16 B units)
  d |= static_cast<uint64_t>(1u) << 46;           // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;           // SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

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

__device__ __forceinline__ float silu_f(float z) { return z / (1.0f + __expf(-z)); }

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
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s.tmem_base)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
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
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * kBN);
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&s.full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(s.a[stage]), b0 = smem_u32(s.b[stage]);
#pragma unroll
          for (int kk = 0; kk < kBK / kUK; ++kk) {
            tc_mma(d_tmem, sdesc_sw128(a0 + kk * kUK * 2), sdesc_sw128(b0 + kk * kUK * 2), idesc,
                   (kb | kk) != 0 ? 1u : 0u);
          }
          tc_commit(&s.empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&s.tfull[acc]);
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
      tc_fence_after();
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
                v.x = pack_bf16x2(silu_f(__uint_as_float(gr[j + 0])) * __uint_as_float(ur[j + 0]),
                                  silu_f(__uint_as_float(gr[j + 1])) * __uint_as_float(ur[j + 1]));
                v.y = pack_bf16x2(silu_f(__uint_as_float(gr[j + 2])) * __uint_as_float(ur[j + 2]),
                                  silu_f(__uint_as_float(gr[j + 3])) * __uint_as_float(ur[j + 3]));
                v.z = pack_bf16x2(silu_f(__uint_as_float(gr[j + 4])) * __uint_as_float(ur[j + 4]),
                                  silu_f(__uint_as_float(gr[j + 5])) * __uint_as_float(ur[j + 5]));
                v.w = pack_bf16x2(silu_f(__uint_as_float(gr[j + 6])) * __uint_as_float(ur[j + 6]),
                                  silu_f(__uint_as_float(gr[j + 7])) * __uint_as_float(ur[j + 7]));
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
      tc_fence_before();
      mbar_arrive(&s.tempty[acc]);
    }
  }

  // ---- teardown ----
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                 : "memory");
  }
}

// ---- host: tensor maps ------------------------------------------------------------------------------
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

readme_status launch_ffn_bf16(const __nv_bfloat16* xs, int64_t rows, int32_t H, int32_t E, int32_t d,
                              int32_t nseg, const int32_t* offsets, const __nv_bfloat16* wg,
                              const __nv_bfloat16* wu, const __nv_bfloat16* wd, __nv_bfloat16* ys,
                              __nv_bfloat16* h_ws, cudaStream_t st) {
  if (rows == 0) return README_OK;
  if (nseg > kMaxSeg) {
    set_error("bf16 expert FFN supports at most %d segments (got %d)", kMaxSeg, nseg);
    return README_ERR_UNSUPPORTED;
  }
  readme_status rs = set_smem_attr();
  if (rs != README_OK) return rs;
  CUtensorMap mA1, mG, mU, mA2, mD;
  bool ok = make_map_2d(&mA1, xs, H, rows, kBK, kBM) && make_map_3d(&mG, wg, H, d, E, kBK, kBN / 2) &&
            make_map_3d(&mU, wu, H, d, E, kBK, kBN / 2) && make_map_2d(&mA2, h_ws, d, rows, kBK, kBM) &&
            make_map_3d(&mD, wd, d, H, E, kBK, kBN);
  if (!ok) {
    set_error("cuTensorMapEncodeTiled failed (driver entry point missing or bad shape/alignment)");
    return README_ERR_CUDA;
  }
  const int64_t mt_ub = nseg + (rows + kBM - 1) / kBM;
  const int nsm = num_sms();
  const int64_t t1 = mt_ub * ((d + kBN / 2 - 1) / (kBN / 2));
  const int64_t t2 = mt_ub * ((H + kBN - 1) / kBN);
  const int g1 = static_cast<int>(t1 < nsm ? t1 : nsm);
  const int g2 = static_cast<int>(t2 < nsm ? t2 : nsm);
  ffn_gemm_kernel<0><<<g1, kThreads, kSmemBytes, st>>>(mA1, mG, mU, H, d, E, nseg, offsets, h_ws);
  README_CUDA(cudaGetLastError());
  ffn_gemm_kernel<1><<<g2, kThreads, kSmemBytes, st>>>(mA2, mD, mD, d, H, E, nseg, offsets, ys);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

}  // namespace readme
