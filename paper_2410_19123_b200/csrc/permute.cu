// permute.cu — a5 dispatch, a8 combine and the setup-time expert slicing.
//
// dispatch  x_sorted[dest[s]] = x[s / k]                         (tokens grouped per expert)
// combine   y[t] = res[t] + sum_{j<k} w[t,j] * y_sorted[dest[t*k+j]]   (Eq. 2's weighted sum)
// slicing   W_gate,e = W_gate[S_e, :], W_up,e = W_up[S_e, :], W_down,e = W_down[:, S_e]
//
// All three are HBM-bound row moves. One warp per row; each lane keeps kUnroll 128-bit loads in flight
// before storing (Little's law: ~6.4 TB/s x ~1 us needs ~45 KB in flight per SM; 64 warps x 32 lanes x
// 4 x 16 B = 128 KB), L1 bypassed for the streamed source.
#include <stdlib.h>

#include <mutex>

#include "kernels.h"
#include "tc_common.cuh"

namespace readme {

namespace {

constexpr int kPermThreads = 256;

// The dispatch kernels let the expert FFN (launched as a programmatic dependent) start its prologue and
// warm L2 with weights while they run; the FFN waits for their completion before reading x_sorted.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void set_offsets_kernel(int32_t* offs, int32_t T) {
  offs[0] = 0;
  offs[1] = T;
}
constexpr int kUnroll = 4;

// One warp moves one row of `vec` uint4 from src_row to dst_row.
template <int U = kUnroll>
__device__ __forceinline__ void copy_row(const uint4* __restrict__ s, uint4* __restrict__ d, int vec, int lane) {
  int i = lane;
  for (; i + (U - 1) * kWarp < vec; i += U * kWarp) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = ld_nc_v4(s + i + u * kWarp);
#pragma unroll
    for (int u = 0; u < U; ++u) st_v4(d + i + u * kWarp, r[u]);
  }
  for (; i < vec; i += kWarp) st_v4(d + i, ld_nc_v4(s + i));
}

template <int U>
__global__ void __launch_bounds__(kPermThreads)
dispatch_kernel(const uint4* __restrict__ x, int vec, int64_t nslots, int k, const int32_t* __restrict__ dest,
                uint4* __restrict__ xs, uint32_t* __restrict__ dev_status) {
  pdl_launch_dependents();
  const int lane = threadIdx.x % kWarp;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kPermThreads / kWarp);
  for (int64_t s = blockIdx.x * static_cast<int64_t>(kPermThreads / kWarp) + threadIdx.x / kWarp; s < nslots;
       s += warps) {
    const int32_t r = __ldg(dest + s);
    if (r < 0 || r >= nslots) {
      if (lane == 0 && dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
      continue;
    }
    copy_row<U>(x + (s / k) * vec, xs + static_cast<int64_t>(r) * vec, vec, lane);
  }
}

// Row moves through the bulk-copy engine (large batches): each of kBulkCopiers single-thread copiers per CTA
// streams its rows global -> shared -> global with cp.async.bulk — a ring of kBulkSlots whole rows,
// loads completing on per-slot mbarriers, stores tracked as bulk groups — so one thread keeps several 8 KB
// rows in flight instead of a warp of 16-byte loads. Rows are byte copies (bit-exact).
constexpr int kBulkCopiers = 4;
constexpr int kBulkSlots = 4;
constexpr size_t kBulkMaxSmem = 192 * 1024;

__device__ __forceinline__ void bulk_load_row(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(dst_smem))),
      "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}
__device__ __forceinline__ void bulk_store_row(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(static_cast<uint32_t>(__cvta_generic_to_shared(src_smem))), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// kGather = false: scatter dispatch, row s of x_sorted's input x[s / k] goes to x_sorted[dest[s]];
// kGather = true: the k = 1 combine without residual, y[t] = y_sorted[dest[t]] (rows = T, k = 1).
template <bool kGather>
__global__ void __launch_bounds__(kBulkCopiers * kWarp)
move_rows_bulk_kernel(const uint8_t* __restrict__ in, uint32_t row_bytes, int64_t nslots, int k,
                      const int32_t* __restrict__ dest, uint8_t* __restrict__ out, uint32_t* __restrict__ dev_status) {
  pdl_launch_dependents();
  extern __shared__ __align__(128) uint8_t bulk_ring[];
  __shared__ __align__(8) uint64_t bar[kBulkCopiers][kBulkSlots];
  const int copier = threadIdx.x / kWarp;
  if (threadIdx.x % kWarp != 0) return;  // one thread per copier; its warp's other lanes have no work
  uint8_t* ring = bulk_ring + static_cast<size_t>(copier) * kBulkSlots * row_bytes;
  uint64_t* b = bar[copier];
  for (int i = 0; i < kBulkSlots; ++i) tc::mbar_init(&b[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const int64_t c = static_cast<int64_t>(blockIdx.x) * kBulkCopiers + copier;
  const int64_t nc = static_cast<int64_t>(gridDim.x) * kBulkCopiers;
  const int64_t mine = c < nslots ? (nslots - 1 - c) / nc + 1 : 0;
  auto valid = [&](int32_t r) { return r >= 0 && r < nslots; };
  auto load = [&](int64_t j) {
    const int slot = static_cast<int>(j % kBulkSlots);
    const int64_t s = c + j * nc;
    int64_t src_row = s / k;
    if constexpr (kGather) {
      const int32_t r = __ldg(dest + s);
      src_row = valid(r) ? r : 0;  // a bad index still fills the slot (row 0); its store is skipped
    }
    tc::mbar_expect_tx(&b[slot], row_bytes);
    bulk_load_row(ring + static_cast<size_t>(slot) * row_bytes, in + src_row * static_cast<int64_t>(row_bytes),
                  row_bytes, &b[slot]);
  };
  for (int64_t j = 0; j < mine && j < kBulkSlots; ++j) load(j);
  for (int64_t j = 0; j < mine; ++j) {
    const int slot = static_cast<int>(j % kBulkSlots);
    const int64_t s = c + j * nc;
    const int32_t r = __ldg(dest + s);
    tc::mbar_wait(&b[slot], static_cast<uint32_t>(j / kBulkSlots) & 1u);
    if (!valid(r)) {
      if (dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
    } else {
      bulk_store_row(out + (kGather ? s : static_cast<int64_t>(r)) * row_bytes,
                     ring + static_cast<size_t>(slot) * row_bytes, row_bytes);
    }
    if (j + kBulkSlots < mine) {
      // the slot is refilled once this row's store has read it out of shared memory
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(j + kBulkSlots);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 v = ld_nc_v4(reinterpret_cast<const uint4*>(p));
  f[0] = bf16_lo(v.x); f[1] = bf16_hi(v.x); f[2] = bf16_lo(v.y); f[3] = bf16_hi(v.y);
  f[4] = bf16_lo(v.z); f[5] = bf16_hi(v.z); f[6] = bf16_lo(v.w); f[7] = bf16_hi(v.w);
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 v;
  v.x = pack_bf16x2(f[0], f[1]); v.y = pack_bf16x2(f[2], f[3]);
  v.z = pack_bf16x2(f[4], f[5]); v.w = pack_bf16x2(f[6], f[7]);
  st_v4(reinterpret_cast<uint4*>(p), v);
}
__device__ __forceinline__ void load8(const float* p, float (&f)[8]) {
  const uint4 a = ld_nc_v4(reinterpret_cast<const uint4*>(p));
  const uint4 b = ld_nc_v4(reinterpret_cast<const uint4*>(p) + 1);
  f[0] = __uint_as_float(a.x); f[1] = __uint_as_float(a.y); f[2] = __uint_as_float(a.z); f[3] = __uint_as_float(a.w);
  f[4] = __uint_as_float(b.x); f[5] = __uint_as_float(b.y); f[6] = __uint_as_float(b.z); f[7] = __uint_as_float(b.w);
}
__device__ __forceinline__ void store8(float* p, const float (&f)[8]) {
  st_v4(reinterpret_cast<uint4*>(p), make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]),
                                                __float_as_uint(f[2]), __float_as_uint(f[3])));
  st_v4(reinterpret_cast<uint4*>(p) + 1, make_uint4(__float_as_uint(f[4]), __float_as_uint(f[5]),
                                                    __float_as_uint(f[6]), __float_as_uint(f[7])));
}

__device__ __forceinline__ void load8_cached(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  f[0] = bf16_lo(v.x); f[1] = bf16_hi(v.x); f[2] = bf16_lo(v.y); f[3] = bf16_hi(v.y);
  f[4] = bf16_lo(v.z); f[5] = bf16_hi(v.z); f[6] = bf16_lo(v.w); f[7] = bf16_hi(v.w);
}
__device__ __forceinline__ void load8_cached(const float* p, float (&f)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// Pre-norm dispatch for the MoE-only stack (reading Q10: x <- x + MoE(RMSNorm(x)), RMSNorm weight 1):
// x_sorted[dest[t*k+j]] = x[t] / sqrt(mean(x[t]^2) + eps), fp32 statistics, one rounding. One warp per token:
// pass 1 sums squares (row stays in L1), pass 2 scales and writes the k destination rows.
template <typename Elt>
__global__ void __launch_bounds__(kPermThreads)
dispatch_rmsnorm_kernel(const Elt* __restrict__ x, int H, int64_t T, int k, const int32_t* __restrict__ dest,
                        float eps, Elt* __restrict__ xs, uint32_t* __restrict__ dev_status) {
  pdl_launch_dependents();
  const int lane = threadIdx.x % kWarp;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kPermThreads / kWarp);
  const int groups = H / 8;
  const int64_t nrows = T * k;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(kPermThreads / kWarp) + threadIdx.x / kWarp; t < T;
       t += warps) {
    const Elt* row = x + t * H;
    float ss = 0.f;
    for (int g = lane; g < groups; g += kWarp) {
      float v[8];
      load8_cached(row + g * 8, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) ss = fmaf(v[i], v[i], ss);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float r = rsqrtf(ss / static_cast<float>(H) + eps);
    for (int g = lane; g < groups; g += kWarp) {
      float v[8];
      load8_cached(row + g * 8, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] *= r;
      for (int j = 0; j < k; ++j) {
        const int32_t dr = __ldg(dest + t * k + j);
        if (dr < 0 || dr >= nrows) {
          if (dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
          continue;
        }
        store8(xs + static_cast<int64_t>(dr) * H + g * 8, v);
      }
    }
  }
}

// Same pre-norm dispatch for bf16 rows of H = 256 * nch <= 4096 elements: the whole row is loaded once into
// registers (nch x 16 B per lane, all in flight) instead of read twice with one load in flight per lane —
// 62.5 us at 16384 x 4096 (0.63 of the copy bandwidth, config 4's per-layer launch list) before. Same sum
// order (lane-strided 8-element groups, then the butterfly) and roundings: bitwise equal to the kernel above.
constexpr int kNormMaxChunks = 16;
__global__ void __launch_bounds__(kPermThreads)
dispatch_rmsnorm_row_kernel(const uint4* __restrict__ x, int nch, int64_t T, int k, const int32_t* __restrict__ dest,
                            float eps, uint4* __restrict__ xs, uint32_t* __restrict__ dev_status) {
  pdl_launch_dependents();
  const int lane = threadIdx.x % kWarp;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kPermThreads / kWarp);
  const int vec = nch * kWarp;  // 16-byte vectors per row
  const int64_t nrows = T * k;
  const float hf = static_cast<float>(vec * 8);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(kPermThreads / kWarp) + threadIdx.x / kWarp; t < T;
       t += warps) {
    const uint4* row = x + t * vec;
    uint4 w[kNormMaxChunks];
#pragma unroll
    for (int j = 0; j < kNormMaxChunks; ++j)
      if (j < nch) w[j] = ld_nc_v4(row + lane + j * kWarp);
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < kNormMaxChunks; ++j) {
      if (j < nch) {
        const float f[8] = {bf16_lo(w[j].x), bf16_hi(w[j].x), bf16_lo(w[j].y), bf16_hi(w[j].y),
                            bf16_lo(w[j].z), bf16_hi(w[j].z), bf16_lo(w[j].w), bf16_hi(w[j].w)};
#pragma unroll
        for (int i = 0; i < 8; ++i) ss = fmaf(f[i], f[i], ss);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float r = rsqrtf(ss / hf + eps);
#pragma unroll
    for (int j = 0; j < kNormMaxChunks; ++j) {
      if (j < nch) {
        uint4 o;
        o.x = pack_bf16x2(bf16_lo(w[j].x) * r, bf16_hi(w[j].x) * r);
        o.y = pack_bf16x2(bf16_lo(w[j].y) * r, bf16_hi(w[j].y) * r);
        o.z = pack_bf16x2(bf16_lo(w[j].z) * r, bf16_hi(w[j].z) * r);
        o.w = pack_bf16x2(bf16_lo(w[j].w) * r, bf16_hi(w[j].w) * r);
        w[j] = o;
      }
    }
    for (int jj = 0; jj < k; ++jj) {
      const int32_t dr = __ldg(dest + t * k + jj);
      if (dr < 0 || dr >= nrows) {
        if (lane == 0 && dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
        continue;
      }
      uint4* drow = xs + static_cast<int64_t>(dr) * vec;
#pragma unroll
      for (int j = 0; j < kNormMaxChunks; ++j)
        if (j < nch) st_v4(drow + lane + j * kWarp, w[j]);
    }
  }
}

// readme_moe_layer's a4-finalize + a5 in one pass: dest holds each slot's rank inside its expert (left by
// route_tile_kernel); row = offsets[e] + rank, then dest/src are finalised and the token row copied there.
__global__ void __launch_bounds__(kPermThreads)
finalize_dispatch_kernel(const uint4* __restrict__ x, int vec, int64_t nslots, int k, int E,
                         const int32_t* __restrict__ topk_idx, const int32_t* __restrict__ offsets,
                         int32_t* __restrict__ dest, int32_t* __restrict__ src, uint4* __restrict__ xs) {
  pdl_launch_dependents();
  __shared__ int s_off[README_MAX_EXPERTS + 1];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) s_off[i] = offsets[i];
  __syncthreads();
  const int lane = threadIdx.x % kWarp;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kPermThreads / kWarp);
  for (int64_t s = blockIdx.x * static_cast<int64_t>(kPermThreads / kWarp) + threadIdx.x / kWarp; s < nslots;
       s += warps) {
    int r = 0;
    if (lane == 0) {
      r = s_off[topk_idx[s]] + dest[s];
      dest[s] = r;
      if (src) src[r] = static_cast<int32_t>(s);
    }
    r = __shfl_sync(0xffffffffu, r, 0);
    copy_row(x + (s / k) * vec, xs + static_cast<int64_t>(r) * vec, vec, lane);
  }
}

// readme_moe_layer's a5 after the single-launch route (dest/src final): gather form x_sorted[r] = x[src[r]/k].
// Warp w of W moves rows w, w + W, w + 2W, ... so the rows complete in ascending waves of W rows; after each
// row the warp publishes xready[r] = 1 (release, gpu scope) and the expert FFN, launched behind this kernel
// as a programmatic dependent and co-resident with it, starts expert 0's gate/up tiles after the first wave
// instead of after the whole dispatch. Co-residency is a register budget per SM sub-partition (16K each):
// the FFN CTA puts up to 2 warps x 152 x 32 registers on one, which leaves room for 3 warps of <= 64
// registers — hence ONE CTA of 12 warps per SM. The TMA (async proxy) reads x_sorted, hence the proxy
// fence before the flag.
constexpr int kGatherUnroll = 8;
#ifndef README_GATHER_THREADS  // lab builds may shrink it (README_NVCC_EXTRA)
#define README_GATHER_THREADS 384
#endif
constexpr int kGatherThreads = README_GATHER_THREADS;
__global__ void __maxnreg__(64)
dispatch_gather_kernel(const uint4* __restrict__ x, int vec, int64_t nrows, int k, const int32_t* __restrict__ src,
                       uint4* __restrict__ xs, uint32_t* __restrict__ xready, uint32_t* __restrict__ dev_status,
                       uint64_t* __restrict__ trace) {
  pdl_launch_dependents();
  if (trace && threadIdx.x == 0) trace_min(trace, 0);
  const int lane = threadIdx.x % kWarp;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kGatherThreads / kWarp);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(kGatherThreads / kWarp) + threadIdx.x / kWarp; r < nrows;
       r += warps) {
    const int32_t sl = __ldg(src + r);
    if (sl < 0 || sl >= nrows) {
      if (lane == 0 && dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
    } else {
      const uint4* srow = x + (sl / k) * static_cast<int64_t>(vec);
      uint4* drow = xs + r * vec;
      int i = lane;
      for (; i + (kGatherUnroll - 1) * kWarp < vec; i += kGatherUnroll * kWarp) {
        uint4 v[kGatherUnroll];
#pragma unroll
        for (int u = 0; u < kGatherUnroll; ++u) v[u] = ld_nc_v4(srow + i + u * kWarp);
#pragma unroll
        for (int u = 0; u < kGatherUnroll; ++u) st_v4(drow + i + u * kWarp, v[u]);
      }
      for (; i < vec; i += kWarp) st_v4(drow + i, ld_nc_v4(srow + i));
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(xready + r), "r"(1u) : "memory");
    }
  }
  if (trace && threadIdx.x % kWarp == 0) trace_max(trace, 1);
}

// The stack's pre-norm dispatch in the same gather form (readme_moe_stack with the fused FFN behind it):
// x_sorted[r] = RMSNorm(x[src[r] / k]) with the row flags of dispatch_gather_kernel. The FFN of the same
// layer updates x in place (residual fused), but only for rows of m-tiles whose flags it has acquired, i.e.
// after this kernel has finished reading those tokens (k == 1: one row per token).
template <typename Elt>
__global__ void __maxnreg__(64)
dispatch_rmsnorm_gather_kernel(const Elt* __restrict__ x, int H, int64_t nrows, int k,
                               const int32_t* __restrict__ src, float eps, Elt* __restrict__ xs,
                               uint32_t* __restrict__ xready, uint32_t* __restrict__ dev_status) {
  pdl_launch_dependents();
  const int lane = threadIdx.x % kWarp;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kGatherThreads / kWarp);
  const int groups = H / 8;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(kGatherThreads / kWarp) + threadIdx.x / kWarp; r < nrows;
       r += warps) {
    const int32_t sl = __ldg(src + r);
    if (sl < 0 || sl >= nrows) {
      if (lane == 0 && dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
    } else {
      const Elt* row = x + static_cast<int64_t>(sl / k) * H;
      float ss = 0.f;
      for (int g = lane; g < groups; g += kWarp) {
        float v[8];
        load8_cached(row + g * 8, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) ss = fmaf(v[i], v[i], ss);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
      const float rs = rsqrtf(ss / static_cast<float>(H) + eps);
      Elt* drow = xs + r * H;
      for (int g = lane; g < groups; g += kWarp) {
        float v[8];
        load8_cached(row + g * 8, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] *= rs;
        store8(drow + g * 8, v);
      }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(xready + r), "r"(1u) : "memory");
    }
  }
}

// src = dest^-1 (plan-in callers that pass only dest)
__global__ void invert_perm_kernel(const int32_t* __restrict__ dest, int64_t n, int32_t* __restrict__ src) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < n;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t r = dest[s];
    if (r >= 0 && r < n) src[r] = static_cast<int32_t>(s);
  }
}

// k == 1, no residual: y[t] = y_sorted[dest[t]] (a bit copy; the weight is exactly 1).
template <int U>
__global__ void __launch_bounds__(kPermThreads)
gather_kernel(const uint4* __restrict__ ys, int vec, int64_t T, const int32_t* __restrict__ dest,
              uint4* __restrict__ y, uint32_t* __restrict__ dev_status) {
  const int lane = threadIdx.x % kWarp;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kPermThreads / kWarp);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(kPermThreads / kWarp) + threadIdx.x / kWarp; t < T;
       t += warps) {
    const int32_t r = __ldg(dest + t);
    if (r < 0 || r >= T) {
      if (lane == 0 && dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
      continue;
    }
    copy_row<U>(ys + static_cast<int64_t>(r) * vec, y + t * vec, vec, lane);
  }
}


// General combine in fp32, j ascending (Q8), one rounding at the end. 8 elements per lane step.
template <typename Elt>
__global__ void __launch_bounds__(kPermThreads)
combine_kernel(const Elt* __restrict__ ys, int H, int64_t T, int k, const int32_t* __restrict__ dest,
               const float* __restrict__ w, const Elt* __restrict__ res, Elt* __restrict__ y,
               uint32_t* __restrict__ dev_status) {
  const int lane = threadIdx.x % kWarp;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kPermThreads / kWarp);
  const int groups = H / 8;
  const int64_t nrows = T * k;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(kPermThreads / kWarp) + threadIdx.x / kWarp; t < T;
       t += warps) {
    for (int g = lane; g < groups; g += kWarp) {
      float acc[8];
      if (res) {
        load8(res + t * H + g * 8, acc);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.f;
      }
      for (int j = 0; j < k; ++j) {
        int32_t r = __ldg(dest + t * k + j);
        if (r < 0 || r >= nrows) {
          if (dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
          continue;
        }
        const float wj = w ? __ldg(w + t * k + j) : 1.0f;
        float v[8];
        load8(ys + static_cast<int64_t>(r) * H + g * 8, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(wj, v[i], acc[i]);
      }
      store8(y + t * H + g * 8, acc);
    }
  }
}

// Expert slicing (setup, not on the timed path). Grid: (E*d) rows for gate/up, (E*H) rows for down.
template <typename Elt>
__global__ void slice_rows_kernel(const Elt* __restrict__ wg, const Elt* __restrict__ wu, int D, int H, int E,
                                  int d, const int32_t* __restrict__ nidx, Elt* __restrict__ eg,
                                  Elt* __restrict__ eu, uint32_t* __restrict__ dev_status) {
  const int64_t row = blockIdx.x;  // e*d + n
  const int e = static_cast<int>(row / d), n = static_cast<int>(row % d);
  const int32_t s = nidx[row];
  const bool ok = s >= 0 && s < D && (n == 0 || s > nidx[row - 1]);
  if (!ok && threadIdx.x == 0 && dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
  (void)e;
  for (int c = threadIdx.x; c < H; c += blockDim.x) {
    eg[row * H + c] = ok ? wg[static_cast<int64_t>(s) * H + c] : Elt(0.f);
    eu[row * H + c] = ok ? wu[static_cast<int64_t>(s) * H + c] : Elt(0.f);
  }
}

template <typename Elt>
__global__ void slice_cols_kernel(const Elt* __restrict__ wd, int D, int H, int E, int d,
                                  const int32_t* __restrict__ nidx, Elt* __restrict__ ed) {
  const int64_t row = blockIdx.x;  // e*H + c
  const int e = static_cast<int>(row / H), c = static_cast<int>(row % H);
  for (int n = threadIdx.x; n < d; n += blockDim.x) {
    const int32_t s = nidx[static_cast<int64_t>(e) * d + n];
    const bool ok = s >= 0 && s < D && (n == 0 || s > nidx[static_cast<int64_t>(e) * d + n - 1]);
    ed[row * d + n] = ok ? wd[static_cast<int64_t>(c) * D + s] : Elt(0.f);
  }
}

// The kernels the expert FFN follows as a programmatic dependent run with the maximum shared-memory carveout:
// an SM's L1/shared split only changes while it is idle, so a dispatch CTA running under an L1-heavy split
// would keep the FFN's CTA (~200 KB of shared memory) off that SM until the dispatch retires there.
void set_dispatch_carveout() {
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  std::call_once(once[dev], [] {
    const void* fns[] = {reinterpret_cast<const void*>(dispatch_gather_kernel),
                         reinterpret_cast<const void*>(finalize_dispatch_kernel),
                         reinterpret_cast<const void*>(dispatch_kernel<4>),
                         reinterpret_cast<const void*>(dispatch_kernel<8>),
                         reinterpret_cast<const void*>(dispatch_rmsnorm_kernel<__nv_bfloat16>),
                         reinterpret_cast<const void*>(dispatch_rmsnorm_kernel<float>),
                         reinterpret_cast<const void*>(dispatch_rmsnorm_gather_kernel<__nv_bfloat16>),
                         reinterpret_cast<const void*>(dispatch_rmsnorm_gather_kernel<float>)};
    for (const void* f : fns)
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaGetLastError();  // a hint only
  });
}

// 128-bit loads in flight per lane: 4 in the scatter dispatch (contiguous reads, scattered row writes),
// 8 in the k = 1 gather combine (scattered row reads) — measured on one box, 3 runs each at 65536 rows:
// dispatch 0.834 vs 0.79 of the copy peak with 4 vs 8, combine 0.89 vs 0.92 (README_PERM_UNROLL_D /
// knobs perm_unroll_c / perm_unroll_d = 4 | 8 override for A/B measurement)
int perm_unroll(bool gather) { return knob(gather ? Knob::kPermUnrollC : Knob::kPermUnrollD) == 4 ? 4 : 8; }

// Bulk-copy row moves (scatter dispatch; k = 1 combine without residual) for >= 4096 rows whose 16-row
// ring fits in shared memory; knobs dispatch_bulk / combine_bulk = 0|1 override (A/B measurement).
bool use_bulk_moves(int64_t rows, size_t row_bytes, Knob which) {
  if (row_bytes % 16 != 0 || static_cast<size_t>(kBulkCopiers) * kBulkSlots * row_bytes > kBulkMaxSmem) return false;
  const int v = knob(which);
  if (v >= 0) return v != 0;
  return rows >= 4096;
}

template <bool kGather>
readme_status launch_move_rows_bulk(const void* in, size_t row_bytes, int64_t rows, int32_t k, const int32_t* dest,
                                    void* out, uint32_t* dev_status, cudaStream_t st) {
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  std::call_once(once[dev], [] {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(move_rows_bulk_kernel<kGather>),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kBulkMaxSmem));
  });
  const size_t smem = static_cast<size_t>(kBulkCopiers) * kBulkSlots * row_bytes;
  const int64_t want = (rows + kBulkCopiers - 1) / kBulkCopiers;
  const int64_t cap = num_sms();
  move_rows_bulk_kernel<kGather><<<static_cast<int>(want < cap ? want : cap), kBulkCopiers * kWarp, smem, st>>>(
      static_cast<const uint8_t*>(in), static_cast<uint32_t>(row_bytes), rows, k, dest, static_cast<uint8_t*>(out),
      dev_status);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

int grid_for_rows(int64_t rows) {
  set_dispatch_carveout();
  const int64_t want = (rows + (kPermThreads / kWarp) - 1) / (kPermThreads / kWarp);
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;  // 8 CTAs x 8 warps = 64 warps per SM
  return static_cast<int>(want < cap ? (want < 1 ? 1 : want) : cap);
}

}  // namespace

readme_status launch_dispatch(const void* x, size_t row_bytes, int64_t T, int32_t k, const int32_t* dest,
                              void* x_sorted, uint32_t* dev_status, cudaStream_t st) {
  const int64_t nslots = T * k;
  if (nslots == 0) return README_OK;
  if (use_bulk_moves(nslots, row_bytes, Knob::kDispatchBulk))
    return launch_move_rows_bulk<false>(x, row_bytes, nslots, k, dest, x_sorted, dev_status, st);
  if (perm_unroll(false) == 8)
    dispatch_kernel<8><<<grid_for_rows(nslots), kPermThreads, 0, st>>>(
        static_cast<const uint4*>(x), static_cast<int>(row_bytes / 16), nslots, k, dest,
        static_cast<uint4*>(x_sorted), dev_status);
  else
    dispatch_kernel<4><<<grid_for_rows(nslots), kPermThreads, 0, st>>>(
        static_cast<const uint4*>(x), static_cast<int>(row_bytes / 16), nslots, k, dest,
        static_cast<uint4*>(x_sorted), dev_status);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_dispatch_gather(const void* x, size_t row_bytes, int64_t rows, int32_t k, const int32_t* src,
                                     void* x_sorted, uint32_t* xready, uint32_t* dev_status, cudaStream_t st) {
  if (rows == 0) return README_OK;
  set_dispatch_carveout();
  const int64_t want = (rows + (kGatherThreads / kWarp) - 1) / (kGatherThreads / kWarp);
  const int64_t cap = num_sms();
  dispatch_gather_kernel<<<static_cast<int>(want < cap ? want : cap), kGatherThreads, 0, st>>>(
      static_cast<const uint4*>(x), static_cast<int>(row_bytes / 16), rows, k, src, static_cast<uint4*>(x_sorted),
      xready, dev_status, g_trace_buf);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

__global__ void debug_mark_kernel(uint64_t* slot) { *slot = globaltimer_ns(); }
readme_status launch_debug_mark(uint64_t* slot, cudaStream_t st) {
  debug_mark_kernel<<<1, 1, 0, st>>>(slot);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

// Test only: occupy whole SMs for `ns` nanoseconds (one CTA per SM: each takes the maximum shared memory),
// so a kernel launched behind it on another stream finds only the remaining SMs.
constexpr int kHoldSmem = 227 * 1024;
__global__ void debug_hold_kernel(int64_t ns) {
  extern __shared__ uint8_t hold_smem[];
  if (threadIdx.x == 0) {
    const uint64_t t0 = globaltimer_ns();
    while (globaltimer_ns() - t0 < static_cast<uint64_t>(ns)) __nanosleep(1000);
    hold_smem[0] = 1;
  }
}
readme_status launch_debug_hold_sms(int32_t n_ctas, int64_t ns, cudaStream_t st) {
  README_CUDA(cudaFuncSetAttribute(debug_hold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHoldSmem));
  debug_hold_kernel<<<n_ctas, 32, kHoldSmem, st>>>(ns);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_dispatch_rmsnorm_gather(const void* x, readme_dtype dt, int64_t rows, int32_t H, int32_t k,
                                             const int32_t* src, float eps, void* x_sorted, uint32_t* xready,
                                             uint32_t* dev_status, cudaStream_t st) {
  if (rows == 0) return README_OK;
  set_dispatch_carveout();
  const int64_t want = (rows + (kGatherThreads / kWarp) - 1) / (kGatherThreads / kWarp);
  const int64_t cap = num_sms();
  const int grid = static_cast<int>(want < cap ? want : cap);
  if (dt == README_BF16)
    dispatch_rmsnorm_gather_kernel<__nv_bfloat16><<<grid, kGatherThreads, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), H, rows, k, src, eps, static_cast<__nv_bfloat16*>(x_sorted), xready,
        dev_status);
  else
    dispatch_rmsnorm_gather_kernel<float><<<grid, kGatherThreads, 0, st>>>(
        static_cast<const float*>(x), H, rows, k, src, eps, static_cast<float*>(x_sorted), xready, dev_status);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_invert_perm(const int32_t* dest, int64_t n, int32_t* src, cudaStream_t st) {
  if (n == 0) return README_OK;
  const int64_t want = (n + 255) / 256, cap = 4LL * num_sms();
  invert_perm_kernel<<<static_cast<int>(want < cap ? want : cap), 256, 0, st>>>(dest, n, src);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_set_offsets(int32_t* offs, int32_t T, cudaStream_t st) {
  set_offsets_kernel<<<1, 1, 0, st>>>(offs, T);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_finalize_dispatch(const void* x, size_t row_bytes, int64_t T, int32_t k, int32_t E,
                                       const int32_t* topk_idx, const int32_t* offsets, int32_t* dest, int32_t* src,
                                       void* x_sorted, cudaStream_t st) {
  const int64_t nslots = T * k;
  if (nslots == 0) return README_OK;
  finalize_dispatch_kernel<<<grid_for_rows(nslots), kPermThreads, 0, st>>>(
      static_cast<const uint4*>(x), static_cast<int>(row_bytes / 16), nslots, k, E, topk_idx, offsets, dest, src,
      static_cast<uint4*>(x_sorted));
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_dispatch_rmsnorm(const void* x, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                                      const int32_t* dest, float eps, void* x_sorted, uint32_t* dev_status,
                                      cudaStream_t st) {
  if (T == 0) return README_OK;
  const int grid = grid_for_rows(T);
  if (dt == README_BF16 && H % 256 == 0 && H / 256 <= kNormMaxChunks)
    dispatch_rmsnorm_row_kernel<<<grid, kPermThreads, 0, st>>>(static_cast<const uint4*>(x), H / 256, T, k, dest, eps,
                                                               static_cast<uint4*>(x_sorted), dev_status);
  else if (dt == README_BF16)
    dispatch_rmsnorm_kernel<__nv_bfloat16><<<grid, kPermThreads, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), H, T, k, dest, eps, static_cast<__nv_bfloat16*>(x_sorted), dev_status);
  else
    dispatch_rmsnorm_kernel<float><<<grid, kPermThreads, 0, st>>>(static_cast<const float*>(x), H, T, k, dest, eps,
                                                                 static_cast<float*>(x_sorted), dev_status);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_combine(const void* y_sorted, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                             const int32_t* dest, const float* topk_w, const void* residual, void* y,
                             uint32_t* dev_status, cudaStream_t st) {
  if (T == 0) return README_OK;
  if (k == 1 && residual == nullptr && use_bulk_moves(T, static_cast<size_t>(H) * dt_size(dt), Knob::kCombineBulk))
    return launch_move_rows_bulk<true>(y_sorted, static_cast<size_t>(H) * dt_size(dt), T, 1, dest, y, dev_status, st);
  const int grid = grid_for_rows(T);
  if (k == 1 && residual == nullptr) {
    if (perm_unroll(true) == 8)
      gather_kernel<8><<<grid, kPermThreads, 0, st>>>(static_cast<const uint4*>(y_sorted),
                                                      static_cast<int>(H * dt_size(dt) / 16), T, dest,
                                                      static_cast<uint4*>(y), dev_status);
    else
      gather_kernel<4><<<grid, kPermThreads, 0, st>>>(static_cast<const uint4*>(y_sorted),
                                                      static_cast<int>(H * dt_size(dt) / 16), T, dest,
                                                      static_cast<uint4*>(y), dev_status);
  } else if (dt == README_BF16) {
    combine_kernel<__nv_bfloat16><<<grid, kPermThreads, 0, st>>>(
        static_cast<const __nv_bfloat16*>(y_sorted), H, T, k, dest, topk_w,
        static_cast<const __nv_bfloat16*>(residual), static_cast<__nv_bfloat16*>(y), dev_status);
  } else {
    combine_kernel<float><<<grid, kPermThreads, 0, st>>>(static_cast<const float*>(y_sorted), H, T, k, dest,
                                                         topk_w, static_cast<const float*>(residual),
                                                         static_cast<float*>(y), dev_status);
  }
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_build_experts(const void* wg, const void* wu, const void* wd, readme_dtype dt, int32_t D,
                                   int32_t H, int32_t E, int32_t d, const int32_t* nidx, void* eg, void* eu,
                                   void* ed, uint32_t* dev_status, cudaStream_t st) {
  const unsigned rows_gu = static_cast<unsigned>(static_cast<int64_t>(E) * d);
  const unsigned rows_d = static_cast<unsigned>(static_cast<int64_t>(E) * H);
  if (dt == README_BF16) {
    slice_rows_kernel<__nv_bfloat16><<<rows_gu, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(wg), static_cast<const __nv_bfloat16*>(wu), D, H, E, d, nidx,
        static_cast<__nv_bfloat16*>(eg), static_cast<__nv_bfloat16*>(eu), dev_status);
    slice_cols_kernel<__nv_bfloat16><<<rows_d, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(wd), D, H, E, d,
                                                             nidx, static_cast<__nv_bfloat16*>(ed));
  } else {
    slice_rows_kernel<float><<<rows_gu, 256, 0, st>>>(static_cast<const float*>(wg), static_cast<const float*>(wu),
                                                     D, H, E, d, nidx, static_cast<float*>(eg),
                                                     static_cast<float*>(eu), dev_status);
    slice_cols_kernel<float><<<rows_d, 256, 0, st>>>(static_cast<const float*>(wd), D, H, E, d, nidx,
                                                     static_cast<float*>(ed));
  }
  README_CUDA(cudaGetLastError());
  return README_OK;
}

}  // namespace readme
