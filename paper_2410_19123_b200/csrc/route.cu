// route.cu — a1-a4 of the hot path: top-K selection + gate weights, per-expert histogram, cross-tile
// exclusive scan (decoupled lookback) and the stable permutation (dest/src).
//
// Paper: Eq. 2's indicator 1(|{j : G_j >= G_i}| <= K) read as "exactly K experts, ties
// to the lower id" (Q2), softmax over the selected logits (Q1); grouping = Alg. 1's ReqQueueByExpert
// with FIFO order inside an expert (Q7).
//
// Design (B200): one CTA per tile of <= 1024 slots (slot s = t*k + j); tile = blockIdx.x (blocks are
// dispatched in index order, so a lookback only ever waits on CTAs that are running or finished).
//   phase A  logits tile -> shared memory (all loads in flight at once), then lane-groups of
//            LPT = min(32, pow2ceil(E)) lanes per token run a warp-shuffle arg-max k times.
//   phase B  per warp, 32 slots at a time: __match_any_sync groups equal experts, popc of the
//            lower-lane mask gives the stable in-warp rank; per-warp per-expert running counts in smem.
//   phase C  per expert: exclusive scan over warps and publication of the tile aggregate, then a
//            decoupled lookback by one warp per expert that reads 32 predecessor tiles at once
//            (64-bit status words: flag << 32 | count; 1 = tile aggregate, 2 = inclusive prefix).
//            The last tile knows the global counts and writes counts[] and offsets[].
//   phase D  dest[s] = (rank of s among its expert's slots); the finalize kernel adds offsets[e] and
//            writes src (offsets need every tile's counts, so a second launch is the cheap barrier).
//            readme_moe_layer fuses that finalize into the dispatch kernel (permute.cu).
#include <math.h>
#include <stdlib.h>

#include "kernels.h"

namespace readme {

namespace {

constexpr int kRouteThreads = 256;
constexpr int kRouteWarps = kRouteThreads / kWarp;
constexpr int kMaxTileSlots = 1024;
constexpr int kMaxLogitFloats = 8192;  // 32 KB of staged logits per tile
constexpr int kMaxItems = README_MAX_EXPERTS / kWarp;  // logits per lane when LPT == 32

struct RouteGeom {
  int tile_tokens;
  int ntiles;
};

RouteGeom route_geom(int64_t T, int32_t E, int32_t k) {
  int tt = kMaxTileSlots / k;
  int by_e = kMaxLogitFloats / E;
  if (by_e < tt) tt = by_e;
  // enough tiles to spread over the SMs (latency-bound: more CTAs in flight), at least 32 tokens per tile
  // so lookback chains stay short; README_ROUTE_TILE overrides (A/B measurement)
  int cap = 256;
  while (cap > 32 && (T + cap - 1) / cap < 148) cap >>= 1;
  if (const char* v = getenv("README_ROUTE_TILE")) cap = atoi(v) > 0 ? atoi(v) : cap;
  if (tt > cap) tt = cap;
  if (tt < 1) tt = 1;
  RouteGeom g;
  g.tile_tokens = tt;
  g.ntiles = static_cast<int>((T + tt - 1) / tt);
  return g;
}

template <typename LogitT>
__device__ __forceinline__ float load_logit(const LogitT* p, int64_t i);
template <>
__device__ __forceinline__ float load_logit<float>(const float* p, int64_t i) {
  return __ldg(p + i);
}
template <>
__device__ __forceinline__ float load_logit<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

// (v, id) "beats" (bv, bid): larger logit, ties to the lower id.
__device__ __forceinline__ bool beats(float v, int id, float bv, int bid) {
  return v > bv || (v == bv && id < bid);
}

template <typename LogitT>
__global__ void __launch_bounds__(kRouteThreads)
route_tile_kernel(const LogitT* __restrict__ logits, int64_t T, int E, int k, int tile_tokens, int ntiles,
                  int lpt, int items, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                  int32_t* __restrict__ counts, int32_t* __restrict__ offsets, int32_t* __restrict__ rank_out,
                  uint32_t* __restrict__ dev_status, uint64_t* __restrict__ status) {
  __shared__ float s_logit[kMaxLogitFloats];
  __shared__ uint8_t s_exp[kMaxTileSlots];
  __shared__ int s_wcount[kRouteWarps][README_MAX_EXPERTS];
  __shared__ int s_prefix[README_MAX_EXPERTS];
  __shared__ int s_run[README_MAX_EXPERTS];
  __shared__ int s_bad;

  const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
  if (tid == 0) s_bad = 0;
  for (int i = tid; i < kRouteWarps * README_MAX_EXPERTS; i += kRouteThreads) (&s_wcount[0][0])[i] = 0;
  __syncthreads();
  const int tile = blockIdx.x;
  const int64_t t0 = static_cast<int64_t>(tile) * tile_tokens;
  const int64_t rem = T - t0;
  const int nt = static_cast<int>(rem < tile_tokens ? rem : tile_tokens);
  const int nslots = nt * k;

  // ---- phase A: stage the tile's logits (every load in flight at once), then top-k per token ----
  const int nlog = nt * E;
  const LogitT* src = logits + t0 * E;
  bool bad = false;
  for (int i = tid; i < nlog; i += kRouteThreads) {
    float v = load_logit(src, i);
    if (!isfinite(v)) {
      bad = true;
      if (isnan(v)) v = -INFINITY;  // Q3: NaN ranks as -inf so ids stay in range
    }
    s_logit[i] = v;
  }
  if (bad) s_bad = 1;
  __syncthreads();
  if (tid == 0 && s_bad && dev_status) atomicOr(dev_status, README_DEV_NONFINITE_LOGIT);

  const int tokens_per_warp_iter = kWarp / lpt;
  const int gl = lane % lpt;  // lane within the token's group
  for (int base = warp * tokens_per_warp_iter; base < nt; base += kRouteWarps * tokens_per_warp_iter) {
    const int tok = base + lane / lpt;
    const bool tok_ok = tok < nt;
    float v[kMaxItems];
    uint32_t taken = 0;
#pragma unroll
    for (int i = 0; i < kMaxItems; ++i) {
      const int e = gl + i * lpt;
      v[i] = (tok_ok && i < items && e < E) ? s_logit[tok * E + e] : -INFINITY;
    }
    float m = 0.f, z = 0.f;
    for (int j = 0; j < k; ++j) {
      float bv = -INFINITY;
      int bid = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < kMaxItems; ++i) {
        const int e = gl + i * lpt;
        if (i < items && e < E && !(taken >> i & 1u) && beats(v[i], e, bv, bid)) {
          bv = v[i];
          bid = e;
        }
      }
      for (int off = lpt >> 1; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oid = __shfl_xor_sync(0xffffffffu, bid, off);
        if (beats(ov, oid, bv, bid)) {
          bv = ov;
          bid = oid;
        }
      }
      if (bid % lpt == gl) taken |= 1u << (bid / lpt);
      if (j == 0) m = bv;
      const float ej = expf(bv - m);
      z += ej;
      if (gl == 0 && tok_ok) {
        const int64_t s = (t0 + tok) * k + j;
        topk_idx[s] = bid;
        topk_w[s] = ej;  // normalised below
        s_exp[tok * k + j] = static_cast<uint8_t>(bid);
      }
    }
    if (gl == 0 && tok_ok) {
      const float inv = 1.0f / z;  // k == 1: z == 1 -> weight exactly 1.0f
      for (int j = 0; j < k; ++j) {
        const int64_t s = (t0 + tok) * k + j;
        topk_w[s] = (k == 1) ? 1.0f : topk_w[s] * inv;
      }
    }
  }
  __syncthreads();

  // ---- phase B: stable in-warp ranks, per-warp per-expert counts ----
  const int chunk = (kMaxTileSlots / kRouteWarps);  // 128 contiguous slots per warp, ascending
  constexpr int kIters = kMaxTileSlots / kRouteWarps / kWarp;
  int local[kIters];
#pragma unroll
  for (int it = 0; it < kIters; ++it) {
    const int sl = warp * chunk + it * kWarp + lane;
    const bool ok = sl < nslots;
    const int e = ok ? s_exp[sl] : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    const int r = __popc(peers & lanemask_lt());
    int base = 0;
    if (ok) base = s_wcount[warp][e];
    __syncwarp();
    if (ok && r == 0) s_wcount[warp][e] = base + __popc(peers);
    __syncwarp();
    local[it] = base + r;
  }
  __syncthreads();

  // ---- phase C: per-expert warp scan, publish the tile aggregate, decoupled lookback ----
  for (int e = tid; e < E; e += kRouteThreads) {
    int run = 0;
#pragma unroll
    for (int w = 0; w < kRouteWarps; ++w) {
      const int c = s_wcount[w][e];
      s_wcount[w][e] = run;
      run += c;
    }
    s_run[e] = run;
    st_relaxed_gpu_u64(status + static_cast<int64_t>(tile) * E + e,
                       ((tile == 0 ? 2ull : 1ull) << 32) | static_cast<uint32_t>(run));
  }
  __syncthreads();
  for (int e = warp; e < E; e += kRouteWarps) {
    int excl = 0;
    int base = tile - 1;  // the window covers tiles base, base-1, ..., base-31 (lane j -> tile base-j)
    while (base >= 0) {
      const int i = base - lane;
      uint64_t w = (2ull << 32);  // lanes past tile 0 read as an empty inclusive prefix
      if (i >= 0) w = ld_relaxed_gpu_u64(status + static_cast<int64_t>(i) * E + e);
      const uint32_t flag = static_cast<uint32_t>(w >> 32);
      if (__any_sync(0xffffffffu, flag == 0)) {  // a predecessor has not published yet
        __nanosleep(32);
        continue;
      }
      const uint32_t pref = __ballot_sync(0xffffffffu, flag == 2);
      const int stop = pref ? __ffs(pref) - 1 : kWarp - 1;  // nearest predecessor with an inclusive prefix
      int v = lane <= stop ? static_cast<int>(static_cast<uint32_t>(w)) : 0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      excl += v;
      if (pref) break;
      base -= kWarp;
    }
    if (lane == 0) {
      const int run = s_run[e];
      if (tile > 0)
        st_relaxed_gpu_u64(status + static_cast<int64_t>(tile) * E + e, (2ull << 32) | static_cast<uint32_t>(excl + run));
      s_prefix[e] = excl;
      if (tile == ntiles - 1) counts[e] = excl + run;
    }
  }
  __syncthreads();
  if (tile == ntiles - 1 && tid == 0) {
    int acc = 0;
    offsets[0] = 0;
    for (int e = 0; e < E; ++e) {
      acc += counts[e];
      offsets[e + 1] = acc;
    }
  }

  // ---- phase D: rank of every slot within its expert (offsets added by the finalize kernel) ----
#pragma unroll
  for (int it = 0; it < kIters; ++it) {
    const int sl = warp * chunk + it * kWarp + lane;
    if (sl < nslots) {
      const int e = s_exp[sl];
      rank_out[t0 * k + sl] = s_prefix[e] + s_wcount[warp][e] + local[it];
    }
  }
}

__global__ void route_finalize_kernel(int64_t nslots, int E, const int32_t* __restrict__ topk_idx,
                                      const int32_t* __restrict__ offsets, int32_t* __restrict__ dest,
                                      int32_t* __restrict__ src) {
  __shared__ int s_off[README_MAX_EXPERTS + 1];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) s_off[i] = offsets[i];
  __syncthreads();
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < nslots;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = s_off[topk_idx[s]] + dest[s];
    dest[s] = r;
    if (src) src[r] = static_cast<int32_t>(s);
  }
}

}  // namespace

size_t route_ws_bytes(int64_t T, int32_t E, int32_t k) {
  if (T <= 0 || E < 1 || k < 1) return 256;
  RouteGeom g = route_geom(T, E, k);
  return align_up(static_cast<size_t>(g.ntiles) * E * sizeof(uint64_t), 256);
}

readme_status launch_route(const void* logits, readme_dtype logits_dt, int64_t T, int32_t E, int32_t k,
                           int32_t* topk_idx, float* topk_w, int32_t* counts, int32_t* offsets, int32_t* dest,
                           int32_t* src, uint32_t* dev_status, void* ws, cudaStream_t st, bool finalize) {
  if (T == 0) {
    README_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, st));
    README_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (E + 1), st));
    return README_OK;
  }
  RouteGeom g = route_geom(T, E, k);
  uint64_t* status = static_cast<uint64_t*>(ws);
  README_CUDA(cudaMemsetAsync(status, 0, static_cast<size_t>(g.ntiles) * E * sizeof(uint64_t), st));
  int lpt = 1;
  while (lpt < E && lpt < kWarp) lpt <<= 1;
  const int items = (E + lpt - 1) / lpt;
  if (logits_dt == README_F32) {
    route_tile_kernel<float><<<g.ntiles, kRouteThreads, 0, st>>>(
        static_cast<const float*>(logits), T, E, k, g.tile_tokens, g.ntiles, lpt, items, topk_idx, topk_w,
        counts, offsets, dest, dev_status, status);
  } else {
    route_tile_kernel<__nv_bfloat16><<<g.ntiles, kRouteThreads, 0, st>>>(
        static_cast<const __nv_bfloat16*>(logits), T, E, k, g.tile_tokens, g.ntiles, lpt, items, topk_idx,
        topk_w, counts, offsets, dest, dev_status, status);
  }
  README_CUDA(cudaGetLastError());
  if (!finalize) return README_OK;  // the caller fuses the finalize into its dispatch
  const int64_t nslots = T * k;
  const int64_t want = (nslots + 255) / 256, cap = 4LL * num_sms();
  const int blocks = static_cast<int>(want < cap ? want : cap);
  route_finalize_kernel<<<blocks, 256, 0, st>>>(nslots, E, topk_idx, offsets, dest, src);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

}  // namespace readme
