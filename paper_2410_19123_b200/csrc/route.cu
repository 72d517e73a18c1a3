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
#include <string.h>

#include "kernels.h"
#include "router_head.cuh"

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
  if (const int v = knob(Knob::kRouteTile)) cap = v > 0 ? v : cap;
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

// Top-k of one token by one thread (E <= NE <= 32): the token's E logits are loaded straight into registers
// (128-bit loads when the row allows), k passes of a register arg-max (ties -> lower id), then the softmax
// over the selected logits. Writes idx/w of the token's k slots and their expert ids to s_exp. For small E
// this costs a few instructions per token, where a lane group per token (the E > 32 path) spends a warp
// pass per 32/lpt tokens.
template <int NE>
__device__ __forceinline__ void topk_select(float (&v)[NE], int E, int k, int32_t* __restrict__ idx_out,
                                            float* __restrict__ w_out, uint8_t* __restrict__ s_exp_out, bool& bad);

template <int NE, typename LogitT>
__device__ __forceinline__ void topk_one_token(const LogitT* __restrict__ row, int E, int k, bool vec,
                                               int32_t* __restrict__ idx_out, float* __restrict__ w_out,
                                               uint8_t* __restrict__ s_exp_out, bool& bad) {
  float v[NE];
  if constexpr (sizeof(LogitT) == 4) {
    if (vec) {  // E % 4 == 0 and the row is 16-B aligned
#pragma unroll
      for (int q = 0; q < NE / 4; ++q) {
        float4 f = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        if (4 * q < E) f = __ldg(reinterpret_cast<const float4*>(row) + q);
        v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < NE; ++e) v[e] = e < E ? load_logit(row, e) : -INFINITY;
    }
  } else {
    if (vec) {  // E % 8 == 0 and the row is 16-B aligned
#pragma unroll
      for (int q = 0; q < NE / 8; ++q) {
        uint4 u = make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u);  // bf16 -inf pairs
        if (8 * q < E) u = __ldg(reinterpret_cast<const uint4*>(row) + q);
        v[8 * q + 0] = bf16_lo(u.x); v[8 * q + 1] = bf16_hi(u.x); v[8 * q + 2] = bf16_lo(u.y);
        v[8 * q + 3] = bf16_hi(u.y); v[8 * q + 4] = bf16_lo(u.z); v[8 * q + 5] = bf16_hi(u.z);
        v[8 * q + 6] = bf16_lo(u.w); v[8 * q + 7] = bf16_hi(u.w);
      }
    } else {
#pragma unroll
      for (int e = 0; e < NE; ++e) v[e] = e < E ? load_logit(row, e) : -INFINITY;
    }
  }
  topk_select<NE>(v, E, k, idx_out, w_out, s_exp_out, bad);
}

// Top-k of one token's E <= NE logits held in registers (ties -> lower id, Q2), softmax weights over the
// selected logits (Q1; k == 1 gives exactly 1.0f), non-finite logits flagged (Q3).
template <int NE>
__device__ __forceinline__ void topk_select(float (&v)[NE], int E, int k, int32_t* __restrict__ idx_out,
                                            float* __restrict__ w_out, uint8_t* __restrict__ s_exp_out, bool& bad) {
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    if (e < E && !isfinite(v[e])) {
      bad = true;
      if (isnan(v[e])) v[e] = -INFINITY;  // Q3: NaN ranks as -inf so ids stay in range
    }
  }
  uint32_t taken = 0;
  float m = 0.f, z = 0.f;
  for (int j = 0; j < k; ++j) {
    float bv = -INFINITY;
    int bid = 0x7fffffff;
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      if (e < E && !(taken >> e & 1u) && beats(v[e], e, bv, bid)) {
        bv = v[e];
        bid = e;
      }
    }
    taken |= 1u << bid;
    if (j == 0) m = bv;
    const float ej = isfinite(m) ? expf(bv - m) : (bv == m ? 1.0f : 0.0f);  // +-inf max: uniform over the tied maxima
    z += ej;
    idx_out[j] = bid;
    if (k > 1) w_out[j] = ej;  // normalised below
    s_exp_out[j] = static_cast<uint8_t>(bid);
  }
  if (k == 1) {
    w_out[0] = 1.0f;  // z == 1: the weight is exactly 1.0f
  } else {
    const float inv = 1.0f / z;
    for (int j = 0; j < k; ++j) w_out[j] *= inv;
  }
}

template <typename LogitT>
__device__ __forceinline__ bool row_vec_ok(const LogitT* logits, int E) {
  return (reinterpret_cast<uintptr_t>(logits) & 15u) == 0 && (E * static_cast<int>(sizeof(LogitT))) % 16 == 0;
}

template <typename LogitT, int NE>
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

  // ---- phase A: top-k per token: a thread per token (E <= 32), or stage the tile's logits (every load in
  // flight at once) and run lane groups per token ----
  const int nlog = nt * E;
  const LogitT* src = logits + t0 * E;
  bool bad = false;
  if constexpr (NE > 0) {
    const bool vec = row_vec_ok(logits, E);
    for (int tok = tid; tok < nt; tok += kRouteThreads)
      topk_one_token<NE>(src + static_cast<int64_t>(tok) * E, E, k, vec, topk_idx + (t0 + tok) * k,
                         topk_w + (t0 + tok) * k, s_exp + tok * k, bad);
    if (bad) s_bad = 1;
    __syncthreads();
    if (tid == 0 && s_bad && dev_status) atomicOr(dev_status, README_DEV_NONFINITE_LOGIT);
  } else {
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
      const float ej = isfinite(m) ? expf(bv - m) : (bv == m ? 1.0f : 0.0f);  // +-inf max: uniform over the tied maxima
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
  }

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

// ===================================================================================================
// Single-launch route for batches up to kClusterMaxSlots slots: ONE thread-block cluster of C <= 16 CTAs
// (1024 threads each) does a1-a4 including the finalize. CTA c owns the contiguous token chunk
// [c*chunk, (c+1)*chunk) and walks it in sub-tiles of <= 1024 slots: phase A and B as in route_tile_kernel
// (one slot per thread), then each slot's rank inside its expert AMONG THE CTA'S SLOTS (running per-expert
// counts carried across sub-tiles). The cross-CTA exclusive scan is a cluster barrier plus distributed
// shared memory: every CTA reads the C per-expert counts of its peers (ld.shared::cluster), so
//   offsets[e] = sum_{e'<e} total[e'],  base_c[e] = offsets[e] + sum_{c'<c} count_{c'}[e],
// and dest[s] = base_c[e_s] + rank_c(s), src[dest[s]] = s — no lookback chain, no status memset, no second
// launch. Chunks are contiguous and ascending, so the order inside an expert is still ascending slot (Q7).
constexpr int kCThreads = 1024;
constexpr int kCWarps = kCThreads / kWarp;
constexpr int kCMaxCluster = 16;
constexpr int64_t kClusterMaxSlots = 256 * 1024;  // beyond: the multi-CTA lookback route
constexpr int kCMaxSmem = (kMaxLogitFloats + kCWarps * README_MAX_EXPERTS) * 4;  // 64 KB
// head mode (E <= 16): s_wcount, W_head in bf16 and the sub-tile's fp32 logits
constexpr int kCHeadMaxE = 16;
constexpr int kCMaxSmemHead = (kCWarps * kCHeadMaxE + kCThreads * kCHeadMaxE) * 4 + kCHeadMaxE * kRouterDim * 2;

struct RouteExtra {
  uint32_t* zero;      // nullable: words zeroed by the launch (the FFN's readiness region)
  int64_t zero_words;
  // head mode (non-null head_h, E <= 16): each sub-tile's logits are computed in the launch from the pre-gating
  // router's last hidden state (router_head.cuh) into shared memory, written out to head_logits, then routed
  const __nv_bfloat16* head_h;  // [T, 512]
  const __nv_bfloat16* head_g;  // [512] final RMSNorm weight
  const __nv_bfloat16* head_w;  // [E, 512] gating head
  float head_eps;
  float* head_logits;           // [T, E] out
};

struct ClusterGeom {
  int C;             // CTAs in the (single) cluster
  int tile_tokens;   // tokens per sub-tile (<= 1024 slots, <= kMaxLogitFloats logits)
  int64_t chunk;     // tokens per CTA
  size_t smem;       // dynamic shared memory bytes
};

template <typename LogitT, int NE>
__global__ void __launch_bounds__(kCThreads, 1)
route_cluster_kernel(const LogitT* __restrict__ logits, int64_t T, int E, int k, int tile_tokens, int64_t chunk,
                     int lpt, int items, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                     int32_t* __restrict__ counts, int32_t* __restrict__ offsets, int32_t* __restrict__ dest,
                     int32_t* __restrict__ src, uint32_t* __restrict__ dev_status, uint64_t* __restrict__ trace,
                     RouteExtra ex) {
  extern __shared__ __align__(16) uint8_t route_smem[];
  if (trace && threadIdx.x == 0) trace_min(trace, 5);
  if (ex.zero) {  // the FFN's readiness counters / row flags (instead of a memset node before this launch)
    uint32_t cr, cs;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
    for (int64_t i = static_cast<int64_t>(cr) * kCThreads + threadIdx.x; i < ex.zero_words;
         i += static_cast<int64_t>(cs) * kCThreads)
      ex.zero[i] = 0u;
  }
  float* s_logit = reinterpret_cast<float*>(route_smem);                             // [tile_tokens * E]
  // [kCWarps][E], after the staged logits (lane-group path only)
  int* s_wcount = reinterpret_cast<int*>(route_smem + (NE > 0 ? 0 : sizeof(float) * tile_tokens * E));
  __shared__ uint8_t s_exp[kCThreads];
  __shared__ int s_run[README_MAX_EXPERTS];   // this CTA's per-expert count (read by the peers)
  __shared__ int s_base[README_MAX_EXPERTS];  // offsets[e] + peers-before count
  __shared__ int s_tot[README_MAX_EXPERTS];
  __shared__ int s_bad;

  const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
  uint32_t crank, csize;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  for (int e = tid; e < E; e += kCThreads) s_run[e] = 0;
  if (tid == 0) s_bad = 0;
  __nv_bfloat16* s_whead = reinterpret_cast<__nv_bfloat16*>(route_smem + sizeof(int) * kCWarps * E);
  float* s_hl = reinterpret_cast<float*>(route_smem + sizeof(int) * kCWarps * E + sizeof(__nv_bfloat16) * E * kRouterDim);
  if (NE > 0 && ex.head_h) {
    for (int i = tid; i < E * kRouterDim; i += kCThreads) s_whead[i] = ex.head_w[i];
    __syncthreads();
  }
  const int64_t tok0 = static_cast<int64_t>(crank) * chunk;
  const int64_t tok1 = tok0 + chunk < T ? tok0 + chunk : T;
  const int tokens_per_warp_iter = kWarp / lpt;
  const int gl = lane % lpt;
  bool bad = false;

  for (int64_t t0 = tok0; t0 < tok1; t0 += tile_tokens) {
    const int nt = static_cast<int>(tok1 - t0 < tile_tokens ? tok1 - t0 : tile_tokens);
    const int nslots = nt * k;
    for (int i = tid; i < kCWarps * E; i += kCThreads) s_wcount[i] = 0;
    // ---- phase A: top-k per token: a thread per token (E <= 32), else logits -> smem and lane groups ----
    const LogitT* lsrc = logits + t0 * E;
    if constexpr (NE > 0) {
      if (ex.head_h) {
        // the sub-tile's logits from the router's hidden state, one warp per token (bit-identical to the
        // separate head kernel), kept in shared memory for the thread-per-token top-k below
        for (int tok = warp; tok < nt; tok += kCWarps) {
          const int64_t t = t0 + tok;
          head_logits_warp(ex.head_h + t * kRouterDim, ex.head_g,
                           [&](int n, int c) { return __bfloat162float(s_whead[n * kRouterDim + c]); }, E,
                           ex.head_eps, lane, [&](int n, float v) {
                             s_hl[tok * E + n] = v;
                             ex.head_logits[t * E + n] = v;
                           });
        }
        __syncthreads();
        if (tid < nt) {
          float v[NE];
#pragma unroll
          for (int e = 0; e < NE; ++e) v[e] = e < E ? s_hl[tid * E + e] : -INFINITY;
          topk_select<NE>(v, E, k, topk_idx + (t0 + tid) * k, topk_w + (t0 + tid) * k, s_exp + tid * k, bad);
        }
      } else if (tid < nt) {
        topk_one_token<NE>(lsrc + static_cast<int64_t>(tid) * E, E, k, row_vec_ok(logits, E),
                           topk_idx + (t0 + tid) * k, topk_w + (t0 + tid) * k, s_exp + tid * k, bad);
      }
    } else {
    for (int i = tid; i < nt * E; i += kCThreads) {
      float v = load_logit(lsrc, i);
      if (!isfinite(v)) {
        bad = true;
        if (isnan(v)) v = -INFINITY;  // Q3
      }
      s_logit[i] = v;
    }
    __syncthreads();
    for (int base = warp * tokens_per_warp_iter; base < nt; base += kCWarps * tokens_per_warp_iter) {
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
        const float ej = isfinite(m) ? expf(bv - m) : (bv == m ? 1.0f : 0.0f);  // +-inf max: uniform over the tied maxima
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
    }
    __syncthreads();
    // ---- phase B: one slot per thread; stable in-warp rank, per-warp per-expert counts ----
    const bool ok = tid < nslots;
    const int e = ok ? s_exp[tid] : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    const int local = __popc(peers & lanemask_lt());
    if (ok && local == 0) s_wcount[warp * E + e] = __popc(peers);
    __syncthreads();
    // ---- phase C: per expert, exclusive scan over the warps on top of the CTA's running count ----
    for (int x = tid; x < E; x += kCThreads) {
      int run = s_run[x];
      for (int w = 0; w < kCWarps; ++w) {
        const int c = s_wcount[w * E + x];
        s_wcount[w * E + x] = run;
        run += c;
      }
      s_run[x] = run;
    }
    __syncthreads();
    if (ok) dest[t0 * k + tid] = s_wcount[warp * E + e] + local;  // rank among this CTA's slots of expert e
    __syncthreads();  // s_exp / s_wcount / s_logit are reused by the next sub-tile
  }
  if (bad) s_bad = 1;

  // ---- cross-CTA scan through distributed shared memory ----
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  for (int x = tid; x < E; x += kCThreads) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&s_run[x]));
    int tot = 0, before = 0;
    for (uint32_t c = 0; c < csize; ++c) {
      uint32_t ra;
      int v;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(c));
      asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
      tot += v;
      if (c < crank) before += v;
    }
    s_tot[x] = tot;
    s_base[x] = before;
  }
  // every peer read of this CTA's s_run is done once all CTAs arrive; the wait is deferred to the exit
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the totals over experts (E <= 256: 8 per lane)
    constexpr int kPer = README_MAX_EXPERTS / kWarp;
    int v[kPer], sum = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int x = lane * kPer + i;
      v[i] = x < E ? s_tot[x] : 0;
      sum += v[i];
    }
    int incl = sum;
#pragma unroll
    for (int off = 1; off < kWarp; off <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    int run = incl - sum;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int x = lane * kPer + i;
      if (x < E) {
        if (crank == 0) {
          counts[x] = v[i];
          offsets[x] = run;
        }
        s_base[x] += run;
      }
      run += v[i];
    }
    if (crank == 0 && lane == kWarp - 1) offsets[E] = incl;
  }
  if (tid == 0 && s_bad && dev_status) atomicOr(dev_status, README_DEV_NONFINITE_LOGIT);
  __syncthreads();
  // ---- finalize: dest = base + rank, src = dest^-1 (this CTA's own writes, ordered by the barriers) ----
  for (int64_t s = tok0 * k + tid; s < tok1 * k; s += kCThreads) {
    const int r = s_base[topk_idx[s]] + dest[s];
    dest[s] = r;
    if (src) src[r] = static_cast<int32_t>(s);
  }
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (trace && threadIdx.x == 0) trace_max(trace, 6);
}

// register-resident top-k width for E experts: 8 / 16 / 32, or 0 = lane groups over staged logits
int topk_ne(int32_t E) { return E <= 8 ? 8 : E <= 16 ? 16 : E <= 32 ? 32 : 0; }

template <typename LogitT>
const void* cluster_fn(int ne) {
  switch (ne) {
    case 8: return reinterpret_cast<const void*>(route_cluster_kernel<LogitT, 8>);
    case 16: return reinterpret_cast<const void*>(route_cluster_kernel<LogitT, 16>);
    case 32: return reinterpret_cast<const void*>(route_cluster_kernel<LogitT, 32>);
    default: return reinterpret_cast<const void*>(route_cluster_kernel<LogitT, 0>);
  }
}

int max_route_cluster() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int c = 8;
    bool ok16 = true;
    for (int ne : {0, 8, 16, 32}) {
      for (const void* f : {cluster_fn<float>(ne), cluster_fn<__nv_bfloat16>(ne)}) {
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kCMaxSmem > kCMaxSmemHead ? kCMaxSmem : kCMaxSmemHead);
        ok16 = ok16 && cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
      }
    }
    if (ok16) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kCMaxCluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(kCMaxCluster);
      cfg.blockDim = dim3(kCThreads);
      cfg.dynamicSmemBytes = kCMaxSmem;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, route_cluster_kernel<float, 0>, &cfg) == cudaSuccess && n > 0)
        c = kCMaxCluster;
    }
    cudaGetLastError();  // an unsupported attribute only lowers the cluster size
    cache[dev] = c;
  }
  return cache[dev];
}

// Which route implementation a batch takes: knob route = 1 (cluster) | 2 (lookback) overrides (A/B
// measurement).
bool use_cluster_route(int64_t T, int32_t k) {
  const int v = knob(Knob::kRoute);
  if (v == 2) return false;
  if (v == 1) return true;
  return T * k <= kClusterMaxSlots;
}

ClusterGeom cluster_geom(int64_t T, int32_t E, int32_t k) {
  ClusterGeom g;
  const bool staged = topk_ne(E) == 0;  // lane groups read the tile's logits from shared memory
  int tt = kCThreads / k;
  const int by_e = kMaxLogitFloats / E;
  if (staged && by_e < tt) tt = by_e;
  if (tt < 1) tt = 1;
  g.tile_tokens = tt;
  const int64_t subtiles = (T + tt - 1) / tt;
  const int cmax = max_route_cluster();
  int C = 1;
  while (C < cmax && C < subtiles) C <<= 1;  // one sub-tile per CTA while the cluster can grow
  if (const int f = knob(Knob::kRouteCluster)) {  // A/B measurement: force the cluster size
    if (f == 1 || f == 2 || f == 4 || f == 8 || (f == 16 && cmax == 16)) C = f;
  }
  g.C = C;
  const int64_t per = (subtiles + C - 1) / C;  // sub-tiles per CTA
  g.chunk = per * tt;
  g.smem = (staged ? sizeof(float) * static_cast<size_t>(tt) * E : 0) + sizeof(int) * static_cast<size_t>(kCWarps) * E;
  return g;
}

}  // namespace

bool route_is_single_launch(int64_t T, int32_t k) { return T > 0 && use_cluster_route(T, k); }

size_t route_ws_bytes(int64_t T, int32_t E, int32_t k) {
  if (T <= 0 || E < 1 || k < 1) return 256;
  RouteGeom g = route_geom(T, E, k);
  return align_up(static_cast<size_t>(g.ntiles) * E * sizeof(uint64_t), 256);
}

readme_status launch_route(const void* logits, readme_dtype logits_dt, int64_t T, int32_t E, int32_t k,
                           int32_t* topk_idx, float* topk_w, int32_t* counts, int32_t* offsets, int32_t* dest,
                           int32_t* src, uint32_t* dev_status, void* ws, cudaStream_t st, bool finalize,
                           uint32_t* zero, int64_t zero_words, const RouteHead* head) {
  if (T == 0) {
    README_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, st));
    README_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (E + 1), st));
    return README_OK;
  }
  if (head) {  // the logits come from the gating head; f32 from here on
    logits = head->logits;
    logits_dt = README_F32;
  }
  // the head runs inside the single-launch route (E <= 16); otherwise as its own kernel first
  bool head_fused = head != nullptr && E <= kCHeadMaxE && use_cluster_route(T, k);
  if (head && !head_fused)
    README_TRY(launch_router_head(head->h, T, head->g, head->w, E, head->eps, head->logits, st));
  int lpt = 1;
  while (lpt < E && lpt < kWarp) lpt <<= 1;
  const int items = (E + lpt - 1) / lpt;
  if (use_cluster_route(T, k)) {
    // one cluster launch: a1-a4 including the finalize (dest = offsets + rank, src)
    const ClusterGeom cg = cluster_geom(T, E, k);
    RouteExtra ex{zero, zero_words, nullptr, nullptr, nullptr, 0.f, nullptr};
    size_t smem = cg.smem;
    if (head_fused) {
      ex.head_h = head->h;
      ex.head_g = head->g;
      ex.head_w = head->w;
      ex.head_eps = head->eps;
      ex.head_logits = head->logits;
      smem += sizeof(__nv_bfloat16) * static_cast<size_t>(E) * kRouterDim + sizeof(float) * cg.tile_tokens * E;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(cg.C);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(static_cast<unsigned>(cg.C));
    cfg.blockDim = dim3(kCThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    void* args[] = {const_cast<void**>(&logits), &T, &E, &k, const_cast<int*>(&cg.tile_tokens),
                    const_cast<int64_t*>(&cg.chunk), &lpt, const_cast<int*>(&items), &topk_idx, &topk_w, &counts,
                    &offsets, &dest, &src, &dev_status, &g_trace_buf, &ex};
    const void* fn = logits_dt == README_F32 ? cluster_fn<float>(topk_ne(E)) : cluster_fn<__nv_bfloat16>(topk_ne(E));
    const cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e == cudaSuccess) return README_OK;
    // the cluster could not be placed (e.g. SMs partitioned away): the multi-CTA route gives the same
    // result, finalized as the caller expects from the single-launch path
    cudaGetLastError();
    finalize = true;
    if (head_fused) README_TRY(launch_router_head(head->h, T, head->g, head->w, E, head->eps, head->logits, st));
  }
  if (zero && zero_words > 0) README_CUDA(cudaMemsetAsync(zero, 0, sizeof(uint32_t) * zero_words, st));
  RouteGeom g = route_geom(T, E, k);
  uint64_t* status = static_cast<uint64_t*>(ws);
  README_CUDA(cudaMemsetAsync(status, 0, static_cast<size_t>(g.ntiles) * E * sizeof(uint64_t), st));
#define README_TILE_LAUNCH(LT, NE)                                                                         \
  route_tile_kernel<LT, NE><<<g.ntiles, kRouteThreads, 0, st>>>(                                           \
      static_cast<const LT*>(logits), T, E, k, g.tile_tokens, g.ntiles, lpt, items, topk_idx, topk_w, counts, \
      offsets, dest, dev_status, status)
  const int ne = topk_ne(E);
  if (logits_dt == README_F32) {
    if (ne == 8) README_TILE_LAUNCH(float, 8);
    else if (ne == 16) README_TILE_LAUNCH(float, 16);
    else if (ne == 32) README_TILE_LAUNCH(float, 32);
    else README_TILE_LAUNCH(float, 0);
  } else {
    if (ne == 8) README_TILE_LAUNCH(__nv_bfloat16, 8);
    else if (ne == 16) README_TILE_LAUNCH(__nv_bfloat16, 16);
    else if (ne == 32) README_TILE_LAUNCH(__nv_bfloat16, 32);
    else README_TILE_LAUNCH(__nv_bfloat16, 0);
  }
#undef README_TILE_LAUNCH
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
