// router.cu — NEXT-1 of SURVEY §8(f): the pre-gating router G (§2.3; table:router_details,
// PAPER.md:276-294): ONE causal transformer block — vocab 32000, embedding/feature dim 512, 4 heads, SwiGLU
// MLP with intermediate dim 512, RoPE, RMSNorm — followed by a linear gating head to the N expert logits
// G(x_<=t). It runs once per token (not per layer: the whole point of pre-gating) and its
// logits feed readme_route (a0 of the hot path).
//
// Readings (Q15): Llama-style pre-norm block h1 = h0 + Attn(RMSNorm_1(h0)), h2 = h1 +
// MLP(RMSNorm_2(h1)), logits = RMSNorm_f(h2) W_head^T; RMSNorm eps 1e-5 with learned weights; RoPE with
// theta 10000 on the (i, i+64) halves of each 128-dim head; no biases.
//
// Kernels here: the embedding gather + first RMSNorm, a weighted RMSNorm, the causal attention with RoPE
// applied on the fly (flash-attention on mma.sync bf16 tensor-core fragments), and the gating head (final RMSNorm + 512 x N dot products per token). The QKV / output / MLP
// projections are dense contractions and run on the tcgen05 CTA-pair GEMM kernels of ffn_sm100_2cta.cu.
#include <math.h>

#include <mutex>

#include "kernels.h"
#include "router_head.cuh"
#include "tc_common.cuh"

namespace readme {

namespace {

constexpr int kD = 512;       // model dim
constexpr int kHeads = 4;
constexpr int kHd = 128;      // head dim
constexpr float kTheta = 10000.f;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// One warp per token: h0 = Emb[id] (copied to the residual stream), a = RMSNorm(h0) * g. The grid also
// writes the one-segment table offs = {0, T} of the block's GEMMs and zeroes the MLP FFN's readiness words
// (so neither needs a launch of its own).
__global__ void router_embed_norm_kernel(const int32_t* __restrict__ ids, int64_t T, int V,
                                         const __nv_bfloat16* __restrict__ emb, const __nv_bfloat16* __restrict__ g,
                                         float eps, __nv_bfloat16* __restrict__ h0, __nv_bfloat16* __restrict__ a,
                                         uint32_t* __restrict__ dev_status, int32_t* __restrict__ offs,
                                         uint32_t* __restrict__ zero, int64_t zero_words) {
  const int lane = threadIdx.x % kWarp;
  const int64_t gtid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (int64_t i = gtid; i < zero_words; i += static_cast<int64_t>(gridDim.x) * blockDim.x) zero[i] = 0u;
  if (gtid == 0) {
    offs[0] = 0;
    offs[1] = static_cast<int32_t>(T);
  }
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x / kWarp) + threadIdx.x / kWarp;
  if (t >= T) return;
  int id = ids[t];
  if (id < 0 || id >= V) {
    if (lane == 0 && dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
    id = 0;
  }
  const __nv_bfloat16* row = emb + static_cast<int64_t>(id) * kD;
  float v[16];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = __bfloat162float(row[lane + 32 * i]);
    ss = fmaf(v[i], v[i], ss);
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / kD + eps);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int c = lane + 32 * i;
    h0[t * kD + c] = __float2bfloat16_rn(v[i]);
    a[t * kD + c] = __float2bfloat16_rn(v[i] * r * __bfloat162float(g[c]));
  }
}

// One warp per token: y = RMSNorm(x) * g.
__global__ void rmsnorm512_kernel(const __nv_bfloat16* __restrict__ x, int64_t T, const __nv_bfloat16* __restrict__ g,
                                  float eps, __nv_bfloat16* __restrict__ y) {
  const int lane = threadIdx.x % kWarp;
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x / kWarp) + threadIdx.x / kWarp;
  if (t >= T) return;
  float v[16];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = __bfloat162float(x[t * kD + lane + 32 * i]);
    ss = fmaf(v[i], v[i], ss);
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / kD + eps);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int c = lane + 32 * i;
    y[t * kD + c] = __float2bfloat16_rn(v[i] * r * __bfloat162float(g[c]));
  }
}

// Gating head: logits[t] = (RMSNorm(h2[t]) * gf) . W_head^T, fp32. One warp per token, W_head in smem
// (router_head.cuh; the fused head + route launch in route.cu computes the same bits).
__global__ void router_head_kernel(const __nv_bfloat16* __restrict__ h2, int64_t T, const __nv_bfloat16* __restrict__ gf,
                                   const __nv_bfloat16* __restrict__ whead, int N, float eps, float* __restrict__ logits) {
  extern __shared__ float s_w[];  // [N][512]
  for (int i = threadIdx.x; i < N * kD; i += blockDim.x) s_w[i] = __bfloat162float(whead[i]);
  __syncthreads();
  const int lane = threadIdx.x % kWarp;
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x / kWarp) + threadIdx.x / kWarp;
  if (t >= T) return;
  head_logits_warp(h2 + t * kD, gf, [&](int n, int c) { return s_w[n * kD + c]; }, N, eps, lane,
                   [&](int n, float v) { logits[t * N + n] = v; });
}

// RoPE applied once per token, in place on the q and k parts of qkv (positions restart per sequence).
// One warp per token; lane i handles angle pairs i and i + 32 (of 64) for all 4 heads of q and k.
__global__ void router_rope_kernel(__nv_bfloat16* __restrict__ qkv, int64_t T, const int32_t* __restrict__ seq_starts,
                                   int nseq) {
  const int lane = threadIdx.x % kWarp;
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x / kWarp) + threadIdx.x / kWarp;
  if (t >= T) return;
  int lo_s = 0, hi_s = nseq;  // find the sequence holding t (binary search on seq_starts)
  while (hi_s - lo_s > 1) {
    const int mid = (lo_s + hi_s) / 2;
    if (seq_starts[mid] <= t) lo_s = mid; else hi_s = mid;
  }
  const int pos = static_cast<int>(t - seq_starts[lo_s]);
  __nv_bfloat16* row = qkv + t * (3 * kD);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = lane + 32 * u;
    const float inv = exp2f(-static_cast<float>(2 * i) / kHd * log2f(kTheta));
    float sn, cs;
    sincosf(static_cast<float>(pos) * inv, &sn, &cs);
#pragma unroll
    for (int part = 0; part < 2; ++part) {  // q, k
#pragma unroll
      for (int h = 0; h < kHeads; ++h) {
        __nv_bfloat16* base = row + part * kD + h * kHd;
        const float a = __bfloat162float(base[i]), b = __bfloat162float(base[i + 64]);
        base[i] = __float2bfloat16_rn(a * cs - b * sn);
        base[i + 64] = __float2bfloat16_rn(b * cs + a * sn);
      }
    }
  }
}

// ---- causal attention on tcgen05 / TMEM (the prefill path) ----------------------------------------------
// One CTA (4 warps) per (128-query tile of a sequence, head). Q, K and V tiles come in with TMA (128-byte
// swizzle, two 64-dim boxes per 128-row tile); per 128-key block: S = Q K^T on the tensor core into TMEM
// (M = 128 queries, N = 128 keys, K = 128 dims); each thread owns one query row (its TMEM lane): causal mask,
// online softmax in base 2, P (bf16) written to shared memory in the swizzled K-major layout; O_b = P V on
// the tensor core into a second TMEM region (V is the MN-major B operand: its tile is used exactly as TMA
// wrote it); the thread folds O_b into its fp32 row accumulator in registers with the softmax rescale. K/V
// blocks are double-buffered (the next block's TMA runs under this block's work).
constexpr int kAQ = 128;                 // queries per CTA
constexpr int kAK = 128;                 // keys per block
constexpr int kABox = 128 * 128;         // one 128-row x 64-dim swizzled box: 16 KB

struct __align__(1024) AttnSmem {
  uint8_t q[2][kABox];        // Q tile: dims [0,64) | [64,128)
  uint8_t k[2][2][kABox];     // [slot][dim half]
  uint8_t v[2][2][kABox];
  uint8_t p[2][kABox];        // P tile: keys [0,64) | [64,128), rows = queries, K-major
  uint64_t qbar, kvbar[2], sbar, pvbar;
  uint32_t tmem_base;
};
constexpr size_t kAttnSmem = sizeof(AttnSmem) + 1024;
static_assert(kAttnSmem <= 232448, "attention shared memory");

// SW128 K-major descriptor as in tc_common.cuh, and the MN-major form for V: 64-element (128 B) rows along
// N (dims), 8-row groups along K (keys) 1024 B apart (SBO), the second 64-dim half 16 KB away (LBO).
__device__ __forceinline__ uint64_t sdesc_sw128_mn(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

__global__ void __launch_bounds__(128, 1)
router_attention_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const int32_t* __restrict__ seq_starts,
                           const int32_t* __restrict__ tile_seq, const int32_t* __restrict__ tile_q0,
                           const int32_t* __restrict__ ntiles, __nv_bfloat16* __restrict__ out) {
  extern __shared__ uint8_t attn_raw[];
  AttnSmem& s = *reinterpret_cast<AttnSmem*>((reinterpret_cast<uintptr_t>(attn_raw) + 1023) & ~uintptr_t(1023));
  const int tile = blockIdx.x, head = blockIdx.y;
  if (tile >= *ntiles) return;
  const int seq = tile_seq[tile];
  const int s0 = seq_starts[seq], s1 = seq_starts[seq + 1];
  const int q0 = tile_q0[tile];
  const int q_last = min(q0 + kAQ, s1) - 1;
  const int nblk = (q_last - s0) / kAK + 1;  // key blocks [s0 + b*128, ...) up to the last query
  const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
  const int qcol = head * kHd, kcol = kD + head * kHd, vcol = 2 * kD + head * kHd;

  if (tid == 0) {
    tc::prefetch_tmap(&tmQKV);
    tc::mbar_init(&s.qbar, 1);
    tc::mbar_init(&s.kvbar[0], 1);
    tc::mbar_init(&s.kvbar[1], 1);
    tc::mbar_init(&s.sbar, 1);
    tc::mbar_init(&s.pvbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tc::tmem_alloc<1>(&s.tmem_base, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = s.tmem_base;
  auto load_kv = [&](int b) {  // thread 0: key block b into slot b & 1
    const int sl = b & 1, k0 = s0 + b * kAK;
    tc::mbar_expect_tx(&s.kvbar[sl], 4u * kABox);
    tc::tma_load_2d(&tmQKV, s.k[sl][0], &s.kvbar[sl], kcol, k0);
    tc::tma_load_2d(&tmQKV, s.k[sl][1], &s.kvbar[sl], kcol + 64, k0);
    tc::tma_load_2d(&tmQKV, s.v[sl][0], &s.kvbar[sl], vcol, k0);
    tc::tma_load_2d(&tmQKV, s.v[sl][1], &s.kvbar[sl], vcol + 64, k0);
  };
  if (tid == 0) {
    tc::mbar_expect_tx(&s.qbar, 2u * kABox);
    tc::tma_load_2d(&tmQKV, s.q[0], &s.qbar, qcol, q0);
    tc::tma_load_2d(&tmQKV, s.q[1], &s.qbar, qcol + 64, q0);
    load_kv(0);
    if (nblk > 1) load_kv(1);
  }
  constexpr uint32_t idesc_s = tc::idesc_bf16(128, 128);
  constexpr uint32_t idesc_pv = tc::idesc_bf16(128, 128) | (1u << 16);  // B (V) MN-major
  const float scale_log2 = rsqrtf(static_cast<float>(kHd)) * 1.4426950408889634f;
  const int qrow = q0 + warp * 32 + lane;  // this thread's query (TMEM lane 32 * warp + lane)
  const uint32_t t_s = tmem + (static_cast<uint32_t>(warp * 32) << 16), t_o = t_s + 128u;
  // O accumulates in TMEM columns [128, 256) across the key blocks (PV MMAs with accumulate); the row's
  // exponent base m only moves when a block's max exceeds it by more than 2^8 (then O and l are rescaled in
  // place), so most blocks need no O round trip (values stay within 2^8 of 1: exact enough in fp32 / bf16)
  float m = -INFINITY, l = 0.f;

  for (int b = 0; b < nblk; ++b) {
    const int sl = b & 1, k0 = s0 + b * kAK;
    if (tid == 0) {
      if (b == 0) tc::mbar_wait(&s.qbar, 0);
      tc::mbar_wait(&s.kvbar[sl], static_cast<uint32_t>(b >> 1) & 1u);
      tc::fence_after();
#pragma unroll
      for (int kk = 0; kk < kHd / 16; ++kk) {  // S = Q K^T over the 128 dims (two 64-dim swizzled halves)
        const uint64_t ad = tc::sdesc_sw128(tc::smem_u32(s.q[kk >> 2])) + static_cast<uint64_t>((kk & 3) * 2);
        const uint64_t bd = tc::sdesc_sw128(tc::smem_u32(s.k[sl][kk >> 2])) + static_cast<uint64_t>((kk & 3) * 2);
        tc::mma_f16<1>(tmem, ad, bd, idesc_s, kk != 0 ? 1u : 0u);
      }
      tc::commit(&s.sbar);
    }
    __syncwarp();
    tc::mbar_wait(&s.sbar, static_cast<uint32_t>(b) & 1u);
    tc::fence_after();
    // ---- this thread's query row over the block's 128 keys: masked max, then p = 2^(s - m) into P ----
    float mx = -INFINITY;
#pragma unroll
    for (int c = 0; c < kAK; c += 32) {
      uint32_t r[32];
      tc::tmem_ld32(t_s + static_cast<uint32_t>(c), r);
      tc::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int key = k0 + c + j;
        if (key <= qrow && key < s1) mx = fmaxf(mx, __uint_as_float(r[j]) * scale_log2);
      }
    }
    // move the base when the block's max exceeds it by more than 2^8 (also the row's first finite max);
    // O is rescaled in TMEM by the warp (tcgen05.ld/st are warp-collective) when any lane's base moved
    const bool up = mx > m + 8.f;
    const float alpha = (up && m != -INFINITY) ? exp2f(m - mx) : 1.f;
    if (up) {
      l *= alpha;
      m = mx;
    }
    if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
      for (int c = 0; c < kHd; c += 32) {
        uint32_t r[32];
        tc::tmem_ld32(t_o + static_cast<uint32_t>(c), r);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
        tc::tmem_st32(t_o + static_cast<uint32_t>(c), r);
      }
      tc::tmem_wait_st();
    }
    float ps = 0.f;
#pragma unroll
    for (int c = 0; c < kAK; c += 32) {
      uint32_t r[32];
      tc::tmem_ld32(t_s + static_cast<uint32_t>(c), r);
      tc::tmem_wait_ld();
#pragma unroll
      for (int c8 = 0; c8 < 32; c8 += 8) {
        float pf[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int key = k0 + c + c8 + j;
          pf[j] = (key <= qrow && key < s1) ? exp2f(__uint_as_float(r[c8 + j]) * scale_log2 - m) : 0.f;
          ps += pf[j];
        }
        uint4 w;
        w.x = pack_bf16x2(pf[0], pf[1]);
        w.y = pack_bf16x2(pf[2], pf[3]);
        w.z = pack_bf16x2(pf[4], pf[5]);
        w.w = pack_bf16x2(pf[6], pf[7]);
        const int row = warp * 32 + lane, kc = c + c8, chunk = (kc & 63) >> 3;  // 128-B swizzle
        *reinterpret_cast<uint4*>(s.p[kc >> 6] + row * 128 + ((chunk ^ (row & 7)) << 4)) = w;
      }
    }
    l += ps;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P (generic stores) -> the tensor core
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 0) {
#pragma unroll
      for (int kk = 0; kk < kAK / 16; ++kk) {  // O += P V over the block's 128 keys
        const uint64_t ad = tc::sdesc_sw128(tc::smem_u32(s.p[kk >> 2])) + static_cast<uint64_t>((kk & 3) * 2);
        const uint64_t bd = sdesc_sw128_mn(tc::smem_u32(s.v[sl][0]) + static_cast<uint32_t>(kk * 16 * 128),
                                           static_cast<uint32_t>(kABox));
        tc::mma_f16<1>(tmem + 128u, ad, bd, idesc_pv, (b | kk) != 0 ? 1u : 0u);
      }
      tc::commit(&s.pvbar);
    }
    __syncwarp();
    tc::mbar_wait(&s.pvbar, static_cast<uint32_t>(b) & 1u);
    tc::fence_after();
    if (tid == 0 && b + 2 < nblk) load_kv(b + 2);  // the slot's K and V have been consumed
  }
  {  // the warp reads its rows' O (warp-collective), the rows of this tile's queries are stored
    const bool store = qrow <= q_last;
    const float il = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* dst = out + static_cast<int64_t>(store ? qrow : 0) * kD + head * kHd;
#pragma unroll
    for (int c = 0; c < kHd; c += 32) {
      uint32_t r[32];
      tc::tmem_ld32(t_o + static_cast<uint32_t>(c), r);
      tc::tmem_wait_ld();
#pragma unroll
      for (int c8 = 0; c8 < 32; c8 += 8) {
        uint4 w;
        w.x = pack_bf16x2(__uint_as_float(r[c8 + 0]) * il, __uint_as_float(r[c8 + 1]) * il);
        w.y = pack_bf16x2(__uint_as_float(r[c8 + 2]) * il, __uint_as_float(r[c8 + 3]) * il);
        w.z = pack_bf16x2(__uint_as_float(r[c8 + 4]) * il, __uint_as_float(r[c8 + 5]) * il);
        w.w = pack_bf16x2(__uint_as_float(r[c8 + 6]) * il, __uint_as_float(r[c8 + 7]) * il);
        if (store) *reinterpret_cast<uint4*>(dst + c + c8) = w;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<1>(tmem, 256);
}

// 128-query tile table for the tcgen05 attention (as router_tiles_kernel).
__global__ void router_tiles128_kernel(const int32_t* __restrict__ seq_starts, int nseq, int32_t* __restrict__ tile_seq,
                                       int32_t* __restrict__ tile_q0, int32_t* __restrict__ ntiles_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int n = 0;
  for (int s = 0; s < nseq; ++s)
    for (int q = seq_starts[s]; q < seq_starts[s + 1]; q += kAQ) {
      tile_seq[n] = s;
      tile_q0[n] = q;
      ++n;
    }
  *ntiles_out = n;
}

// ---- incremental evaluation (decode): one or more new tokens per request against a key/value cache ----

// One warp per new token t at position pos[t] of request slot[t]: RoPE on q in place (as the prefill path),
// RoPE'd k and raw v appended to the cache row kv[slot][pos] = [k (512) | v (512)].
__global__ void router_rope_append_kernel(__nv_bfloat16* __restrict__ qkv, int64_t n, const int32_t* __restrict__ slot,
                                          const int32_t* __restrict__ pos, __nv_bfloat16* __restrict__ kv,
                                          int n_slots, int max_len, uint32_t* __restrict__ dev_status) {
  const int lane = threadIdx.x % kWarp;
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x / kWarp) + threadIdx.x / kWarp;
  if (t >= n) return;
  const int sl = slot[t], p = pos[t];
  const bool ok = sl >= 0 && sl < n_slots && p >= 0 && p < max_len;
  if (!ok) {
    if (lane == 0 && dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
    return;
  }
  __nv_bfloat16* row = qkv + t * (3 * kD);
  __nv_bfloat16* cache = kv + (static_cast<int64_t>(sl) * max_len + p) * (2 * kD);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = lane + 32 * u;
    const float inv = exp2f(-static_cast<float>(2 * i) / kHd * log2f(kTheta));
    float sn, cs;
    sincosf(static_cast<float>(p) * inv, &sn, &cs);
#pragma unroll
    for (int h = 0; h < kHeads; ++h) {
      __nv_bfloat16* q = row + h * kHd;
      float a = __bfloat162float(q[i]), b = __bfloat162float(q[i + 64]);
      q[i] = __float2bfloat16_rn(a * cs - b * sn);
      q[i + 64] = __float2bfloat16_rn(b * cs + a * sn);
      const __nv_bfloat16* k = row + kD + h * kHd;
      a = __bfloat162float(k[i]);
      b = __bfloat162float(k[i + 64]);
      cache[h * kHd + i] = __float2bfloat16_rn(a * cs - b * sn);
      cache[h * kHd + i + 64] = __float2bfloat16_rn(b * cs + a * sn);
    }
  }
  for (int c = lane; c < kD; c += kWarp) cache[kD + c] = row[2 * kD + c];
}

// Split-K decode attention (flash-decoding), KV-bandwidth bound (2 x 256 B per cached key per head). One
// CTA (128 threads) per (new token, head, chunk of kChunk cached positions): 8 groups of 16 threads, group g
// takes keys g, g+8, ... of the chunk and a thread owns 8 of the 128 dims, so every K / V row is read as 16
// coalesced 16-byte pieces. Each CTA leaves its chunk's (max m, sum l, o = sum_j e^(s_j - m) v_j); the merge
// kernel combines the chunks. Long histories thus spread over many SMs instead of serialising in one CTA.
constexpr int kChunk = 256;
constexpr int kPart = kHd + 2;  // floats per partial: o[128], m, l

__global__ void __launch_bounds__(128)
router_decode_attention_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t n, const int32_t* __restrict__ slot,
                               const int32_t* __restrict__ pos, const __nv_bfloat16* __restrict__ kv, int n_slots,
                               int max_len, int nchunk, float* __restrict__ part) {
  __shared__ float s_sc[kChunk];
  __shared__ float s_o[8][kHd];
  __shared__ float s_red[4];
  const int64_t t = blockIdx.x;
  const int head = blockIdx.y, c = blockIdx.z, tid = threadIdx.x, lane = tid % kWarp, warp = tid / kWarp;
  const int grp = tid / 16, l16 = tid % 16;
  const int sl = slot[t], p = pos[t];
  float* pp = part + ((t * kHeads + head) * nchunk + c) * kPart;
  if (sl < 0 || sl >= n_slots || p < 0 || p >= max_len || c * kChunk > p) {  // empty chunk (or bad index)
    if (tid == 0) {
      pp[kHd] = -INFINITY;
      pp[kHd + 1] = 0.f;
    }
    return;
  }
  const int j_lo = c * kChunk, j_hi = min(p, j_lo + kChunk - 1);  // inclusive
  float q[8];
  {
    const uint4 w = *reinterpret_cast<const uint4*>(qkv + t * (3 * kD) + head * kHd + 8 * l16);
    q[0] = bf16_lo(w.x); q[1] = bf16_hi(w.x); q[2] = bf16_lo(w.y); q[3] = bf16_hi(w.y);
    q[4] = bf16_lo(w.z); q[5] = bf16_hi(w.z); q[6] = bf16_lo(w.w); q[7] = bf16_hi(w.w);
  }
  const float scale = rsqrtf(static_cast<float>(kHd));
  const int64_t rs = 2 * kD;  // cache row stride (elements)
  const __nv_bfloat16* kbase = kv + static_cast<int64_t>(sl) * max_len * rs + head * kHd + 8 * l16;
  const __nv_bfloat16* vbase = kbase + kD;
  float mx = -INFINITY;
  // uniform trip count for the whole CTA (the 16-lane shuffles below need both half-warps present)
  for (int jb = j_lo; jb <= j_hi; jb += 32) {
    uint4 w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = jb + grp + 8 * u;
      w[u] = j <= j_hi ? ld_nc_v4(reinterpret_cast<const uint4*>(kbase + j * rs)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float acc = q[0] * bf16_lo(w[u].x);
      acc = fmaf(q[1], bf16_hi(w[u].x), acc); acc = fmaf(q[2], bf16_lo(w[u].y), acc);
      acc = fmaf(q[3], bf16_hi(w[u].y), acc); acc = fmaf(q[4], bf16_lo(w[u].z), acc);
      acc = fmaf(q[5], bf16_hi(w[u].z), acc); acc = fmaf(q[6], bf16_lo(w[u].w), acc);
      acc = fmaf(q[7], bf16_hi(w[u].w), acc);
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      const int j = jb + grp + 8 * u;
      if (j <= j_hi) {
        acc *= scale;
        if (l16 == 0) s_sc[j - j_lo] = acc;
        mx = fmaxf(mx, acc);
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 0) s_red[warp] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(s_red[0], s_red[1]), fmaxf(s_red[2], s_red[3]));
  __syncthreads();
  float sum = 0.f;
  for (int j = j_lo + tid; j <= j_hi; j += 128) {
    const float e = __expf(s_sc[j - j_lo] - mx);
    s_sc[j - j_lo] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  if (lane == 0) s_red[warp] = sum;
  __syncthreads();
  sum = s_red[0] + s_red[1] + s_red[2] + s_red[3];
  float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int jb = j_lo; jb <= j_hi; jb += 32) {
    uint4 w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = jb + grp + 8 * u;
      w[u] = j <= j_hi ? ld_nc_v4(reinterpret_cast<const uint4*>(vbase + j * rs)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = jb + grp + 8 * u;
      const float pj = j <= j_hi ? s_sc[j - j_lo] : 0.f;
      o[0] = fmaf(pj, bf16_lo(w[u].x), o[0]); o[1] = fmaf(pj, bf16_hi(w[u].x), o[1]);
      o[2] = fmaf(pj, bf16_lo(w[u].y), o[2]); o[3] = fmaf(pj, bf16_hi(w[u].y), o[3]);
      o[4] = fmaf(pj, bf16_lo(w[u].z), o[4]); o[5] = fmaf(pj, bf16_hi(w[u].z), o[5]);
      o[6] = fmaf(pj, bf16_lo(w[u].w), o[6]); o[7] = fmaf(pj, bf16_hi(w[u].w), o[7]);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) s_o[grp][8 * l16 + i] = o[i];
  __syncthreads();
  float acc = 0.f;
#pragma unroll
  for (int g = 0; g < 8; ++g) acc += s_o[g][tid];
  pp[tid] = acc;
  if (tid == 0) {
    pp[kHd] = mx;
    pp[kHd + 1] = sum;
  }
}

// Merge the chunks of one (token, head): o = sum_c e^(m_c - M) o_c / sum_c e^(m_c - M) l_c, c ascending.
__global__ void __launch_bounds__(128)
router_decode_merge_kernel(const float* __restrict__ part, int nchunk, __nv_bfloat16* __restrict__ out) {
  const int64_t t = blockIdx.x;
  const int head = blockIdx.y, tid = threadIdx.x;
  const float* pp = part + (t * kHeads + head) * nchunk * kPart;
  float M = -INFINITY;
  for (int c = 0; c < nchunk; ++c) M = fmaxf(M, pp[c * kPart + kHd]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int c = 0; c < nchunk; ++c) {
      const float m = pp[c * kPart + kHd];
      if (m == -INFINITY) continue;
      const float f = __expf(m - M);
      L = fmaf(f, pp[c * kPart + kHd + 1], L);
      O = fmaf(f, pp[c * kPart + tid], O);
    }
  }
  out[t * kD + head * kHd + tid] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
}



}  // namespace

// Workspace layout: offsets (256 B) | h0 | a | qkv (3x) | att | h1 | h2 | tile_seq | tile_q0 | ntiles |
// expert-FFN scratch (h [T, 512] + readiness counters).
namespace {
// h1 = h0 + att . Wo^T; h2 = h1 + MLP(RMSNorm_2(h1)); logits = RMSNorm_f(h2) . W_head^T.
readme_status router_tail(int64_t T, const RouterWeights& w, float eps, float* logits, const int32_t* offs,
                          const __nv_bfloat16* h0, __nv_bfloat16* a, const __nv_bfloat16* att, __nv_bfloat16* h1,
                          __nv_bfloat16* h2, __nv_bfloat16* hff, uint32_t* ready, uint32_t* dev_status,
                          cudaStream_t st, const RoutePlanOut* plan) {
  const int wpb = 8;
  const unsigned gblocks = static_cast<unsigned>((T + wpb - 1) / wpb);
  // h1 = h0 + att . Wo^T (the residual add fused into the GEMM epilogue)
  README_TRY(launch_gemm_2cta(1, att, T, kD, kD, 1, 1, offs, w.wo, nullptr, h1, nullptr, h0, st));
  // h2 = h1 + MLP(RMSNorm_2(h1)): the SwiGLU MLP is an expert FFN with one segment (E = 1, d = 512)
  rmsnorm512_kernel<<<gblocks, 32 * wpb, 0, st>>>(h1, T, w.g2, eps, a);
  README_CUDA(cudaGetLastError());
  // `ready` was zeroed by the embed launch (pdl = true: no memset node; the FFN waits on the RMSNorm grid)
  README_TRY(launch_ffn_layer_2cta(a, T, kD, 1, kD, 1, offs, w.wg, w.wu, w.wd, hff, h2, nullptr, h1, ready,
                                   dev_status, st, nullptr, 0, nullptr, true, nullptr));
  if (plan) {
    // NEXT-1 fusion: the final RMSNorm + gating head + top-k / histogram / scan / permutation in ONE route
    // launch that consumes h2 (logits still written, bit-identical to the head kernel's)
    const RouteHead head{h2, w.gf, w.whead, eps, logits};
    return launch_route(logits, README_F32, T, w.n_experts, plan->k, plan->topk_idx, plan->topk_w, plan->counts,
                        plan->offsets, plan->dest, plan->src, dev_status, plan->ws, st, true, nullptr, 0, &head);
  }
  return launch_router_head(h2, T, w.gf, w.whead, w.n_experts, eps, logits, st);
}
}  // namespace

size_t router_ws_bytes(int64_t T, int32_t nseq) {
  const size_t act = align_up(static_cast<size_t>(T) * kD * 2, 256);
  const size_t tiles = align_up(static_cast<size_t>(T / kAQ + nseq + 1) * sizeof(int32_t), 256);
  return 256 + 8 * act + 2 * tiles + 256 + act + ffn_layer_ready_bytes(T, 1) + 256;
}

readme_status launch_router_head(const __nv_bfloat16* h2, int64_t T, const __nv_bfloat16* gf,
                                 const __nv_bfloat16* whead, int N, float eps, float* logits, cudaStream_t st) {
  if (T == 0) return README_OK;
  const int wpb = 8;
  const unsigned gblocks = static_cast<unsigned>((T + wpb - 1) / wpb);
  router_head_kernel<<<gblocks, 32 * wpb, N * kD * sizeof(float), st>>>(h2, T, gf, whead, N, eps, logits);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_router_forward(const int32_t* ids, int64_t T, const int32_t* seq_starts, int32_t nseq,
                                    const RouterWeights& w, float eps, float* logits, void* ws,
                                    uint32_t* dev_status, cudaStream_t st, const RoutePlanOut* plan) {
  if (T == 0) return README_OK;
  const size_t act = align_up(static_cast<size_t>(T) * kD * 2, 256);
  const size_t tiles_b = align_up(static_cast<size_t>(T / kAQ + nseq + 1) * sizeof(int32_t), 256);
  char* p = static_cast<char*>(ws);
  int32_t* offs = reinterpret_cast<int32_t*>(p);
  p += 256;
  auto* h0 = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  auto* a = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  auto* qkv = reinterpret_cast<__nv_bfloat16*>(p); p += 3 * act;
  auto* att = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  auto* h1 = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  auto* h2 = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  int32_t* tile_seq = reinterpret_cast<int32_t*>(p); p += tiles_b;
  int32_t* tile_q0 = reinterpret_cast<int32_t*>(p); p += tiles_b;
  int32_t* ntiles = reinterpret_cast<int32_t*>(p); p += 256;
  auto* hff = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  uint32_t* ready = reinterpret_cast<uint32_t*>(p);
  const int64_t zero_words = static_cast<int64_t>(ffn_layer_ready_bytes(T, 1) / sizeof(uint32_t));

  const int wpb = 8;
  const unsigned gblocks = static_cast<unsigned>((T + wpb - 1) / wpb);
  router_embed_norm_kernel<<<gblocks, 32 * wpb, 0, st>>>(ids, T, w.vocab, w.emb, w.g1, eps, h0, a, dev_status,
                                                         offs, ready, zero_words);
  README_CUDA(cudaGetLastError());
  // q | k | v = a . Wqkv^T (tcgen05 CTA-pair GEMM over one segment)
  README_TRY(launch_gemm_2cta(1, a, T, kD, 3 * kD, 1, 1, offs, w.wqkv, nullptr, qkv, nullptr, nullptr, st));
  router_rope_kernel<<<gblocks, 32 * wpb, 0, st>>>(qkv, T, seq_starts, nseq);
  README_CUDA(cudaGetLastError());
  {
    static std::once_flag once[64];
    static cudaError_t attr_err[64];
    int dev = 0;
    README_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) dev = 0;
    std::call_once(once[dev], [&] {
      attr_err[dev] = cudaFuncSetAttribute(router_attention_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(kAttnSmem));
    });
    if (attr_err[dev] != cudaSuccess) return cuda_fail(attr_err[dev], "cudaFuncSetAttribute(router_attention_tc_kernel)");
    CUtensorMap mq;
    if (!tc::make_map_2d(&mq, qkv, 3 * kD, static_cast<uint64_t>(T), 64, 128)) {
      set_error("cuTensorMapEncodeTiled failed for the router's qkv");
      return README_ERR_CUDA;
    }
    router_tiles128_kernel<<<1, 1, 0, st>>>(seq_starts, nseq, tile_seq, tile_q0, ntiles);
    README_CUDA(cudaGetLastError());
    dim3 ag(static_cast<unsigned>(T / kAQ + nseq), kHeads);
    router_attention_tc_kernel<<<ag, 128, kAttnSmem, st>>>(mq, seq_starts, tile_seq, tile_q0, ntiles, att);
    README_CUDA(cudaGetLastError());
  }
  return router_tail(T, w, eps, logits, offs, h0, a, att, h1, h2, hff, ready, dev_status, st, plan);
}

size_t router_step_ws_bytes(int64_t n, int32_t max_len) {
  const int nchunk = (max_len + kChunk - 1) / kChunk;
  return router_ws_bytes(n, 1) + align_up(static_cast<size_t>(n) * kHeads * nchunk * kPart * sizeof(float), 256);
}

readme_status launch_router_step(const int32_t* ids, int64_t n, const int32_t* slot, const int32_t* pos,
                                 __nv_bfloat16* kv, int32_t n_slots, int32_t max_len, const RouterWeights& w,
                                 float eps, float* logits, void* ws, uint32_t* dev_status, cudaStream_t st) {
  if (n == 0) return README_OK;
  const size_t act = align_up(static_cast<size_t>(n) * kD * 2, 256);
  const size_t tiles_b = align_up(static_cast<size_t>(n / kAQ + 2) * sizeof(int32_t), 256);
  char* p = static_cast<char*>(ws);
  int32_t* offs = reinterpret_cast<int32_t*>(p);
  p += 256;
  auto* h0 = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  auto* a = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  auto* qkv = reinterpret_cast<__nv_bfloat16*>(p); p += 3 * act;
  auto* att = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  auto* h1 = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  auto* h2 = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  p += 2 * tiles_b + 256;
  auto* hff = reinterpret_cast<__nv_bfloat16*>(p); p += act;
  uint32_t* ready = reinterpret_cast<uint32_t*>(p);
  const int64_t zero_words = static_cast<int64_t>(ffn_layer_ready_bytes(n, 1) / sizeof(uint32_t));
  float* part = reinterpret_cast<float*>(static_cast<char*>(ws) + router_ws_bytes(n, 1));
  const int nchunk = (max_len + kChunk - 1) / kChunk;

  const int wpb = 8;
  const unsigned gblocks = static_cast<unsigned>((n + wpb - 1) / wpb);
  router_embed_norm_kernel<<<gblocks, 32 * wpb, 0, st>>>(ids, n, w.vocab, w.emb, w.g1, eps, h0, a, dev_status,
                                                         offs, ready, zero_words);
  README_CUDA(cudaGetLastError());
  README_TRY(launch_gemm_2cta(1, a, n, kD, 3 * kD, 1, 1, offs, w.wqkv, nullptr, qkv, nullptr, nullptr, st));
  // every new token's k/v reach the cache before any attention of this call reads it (causal within the
  // call too: token t only reads positions <= pos[t])
  router_rope_append_kernel<<<gblocks, 32 * wpb, 0, st>>>(qkv, n, slot, pos, kv, n_slots, max_len, dev_status);
  README_CUDA(cudaGetLastError());
  router_decode_attention_kernel<<<dim3(static_cast<unsigned>(n), kHeads, nchunk), 128, 0, st>>>(
      qkv, n, slot, pos, kv, n_slots, max_len, nchunk, part);
  README_CUDA(cudaGetLastError());
  router_decode_merge_kernel<<<dim3(static_cast<unsigned>(n), kHeads), 128, 0, st>>>(part, nchunk, att);
  README_CUDA(cudaGetLastError());
  return router_tail(n, w, eps, logits, offs, h0, a, att, h1, h2, hff, ready, dev_status, st, nullptr);
}

}  // namespace readme
