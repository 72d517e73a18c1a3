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
// applied on the fly (SIMT fp32 flash-style tiles: the router is ~50 GFLOP for 8192 tokens, off the hot
// path), and the gating head (final RMSNorm + 512 x N dot products per token). The QKV / output / MLP
// projections are dense contractions and run on the tcgen05 CTA-pair GEMM kernels of ffn_sm100_2cta.cu.
#include <math.h>

#include "kernels.h"

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

// One warp per token: h0 = Emb[id] (copied to the residual stream), a = RMSNorm(h0) * g.
__global__ void router_embed_norm_kernel(const int32_t* __restrict__ ids, int64_t T, int V,
                                         const __nv_bfloat16* __restrict__ emb, const __nv_bfloat16* __restrict__ g,
                                         float eps, __nv_bfloat16* __restrict__ h0, __nv_bfloat16* __restrict__ a,
                                         uint32_t* __restrict__ dev_status) {
  const int lane = threadIdx.x % kWarp;
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

// Gating head: logits[t] = (RMSNorm(h2[t]) * gf) . W_head^T, fp32. One warp per token, W_head in smem.
__global__ void router_head_kernel(const __nv_bfloat16* __restrict__ h2, int64_t T, const __nv_bfloat16* __restrict__ gf,
                                   const __nv_bfloat16* __restrict__ whead, int N, float eps, float* __restrict__ logits) {
  extern __shared__ float s_w[];  // [N][512]
  for (int i = threadIdx.x; i < N * kD; i += blockDim.x) s_w[i] = __bfloat162float(whead[i]);
  __syncthreads();
  const int lane = threadIdx.x % kWarp;
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x / kWarp) + threadIdx.x / kWarp;
  if (t >= T) return;
  float v[16];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = __bfloat162float(h2[t * kD + lane + 32 * i]);
    ss = fmaf(v[i], v[i], ss);
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / kD + eps);
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] *= r * __bfloat162float(gf[lane + 32 * i]);
  for (int n = 0; n < N; ++n) {
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) acc = fmaf(v[i], s_w[n * kD + lane + 32 * i], acc);
    acc = warp_sum(acc);
    if (lane == 0) logits[t * N + n] = acc;
  }
}

// Causal attention with RoPE, per (sequence, head, 32-query tile); K/V streamed in 32-key tiles.
// qkv [T, 1536] bf16 (q | k | v, head h = columns h*128..), seq_starts [nseq+1] (device), out [T, 512] bf16.
// Thread (r = tid / 8, s = tid % 8): scores of row r for keys 4s..4s+3 and output dims 16s..16s+15.
constexpr int kQT = 32, kKT = 32;

__device__ __forceinline__ void rope_pair(float& lo, float& hi, int pos, int i) {
  // rotate dims (i, i + 64) of a head by angle pos * theta^(-2i/128)
  const float inv = exp2f(-static_cast<float>(2 * i) / kHd * log2f(kTheta));
  float sn, cs;
  sincosf(static_cast<float>(pos) * inv, &sn, &cs);
  const float a = lo, b = hi;
  lo = a * cs - b * sn;
  hi = b * cs + a * sn;
}

__global__ void __launch_bounds__(256)
router_attention_kernel(const __nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ seq_starts,
                        const int32_t* __restrict__ tile_seq, const int32_t* __restrict__ tile_q0,
                        const int32_t* __restrict__ ntiles, __nv_bfloat16* __restrict__ out) {
  extern __shared__ float att_smem[];
  float(*sQ)[kHd + 1] = reinterpret_cast<float(*)[kHd + 1]>(att_smem);
  float(*sK)[kHd + 1] = reinterpret_cast<float(*)[kHd + 1]>(att_smem + kQT * (kHd + 1));
  float(*sV)[kHd] = reinterpret_cast<float(*)[kHd]>(att_smem + (kQT + kKT) * (kHd + 1));
  float(*sP)[kKT + 1] = reinterpret_cast<float(*)[kKT + 1]>(att_smem + (kQT + kKT) * (kHd + 1) + kKT * kHd);
  const int tile = blockIdx.x, head = blockIdx.y;
  if (tile >= *ntiles) return;
  const int seq = tile_seq[tile];
  const int s0 = seq_starts[seq], s1 = seq_starts[seq + 1];
  const int q0 = tile_q0[tile];  // absolute first query row
  const int nq = min(kQT, s1 - q0);
  const int tid = threadIdx.x, r = tid / 8, sub = tid % 8;
  const float scale = rsqrtf(static_cast<float>(kHd));
  const int ld = 3 * kD;

  // Q tile with RoPE (positions relative to the sequence start)
  for (int i = tid; i < kQT * (kHd / 2); i += blockDim.x) {
    const int rr = i / (kHd / 2), c = i % (kHd / 2);
    float lo = 0.f, hi = 0.f;
    if (rr < nq) {
      const int64_t row = q0 + rr;
      lo = __bfloat162float(qkv[row * ld + head * kHd + c]);
      hi = __bfloat162float(qkv[row * ld + head * kHd + c + 64]);
      rope_pair(lo, hi, static_cast<int>(row - s0), c);
    }
    sQ[rr][c] = lo * scale;
    sQ[rr][c + 64] = hi * scale;
  }
  float m_i = -INFINITY, l_i = 0.f;
  float o[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j] = 0.f;

  const int q_last = q0 + nq - 1;
  for (int k0 = s0; k0 <= q_last; k0 += kKT) {
    const int nk = min(kKT, s1 - k0);
    __syncthreads();
    for (int i = tid; i < kKT * (kHd / 2); i += blockDim.x) {
      const int kk = i / (kHd / 2), c = i % (kHd / 2);
      float lo = 0.f, hi = 0.f, vlo = 0.f, vhi = 0.f;
      if (kk < nk) {
        const int64_t row = k0 + kk;
        lo = __bfloat162float(qkv[row * ld + kD + head * kHd + c]);
        hi = __bfloat162float(qkv[row * ld + kD + head * kHd + c + 64]);
        rope_pair(lo, hi, static_cast<int>(row - s0), c);
        vlo = __bfloat162float(qkv[row * ld + 2 * kD + head * kHd + c]);
        vhi = __bfloat162float(qkv[row * ld + 2 * kD + head * kHd + c + 64]);
      }
      sK[kk][c] = lo;
      sK[kk][c + 64] = hi;
      sV[kk][c] = vlo;
      sV[kk][c + 64] = vhi;
    }
    __syncthreads();
    // scores for row r, keys 4*sub .. 4*sub+3 (causal: key <= query)
    float sc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int kk = 4 * sub + j;
      float acc = 0.f;
#pragma unroll 8
      for (int c = 0; c < kHd; ++c) acc = fmaf(sQ[r][c], sK[kk][c], acc);
      const bool ok = r < nq && kk < nk && (k0 + kk) <= (q0 + r);
      sc[j] = ok ? acc : -INFINITY;
    }
    float mx = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float m_new = fmaxf(m_i, mx);
    const float corr = (m_i == -INFINITY) ? 0.f : expf(m_i - m_new);
    float ps = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float p = (sc[j] == -INFINITY) ? 0.f : expf(sc[j] - m_new);
      sP[r][4 * sub + j] = p;
      ps += p;
    }
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
    l_i = l_i * corr + ps;
    m_i = m_new;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j] *= corr;
    for (int kk = 0; kk < nk; ++kk) {
      const float p = sP[r][kk];
#pragma unroll
      for (int j = 0; j < 16; ++j) o[j] = fmaf(p, sV[kk][16 * sub + j], o[j]);
    }
  }
  if (r < nq) {
    const float inv = 1.f / l_i;
    const int64_t row = q0 + r;
#pragma unroll
    for (int j = 0; j < 16; ++j) out[row * kD + head * kHd + 16 * sub + j] = __float2bfloat16_rn(o[j] * inv);
  }
}

// Query-tile table: for each sequence, ceil(len/32) tiles (seq id, first row). Built on the device.
constexpr size_t kAttSmem = sizeof(float) * ((kQT + kKT) * (kHd + 1) + kKT * kHd + kQT * (kKT + 1));

__global__ void router_tiles_kernel(const int32_t* __restrict__ seq_starts, int nseq, int32_t* __restrict__ tile_seq,
                                    int32_t* __restrict__ tile_q0, int32_t* __restrict__ ntiles_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int n = 0;
  for (int s = 0; s < nseq; ++s)
    for (int q = seq_starts[s]; q < seq_starts[s + 1]; q += kQT) {
      tile_seq[n] = s;
      tile_q0[n] = q;
      ++n;
    }
  *ntiles_out = n;
}

}  // namespace

// Workspace layout: offsets (256 B) | h0 | a | qkv (3x) | att | h1 | h2 | tile_seq | tile_q0 | ntiles |
// expert-FFN scratch (h [T, 512] + readiness counters).
size_t router_ws_bytes(int64_t T, int32_t nseq) {
  const size_t act = align_up(static_cast<size_t>(T) * kD * 2, 256);
  const size_t tiles = align_up(static_cast<size_t>(T / kQT + nseq + 1) * sizeof(int32_t), 256);
  return 256 + 8 * act + 2 * tiles + 256 + act + ffn_layer_ready_bytes(T, 1) + 256;
}

readme_status launch_router_forward(const int32_t* ids, int64_t T, const int32_t* seq_starts, int32_t nseq,
                                    const RouterWeights& w, float eps, float* logits, void* ws,
                                    uint32_t* dev_status, cudaStream_t st) {
  if (T == 0) return README_OK;
  const size_t act = align_up(static_cast<size_t>(T) * kD * 2, 256);
  const size_t tiles_b = align_up(static_cast<size_t>(T / kQT + nseq + 1) * sizeof(int32_t), 256);
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

  const int wpb = 8;
  const unsigned gblocks = static_cast<unsigned>((T + wpb - 1) / wpb);
  README_TRY(launch_set_offsets(offs, static_cast<int32_t>(T), st));
  router_embed_norm_kernel<<<gblocks, 32 * wpb, 0, st>>>(ids, T, w.vocab, w.emb, w.g1, eps, h0, a, dev_status);
  README_CUDA(cudaGetLastError());
  // q | k | v = a . Wqkv^T (tcgen05 CTA-pair GEMM over one segment)
  README_TRY(launch_gemm_2cta(1, a, T, kD, 3 * kD, 1, 1, offs, w.wqkv, nullptr, qkv, nullptr, nullptr, st));
  router_tiles_kernel<<<1, 1, 0, st>>>(seq_starts, nseq, tile_seq, tile_q0, ntiles);
  README_CUDA(cudaGetLastError());
  const int64_t max_tiles = T / kQT + nseq;
  dim3 ag(static_cast<unsigned>(max_tiles), kHeads);
  static bool attr_set[64] = {false};
  int dev = 0;
  README_CUDA(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    README_CUDA(cudaFuncSetAttribute(router_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kAttSmem)));
    attr_set[dev] = true;
  }
  router_attention_kernel<<<ag, 256, kAttSmem, st>>>(qkv, seq_starts, tile_seq, tile_q0, ntiles, att);
  README_CUDA(cudaGetLastError());
  // h1 = h0 + att . Wo^T (the residual add fused into the GEMM epilogue)
  README_TRY(launch_gemm_2cta(1, att, T, kD, kD, 1, 1, offs, w.wo, nullptr, h1, nullptr, h0, st));
  // h2 = h1 + MLP(RMSNorm_2(h1)): the SwiGLU MLP is an expert FFN with one segment (E = 1, d = 512)
  rmsnorm512_kernel<<<gblocks, 32 * wpb, 0, st>>>(h1, T, w.g2, eps, a);
  README_CUDA(cudaGetLastError());
  README_TRY(launch_ffn_layer_2cta(a, T, kD, 1, kD, 1, offs, w.wg, w.wu, w.wd, hff, h2, nullptr, h1, ready,
                                   dev_status, st));
  router_head_kernel<<<gblocks, 32 * wpb, w.n_experts * kD * sizeof(float), st>>>(h2, T, w.gf, w.whead,
                                                                                   w.n_experts, eps, logits);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

}  // namespace readme
