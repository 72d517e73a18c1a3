// kernels.h — internal launchers (host functions) behind the C ABI in capi.cu. Not exported.
#pragma once
#include "common.cuh"

namespace readme {

// knobs.cpp: lab/test switches, read from the environment once, overridable by readme_debug_set_knob.
enum class Knob : int {
  kRoute, kRouteCluster, kRouteTile, kDispatch, kDispatchBulk, kCombineBulk, kPermUnrollD, kPermUnrollC,
  kFfnKernel, kFfnMt, kFfnPairs, kFfnAskip, kFfnOrder, kFfnSwap, kFfnSpin, kFfnMerge, kFfnDyn, kFfnClaim, kCount
};
int knob(Knob k);

// route.cu
// The pre-gating router's gating head as the route's input (NEXT-1 fusion): logits = RMSNorm(h)*g . W^T are
// computed inside the route launch (E <= 16 and the single-launch route; else by the head kernel first) and
// written to `logits` [T, E] f32.
struct RouteHead {
  const __nv_bfloat16* h;  // [T, 512] the router block's output hidden state
  const __nv_bfloat16* g;  // [512]
  const __nv_bfloat16* w;  // [E, 512]
  float eps;
  float* logits;           // [T, E] out
};
size_t route_ws_bytes(int64_t T, int32_t E, int32_t k);
readme_status launch_route(const void* logits, readme_dtype logits_dt, int64_t T, int32_t E, int32_t k,
                           int32_t* topk_idx, float* topk_w, int32_t* counts, int32_t* offsets, int32_t* dest,
                           int32_t* src, uint32_t* dev_status, void* ws, cudaStream_t st, bool finalize = true,
                           uint32_t* zero = nullptr, int64_t zero_words = 0, const RouteHead* head = nullptr);
// router.cu: the separate gating-head kernel (logits [T, N] f32 from the hidden state)
readme_status launch_router_head(const __nv_bfloat16* h2, int64_t T, const __nv_bfloat16* gf,
                                 const __nv_bfloat16* whead, int N, float eps, float* logits, cudaStream_t st);
// zero/zero_words: words the launch zeroes (the FFN's readiness region, so no memset node precedes it; a
// memset on the multi-CTA path).
// true when launch_route runs the single-launch cluster route for this batch: it then always finalizes
// (dest = offsets + rank, src) regardless of `finalize`.
bool route_is_single_launch(int64_t T, int32_t k);

// permute.cu
readme_status launch_dispatch(const void* x, size_t row_bytes, int64_t T, int32_t k, const int32_t* dest,
                              void* x_sorted, uint32_t* dev_status, cudaStream_t st);
// Gather form of a5 for readme_moe_layer after the single-launch route: x_sorted[r] = x[src[r] / k], rows
// in ascending waves, xready[r] set (release) once row r is written; the expert FFN launched behind it
// (PDL) waits on those flags per tile instead of on the whole dispatch.
readme_status launch_dispatch_gather(const void* x, size_t row_bytes, int64_t rows, int32_t k, const int32_t* src,
                                     void* x_sorted, uint32_t* xready, uint32_t* dev_status, cudaStream_t st);
readme_status launch_dispatch_rmsnorm_gather(const void* x, readme_dtype dt, int64_t rows, int32_t H, int32_t k,
                                             const int32_t* src, float eps, void* x_sorted, uint32_t* xready,
                                             uint32_t* dev_status, cudaStream_t st);
readme_status launch_invert_perm(const int32_t* dest, int64_t n, int32_t* src, cudaStream_t st);  // src = dest^-1
readme_status launch_set_offsets(int32_t* offs, int32_t T, cudaStream_t st);  // {0, T}
readme_status launch_debug_mark(uint64_t* slot, cudaStream_t st);  // measurement only
readme_status launch_debug_hold_sms(int32_t n_ctas, int64_t ns, cudaStream_t st);  // test only
readme_status launch_finalize_dispatch(const void* x, size_t row_bytes, int64_t T, int32_t k, int32_t E,
                                       const int32_t* topk_idx, const int32_t* offsets, int32_t* dest, int32_t* src,
                                       void* x_sorted, cudaStream_t st);
readme_status launch_dispatch_rmsnorm(const void* x, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                                      const int32_t* dest, float eps, void* x_sorted, uint32_t* dev_status,
                                      cudaStream_t st);
readme_status launch_combine(const void* y_sorted, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                             const int32_t* dest, const float* topk_w, const void* residual, void* y,
                             uint32_t* dev_status, cudaStream_t st);
readme_status launch_build_experts(const void* wg, const void* wu, const void* wd, readme_dtype dt, int32_t D,
                                   int32_t H, int32_t E, int32_t d, const int32_t* nidx, void* eg, void* eu,
                                   void* ed, uint32_t* dev_status, cudaStream_t st);

// ffn_f32.cu (SIMT fp32, no TF32). a6: h = silu(xs Wg^T) * (xs Wu^T); a7: out = h Wd^T, or with
// src != null row r -> out[src[r]] (+ residual).
readme_status launch_gate_up_f32(const float* xs, int64_t rows, int32_t H, int32_t E, int32_t d, int32_t nseg,
                                 const int32_t* offsets, const float* wg, const float* wu, float* h, cudaStream_t st);
readme_status launch_down_f32(const float* h, int64_t rows, int32_t H, int32_t E, int32_t d, int32_t nseg,
                              const int32_t* offsets, const float* wd, float* out, const int32_t* src,
                              const float* residual, cudaStream_t st);
// a6 + a7 (+ fused combine: y[src[r]] (+ residual) when src is set; + a5 as a gather of x[gsrc[r] / k] when x
// is set, else rows of xs) in one launch, for H, d <= 128 (ffn_f32_fusable); bitwise equal to the two launches
bool ffn_f32_fusable(int32_t H, int32_t d);
readme_status launch_ffn_f32_fused(const float* xs, const float* x, const int32_t* gsrc, int32_t k, int64_t rows,
                                   int32_t H, int32_t E, int32_t d, int32_t nseg, const int32_t* offsets, const float* wg,
                                   const float* wu, const float* wd, float* out, const int32_t* src,
                                   const float* residual, cudaStream_t st);

// ffn_sm100.cu / ffn_sm100_2cta.cu (tcgen05 / TMEM / TMA grouped GEMMs, bf16)
readme_status launch_gemm_1cta(int mode, const __nv_bfloat16* A, int64_t rows, int32_t K, int32_t N, int32_t E,
                               int32_t nseg, const int32_t* offsets, const __nv_bfloat16* B0,
                               const __nv_bfloat16* B1, __nv_bfloat16* out, cudaStream_t st);
readme_status launch_gemm_2cta(int mode, const __nv_bfloat16* A, int64_t rows, int32_t K, int32_t N, int32_t E,
                               int32_t nseg, const int32_t* offsets, const __nv_bfloat16* B0,
                               const __nv_bfloat16* B1, __nv_bfloat16* out, const int32_t* src,
                               const __nv_bfloat16* residual, cudaStream_t st);
// a6 + a7 (+ a8 when src != null, k == 1) in one persistent CTA-pair launch; `ready` is a device scratch of
// ffn_layer_ready_bytes() bytes (zeroed by the launcher). With `peers`, received row r is stored to rank
// p's output (peer memory) as described on LayerArgs (expert parallelism, ep.cu).
constexpr int kMaxPeers = 8;
struct PeerOut {
  __nv_bfloat16* y[kMaxPeers];
  const __nv_bfloat16* res[kMaxPeers];
  int npeer;
  int64_t vrows;
};
// a5 fused into the single-launch FFN (launched as a programmatic dependent of the route): x_sorted[r] =
// x[src[r] / k] gathered by the kernel's epilogue warps before their first tile, published per row in xready.
struct SelfDispatch {
  const __nv_bfloat16* x;  // [T, H] tokens
  const int32_t* src;      // [T * k] slot of expert-contiguous row r
  int32_t k;
};
size_t ffn_layer_ready_bytes(int64_t rows, int32_t nseg);
size_t ffn_layer_xready_offset(int64_t rows);  // byte offset of the x_sorted row flags in `ready`

// Expert parallelism over peer memory (ep.cu).
readme_status launch_ep_signal(uint64_t* const* peer_flags, int G, int me, uint64_t* epoch, cudaStream_t st);
readme_status launch_ep_wait(const uint64_t* flags, int G, const uint64_t* epoch, uint32_t* dev_status,
                             cudaStream_t st);
readme_status launch_ep_publish(const int32_t* counts, int E, int32_t* const* peer_tables, int G, int me,
                                cudaStream_t st);
readme_status launch_ep_plan(const int32_t* table, int G, int E, int me, int32_t* seg_offsets, int32_t* row_base,
                             cudaStream_t st);
readme_status launch_ep_dispatch(const void* x, size_t row_bytes, int64_t T, int k, const int32_t* dest,
                                 const int32_t* offsets, const int32_t* row_base, int E, int G, int me,
                                 void* const* peer_x, int32_t* const* peer_map, int64_t vrows, int to_token,
                                 uint32_t* dev_status, cudaStream_t st);
readme_status launch_ffn_layer_2cta(const __nv_bfloat16* xs, int64_t rows, int32_t H, int32_t E, int32_t d,
                                    int32_t nseg, const int32_t* offsets, const __nv_bfloat16* wg,
                                    const __nv_bfloat16* wu, const __nv_bfloat16* wd, __nv_bfloat16* h,
                                    __nv_bfloat16* y, const int32_t* src, const __nv_bfloat16* residual,
                                    uint32_t* ready, uint32_t* dev_status, cudaStream_t st,
                                    const int32_t* expert_slot = nullptr, int32_t n_slots = 0,
                                    const PeerOut* peers = nullptr, bool pdl = false,
                                    const uint32_t* xready = nullptr, const SelfDispatch* sd = nullptr);
readme_status launch_gate_up_bf16(const __nv_bfloat16* xs, int64_t rows, int32_t H, int32_t E, int32_t d,
                                  int32_t nseg, const int32_t* offsets, const __nv_bfloat16* wg,
                                  const __nv_bfloat16* wu, __nv_bfloat16* h, cudaStream_t st);
readme_status launch_down_bf16(const __nv_bfloat16* h, int64_t rows, int32_t H, int32_t E, int32_t d, int32_t nseg,
                               const int32_t* offsets, const __nv_bfloat16* wd, __nv_bfloat16* out,
                               const int32_t* src, const __nv_bfloat16* residual, cudaStream_t st);

// router.cu: the pre-gating router G (one causal transformer block + gating head), NEXT-1.
struct RouterWeights {
  int vocab, n_experts;
  const __nv_bfloat16 *emb, *g1, *wqkv, *wo, *g2, *wg, *wu, *wd, *gf, *whead;
};
size_t router_ws_bytes(int64_t T, int32_t nseq);
// plan != null: instead of the head kernel, the routing plan is built by the route launch that consumes the
// block's hidden state (head fused into a1-a4); logits are still written.
struct RoutePlanOut {
  int32_t k;
  int32_t *topk_idx, *counts, *offsets, *dest, *src;
  float* topk_w;
  void* ws;  // route workspace (route_ws_bytes)
};
readme_status launch_router_forward(const int32_t* ids, int64_t T, const int32_t* seq_starts, int32_t nseq,
                                    const RouterWeights& w, float eps, float* logits, void* ws,
                                    uint32_t* dev_status, cudaStream_t st, const RoutePlanOut* plan = nullptr);
size_t router_step_ws_bytes(int64_t n, int32_t max_len);
readme_status launch_router_step(const int32_t* ids, int64_t n, const int32_t* slot, const int32_t* pos,
                                 __nv_bfloat16* kv, int32_t n_slots, int32_t max_len, const RouterWeights& w,
                                 float eps, float* logits, void* ws, uint32_t* dev_status, cudaStream_t st);

}  // namespace readme
