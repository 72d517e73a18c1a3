/* include/readme.h — C ABI of the B200-native READ-ME pre-gated MoE layer (libreadme_b200.so).
 *
 * READ-ME (arXiv 2410.19123) refactors a dense FFN into N experts, each a subset of the dense FFN's
 * neurons (§3: F_i(x) = W_2 M_i^T sigma(M_i W_1 x)), and routes every token ONCE with a
 * pre-gating router G that is independent of the layer (§2.3, Eq. 2):
 *
 *     y_t = sum_i 1( |{j : G(x_<=t)_j >= G(x_<=t)_i}| <= K ) * G(x_<=t)_i * F_i^(l)(x_t)
 *
 * This library implements the data-parallel hot path of one such layer on an NVIDIA B200 (sm_100a):
 *   readme_route      a1-a4  top-K + gate weights, per-expert histogram, exclusive scan, stable permutation
 *   readme_dispatch   a5     scatter tokens into expert-contiguous rows
 *   readme_expert_ffn a6-a7  grouped SwiGLU expert GEMMs (tcgen05/TMEM for bf16, SIMT fp32 for f32), also
 *                            split as readme_expert_gate_up (a6) and readme_expert_down (a7, optional fused a8)
 *   readme_combine    a8     gather back to token order, weight, add residual
 *   readme_moe_layer  a1-a8  the whole layer; with logits == NULL it reuses a routing plan (a9: route
 *                            once, reuse across all L layers)
 *   readme_moe_stack         L pre-norm MoE layers routed once (config 4), in place
 *   readme_router_forward    the pre-gating router G itself (one causal transformer block + gating head)
 *   readme_build_experts     setup: slice expert stacks out of the dense FFN
 * Readings of the paper (Q1..Q14) are listed in DESIGN.md; they are cited below where they decide a
 * behaviour.
 *
 * Conventions for every entry point:
 *   - Tensor pointers are CUDA DEVICE pointers (unless stated), row-major, contiguous, 16-byte aligned.
 *   - Calls are stream-ordered on `stream` (a cudaStream_t), never synchronise the host, never allocate
 *     device or host memory, and retain no pointer after returning: they are CUDA-graph capturable.
 *   - Ownership: the caller owns every buffer and the workspace; the library borrows them for the
 *     stream-ordered duration of the call. Outputs are fully overwritten (no pre-zeroing needed).
 *   - Errors: argument errors are reported synchronously by the return code and nothing is launched;
 *     readme_last_error() gives a thread-local message. Data errors only visible on the device
 *     (non-finite logits, out-of-range ids in a caller-supplied plan) are OR-ed as README_DEV_* bits into
 *     *dev_status (if non-NULL); indices are clamped so nothing faults. No exception crosses the ABI and
 *     nothing calls exit/abort.
 *   - T == 0 is a valid no-op (counts/offsets are still written as zeros).
 *   - Thread safety: reentrant. The only global state is per-device kernel attributes and cached driver
 *     entry points, initialised once under std::call_once.
 */
#ifndef README_B200_H_
#define README_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same object as cudaStream_t (struct CUstream_st*); NULL = the legacy default stream. */
typedef struct CUstream_st* readme_stream_t;

typedef enum {
  README_OK = 0,
  README_ERR_INVALID_ARG = 1,  /* null required pointer, bad size, misalignment */
  README_ERR_UNSUPPORTED = 2,  /* a dtype / shape combination this build does not provide */
  README_ERR_WORKSPACE = 3,    /* ws_bytes smaller than the matching *_workspace_bytes() */
  README_ERR_CUDA = 4          /* a CUDA launch or driver call failed (see readme_last_error) */
} readme_status;

typedef enum { README_F32 = 0, README_BF16 = 1 } readme_dtype;

#define README_DEV_NONFINITE_LOGIT 0x1u /* some logit was NaN/Inf (Q3: NaN ranks as -inf) */
#define README_DEV_BAD_INDEX 0x2u       /* a caller-supplied plan held an id/row out of range */
#define README_DEV_SCHED_TIMEOUT 0x4u   /* the single-launch expert FFN could not co-schedule its CTA pairs: a
                                          readiness wait gave up, and every output element is then either its
                                          correct value or left untouched (never computed from unready rows) */
#define README_DEV_EP_TIMEOUT 0x8u      /* readme_ep_wait gave up on a peer (~10 s) instead of hanging */

#define README_MAX_EXPERTS 256

/* ---------------------------------------------------------------------------------------------- */
/* a1-a4: routing plan.  PAPER.md:136-138 (Eq. 2 indicator), Alg. 1 ReqQueueByExpert.
 *
 * logits   [T,E] f32 or bf16 (logits_dt): G(x_<=t), produced once per token by the pre-gating router.
 * topk_idx [T,k] int32 out: the k experts of each token in descending logit order; ties go to the
 *          lower expert id (Q2). Exactly k distinct ids per token.
 * topk_w   [T,k] f32 out: softmax over the k selected logits (Q1); k == 1 gives exactly 1.0f.
 * counts   [E]   int32 out: #{(t,j) : topk_idx[t,j] == e}.
 * offsets  [E+1] int32 out: exclusive prefix sum of counts; offsets[E] == T*k.
 * dest     [T*k] int32 out: for flat slot s = t*k + j, the row of x_sorted that holds it:
 *          dest[s] = offsets[e] + #{s' < s : expert(s') == e}  (stable / FIFO within an expert, Q7).
 * src      [T*k] int32 out, nullable: inverse permutation, src[dest[s]] = s.
 * dev_status nullable: README_DEV_NONFINITE_LOGIT is OR-ed in if any logit is NaN/Inf.
 * ws       device workspace of readme_route_workspace_bytes(T,E,k) bytes (zeroed by the call itself).
 * Requires 1 <= E <= 256, 1 <= k <= E, T*k < 2^31.
 */
size_t readme_route_workspace_bytes(int64_t T, int32_t E, int32_t k);
readme_status readme_route(const void* logits, readme_dtype logits_dt, int64_t T, int32_t E, int32_t k,
                           int32_t* topk_idx, float* topk_w, int32_t* counts, int32_t* offsets,
                           int32_t* dest, int32_t* src, uint32_t* dev_status, void* ws, size_t ws_bytes,
                           readme_stream_t stream);

/* a5: dispatch.  x_sorted[dest[s]] = x[s / k] for every slot s < T*k (a bit copy of whole rows).
 * x [T,H] and x_sorted [T*k,H] of dtype dt; H*sizeof(dt) must be a multiple of 16 bytes.
 * Out-of-range dest entries set README_DEV_BAD_INDEX in dev_status (nullable) and are skipped. */
readme_status readme_dispatch(const void* x, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                              const int32_t* dest, void* x_sorted, uint32_t* dev_status,
                              readme_stream_t stream);

/* a6-a7: grouped expert FFN over expert-contiguous rows (PAPER.md:159 with sigma = SwiGLU, Q4):
 *     for segment g, rows r in [offsets[g], offsets[g+1]), expert e = g % E:
 *         h_r = silu(x_r W_gate[e]^T) * (x_r W_up[e]^T)      silu(z) = z / (1 + e^-z)
 *         y_sorted_r = h_r W_down[e]^T
 * n_src segment groups of E segments each (n_src = 1 on one GPU; n_src = G for the expert-parallel
 * receive buffer, which is ordered by source rank then expert).
 * x_sorted [rows,H], w_gate/w_up [E,d,H] (the expert's neurons = rows of the dense W_gate/W_up),
 * w_down [E,H,d] (columns of the dense W_down), y_sorted [rows,H]; all of dtype dt.
 * offsets: DEVICE int32 [n_src*E+1], non-decreasing, offsets[0] == 0, offsets[n_src*E] == rows.
 * bf16: tcgen05 tensor cores, fp32 accumulation in TMEM, fp32 SiLU, h rounded once to bf16 (Q11), y
 *       rounded once to bf16; requires H % 8 == 0 and d % 8 == 0.
 * f32:  CUDA-core FMA in fp32 (no TF32), for the tiny config.
 * Segments with no rows read no weights. ws: readme_expert_ffn_workspace_bytes(...) bytes.
 * bf16 runs a6 and a7 in ONE persistent launch whose down tiles wait on other CTA pairs' gate/up tiles; its
 * grid never exceeds the CTA pairs that can be co-resident (cudaOccupancyMaxActiveClusters). If SMs are
 * held elsewhere (another stream or process) for seconds, a wait gives up: README_DEV_SCHED_TIMEOUT is
 * OR-ed into dev_status (nullable) and the launch stores nothing more, so every element of y_sorted is
 * either correct or untouched. */
size_t readme_expert_ffn_workspace_bytes(int64_t rows, int32_t H, int32_t E, int32_t d, readme_dtype dt);
readme_status readme_expert_ffn(const void* x_sorted, readme_dtype dt, int64_t rows, int32_t H, int32_t E,
                                int32_t d, int32_t n_src, const int32_t* offsets, const void* w_gate,
                                const void* w_up, const void* w_down, void* y_sorted, uint32_t* dev_status,
                                void* ws, size_t ws_bytes, readme_stream_t stream);

/* a6 alone: h = silu(x_sorted W_gate[e]^T) * (x_sorted W_up[e]^T) per segment; h [rows,d] of dtype dt (bf16 h is
 * rounded once, Q11). Same arguments as readme_expert_ffn; no workspace. */
readme_status readme_expert_gate_up(const void* x_sorted, readme_dtype dt, int64_t rows, int32_t H, int32_t E,
                                    int32_t d, int32_t n_src, const int32_t* offsets, const void* w_gate,
                                    const void* w_up, void* h, readme_stream_t stream);

/* a7 alone: y_sorted_r = h_r W_down[e]^T per segment, out [rows,H]. With src != NULL (a layer with k == 1, whose
 * combine weight is exactly 1) row r is instead written to out[src[r]] + residual[src[r]] (residual nullable;
 * out is then y [T = rows, H]): the combine a8 fused into the epilogue, fp32 add, one rounding. Rows whose
 * src is out of range are skipped. With src == NULL and residual != NULL: out[r] = residual[r] + y_r. */
readme_status readme_expert_down(const void* h, readme_dtype dt, int64_t rows, int32_t H, int32_t E, int32_t d,
                                 int32_t n_src, const int32_t* offsets, const void* w_down, const int32_t* src,
                                 const void* residual, void* out, readme_stream_t stream);

/* The expert FFN over an expert CACHE (memory-constrained mode, §4.1; NEXT-4): the weights
 * are slot pools w_gate/w_up [n_slots,d,H], w_down [n_slots,H,d] and expert e's weights sit in slot
 * expert_slot[e] (DEVICE int32 [E]); only experts with rows are read, so slots of untouched experts may hold
 * anything. One segment group (n_src = 1). src/residual/out as in readme_expert_down (src == NULL and
 * residual == NULL: out = y_sorted). bf16 only. ws: readme_expert_ffn_workspace_bytes(...). */
readme_status readme_expert_ffn_slots(const void* x_sorted, readme_dtype dt, int64_t rows, int32_t H, int32_t E,
                                      int32_t d, const int32_t* offsets, const int32_t* expert_slot, int32_t n_slots,
                                      const void* w_gate, const void* w_up, const void* w_down, const int32_t* src,
                                      const void* residual, void* out, uint32_t* dev_status, void* ws,
                                      size_t ws_bytes, readme_stream_t stream);

/* a8: combine (Eq. 2's weighted sum):
 *     y[t] = residual[t] + sum_{j<k} topk_w[t,j] * y_sorted[dest[t*k+j]]   (j ascending, fp32, Q8)
 * topk_w is nullable iff k == 1 (weight 1); residual [T,H] nullable. With k == 1 and no residual the
 * result is a bit copy. y_sorted [T*k,H], y [T,H] of dtype dt (residual too). */
readme_status readme_combine(const void* y_sorted, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                             const int32_t* dest, const float* topk_w, const void* residual, void* y,
                             uint32_t* dev_status, readme_stream_t stream);

/* The whole layer (a1-a8).  If logits != NULL the plan (topk_idx..src) is computed and written (src may be
 * NULL: the library then keeps it in the workspace); if
 * logits == NULL the plan arrays are INPUTS from an earlier call (plan-in mode: route once per batch,
 * reuse for every layer). x, residual, y: [T,H] of dtype dt; weights as in
 * readme_expert_ffn. ws: readme_moe_layer_workspace_bytes(...) bytes. With k == 1 and a src available, the
 * combine is fused into the down projection's epilogue (one rounding of residual + y instead of two). */
size_t readme_moe_layer_workspace_bytes(int64_t T, int32_t H, int32_t E, int32_t d, int32_t k, readme_dtype dt);
readme_status readme_moe_layer(const void* x, readme_dtype dt, int64_t T, int32_t H, const void* logits,
                               readme_dtype logits_dt, int32_t E, int32_t k, int32_t d, const void* w_gate,
                               const void* w_up, const void* w_down, const void* residual, void* y,
                               int32_t* topk_idx, float* topk_w, int32_t* counts, int32_t* offsets,
                               int32_t* dest, int32_t* src, uint32_t* dev_status, void* ws, size_t ws_bytes,
                               readme_stream_t stream);

/* The 32-layer refactored stack (BASELINE config 4; reading Q10 in DESIGN.md): a MoE-only pre-norm stack
 *     x <- x + MoE_l(RMSNorm(x)),  l = 0..L-1,  RMSNorm(x) = x / sqrt(mean(x^2) + eps) (weight 1),
 * routed ONCE for all layers ("expert selection can be determined at the outset";
 * :237: "routed to Expert 1 in every layer"). x [T,H] is updated in place. w_gate/w_up/w_down are HOST
 * arrays of L device pointers (each as in readme_expert_ffn). logits == NULL: plan-in mode as in
 * readme_moe_layer. The attention blocks of the paper's model are outside this path.
 * readme_dispatch_rmsnorm is its pre-norm dispatch: x_sorted[dest[t*k+j]] = RMSNorm(x[t]), fp32 statistics. */
readme_status readme_dispatch_rmsnorm(const void* x, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                                      const int32_t* dest, float eps, void* x_sorted, uint32_t* dev_status,
                                      readme_stream_t stream);
size_t readme_moe_stack_workspace_bytes(int64_t T, int32_t H, int32_t E, int32_t d, int32_t k, readme_dtype dt);
readme_status readme_moe_stack(void* x, readme_dtype dt, int64_t T, int32_t H, const void* logits,
                               readme_dtype logits_dt, int32_t E, int32_t k, int32_t d, int32_t L,
                               const void* const* w_gate, const void* const* w_up, const void* const* w_down,
                               float eps, int32_t* topk_idx, float* topk_w, int32_t* counts, int32_t* offsets,
                               int32_t* dest, int32_t* src, uint32_t* dev_status, void* ws, size_t ws_bytes,
                               readme_stream_t stream);

/* The permanent expert (§3: neurons "activated for all tokens", NEXT-3 of SURVEY §8(f)):
 *     y[t] <- y[t] + F_perm(x[t]),   F_perm(x) = W_down,p (silu(W_gate,p x) * (W_up,p x))   for EVERY token,
 * added in place to y (call it after readme_moe_layer). w_gate/w_up [d_perm,H], w_down [H,d_perm] of dtype
 * dt; runs the same grouped-GEMM kernels over one segment of T rows (no dispatch: token order), with the
 * add fused into the down projection's epilogue. ws: readme_permanent_expert_workspace_bytes(...).
 * dev_status (nullable): README_DEV_SCHED_TIMEOUT as for readme_expert_ffn. */
size_t readme_permanent_expert_workspace_bytes(int64_t T, int32_t H, int32_t d_perm, readme_dtype dt);
readme_status readme_permanent_expert(const void* x, readme_dtype dt, int64_t T, int32_t H, int32_t d_perm,
                                      const void* w_gate, const void* w_up, const void* w_down, void* y,
                                      uint32_t* dev_status, void* ws, size_t ws_bytes, readme_stream_t stream);

/* ---------------------------------------------------------------------------------------------- */
/* The pre-gating router G (NEXT-1 of SURVEY §8(f)): PAPER.md:130-133 (§2.3, "one transformer block with
 * causal attention"), table:router_details (1 layer, 4 heads, vocab 32000, embedding and
 * feature dim 512, MLP intermediate dim 512, SwiGLU, RoPE, RMSNorm, 18.0 M parameters) and a linear gating
 * head to the N expert logits G(x_<=t) that readme_route consumes. Readings (Q15): Llama-style
 * pre-norm block h1 = h0 + Attn(RMSNorm_1(h0)), h2 = h1 + MLP(RMSNorm_2(h1)),
 * logits = RMSNorm_f(h2) W_head^T; RoPE theta 10000 on the (i, i+64) halves of each 128-dim head; no biases.
 * Run once per token, never per layer. All weights bf16 DEVICE pointers, nn.Linear
 * [out, in] layout; the struct itself is a host object read during the call. */
typedef struct {
  int32_t vocab;       /* rows of emb (32000 in the paper) */
  int32_t n_experts;   /* N, rows of w_head (1..16) */
  const void* emb;     /* [vocab, 512] */
  const void* norm1;   /* [512] RMSNorm weight before attention */
  const void* w_qkv;   /* [1536, 512]: rows 0..511 W_q, 512..1023 W_k, 1024..1535 W_v */
  const void* w_o;     /* [512, 512] */
  const void* norm2;   /* [512] RMSNorm weight before the MLP */
  const void* w_gate;  /* [512, 512] SwiGLU MLP */
  const void* w_up;    /* [512, 512] */
  const void* w_down;  /* [512, 512] */
  const void* norm_f;  /* [512] final RMSNorm weight */
  const void* w_head;  /* [n_experts, 512] gating head */
} readme_router_weights;

/* token_ids [T] int32 (device), sequences concatenated: seq_starts [nseq+1] int32 (DEVICE), seq_starts[0] = 0,
 * non-decreasing, seq_starts[nseq] = T; attention is causal inside each sequence and positions restart at 0
 * for each one. logits [T, n_experts] f32 out. Out-of-vocabulary ids set README_DEV_BAD_INDEX (id 0 used). */
size_t readme_router_workspace_bytes(int64_t T, int32_t nseq);
readme_status readme_router_forward(const int32_t* token_ids, int64_t T, const int32_t* seq_starts, int32_t nseq,
                                    const readme_router_weights* w, float eps, float* logits, uint32_t* dev_status,
                                    void* ws, size_t ws_bytes, readme_stream_t stream);

/* The router AND the routing plan in one call (NEXT-1 fusion: "fuse the gating head and
 * top-k into route"): the block runs as in readme_router_forward, then ONE launch consumes its last hidden
 * state and computes the final RMSNorm, the gating head (logits written to `logits`, bit-identical to
 * readme_router_forward's), the top-k / weights, the per-expert histogram, the exclusive scan and the stable
 * permutation (readme_route's a1-a4 on those logits, bit-identical to calling readme_route on them). Plan
 * arrays as in readme_route (src required). k in [1, n_experts]. The one-launch form covers batches the
 * single-launch route takes (T*k <= 256K slots); larger batches run the head kernel, then readme_route's
 * multi-CTA form, with the same results. ws: readme_router_route_workspace_bytes(T, nseq, n_experts, k). */
size_t readme_router_route_workspace_bytes(int64_t T, int32_t nseq, int32_t E, int32_t k);
readme_status readme_router_forward_route(const int32_t* token_ids, int64_t T, const int32_t* seq_starts,
                                          int32_t nseq, const readme_router_weights* w, float eps, int32_t k,
                                          float* logits, int32_t* topk_idx, float* topk_w, int32_t* counts,
                                          int32_t* offsets, int32_t* dest, int32_t* src, uint32_t* dev_status,
                                          void* ws, size_t ws_bytes, readme_stream_t stream);

/* Incremental evaluation (decode; SURVEY §8(f) NEXT-1 "run once per request, incrementally only for new
 * tokens"): n new tokens, token i of request slot[i] at position pos[i] (0-based within its request). Each
 * token's RoPE'd key and value are appended to kv_cache[slot][pos] (bf16 [n_slots, max_len, 2, 512]: k then v
 * of all 4 heads; caller-owned, persists across calls), then every token attends to positions 0..pos[i] of
 * its request (all appends of the call happen first, so several tokens of one request may be passed
 * together, in any order), and logits [n, n_experts] f32 are written. Same block and readings as
 * readme_router_forward; equal to it up to bf16 rounding order. Bad slot/pos set README_DEV_BAD_INDEX (that
 * token's attention output is zero). max_len <= 32768. ws: readme_router_step_workspace_bytes(n, max_len). Attention is split over chunks of
 * 256 cached positions (flash-decoding) and merged. */
size_t readme_router_step_workspace_bytes(int64_t n, int32_t max_len);
readme_status readme_router_step(const int32_t* token_ids, int64_t n, const int32_t* slot, const int32_t* pos,
                                 void* kv_cache, int32_t n_slots, int32_t max_len, const readme_router_weights* w,
                                 float eps, float* logits, uint32_t* dev_status, void* ws, size_t ws_bytes,
                                 readme_stream_t stream);

/* Setup (once per model load, not on the timed path): expert slicing, PAPER.md:159-163 (M_i is a
 * selection matrix without replacement).  dense_w_gate/up [D,H], dense_w_down [H,D] of dtype dt;
 * neuron_idx DEVICE int32 [E,d], each row strictly increasing in [0,D) (violations set
 * README_DEV_BAD_INDEX and the offending rows are zero-filled). Outputs w_gate/w_up [E,d,H],
 * w_down [E,H,d]. Bit copies. */
readme_status readme_build_experts(const void* dense_w_gate, const void* dense_w_up, const void* dense_w_down,
                                   readme_dtype dt, int32_t D, int32_t H, int32_t E, int32_t d,
                                   const int32_t* neuron_idx, void* w_gate, void* w_up, void* w_down,
                                   uint32_t* dev_status, readme_stream_t stream);

/* ---------------------------------------------------------------------------------------------- */
/* Host runtime: expert-aware batching (Alg. 1). Pre-gated tokens wait in one FIFO per
 * expert ("ReqQueueByExpert"); readme_scheduler_next_batch forms the next batch of at most
 * max_tokens by repeatedly taking the largest queue (ties -> lower id) whole while it fits, then a prefix of
 * the next largest to fill the batch, and stops (readings Q12: `k` at PAPER.md:250/:256-257 read as `E`;
 * stop when the largest queue is empty). token_ids/experts are HOST arrays of >= max_tokens entries; the
 * batch comes out grouped by expert in the order the queues were taken; returns its size (-1 on a bad
 * argument). Thread-safe (one mutex per scheduler). No GPU involved. */
typedef struct readme_scheduler readme_scheduler;
readme_scheduler* readme_scheduler_create(int32_t E); /* NULL if E is outside [1, 256] or out of memory */
void readme_scheduler_destroy(readme_scheduler* s);
readme_status readme_scheduler_push(readme_scheduler* s, const int64_t* token_ids, const int32_t* experts, int64_t n);
int64_t readme_scheduler_queued(readme_scheduler* s, int32_t e); /* e = -1: all queues */
int64_t readme_scheduler_next_batch(readme_scheduler* s, int64_t max_tokens, int64_t* token_ids, int32_t* experts);

/* Host runtime: the expert cache of the memory-constrained mode (§4.1). `capacity` slots;
 * policy 0 = LRU, 1 = Belady-inspired (evict argmax_{e in C} F(e,t), the resident whose next access after t
 * is farthest, never-again first; PAPER.md:208 — requires the pre-gated future reference string from
 * readme_cache_set_future), 2 = Random (seeded). Ties go to the lowest key (reading Q17). Keys are int64
 * (layer * E + expert). readme_cache_access returns 1 on a hit, 0 on a miss (the key is then resident, in the
 * slot of the evicted key if the cache was full; *evicted = that key or -1), -1 on a bad argument, -2 if the
 * cache is full of protected keys; *slot = the key's slot in [0, capacity). Residents last accessed at or
 * after `protect_since` are never evicted (the experts of the layer being assembled; pass INT64_MAX for none).
 * Host-only, thread-safe. */
typedef struct readme_expert_cache readme_expert_cache;
readme_expert_cache* readme_cache_create(int32_t capacity, int32_t policy, uint64_t seed);
void readme_cache_destroy(readme_expert_cache* c);
readme_status readme_cache_set_future(readme_expert_cache* c, const int64_t* keys, const int64_t* times, int64_t n);
int32_t readme_cache_access(readme_expert_cache* c, int64_t key, int64_t t, int64_t protect_since, int64_t* evicted,
                            int32_t* slot);
int32_t readme_cache_lookup(readme_expert_cache* c, int64_t key); /* slot or -1 */
void readme_cache_stats(readme_expert_cache* c, int64_t* hits, int64_t* misses);

/* ---------------------------------------------------------------------------------------------- */
/* Expert parallelism over peer memory (stretch C4). G <= README_EP_MAX_RANKS ranks, one
 * process per GPU, experts contiguous per rank (rank q owns [q*E/G, (q+1)*E/G)), tokens data-parallel.
 * Instead of NCCL all-to-alls, rows move by stores into the peer's memory: the dispatch kernel writes each
 * token row into the owning rank's receive buffer, and the down projection's epilogue writes each result
 * row back into its source rank's output (+ the source's residual) — the combine all-to-all fused into
 * the GEMM. Ranks order the phases with flag words (release/acquire at system scope). Because pre-gating
 * fixes every token's expert for all layers, counts are exchanged once per batch
 * (readme_ep_publish_counts + readme_ep_plan) and each layer is: readme_ep_dispatch, readme_ep_signal,
 * readme_ep_wait, readme_ep_expert_ffn, readme_ep_signal, readme_ep_wait (k == 1; for k > 1 the rows
 * return into the source's y_sorted and a local readme_combine follows). Nothing here synchronises the
 * host; every call is stream-ordered and graph-capturable.
 * Every buffer another rank writes or reads must come from readme_ep_alloc and be mapped into that rank with
 * readme_ipc_handle / readme_ipc_open (CUDA IPC; peer access enabled lazily). "peer_*" arguments are HOST
 * arrays of G DEVICE pointers, entry q = rank q's buffer as mapped in this process (entry me = own). */
#define README_EP_MAX_RANKS 8
#define README_IPC_HANDLE_BYTES 64
readme_status readme_ep_alloc(size_t bytes, void** ptr); /* zero-filled device memory on the current device */
readme_status readme_ep_free(void* ptr);
readme_status readme_ipc_handle(const void* ptr, void* handle); /* handle: README_IPC_HANDLE_BYTES host bytes */
/* readme_ipc_open maps a handle from another process; a buffer on another GPU that this one cannot reach by
 * peer access (cudaDeviceCanAccessPeer) is refused with README_ERR_UNSUPPORTED (nothing stays mapped). */
readme_status readme_ipc_open(const void* handle, void** ptr);
readme_status readme_ipc_close(void* ptr);
/* Phase flags: peer_flags[q] -> rank q's uint64 [G] flag array for this phase; epoch -> this rank's uint64
 * counter for the phase (device memory, zero-initialised, private to the rank). readme_ep_signal bumps
 * *epoch and sets peer_flags[q][me] = *epoch for every q (release, system scope) after all earlier work on
 * `stream`; readme_ep_wait blocks `stream` until flags[p] >= *epoch for every p (acquire), or sets
 * README_DEV_EP_TIMEOUT after ~10 s instead of hanging. The epoch is read on the device, so a CUDA graph
 * of a whole layer replays correctly. */
readme_status readme_ep_signal(uint64_t* const* peer_flags, int32_t G, int32_t me, uint64_t* epoch,
                               readme_stream_t stream);
readme_status readme_ep_wait(const uint64_t* flags, int32_t G, const uint64_t* epoch, uint32_t* dev_status,
                             readme_stream_t stream);
/* Once per batch: counts [E] (this rank's readme_route histogram) -> peer_tables[q][me*E + e] for every q
 * (each table int32 [G][E]); signal + wait, then readme_ep_plan turns the complete table into
 * seg_offsets [G*E/G + 1] (this rank's receive layout: segment (source p, local expert el), source-major, so
 * each expert's rows arrive in global token order — P12) and row_base [E] (where this rank's rows for
 * global expert e start in the owner's receive buffer). E % G == 0 required. */
readme_status readme_ep_publish_counts(const int32_t* counts, int32_t E, int32_t* const* peer_tables, int32_t G,
                                       int32_t me, readme_stream_t stream);
readme_status readme_ep_plan(const int32_t* table, int32_t G, int32_t E, int32_t me, int32_t* seg_offsets,
                             int32_t* row_base, readme_stream_t stream);
/* a5 fused with the dispatch all-to-all: slot s = t*k + j with sorted row r = dest[s] of expert e (offsets:
 * this rank's readme_route offsets [E+1]) is stored to rank q = e/(E/G) at row row_base[e] + r - offsets[e]
 * of peer_x[q] ([rows_cap, H] of dt), and peer_map[q][that row] = me*vrows + (to_token ? t : r): where the
 * result must return (to_token = 1 with vrows = T for k == 1; to_token = 0 with vrows = T*k for k > 1).
 * Out-of-range dest entries set README_DEV_BAD_INDEX and are skipped. */
readme_status readme_ep_dispatch(const void* x, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                                 const int32_t* dest, const int32_t* offsets, const int32_t* row_base, int32_t E,
                                 int32_t G, int32_t me, void* const* peer_x, int32_t* const* peer_map,
                                 int64_t vrows, int32_t to_token, uint32_t* dev_status, readme_stream_t stream);
/* a6 + a7 (+ a8) fused with the combine all-to-all (bf16): the grouped SwiGLU FFN over this rank's receive
 * buffer x_recv [rows_cap, H] (segments from seg_offsets [G*E_local+1], expert g % E_local), whose result
 * row r is stored to peer_out[p] + i*H (+ peer_res[p] + i*H when peer_res and its entry are non-NULL),
 * with v = row_map[r], p = v / vrows, i = v % vrows. Weights as readme_expert_ffn (E_local experts).
 * ws: readme_expert_ffn_workspace_bytes(rows_cap, H, E_local, d, dt). */
readme_status readme_ep_expert_ffn(const void* x_recv, readme_dtype dt, int64_t rows_cap, int32_t H,
                                   int32_t E_local, int32_t d, int32_t G, const int32_t* seg_offsets,
                                   const void* w_gate, const void* w_up, const void* w_down, const int32_t* row_map,
                                   void* const* peer_out, const void* const* peer_res, int64_t vrows,
                                   uint32_t* dev_status, void* ws, size_t ws_bytes, readme_stream_t stream);

/* Helpers. */
/* The library links its own (static) CUDA runtime: bind the calling host thread to `device` before
 * calling the entry points above from that thread (the Python binding does this per call). */
readme_status readme_set_device(int device);
const char* readme_status_string(readme_status s);
const char* readme_last_error(void); /* thread-local detail for the last non-OK return */
int readme_version(void);

/* Measurement only (not part of the hot-path contract): register a device buffer of 16 uint64 into which
   the dispatch, route and expert-FFN kernels record %globaltimer extremes, or NULL to stop. Slots: 0/1
   dispatch start (min) / end (max), 2 FFN past prologue (min), 3 first gate/up tile with its rows ready
   (min), 4 FFN end (max), 5/6 route start (min) / end (max). */
void readme_debug_trace(void* dev_buf);
/* Measurement only: store %globaltimer into slot `slot` (8..15) of the registered trace buffer from a
   one-thread kernel on `stream`. README_ERR_INVALID_ARG without a buffer or for another slot. */
readme_status readme_debug_mark(int32_t slot, readme_stream_t stream);
/* Lab / test switches that select measured-slower kernel variants for A/B measurement (DESIGN.md §6 lists
   every name, its values and its default). Each is read once from its README_* environment variable at the
   first launch; set_knob overrides it for the whole process (not thread-safe against running launches),
   reset_knob restores the environment's value. README_ERR_INVALID_ARG for an unknown name. */
readme_status readme_debug_set_knob(const char* name, int32_t value);
/* Test only: occupy n_ctas SMs (one CTA per SM, maximum shared memory) for ns nanoseconds on `stream`, so
   a kernel launched behind it on another stream finds only the remaining SMs (the co-residency tests of
   the single-launch expert FFN). */
readme_status readme_debug_hold_sms(int32_t n_ctas, int64_t ns, readme_stream_t stream);
readme_status readme_debug_get_knob(const char* name, int32_t* value);
readme_status readme_debug_reset_knob(const char* name);
/* Measurement only: register a device buffer of npairs * max_tiles * 8 uint64 into which the single-launch
   expert FFN records, for the first max_tiles tiles of every CTA pair (record [pair][i][0..7]): 0 %globaltimer
   when the MMA warp starts the tile, 1/2 its SM clock then and after issuing the tile's last MMA, 3/4 the
   clock when the leader's first epilogue warp sees the accumulator full / has stored it, 5 %globaltimer at
   that point, 6 the MMA warp's cycles waiting on loaded stages in the tile, 7 the tile index | (cycles the
   MMA warp waited for a free accumulator) << 32. NULL (or max_tiles <= 0) stops it. */
void readme_debug_tile_trace(void* dev_buf, int32_t max_tiles);

#ifdef __cplusplus
}
#endif
#endif /* README_B200_H_ */
