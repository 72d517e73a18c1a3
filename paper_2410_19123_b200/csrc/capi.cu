// capi.cu — the C ABI of libreadme_b200.so (include/readme.h): argument validation, workspace sizing
// and stream-ordered launches of the kernels in route.cu / permute.cu / ffn_*.cu. No allocation, no host
// synchronisation, no exception crosses the boundary.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <exception>
#include <mutex>

#include "kernels.h"

#define README_VERSION 1

namespace readme {

namespace {
thread_local char g_err[512] = {0};
}
uint64_t* g_trace_buf = nullptr;
uint64_t* g_tile_trace = nullptr;
int32_t g_tile_trace_max = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

readme_status cuda_fail(cudaError_t e, const char* where) {
  set_error("%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
  return README_ERR_CUDA;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

namespace {

readme_status check_route_args(int64_t T, int32_t E, int32_t k) {
  README_CHECK_ARG(T >= 0, "T must be >= 0 (got %lld)", static_cast<long long>(T));
  README_CHECK_ARG(E >= 1 && E <= README_MAX_EXPERTS, "E must be in [1, %d] (got %d)", README_MAX_EXPERTS, E);
  README_CHECK_ARG(k >= 1 && k <= E, "k must be in [1, E] (got k=%d, E=%d)", k, E);
  README_CHECK_ARG(T * static_cast<int64_t>(k) < (int64_t(1) << 31), "T*k must be < 2^31");
  return README_OK;
}

readme_status check_rows(readme_dtype dt, int32_t H) {
  if (dt != README_F32 && dt != README_BF16) {
    set_error("unknown dtype %d", static_cast<int>(dt));
    return README_ERR_UNSUPPORTED;
  }
  README_CHECK_ARG(H >= 8 && H % 8 == 0, "H must be a positive multiple of 8 (got %d)", H);
  return README_OK;
}


// expert-FFN workspace: h [rows, d] then the merged kernel's readiness counters (sized for 512 segments)
size_t ffn_h_bytes(int64_t rows, int32_t d, readme_dtype dt) {
  return align_up(static_cast<size_t>(rows) * d * dt_size(dt), 256);
}
size_t ffn_ws_bytes(int64_t rows, int32_t d, readme_dtype dt) {
  return ffn_h_bytes(rows, d, dt) + ffn_layer_ready_bytes(rows, 512) + 256;
}

// Which bf16 kernel family runs the expert FFN: the single-launch CTA-pair kernel by default; knob
// ffn_kernel = 1 (split: two CTA-pair launches) or 2 (unfused: split, and no fused combine in
// readme_moe_layer) for A/B measurement.
enum class FfnPath { kMerged, kSplit, kUnfused };
FfnPath ffn_path() {
  const int v = knob(Knob::kFfnKernel);
  return v == 1 ? FfnPath::kSplit : (v == 2 ? FfnPath::kUnfused : FfnPath::kMerged);
}

// a6 + a7 (+ fused a8 when src != null) over the workspace `ws` (ffn_ws_bytes).
// Whether the single-launch kernel runs (and may be launched as a programmatic dependent of the dispatch:
// the caller then zeroes its readiness counters with zero_ready() BEFORE the dispatch, not between).
bool merged_ffn(readme_dtype dt) { return dt == README_BF16 && ffn_path() == FfnPath::kMerged; }
readme_status zero_ready(void* ws, int64_t rows, int32_t d, readme_dtype dt, int32_t nseg, cudaStream_t st) {
  README_CUDA(cudaMemsetAsync(static_cast<char*>(ws) + ffn_h_bytes(rows, d, dt), 0, ffn_layer_ready_bytes(rows, nseg),
                              st));
  return README_OK;
}

// Whether the dispatch runs in gather form with per-row readiness flags (the FFN starting before it ends) or
// in scatter form behind the FFN's whole-grid PDL wait. The gather form only overlaps while the FFN's CTAs
// can be resident beside the dispatch's: with the FFN at 255 registers per thread (merged tails, dynamic tile
// order) two of its warps fill an SM sub-partition's register file, so the FFN started only once the gather
// kernel had ended; run inside the FFN launch instead (its epilogue warps gather the rows before their first
// tile) the dispatch's traffic slowed the first tiles more than it saved. A/B on one box (bench.py, r02):
// config 2 step 0.777 ms scatter / 0.786-0.789 fused / 0.796 gather kernel; config 4 58.05 / - / 58.85 ms.
// The in-FFN gather was then paced (rows of the next segment copied while an epilogue warp waits for an
// accumulator; one copied-row counter per segment instead of per-row flags): config 2 step 0.785-0.786 ms vs
// 0.783-0.787 scatter on one box — level, not better. So the default stays scatter; knob dispatch = 2 (gather
// kernel) | 3 (gather inside the FFN) | 1 (scatter).
bool gather_dispatch(int64_t rows) {
  (void)rows;
  return knob(Knob::kDispatch) >= 2;
}
bool fused_gather_dispatch() { return knob(Knob::kDispatch) != 2; }

// x_sorted row flags inside the FFN workspace (see ffn_layer_ready_bytes)
uint32_t* ffn_xready(void* ws, int64_t rows, int32_t d, readme_dtype dt) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + ffn_h_bytes(rows, d, dt) + ffn_layer_xready_offset(rows));
}

readme_status run_ffn(const void* x_sorted, readme_dtype dt, int64_t rows, int32_t H, int32_t E, int32_t d,
                      int32_t n_src, const int32_t* offsets, const void* w_gate, const void* w_up,
                      const void* w_down, const int32_t* src, const void* residual, void* out, void* ws,
                      uint32_t* dev_status, cudaStream_t st, bool pdl = false, bool xready = false,
                      const SelfDispatch* sd = nullptr) {
  readme_stream_t stream = reinterpret_cast<readme_stream_t>(st);
  if (merged_ffn(dt)) {
    uint32_t* ready = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + ffn_h_bytes(rows, d, dt));
    return launch_ffn_layer_2cta(static_cast<const __nv_bfloat16*>(x_sorted), rows, H, E, d, n_src * E, offsets,
                                 static_cast<const __nv_bfloat16*>(w_gate), static_cast<const __nv_bfloat16*>(w_up),
                                 static_cast<const __nv_bfloat16*>(w_down), static_cast<__nv_bfloat16*>(ws),
                                 static_cast<__nv_bfloat16*>(out), src,
                                 static_cast<const __nv_bfloat16*>(residual), ready, dev_status, st, nullptr, 0,
                                 nullptr, pdl, xready ? ffn_xready(ws, rows, d, dt) : nullptr, sd);
  }
  if (dt == README_F32 && ffn_f32_fusable(H, d))  // small fp32 layers: a6 + a7 in one launch, h in shared memory
    return launch_ffn_f32_fused(static_cast<const float*>(x_sorted), nullptr, nullptr, 1, rows, H, E, d, n_src * E,
                                offsets, static_cast<const float*>(w_gate), static_cast<const float*>(w_up),
                                static_cast<const float*>(w_down), static_cast<float*>(out), src,
                                static_cast<const float*>(residual), st);
  README_TRY(readme_expert_gate_up(x_sorted, dt, rows, H, E, d, n_src, offsets, w_gate, w_up, ws, stream));
  return readme_expert_down(ws, dt, rows, H, E, d, n_src, offsets, w_down, src, residual, out, stream);
}


}  // namespace
}  // namespace readme

using namespace readme;

#pragma GCC visibility push(default)
extern "C" {

const char* readme_status_string(readme_status s) {
  switch (s) {
    case README_OK: return "README_OK";
    case README_ERR_INVALID_ARG: return "README_ERR_INVALID_ARG";
    case README_ERR_UNSUPPORTED: return "README_ERR_UNSUPPORTED";
    case README_ERR_WORKSPACE: return "README_ERR_WORKSPACE";
    case README_ERR_CUDA: return "README_ERR_CUDA";
  }
  return "README_ERR_UNKNOWN";
}

const char* readme_last_error(void) { return g_err; }

int readme_version(void) { return README_VERSION; }

// Measurement only: register (or clear, with NULL) a device buffer of 16 uint64 the hot-path kernels
// record %globaltimer extremes into: [0] dispatch first CTA start (min), [1] dispatch last CTA end (max),
// [2] expert FFN first CTA past its prologue (min), [3] first gate/up tile whose rows were ready (min),
// [4] expert FFN last CTA end (max), [5] route start (min), [6] route end (max). The caller initialises
// min slots to ~0 and max slots to 0. Not thread-safe; not for production use.
void readme_debug_trace(void* dev_buf) { g_trace_buf = static_cast<uint64_t*>(dev_buf); }

// Measurement only: per-tile records of the single-launch expert FFN (layout in include/readme.h).
void readme_debug_tile_trace(void* dev_buf, int32_t max_tiles) {
  g_tile_trace = max_tiles > 0 ? static_cast<uint64_t*>(dev_buf) : nullptr;
  g_tile_trace_max = max_tiles > 0 ? max_tiles : 0;
}

// Measurement only: a one-thread kernel that stores %globaltimer into slot `slot` (8..15) of the registered
// trace buffer, stream-ordered (marks where a timed region starts / ends on the device clock).
readme_status readme_debug_mark(int32_t slot, readme_stream_t stream) {
  README_CHECK_ARG(g_trace_buf != nullptr && slot >= 8 && slot < 16, "no trace buffer, or slot not in [8, 16)");
  return launch_debug_mark(g_trace_buf + slot, reinterpret_cast<cudaStream_t>(stream));
}

// Test only: hold n_ctas SMs (one CTA each, maximum shared memory) for ns nanoseconds on `stream`.
readme_status readme_debug_hold_sms(int32_t n_ctas, int64_t ns, readme_stream_t stream) {
  README_CHECK_ARG(n_ctas >= 1 && n_ctas <= 4096 && ns >= 0 && ns <= 60000000000LL, "n_ctas in [1, 4096], ns in [0, 60 s]");
  return launch_debug_hold_sms(n_ctas, ns, reinterpret_cast<cudaStream_t>(stream));
}

readme_status readme_set_device(int device) {
  int cur = -1;
  if (cudaGetDevice(&cur) == cudaSuccess && cur == device) return README_OK;
  README_CUDA(cudaSetDevice(device));
  return README_OK;
}

size_t readme_route_workspace_bytes(int64_t T, int32_t E, int32_t k) { return route_ws_bytes(T, E, k); }

namespace readme {
namespace {
readme_status check_route_call(const void* logits, readme_dtype logits_dt, int64_t T, int32_t E, int32_t k,
                               int32_t* topk_idx, float* topk_w, int32_t* counts, int32_t* offsets, int32_t* dest,
                               void* ws, size_t ws_bytes) {
  README_TRY(check_route_args(T, E, k));
  README_CHECK_ARG(counts && offsets, "counts and offsets are required");
  if (T > 0) {
    README_CHECK_ARG(logits && topk_idx && topk_w && dest, "logits, topk_idx, topk_w, dest are required");
    README_CHECK_ARG(logits_dt == README_F32 || logits_dt == README_BF16, "logits_dt must be F32 or BF16");
    README_CHECK_ARG(ws != nullptr, "workspace is required");
    if (ws_bytes < route_ws_bytes(T, E, k)) {
      set_error("route workspace too small: %zu < %zu", ws_bytes, route_ws_bytes(T, E, k));
      return README_ERR_WORKSPACE;
    }
  }
  return README_OK;
}
}  // namespace
}  // namespace readme

readme_status readme_route(const void* logits, readme_dtype logits_dt, int64_t T, int32_t E, int32_t k,
                           int32_t* topk_idx, float* topk_w, int32_t* counts, int32_t* offsets, int32_t* dest,
                           int32_t* src, uint32_t* dev_status, void* ws, size_t ws_bytes,
                           readme_stream_t stream) {
  try {
    README_TRY(check_route_call(logits, logits_dt, T, E, k, topk_idx, topk_w, counts, offsets, dest, ws, ws_bytes));
    return launch_route(logits, logits_dt, T, E, k, topk_idx, topk_w, counts, offsets, dest, src, dev_status, ws,
                        reinterpret_cast<cudaStream_t>(stream));
  } catch (const std::exception& e) {
    set_error("exception: %s", e.what());
    return README_ERR_CUDA;
  } catch (...) {
    set_error("unknown exception");
    return README_ERR_CUDA;
  }
}

readme_status readme_dispatch(const void* x, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                              const int32_t* dest, void* x_sorted, uint32_t* dev_status, readme_stream_t stream) {
  README_TRY(check_rows(dt, H));
  README_CHECK_ARG(T >= 0 && k >= 1 && T * static_cast<int64_t>(k) < (int64_t(1) << 31), "bad T/k");
  if (T == 0) return README_OK;
  README_CHECK_ARG(x && dest && x_sorted, "x, dest and x_sorted are required");
  README_CHECK_ARG(aligned16(x) && aligned16(x_sorted), "x and x_sorted must be 16-byte aligned");
  return launch_dispatch(x, static_cast<size_t>(H) * dt_size(dt), T, k, dest, x_sorted, dev_status,
                         reinterpret_cast<cudaStream_t>(stream));
}

size_t readme_expert_ffn_workspace_bytes(int64_t rows, int32_t H, int32_t E, int32_t d, readme_dtype dt) {
  (void)H;
  (void)E;
  return ffn_ws_bytes(rows < 0 ? 0 : rows, d < 0 ? 0 : d, dt);
}

namespace {
readme_status check_ffn_args(readme_dtype dt, int64_t rows, int32_t H, int32_t E, int32_t d, int32_t n_src,
                             const int32_t* offsets) {
  README_TRY(check_rows(dt, H));
  README_CHECK_ARG(rows >= 0 && rows < (int64_t(1) << 31), "rows out of range");
  README_CHECK_ARG(E >= 1 && E <= README_MAX_EXPERTS, "E must be in [1, %d]", README_MAX_EXPERTS);
  README_CHECK_ARG(n_src >= 1 && static_cast<int64_t>(n_src) * E <= 512, "n_src*E must be in [1, 512]");
  README_CHECK_ARG(d >= 8 && d % 8 == 0, "d must be a positive multiple of 8 (got %d)", d);
  README_CHECK_ARG(offsets != nullptr, "offsets are required");
  return README_OK;
}
}  // namespace

readme_status readme_expert_gate_up(const void* x_sorted, readme_dtype dt, int64_t rows, int32_t H, int32_t E,
                                    int32_t d, int32_t n_src, const int32_t* offsets, const void* w_gate,
                                    const void* w_up, void* h, readme_stream_t stream) {
  README_TRY(check_ffn_args(dt, rows, H, E, d, n_src, offsets));
  if (rows == 0) return README_OK;
  README_CHECK_ARG(x_sorted && w_gate && w_up && h, "null pointer argument");
  README_CHECK_ARG(aligned16(x_sorted) && aligned16(w_gate) && aligned16(w_up) && aligned16(h),
                   "all tensors must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dt == README_BF16)
    return launch_gate_up_bf16(static_cast<const __nv_bfloat16*>(x_sorted), rows, H, E, d, n_src * E, offsets,
                               static_cast<const __nv_bfloat16*>(w_gate), static_cast<const __nv_bfloat16*>(w_up),
                               static_cast<__nv_bfloat16*>(h), st);
  return launch_gate_up_f32(static_cast<const float*>(x_sorted), rows, H, E, d, n_src * E, offsets,
                            static_cast<const float*>(w_gate), static_cast<const float*>(w_up),
                            static_cast<float*>(h), st);
}

readme_status readme_expert_down(const void* h, readme_dtype dt, int64_t rows, int32_t H, int32_t E, int32_t d,
                                 int32_t n_src, const int32_t* offsets, const void* w_down, const int32_t* src,
                                 const void* residual, void* out, readme_stream_t stream) {
  README_TRY(check_ffn_args(dt, rows, H, E, d, n_src, offsets));
  if (rows == 0) return README_OK;
  README_CHECK_ARG(h && w_down && out, "null pointer argument");
  README_CHECK_ARG(aligned16(h) && aligned16(w_down) && aligned16(out) && (!residual || aligned16(residual)),
                   "all tensors must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dt == README_BF16)
    return launch_down_bf16(static_cast<const __nv_bfloat16*>(h), rows, H, E, d, n_src * E, offsets,
                            static_cast<const __nv_bfloat16*>(w_down), static_cast<__nv_bfloat16*>(out), src,
                            static_cast<const __nv_bfloat16*>(residual), st);
  return launch_down_f32(static_cast<const float*>(h), rows, H, E, d, n_src * E, offsets,
                         static_cast<const float*>(w_down), static_cast<float*>(out), src,
                         static_cast<const float*>(residual), st);
}

readme_status readme_expert_ffn(const void* x_sorted, readme_dtype dt, int64_t rows, int32_t H, int32_t E,
                                int32_t d, int32_t n_src, const int32_t* offsets, const void* w_gate,
                                const void* w_up, const void* w_down, void* y_sorted, uint32_t* dev_status, void* ws,
                                size_t ws_bytes, readme_stream_t stream) {
  README_TRY(check_ffn_args(dt, rows, H, E, d, n_src, offsets));
  if (rows == 0) return README_OK;
  README_CHECK_ARG(ws != nullptr && aligned16(ws), "workspace is required (16-byte aligned)");
  if (ws_bytes < ffn_ws_bytes(rows, d, dt)) {
    set_error("expert_ffn workspace too small: %zu < %zu", ws_bytes, ffn_ws_bytes(rows, d, dt));
    return README_ERR_WORKSPACE;
  }
  README_CHECK_ARG(x_sorted && w_gate && w_up && w_down && y_sorted, "null pointer argument");
  README_CHECK_ARG(aligned16(x_sorted) && aligned16(w_gate) && aligned16(w_up) && aligned16(w_down) &&
                       aligned16(y_sorted),
                   "all tensors must be 16-byte aligned");
  return run_ffn(x_sorted, dt, rows, H, E, d, n_src, offsets, w_gate, w_up, w_down, nullptr, nullptr, y_sorted, ws,
                 dev_status, reinterpret_cast<cudaStream_t>(stream));
}



readme_status readme_expert_ffn_slots(const void* x_sorted, readme_dtype dt, int64_t rows, int32_t H, int32_t E,
                                      int32_t d, const int32_t* offsets, const int32_t* expert_slot, int32_t n_slots,
                                      const void* w_gate, const void* w_up, const void* w_down, const int32_t* src,
                                      const void* residual, void* out, uint32_t* dev_status, void* ws,
                                      size_t ws_bytes, readme_stream_t stream) {
  README_TRY(check_ffn_args(dt, rows, H, E, d, 1, offsets));
  if (dt != README_BF16) {
    set_error("readme_expert_ffn_slots is bf16-only");
    return README_ERR_UNSUPPORTED;
  }
  README_CHECK_ARG(expert_slot != nullptr && n_slots >= 1, "expert_slot and n_slots >= 1 are required");
  if (rows == 0) return README_OK;
  README_CHECK_ARG(x_sorted && w_gate && w_up && w_down && out && ws, "null pointer argument");
  README_CHECK_ARG(aligned16(x_sorted) && aligned16(w_gate) && aligned16(w_up) && aligned16(w_down) &&
                       aligned16(out) && aligned16(ws) && (!residual || aligned16(residual)),
                   "all tensors must be 16-byte aligned");
  if (ws_bytes < ffn_ws_bytes(rows, d, dt)) {
    set_error("expert_ffn_slots workspace too small: %zu < %zu", ws_bytes, ffn_ws_bytes(rows, d, dt));
    return README_ERR_WORKSPACE;
  }
  uint32_t* ready = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + ffn_h_bytes(rows, d, dt));
  return launch_ffn_layer_2cta(static_cast<const __nv_bfloat16*>(x_sorted), rows, H, E, d, E, offsets,
                               static_cast<const __nv_bfloat16*>(w_gate), static_cast<const __nv_bfloat16*>(w_up),
                               static_cast<const __nv_bfloat16*>(w_down), static_cast<__nv_bfloat16*>(ws),
                               static_cast<__nv_bfloat16*>(out), src, static_cast<const __nv_bfloat16*>(residual),
                               ready, dev_status, reinterpret_cast<cudaStream_t>(stream), expert_slot, n_slots);
}

readme_status readme_combine(const void* y_sorted, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                             const int32_t* dest, const float* topk_w, const void* residual, void* y,
                             uint32_t* dev_status, readme_stream_t stream) {
  README_TRY(check_rows(dt, H));
  README_CHECK_ARG(T >= 0 && k >= 1 && T * static_cast<int64_t>(k) < (int64_t(1) << 31), "bad T/k");
  if (T == 0) return README_OK;
  README_CHECK_ARG(y_sorted && dest && y, "y_sorted, dest and y are required");
  README_CHECK_ARG(k == 1 || topk_w, "topk_w is required when k > 1");
  README_CHECK_ARG(aligned16(y_sorted) && aligned16(y) && (!residual || aligned16(residual)),
                   "tensors must be 16-byte aligned");
  return launch_combine(y_sorted, dt, T, H, k, dest, topk_w, residual, y, dev_status,
                        reinterpret_cast<cudaStream_t>(stream));
}

size_t readme_moe_layer_workspace_bytes(int64_t T, int32_t H, int32_t E, int32_t d, int32_t k, readme_dtype dt) {
  if (T < 0 || k < 1 || H < 0) return 0;
  const int64_t rows = T * k;
  const size_t act = align_up(static_cast<size_t>(rows) * H * dt_size(dt), 256);
  return align_up(route_ws_bytes(T, E, k), 256) + 2 * act + ffn_ws_bytes(rows, d, dt) +
         align_up(static_cast<size_t>(rows) * sizeof(int32_t), 256);
}

readme_status readme_moe_layer(const void* x, readme_dtype dt, int64_t T, int32_t H, const void* logits,
                               readme_dtype logits_dt, int32_t E, int32_t k, int32_t d, const void* w_gate,
                               const void* w_up, const void* w_down, const void* residual, void* y,
                               int32_t* topk_idx, float* topk_w, int32_t* counts, int32_t* offsets,
                               int32_t* dest, int32_t* src, uint32_t* dev_status, void* ws, size_t ws_bytes,
                               readme_stream_t stream) {
  README_TRY(check_route_args(T, E, k));
  README_TRY(check_rows(dt, H));
  README_CHECK_ARG(d >= 8 && d % 8 == 0, "d must be a positive multiple of 8 (got %d)", d);
  README_CHECK_ARG(counts && offsets, "counts and offsets are required");
  if (T == 0) {
    if (logits) return readme_route(nullptr, logits_dt, 0, E, k, nullptr, nullptr, counts, offsets, nullptr,
                                    nullptr, dev_status, ws, ws_bytes, stream);
    return README_OK;
  }
  README_CHECK_ARG(x && y && topk_idx && topk_w && dest && w_gate && w_up && w_down && ws,
                   "null pointer argument");
  const size_t need = readme_moe_layer_workspace_bytes(T, H, E, d, k, dt);
  if (ws_bytes < need) {
    set_error("moe_layer workspace too small: %zu < %zu", ws_bytes, need);
    return README_ERR_WORKSPACE;
  }
  const int64_t rows = T * k;
  char* w = static_cast<char*>(ws);
  void* ws_route = w;
  w += align_up(route_ws_bytes(T, E, k), 256);
  void* x_sorted = w;
  w += align_up(static_cast<size_t>(rows) * H * dt_size(dt), 256);
  void* y_sorted = w;
  w += align_up(static_cast<size_t>(rows) * H * dt_size(dt), 256);
  void* ws_ffn = w;
  w += ffn_ws_bytes(rows, d, dt);
  int32_t* src_ws = reinterpret_cast<int32_t*>(w);
  const FfnPath path = ffn_path();
  const bool fused = k == 1 && (src != nullptr || logits != nullptr) && path != FfnPath::kUnfused;
  // the single-launch FFN follows the dispatch as a programmatic dependent (PDL), fused combine or not
  const bool pdl = merged_ffn(dt);
  // every argument check precedes the first launch: an error return leaves no partial step behind
  README_CHECK_ARG(aligned16(x) && aligned16(w_gate) && aligned16(w_up) && aligned16(w_down) && aligned16(y) &&
                       (!residual || aligned16(residual)),
                   "x, weights, residual and y must be 16-byte aligned");
  bool xready = false;
  SelfDispatch sd_store{};
  const SelfDispatch* sd = nullptr;  // a5 inside the FFN launch
  if (logits) {
    if (!src) src = src_ws;  // the fused path needs the inverse permutation
    README_TRY(check_route_call(logits, logits_dt, T, E, k, topk_idx, topk_w, counts, offsets, dest, ws_route,
                                route_ws_bytes(T, E, k)));
    README_CHECK_ARG(aligned16(x) && aligned16(x_sorted), "x must be 16-byte aligned");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (route_is_single_launch(T, k)) {
      // a1-a4 in one cluster launch (dest and src final), which also zeroes the FFN's readiness region (no
      // memset node). Large batches: a5 in gather form publishing per-row flags, the fused FFN behind it
      // (PDL) starting each gate/up tile as soon as its rows have landed; small batches: scatter form.
      // (Running a5 inside the route launch for small batches, with the FFN as the route's programmatic
      // dependent, measured no faster: the <= 16-CTA cluster copies 2 MB in ~4.5 us.)
      uint32_t* ready = pdl ? reinterpret_cast<uint32_t*>(static_cast<char*>(ws_ffn) + ffn_h_bytes(rows, d, dt))
                            : nullptr;
      const int64_t ready_words = pdl ? static_cast<int64_t>(ffn_layer_ready_bytes(rows, E) / 4) : 0;
      xready = pdl && gather_dispatch(rows);
      README_TRY(launch_route(logits, logits_dt, T, E, k, topk_idx, topk_w, counts, offsets, dest, src, dev_status,
                              ws_route, st, true, ready, ready_words));
      if (fused && dt == README_F32 && ffn_f32_fusable(H, d)) {
        // small fp32 layer: a5 as a row gather inside the one-launch FFN (x[src[r] / k]), a8 in its epilogue
        return launch_ffn_f32_fused(nullptr, static_cast<const float*>(x), src, k, rows, H, E, d, E, offsets,
                                    static_cast<const float*>(w_gate), static_cast<const float*>(w_up),
                                    static_cast<const float*>(w_down), static_cast<float*>(y), src,
                                    static_cast<const float*>(residual), st);
      }
      if (xready && fused_gather_dispatch()) {
        sd_store = SelfDispatch{static_cast<const __nv_bfloat16*>(x), src, k};
        sd = &sd_store;
      } else if (xready)
        README_TRY(launch_dispatch_gather(x, static_cast<size_t>(H) * dt_size(dt), rows, k, src, x_sorted,
                                          ffn_xready(ws_ffn, rows, d, dt), dev_status, st));
      else
        README_TRY(launch_dispatch(x, static_cast<size_t>(H) * dt_size(dt), T, k, dest, x_sorted, dev_status, st));
    } else {
      if (pdl) README_TRY(zero_ready(ws_ffn, rows, d, dt, E, st));
      // a1-a4 with the finalize (offsets[e] + rank, src) fused into the a5 dispatch pass
      README_TRY(launch_route(logits, logits_dt, T, E, k, topk_idx, topk_w, counts, offsets, dest, src, dev_status,
                              ws_route, st, /*finalize=*/false));
      README_TRY(launch_finalize_dispatch(x, static_cast<size_t>(H) * dt_size(dt), T, k, E, topk_idx, offsets, dest,
                                          src, x_sorted, st));
    }
  } else {
    if (pdl) README_TRY(zero_ready(ws_ffn, rows, d, dt, E, reinterpret_cast<cudaStream_t>(stream)));
    README_TRY(readme_dispatch(x, dt, T, H, k, dest, x_sorted, dev_status, stream));
  }
  if (fused) {
    // a6, then a7 with a8 fused into its epilogue: y[src[r]] = residual + h_r W_down^T (k == 1, weight 1).
    return run_ffn(x_sorted, dt, rows, H, E, d, 1, offsets, w_gate, w_up, w_down, src, residual, y, ws_ffn,
                   dev_status, reinterpret_cast<cudaStream_t>(stream), pdl, xready, sd);
  }
  if (pdl) {
    README_TRY(run_ffn(x_sorted, dt, rows, H, E, d, 1, offsets, w_gate, w_up, w_down, nullptr, nullptr, y_sorted,
                       ws_ffn, dev_status, reinterpret_cast<cudaStream_t>(stream), true, xready, sd));
  } else {
    README_TRY(readme_expert_ffn(x_sorted, dt, rows, H, E, d, 1, offsets, w_gate, w_up, w_down, y_sorted,
                                 dev_status, ws_ffn, ffn_ws_bytes(rows, d, dt), stream));
  }
  return readme_combine(y_sorted, dt, T, H, k, dest, topk_w, residual, y, dev_status, stream);
}

readme_status readme_dispatch_rmsnorm(const void* x, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                                      const int32_t* dest, float eps, void* x_sorted, uint32_t* dev_status,
                                      readme_stream_t stream) {
  README_TRY(check_rows(dt, H));
  README_CHECK_ARG(T >= 0 && k >= 1 && T * static_cast<int64_t>(k) < (int64_t(1) << 31), "bad T/k");
  README_CHECK_ARG(eps >= 0.f, "eps must be >= 0");
  if (T == 0) return README_OK;
  README_CHECK_ARG(x && dest && x_sorted, "x, dest and x_sorted are required");
  README_CHECK_ARG(aligned16(x) && aligned16(x_sorted), "x and x_sorted must be 16-byte aligned");
  return launch_dispatch_rmsnorm(x, dt, T, H, k, dest, eps, x_sorted, dev_status,
                                 reinterpret_cast<cudaStream_t>(stream));
}

size_t readme_moe_stack_workspace_bytes(int64_t T, int32_t H, int32_t E, int32_t d, int32_t k, readme_dtype dt) {
  return readme_moe_layer_workspace_bytes(T, H, E, d, k, dt);
}

readme_status readme_moe_stack(void* x, readme_dtype dt, int64_t T, int32_t H, const void* logits,
                               readme_dtype logits_dt, int32_t E, int32_t k, int32_t d, int32_t L,
                               const void* const* w_gate, const void* const* w_up, const void* const* w_down,
                               float eps, int32_t* topk_idx, float* topk_w, int32_t* counts, int32_t* offsets,
                               int32_t* dest, int32_t* src, uint32_t* dev_status, void* ws, size_t ws_bytes,
                               readme_stream_t stream) {
  README_TRY(check_route_args(T, E, k));
  README_TRY(check_rows(dt, H));
  README_CHECK_ARG(d >= 8 && d % 8 == 0, "d must be a positive multiple of 8 (got %d)", d);
  README_CHECK_ARG(L >= 0, "L must be >= 0");
  README_CHECK_ARG(counts && offsets, "counts and offsets are required");
  if (T == 0) {
    if (logits) return readme_route(nullptr, logits_dt, 0, E, k, nullptr, nullptr, counts, offsets, nullptr, nullptr,
                                    dev_status, ws, ws_bytes, stream);
    return README_OK;
  }
  README_CHECK_ARG(x && topk_idx && topk_w && dest && ws && (L == 0 || (w_gate && w_up && w_down)),
                   "null pointer argument");
  const size_t need = readme_moe_stack_workspace_bytes(T, H, E, d, k, dt);
  if (ws_bytes < need) {
    set_error("moe_stack workspace too small: %zu < %zu", ws_bytes, need);
    return README_ERR_WORKSPACE;
  }
  const int64_t rows = T * k;
  char* w = static_cast<char*>(ws);
  void* ws_route = w;
  w += align_up(route_ws_bytes(T, E, k), 256);
  void* x_sorted = w;
  w += align_up(static_cast<size_t>(rows) * H * dt_size(dt), 256);
  void* y_sorted = w;
  w += align_up(static_cast<size_t>(rows) * H * dt_size(dt), 256);
  void* h = w;
  w += ffn_ws_bytes(rows, d, dt);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // every argument check precedes the first launch (x is updated in place: no partial stack on an error)
  README_CHECK_ARG(aligned16(x), "x must be 16-byte aligned");
  for (int32_t l = 0; l < L; ++l) {
    README_CHECK_ARG(w_gate[l] && w_up[l] && w_down[l], "layer %d: null weight pointer", l);
    README_CHECK_ARG(aligned16(w_gate[l]) && aligned16(w_up[l]) && aligned16(w_down[l]),
                     "layer %d: weights must be 16-byte aligned", l);
  }
  if (logits)
    README_TRY(check_route_call(logits, logits_dt, T, E, k, topk_idx, topk_w, counts, offsets, dest, ws_route,
                                route_ws_bytes(T, E, k)));
  const bool own_src = src == nullptr;
  if (own_src) src = reinterpret_cast<int32_t*>(w);
  // a1-a4 once for the whole stack: the router does not depend on the layer.
  if (logits)
    README_TRY(readme_route(logits, logits_dt, T, E, k, topk_idx, topk_w, counts, offsets, dest, src, dev_status,
                            ws_route, route_ws_bytes(T, E, k), stream));
  else if (own_src)
    README_TRY(launch_invert_perm(dest, rows, src, st));  // plan-in with dest only
  const bool pdl = k == 1 && merged_ffn(dt);
  for (int32_t l = 0; l < L; ++l) {
    if (pdl && gather_dispatch(rows)) {
      // pre-norm dispatch in gather form with per-row flags; the FFN behind it starts tiles as rows land
      README_TRY(zero_ready(h, rows, d, dt, E, st));
      README_TRY(launch_dispatch_rmsnorm_gather(x, dt, rows, H, k, src, eps, x_sorted, ffn_xready(h, rows, d, dt),
                                                dev_status, st));
      README_TRY(run_ffn(x_sorted, dt, rows, H, E, d, 1, offsets, w_gate[l], w_up[l], w_down[l], src, x, x, h,
                         dev_status, st, true, true));
      continue;
    }
    if (pdl) README_TRY(zero_ready(h, rows, d, dt, E, st));  // before the dispatch (see zero_ready)
    README_TRY(readme_dispatch_rmsnorm(x, dt, T, H, k, dest, eps, x_sorted, dev_status, stream));
    if (k == 1) {  // x <- x + MoE(RMSNorm(x)): the residual add is fused into the down epilogue, in place
      README_TRY(run_ffn(x_sorted, dt, rows, H, E, d, 1, offsets, w_gate[l], w_up[l], w_down[l], src, x, x, h,
                         dev_status, reinterpret_cast<cudaStream_t>(stream), pdl));
    } else {
      README_TRY(run_ffn(x_sorted, dt, rows, H, E, d, 1, offsets, w_gate[l], w_up[l], w_down[l], nullptr, nullptr,
                         y_sorted, h, dev_status, reinterpret_cast<cudaStream_t>(stream)));
      README_TRY(readme_combine(y_sorted, dt, T, H, k, dest, topk_w, x, x, dev_status, stream));
    }
  }
  return README_OK;
}

readme_status readme_permanent_expert(const void* x, readme_dtype dt, int64_t T, int32_t H, int32_t d_perm,
                                      const void* w_gate, const void* w_up, const void* w_down, void* y,
                                      uint32_t* dev_status, void* ws, size_t ws_bytes, readme_stream_t stream) {
  README_TRY(check_rows(dt, H));
  README_CHECK_ARG(T >= 0 && T < (int64_t(1) << 31), "T out of range");
  README_CHECK_ARG(d_perm >= 8 && d_perm % 8 == 0, "d_perm must be a positive multiple of 8 (got %d)", d_perm);
  if (T == 0) return README_OK;
  README_CHECK_ARG(x && w_gate && w_up && w_down && y && ws, "null pointer argument");
  README_CHECK_ARG(aligned16(x) && aligned16(w_gate) && aligned16(w_up) && aligned16(w_down) && aligned16(y) &&
                       aligned16(ws),
                   "all tensors must be 16-byte aligned");
  const size_t need = readme_permanent_expert_workspace_bytes(T, H, d_perm, dt);
  if (ws_bytes < need) {
    set_error("permanent_expert workspace too small: %zu < %zu", ws_bytes, need);
    return README_ERR_WORKSPACE;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // one segment covering every token in token order: offsets = {0, T} (kept at the front of ws)
  int32_t* offs = static_cast<int32_t*>(ws);
  README_TRY(launch_set_offsets(offs, static_cast<int32_t>(T), st));
  void* ws_ffn = static_cast<char*>(ws) + 256;
  // y <- y + F_perm(x): the down projection adds the residual y in its epilogue, in place (identity rows)
  return run_ffn(x, dt, T, H, 1, d_perm, 1, offs, w_gate, w_up, w_down, nullptr, y, y, ws_ffn, dev_status, st);
}

size_t readme_permanent_expert_workspace_bytes(int64_t T, int32_t H, int32_t d_perm, readme_dtype dt) {
  (void)H;
  return 256 + ffn_ws_bytes(T < 0 ? 0 : T, d_perm < 0 ? 0 : d_perm, dt);
}

size_t readme_router_workspace_bytes(int64_t T, int32_t nseq) {
  return router_ws_bytes(T < 0 ? 0 : T, nseq < 1 ? 1 : nseq);
}

namespace {
readme_status check_router_weights(const readme_router_weights* w, float eps, RouterWeights* rw) {
  README_CHECK_ARG(w != nullptr, "weights are required");
  README_CHECK_ARG(w->vocab >= 1, "vocab must be >= 1");
  if (w->n_experts < 1 || w->n_experts > 16) {
    set_error("router gating head supports 1..16 experts (got %d)", w->n_experts);
    return README_ERR_UNSUPPORTED;
  }
  README_CHECK_ARG(eps >= 0.f, "eps must be >= 0");
  README_CHECK_ARG(w->emb && w->norm1 && w->w_qkv && w->w_o && w->norm2 && w->w_gate && w->w_up && w->w_down &&
                       w->norm_f && w->w_head,
                   "null weight pointer");
  README_CHECK_ARG(aligned16(w->w_qkv) && aligned16(w->w_o) && aligned16(w->w_gate) && aligned16(w->w_up) &&
                       aligned16(w->w_down),
                   "projection weights must be 16-byte aligned");
  rw->vocab = w->vocab;
  rw->n_experts = w->n_experts;
  rw->emb = static_cast<const __nv_bfloat16*>(w->emb);
  rw->g1 = static_cast<const __nv_bfloat16*>(w->norm1);
  rw->wqkv = static_cast<const __nv_bfloat16*>(w->w_qkv);
  rw->wo = static_cast<const __nv_bfloat16*>(w->w_o);
  rw->g2 = static_cast<const __nv_bfloat16*>(w->norm2);
  rw->wg = static_cast<const __nv_bfloat16*>(w->w_gate);
  rw->wu = static_cast<const __nv_bfloat16*>(w->w_up);
  rw->wd = static_cast<const __nv_bfloat16*>(w->w_down);
  rw->gf = static_cast<const __nv_bfloat16*>(w->norm_f);
  rw->whead = static_cast<const __nv_bfloat16*>(w->w_head);
  return README_OK;
}
}  // namespace

size_t readme_router_step_workspace_bytes(int64_t n, int32_t max_len) {
  return router_step_ws_bytes(n < 0 ? 0 : n, max_len < 1 ? 1 : max_len);
}

readme_status readme_router_step(const int32_t* token_ids, int64_t n, const int32_t* slot, const int32_t* pos,
                                 void* kv_cache, int32_t n_slots, int32_t max_len, const readme_router_weights* w,
                                 float eps, float* logits, uint32_t* dev_status, void* ws, size_t ws_bytes,
                                 readme_stream_t stream) {
  README_CHECK_ARG(n >= 0 && n < (int64_t(1) << 31), "n out of range");
  README_CHECK_ARG(n_slots >= 1 && max_len >= 1 && max_len <= 32768, "need n_slots >= 1 and 1 <= max_len <= 32768");
  RouterWeights rw;
  README_TRY(check_router_weights(w, eps, &rw));
  if (n == 0) return README_OK;
  README_CHECK_ARG(token_ids && slot && pos && kv_cache && logits && ws && aligned16(ws) && aligned16(kv_cache),
                   "null pointer argument (or unaligned workspace / cache)");
  if (ws_bytes < router_step_ws_bytes(n, max_len)) {
    set_error("router step workspace too small: %zu < %zu", ws_bytes, router_step_ws_bytes(n, max_len));
    return README_ERR_WORKSPACE;
  }
  return launch_router_step(token_ids, n, slot, pos, static_cast<__nv_bfloat16*>(kv_cache), n_slots, max_len, rw, eps,
                            logits, ws, dev_status, reinterpret_cast<cudaStream_t>(stream));
}

readme_status readme_router_forward(const int32_t* token_ids, int64_t T, const int32_t* seq_starts, int32_t nseq,
                                    const readme_router_weights* w, float eps, float* logits, uint32_t* dev_status,
                                    void* ws, size_t ws_bytes, readme_stream_t stream) {
  README_CHECK_ARG(T >= 0 && T < (int64_t(1) << 31), "T out of range");
  README_CHECK_ARG(nseq >= 1, "nseq must be >= 1");
  RouterWeights rw;
  README_TRY(check_router_weights(w, eps, &rw));
  if (T == 0) return README_OK;
  README_CHECK_ARG(token_ids && seq_starts && logits && ws && aligned16(ws),
                   "null pointer argument (or unaligned workspace)");
  if (ws_bytes < router_ws_bytes(T, nseq)) {
    set_error("router workspace too small: %zu < %zu", ws_bytes, router_ws_bytes(T, nseq));
    return README_ERR_WORKSPACE;
  }
  return launch_router_forward(token_ids, T, seq_starts, nseq, rw, eps, logits, ws, dev_status,
                               reinterpret_cast<cudaStream_t>(stream));
}

size_t readme_router_route_workspace_bytes(int64_t T, int32_t nseq, int32_t E, int32_t k) {
  return align_up(router_ws_bytes(T < 0 ? 0 : T, nseq < 1 ? 1 : nseq), 256) +
         route_ws_bytes(T < 0 ? 0 : T, E < 1 ? 1 : E, k < 1 ? 1 : k);
}

readme_status readme_router_forward_route(const int32_t* token_ids, int64_t T, const int32_t* seq_starts,
                                          int32_t nseq, const readme_router_weights* w, float eps, int32_t k,
                                          float* logits, int32_t* topk_idx, float* topk_w, int32_t* counts,
                                          int32_t* offsets, int32_t* dest, int32_t* src, uint32_t* dev_status,
                                          void* ws, size_t ws_bytes, readme_stream_t stream) {
  README_CHECK_ARG(T >= 0 && T < (int64_t(1) << 31), "T out of range");
  README_CHECK_ARG(nseq >= 1, "nseq must be >= 1");
  RouterWeights rw;
  README_TRY(check_router_weights(w, eps, &rw));
  README_TRY(check_route_args(T, rw.n_experts, k));
  README_CHECK_ARG(counts && offsets, "counts and offsets are required");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (T == 0) return launch_route(nullptr, README_F32, 0, rw.n_experts, k, nullptr, nullptr, counts, offsets, nullptr,
                                  nullptr, dev_status, ws, st);
  README_CHECK_ARG(token_ids && seq_starts && logits && topk_idx && topk_w && dest && src && ws && aligned16(ws),
                   "null pointer argument (or unaligned workspace)");
  const size_t need = readme_router_route_workspace_bytes(T, nseq, rw.n_experts, k);
  if (ws_bytes < need) {
    set_error("router+route workspace too small: %zu < %zu", ws_bytes, need);
    return README_ERR_WORKSPACE;
  }
  const RoutePlanOut plan{k, topk_idx, counts, offsets, dest, src, topk_w,
                          static_cast<char*>(ws) + align_up(router_ws_bytes(T, nseq), 256)};
  return launch_router_forward(token_ids, T, seq_starts, nseq, rw, eps, logits, ws, dev_status, st, &plan);
}

readme_status readme_build_experts(const void* dense_w_gate, const void* dense_w_up, const void* dense_w_down,
                                   readme_dtype dt, int32_t D, int32_t H, int32_t E, int32_t d,
                                   const int32_t* neuron_idx, void* w_gate, void* w_up, void* w_down,
                                   uint32_t* dev_status, readme_stream_t stream) {
  README_CHECK_ARG(dt == README_F32 || dt == README_BF16, "dt must be F32 or BF16");
  README_CHECK_ARG(D >= 1 && H >= 1 && E >= 1 && d >= 1 && d <= D, "bad D/H/E/d");
  README_CHECK_ARG(dense_w_gate && dense_w_up && dense_w_down && neuron_idx && w_gate && w_up && w_down,
                   "null pointer argument");
  return launch_build_experts(dense_w_gate, dense_w_up, dense_w_down, dt, D, H, E, d, neuron_idx, w_gate, w_up,
                              w_down, dev_status, reinterpret_cast<cudaStream_t>(stream));
}

// ---- expert parallelism over peer memory (ep.cu) ----------------------------------------------------

readme_status readme_ep_alloc(size_t bytes, void** ptr) {
  README_CHECK_ARG(ptr != nullptr && bytes > 0, "ptr required, bytes > 0");
  *ptr = nullptr;
  README_CUDA(cudaMalloc(ptr, bytes));
  cudaError_t e = cudaMemset(*ptr, 0, bytes);
  if (e != cudaSuccess) {
    cudaFree(*ptr);
    *ptr = nullptr;
    return cuda_fail(e, "cudaMemset(ep arena)");
  }
  return README_OK;
}

readme_status readme_ep_free(void* ptr) {
  if (ptr) README_CUDA(cudaFree(ptr));
  return README_OK;
}

readme_status readme_ipc_handle(const void* ptr, void* handle) {
  static_assert(sizeof(cudaIpcMemHandle_t) == README_IPC_HANDLE_BYTES, "IPC handle size");
  README_CHECK_ARG(ptr && handle, "ptr and handle are required");
  cudaIpcMemHandle_t h;
  README_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)));
  memcpy(handle, &h, sizeof(h));
  return README_OK;
}

readme_status readme_ipc_open(const void* handle, void** ptr) {
  README_CHECK_ARG(ptr && handle, "ptr and handle are required");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  *ptr = nullptr;
  README_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  // The kernels load and store through this mapping directly: a buffer on another GPU must be reachable over
  // NVLink / PCIe peer access from this one, else the mapping is refused (the caller falls back to NCCL).
  int cur = -1;
  cudaPointerAttributes at;
  cudaError_t e = cudaGetDevice(&cur);
  if (e == cudaSuccess) e = cudaPointerGetAttributes(&at, *ptr);
  if (e != cudaSuccess) {
    cudaIpcCloseMemHandle(*ptr);
    *ptr = nullptr;
    return cuda_fail(e, "cudaPointerGetAttributes(ipc mapping)");
  }
  if (at.device != cur) {
    int ok = 0;
    e = cudaDeviceCanAccessPeer(&ok, cur, at.device);
    if (e != cudaSuccess || !ok) {
      cudaIpcCloseMemHandle(*ptr);
      *ptr = nullptr;
      set_error("device %d cannot access peer device %d (no P2P path): use the NCCL exchange", cur, at.device);
      return README_ERR_UNSUPPORTED;
    }
  }
  return README_OK;
}

readme_status readme_ipc_close(void* ptr) {
  if (ptr) README_CUDA(cudaIpcCloseMemHandle(ptr));
  return README_OK;
}

namespace {
readme_status check_peers(const void* const* v, int32_t G) {
  README_CHECK_ARG(G >= 1 && G <= README_EP_MAX_RANKS, "G must be in [1, %d]", README_EP_MAX_RANKS);
  README_CHECK_ARG(v != nullptr, "peer pointer array is required");
  for (int i = 0; i < G; ++i) README_CHECK_ARG(v[i] != nullptr, "peer pointer %d is NULL", i);
  return README_OK;
}
}  // namespace

readme_status readme_ep_signal(uint64_t* const* peer_flags, int32_t G, int32_t me, uint64_t* epoch,
                               readme_stream_t stream) {
  README_TRY(check_peers(reinterpret_cast<const void* const*>(peer_flags), G));
  README_CHECK_ARG(me >= 0 && me < G && epoch != nullptr, "me out of range or epoch missing");
  return launch_ep_signal(peer_flags, G, me, epoch, reinterpret_cast<cudaStream_t>(stream));
}

readme_status readme_ep_wait(const uint64_t* flags, int32_t G, const uint64_t* epoch, uint32_t* dev_status,
                             readme_stream_t stream) {
  README_CHECK_ARG(flags != nullptr && epoch != nullptr && G >= 1 && G <= README_EP_MAX_RANKS,
                   "flags and epoch required, G in [1, 8]");
  return launch_ep_wait(flags, G, epoch, dev_status, reinterpret_cast<cudaStream_t>(stream));
}

readme_status readme_ep_publish_counts(const int32_t* counts, int32_t E, int32_t* const* peer_tables, int32_t G,
                                       int32_t me, readme_stream_t stream) {
  README_TRY(check_peers(reinterpret_cast<const void* const*>(peer_tables), G));
  README_CHECK_ARG(counts && E >= 1 && E <= README_MAX_EXPERTS && E % G == 0 && me >= 0 && me < G,
                   "need counts, E in [1, 256] divisible by G, 0 <= me < G");
  return launch_ep_publish(counts, E, peer_tables, G, me, reinterpret_cast<cudaStream_t>(stream));
}

readme_status readme_ep_plan(const int32_t* table, int32_t G, int32_t E, int32_t me, int32_t* seg_offsets,
                             int32_t* row_base, readme_stream_t stream) {
  README_CHECK_ARG(table && seg_offsets && row_base, "table, seg_offsets and row_base are required");
  README_CHECK_ARG(G >= 1 && G <= README_EP_MAX_RANKS && E >= 1 && E <= README_MAX_EXPERTS && E % G == 0 &&
                       me >= 0 && me < G,
                   "need G in [1, 8], E in [1, 256] divisible by G, 0 <= me < G");
  return launch_ep_plan(table, G, E, me, seg_offsets, row_base, reinterpret_cast<cudaStream_t>(stream));
}

readme_status readme_ep_dispatch(const void* x, readme_dtype dt, int64_t T, int32_t H, int32_t k,
                                 const int32_t* dest, const int32_t* offsets, const int32_t* row_base, int32_t E,
                                 int32_t G, int32_t me, void* const* peer_x, int32_t* const* peer_map,
                                 int64_t vrows, int32_t to_token, uint32_t* dev_status, readme_stream_t stream) {
  README_TRY(check_rows(dt, H));
  README_CHECK_ARG(T >= 0 && k >= 1 && T * static_cast<int64_t>(k) < (int64_t(1) << 31), "bad T/k");
  README_CHECK_ARG(E >= 1 && E <= README_MAX_EXPERTS && G >= 1 && E % G == 0 && me >= 0 && me < G,
                   "need E in [1, 256] divisible by G and 0 <= me < G");
  README_CHECK_ARG(vrows >= (to_token ? T : T * k) && vrows * G < (int64_t(1) << 31), "vrows out of range");
  if (T == 0) return README_OK;
  README_TRY(check_peers(peer_x, G));
  README_TRY(check_peers(reinterpret_cast<const void* const*>(peer_map), G));
  README_CHECK_ARG(x && dest && offsets && row_base && aligned16(x), "x (16-byte aligned), dest, offsets, row_base");
  for (int i = 0; i < G; ++i) README_CHECK_ARG(aligned16(peer_x[i]), "peer_x must be 16-byte aligned");
  return launch_ep_dispatch(x, static_cast<size_t>(H) * dt_size(dt), T, k, dest, offsets, row_base, E, G, me,
                            peer_x, peer_map, vrows, to_token, dev_status, reinterpret_cast<cudaStream_t>(stream));
}

readme_status readme_ep_expert_ffn(const void* x_recv, readme_dtype dt, int64_t rows_cap, int32_t H,
                                   int32_t E_local, int32_t d, int32_t G, const int32_t* seg_offsets,
                                   const void* w_gate, const void* w_up, const void* w_down, const int32_t* row_map,
                                   void* const* peer_out, const void* const* peer_res, int64_t vrows,
                                   uint32_t* dev_status, void* ws, size_t ws_bytes, readme_stream_t stream) {
  README_TRY(check_ffn_args(dt, rows_cap, H, E_local, d, G, seg_offsets));
  if (dt != README_BF16) {
    set_error("readme_ep_expert_ffn is bf16-only");
    return README_ERR_UNSUPPORTED;
  }
  if (rows_cap == 0) return README_OK;
  README_TRY(check_peers(peer_out, G));
  README_CHECK_ARG(x_recv && w_gate && w_up && w_down && row_map && ws, "null pointer argument");
  README_CHECK_ARG(vrows >= 1 && vrows * G < (int64_t(1) << 31), "vrows out of range");
  README_CHECK_ARG(aligned16(x_recv) && aligned16(w_gate) && aligned16(w_up) && aligned16(w_down) && aligned16(ws),
                   "all tensors must be 16-byte aligned");
  if (ws_bytes < ffn_ws_bytes(rows_cap, d, dt)) {
    set_error("ep_expert_ffn workspace too small: %zu < %zu", ws_bytes, ffn_ws_bytes(rows_cap, d, dt));
    return README_ERR_WORKSPACE;
  }
  PeerOut po{};
  for (int i = 0; i < G; ++i) {
    po.y[i] = static_cast<__nv_bfloat16*>(peer_out[i]);
    po.res[i] = peer_res ? static_cast<const __nv_bfloat16*>(peer_res[i]) : nullptr;
  }
  po.npeer = G;
  po.vrows = vrows;
  uint32_t* ready = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + ffn_h_bytes(rows_cap, d, dt));
  return launch_ffn_layer_2cta(static_cast<const __nv_bfloat16*>(x_recv), rows_cap, H, E_local, d, G * E_local,
                               seg_offsets, static_cast<const __nv_bfloat16*>(w_gate),
                               static_cast<const __nv_bfloat16*>(w_up), static_cast<const __nv_bfloat16*>(w_down),
                               static_cast<__nv_bfloat16*>(ws), nullptr, row_map, nullptr, ready, dev_status,
                               reinterpret_cast<cudaStream_t>(stream), nullptr, 0, &po);
}

}  // extern "C"
#pragma GCC visibility pop
