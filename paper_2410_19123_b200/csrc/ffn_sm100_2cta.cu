// ffn_sm100_2cta.cu — a6/a7 (+ a8 for k = 1) grouped expert GEMMs on CTA pairs (tcgen05.mma.cta_group::2), bf16.
//
//     a6:  h_r = silu(x_r . W_gate[e]^T) * (x_r . W_up[e]^T)        a7:  y_r = h_r . W_down[e]^T
// (PAPER.md:159 with the SwiGLU reading Q4; e = the expert owning row r's segment). Every tile is computed by a
// CLUSTER OF TWO CTAs on the two SMs of a TPC: one tcgen05.mma.cta_group::2 (issued by the even CTA) multiplies
// A rows held in both CTAs' shared memory by a 256-column B tile whose halves live in the two CTAs, accumulating
// into both CTAs' TMEM — per SM 32 KB of TMA traffic per 64-deep K stage for a 256 x 256 pair tile.
//
// Two kernels:
//   ffn_gemm2_kernel   one projection per launch (readme_expert_gate_up / readme_expert_down, the split form);
//   ffn_layer2_kernel  the whole expert FFN in ONE persistent launch (readme_expert_ffn, moe_layer, moe_stack,
//                      the permanent expert, expert parallelism): [gate/up tiles][down tiles], down tiles waiting
//                      on per-m-tile readiness counters; 256-row m-tiles for prefill (segment tails of <= 64 rows
//                      merged into full m-tiles, dynamic tile order, at <= 16384 rows) and 128-row m-tiles with a
//                      9-stage ring for decode. DESIGN.md §6 has the design and the measurements behind it.
// Tile shapes: 256 rows x 256 accumulator columns (M=256 MMA, each CTA 128 rows, TMEM lane = row); an m-tile of
// <= 128 rows runs as an M=128 MMA (each CTA 64 rows; the "2x2" TMEM layout: lanes 0-63 hold accumulator
// columns [0,128), lanes 64-127 columns [128,256) of the same rows). Gate/up B operand per CTA r: 64 rows of
// W_gate then the same 64 rows of W_up (neurons n0+64r ..), so in accumulator column space gate column c pairs
// with up column c+64 inside every 128-column window.
#include <stdlib.h>

#include <mutex>
#include <type_traits>

#include "kernels.h"
#include "tc_common.cuh"

namespace readme {

namespace {

constexpr int kBK = 64;
constexpr int kUK = 16;
constexpr int kStages = 6;
constexpr int kThreads = 192;
constexpr int kMaxSeg = 512;
constexpr int kStageA = 128 * 128;  // up to 128 rows x 128 B per CTA
constexpr int kStageB = 128 * 128;  // 128 rows x 128 B per CTA (its half of N = 256)
constexpr int kTmemCols = 512;      // two accumulators of 256 columns
constexpr int kPrefetchK = 32;      // K stages of the first weight tile warmed in L2 before the PDL wait
constexpr int kXokWords = 64;       // m-tiles whose x readiness is cached in shared memory (2048)

// Decode-sized launches use 128-row m-tiles only (M = 128 pair MMAs, 64 A rows per CTA): the A slot halves,
// so the ring holds more stages (more weight bytes in flight per SM).
constexpr int kStageAD = 64 * 128;
constexpr int64_t kDecodeRows = 1024;  // launches up to this many rows use the 128-row m-tile variant
constexpr int64_t kDynRows = 16384;    // 256-row m-tile launches up to this many rows: dynamic order, merged tails

template <int S, int SA>
struct __align__(8) SmemT {
  uint8_t a[S][SA];
  uint8_t b[S][kStageB];
  uint64_t full[S];
  uint64_t empty[S];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  alignas(16) uint8_t stg[4][32 * 128];  // epilogue staging, one 4 KB tile per epilogue warp
  int seg_off[kMaxSeg + 1];
  int tile_start[kMaxSeg + 1];
};
using Smem = SmemT<kStages, kStageA>;
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;
static_assert(kSmemBytes <= 232448, "shared memory");

struct Tile {
  int g, m0, rows, n0;
  bool m256;
};

__device__ __forceinline__ Tile decode_tile(const Smem& s, int t, int nseg, int bn_out, int& gcur, int NT,
                                           bool n_fastest) {
  while (gcur + 1 < nseg && s.tile_start[gcur + 1] <= t) ++gcur;
  const int g = gcur;
  const int cnt = s.seg_off[g + 1] - s.seg_off[g];
  const int mt_g = (cnt + 255) / 256;
  const int local = t - s.tile_start[g];
  const int nt = n_fastest ? local % NT : local / mt_g, mt = n_fastest ? local / NT : local % mt_g;
  Tile tl;
  tl.g = g;
  tl.m0 = s.seg_off[g] + mt * 256;
  tl.rows = min(256, cnt - mt * 256);
  tl.m256 = tl.rows > 128;
  tl.n0 = nt * bn_out;
  return tl;
}

// Fusion of the combine into GEMM2 (readme_moe_layer's path, k == 1): kFuse == 1 makes the epilogue
// write row r to y[src[r]] (+ residual, one fp32 add and one rounding) -> no y_sorted and no separate
// combine (Eq. 2's sum has one term with weight exactly 1). (Fusing the dispatch into GEMM1 with TMA
// tile::gather4 was measured 3x slower than dispatch + tiled loads: every 256-row A tile is re-gathered
// for each of the 43 N tiles, 32 gather4 ops per stage — see profiles/SUMMARY.md.)
struct Fuse {
  const int32_t* src;                 // [rows] expert-contiguous row -> token (= dest^-1, k == 1)
  int rows;                           // T
  const __nv_bfloat16* residual;      // [T, N] or null (GEMM2 scatter only)
};

// Epilogue staging (per epilogue warp: 32 rows x 128 B; 16-byte chunks XOR-swizzled by row & 7 so the
// row-per-thread writes and the row-cooperative reads are both bank-conflict-light).
__device__ __forceinline__ void stage_row_bf16x32(uint8_t* stg, int row, int chunk0, const float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 w;
    w.x = pack_bf16x2(v[8 * j + 0], v[8 * j + 1]);
    w.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
    w.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
    w.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
    const int c = chunk0 + j;
    *reinterpret_cast<uint4*>(stg + row * 128 + ((c ^ (row & 7)) << 4)) = w;
  }
}
// Write the warp's 32 staged rows: lane l moves 16 B chunk (l & 7) of row 4i + (l >> 3); row r goes to the
// global address held by lane r (0 = skip the row); chunks at or past `bytes_left` are not written.
__device__ __forceinline__ void stage_flush(const uint8_t* stg, int lane, uint64_t my_row, int bytes_left,
                                            bool evict_first) {
  __syncwarp();
  uint64_t pol = 0;
  if (evict_first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = i * 4 + (lane >> 3), c = lane & 7;
    const uint64_t dst = __shfl_sync(0xffffffffu, my_row, r);
    if (dst && c * 16 < bytes_left) {
      const uint4 v = *reinterpret_cast<const uint4*>(stg + r * 128 + ((c ^ (r & 7)) << 4));
      if (evict_first)
        asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(reinterpret_cast<uint4*>(dst) + c),
                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                     : "memory");
      else
        st_v4(reinterpret_cast<uint4*>(dst) + c, v);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void add_bf16x32(const __nv_bfloat16* src, float (&v)[32], int ncols_left) {
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    if (j < ncols_left) {
      const uint4 w = ld_nc_v4(reinterpret_cast<const uint4*>(src + j));
      v[j + 0] += bf16_lo(w.x); v[j + 1] += bf16_hi(w.x); v[j + 2] += bf16_lo(w.y); v[j + 3] += bf16_hi(w.y);
      v[j + 4] += bf16_lo(w.z); v[j + 5] += bf16_hi(w.z); v[j + 6] += bf16_lo(w.w); v[j + 7] += bf16_hi(w.w);
    }
  }
}

template <int kMode, int kFuse>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
ffn_gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                 const __grid_constant__ CUtensorMap tmB1, int K, int N, int E, int nseg,
                 const int32_t* __restrict__ offsets, __nv_bfloat16* __restrict__ out, Fuse fz) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
  const uint32_t cta = tc::cluster_ctarank();
  const bool leader = cta == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  constexpr int kBnOut = kMode == 0 ? 128 : 256;
  const int NT = (N + kBnOut - 1) / kBnOut;
  const int KB = (K + kBK - 1) / kBK;

  for (int i = tid; i <= nseg; i += kThreads) s.seg_off[i] = offsets[i];
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB0);
    if (kMode == 0) tc::prefetch_tmap(&tmB1);
  }
  if (warp == 1) tc::tmem_alloc<2>(&s.tmem_base, kTmemCols);
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int g = 0; g < nseg; ++g) {
      s.tile_start[g] = acc;
      acc += (s.seg_off[g + 1] - s.seg_off[g] + 255) / 256 * NT;
    }
    s.tile_start[nseg] = acc;
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&s.full[i], 1);   // the leader's producer arms it with both CTAs' bytes
      tc::mbar_init(&s.empty[i], 1);  // one multicast commit per consumed stage
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s.tfull[i], 1);
      tc::mbar_init(&s.tempty[i], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is the one used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after();
  const int ntiles = s.tile_start[nseg];
  const uint32_t tmem_base = s.tmem_base;

  if (warp == 0) {
    // ===== TMA producer (both CTAs; completion counted on the leader's barrier) =====
    // The whole warp runs the loop; lane 0 arms the barrier and issues the loads.
    int stage = 0;
    uint32_t phase = 0;
    int gcur = 0;
    for (int t = pair; t < ntiles; t += npairs) {
      const Tile tl = decode_tile(s, t, nseg, kBnOut, gcur, NT, false);
      const int e = tl.g % E;
      const int a_rows = tl.m256 ? 128 : 64;
      const int a_row0 = tl.m0 + static_cast<int>(cta) * a_rows;
      const uint32_t bytes = 2u * static_cast<uint32_t>(a_rows * 128 + kStageB);
      for (int kb = 0; kb < KB; ++kb) {
        tc::mbar_wait(&s.empty[stage], phase ^ 1);
        const uint32_t fb = tc::mapa(&s.full[stage], 0);
        const int k0 = kb * kBK;
        if (tc::elect_one()) {  // one elected lane of the converged warp (uniform operands)
          if (leader) tc::mbar_expect_tx(&s.full[stage], bytes);
          tc::tma_load_2d_2sm(&tmA, s.a[stage], fb, k0, a_row0);
          if (tl.m256) tc::tma_load_2d_2sm(&tmA, s.a[stage] + 64 * 128, fb, k0, a_row0 + 64);
          if (kMode == 0) {
            tc::tma_load_3d_2sm(&tmB0, s.b[stage], fb, k0, tl.n0 + 64 * static_cast<int>(cta), e);
            tc::tma_load_3d_2sm(&tmB1, s.b[stage] + 64 * 128, fb, k0, tl.n0 + 64 * static_cast<int>(cta), e);
          } else {
            tc::tma_load_3d_2sm(&tmB0, s.b[stage], fb, k0, tl.n0 + 128 * static_cast<int>(cta), e);
            tc::tma_load_3d_2sm(&tmB0, s.b[stage] + 64 * 128, fb, k0, tl.n0 + 128 * static_cast<int>(cta) + 64, e);
          }
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ===== MMA issuer (leader CTA): the whole warp walks the loop, one elected lane issues =====
      constexpr uint32_t idesc256 = tc::idesc_bf16(256, 256);
      constexpr uint32_t idesc128 = tc::idesc_bf16(128, 256);
      const uint64_t adesc0 = tc::sdesc_sw128(tc::smem_u32(s.a[0])), bdesc0 = tc::sdesc_sw128(tc::smem_u32(s.b[0]));
      int stage = 0;
      uint32_t phase = 0;
      int gcur = 0, i = 0;
      for (int t = pair; t < ntiles; t += npairs, ++i) {
        const Tile tl = decode_tile(s, t, nseg, kBnOut, gcur, NT, false);
        const uint32_t idesc = tl.m256 ? idesc256 : idesc128;
        const int acc = i & 1;
        const uint32_t use = static_cast<uint32_t>(i >> 1);
        tc::mbar_wait_cluster(&s.tempty[acc], (use & 1u) ^ 1u);
        tc::fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * 256);
        for (int kb = 0; kb < KB; ++kb) {
          tc::mbar_wait_cluster(&s.full[stage], phase);
          tc::fence_after();
          const uint64_t ad = adesc0 + static_cast<uint64_t>(stage * (kStageA >> 4));
          const uint64_t bd = bdesc0 + static_cast<uint64_t>(stage * (kStageB >> 4));
          if (tc::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kBK / kUK; ++kk)
              tc::mma_f16<2>(d_tmem, ad + static_cast<uint64_t>(kk * 2), bd + static_cast<uint64_t>(kk * 2), idesc,
                             (kb | kk) != 0 ? 1u : 0u);
            tc::commit_2sm_mc(&s.empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (tc::elect_one()) tc::commit_2sm_mc(&s.tfull[acc], 0x3);
        __syncwarp();
      }
    }
  } else {
    // ===== epilogue: warps 2..5 of both CTAs; warp's TMEM lane quarter = warp % 4 =====
    const int q = warp & 3;
    int gcur = 0, i = 0;
    for (int t = pair; t < ntiles; t += npairs, ++i) {
      const Tile tl = decode_tile(s, t, nseg, kBnOut, gcur, NT, false);
      const int acc = i & 1;
      const uint32_t use = static_cast<uint32_t>(i >> 1);
      tc::mbar_wait_cluster(&s.tfull[acc], use & 1u);
      tc::fence_after();
      const uint32_t tacc = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * 256);
      int row_in_tile, col_base, n_windows, out_off;
      if (tl.m256) {  // "4x1": lane = row, all 256 columns
        row_in_tile = static_cast<int>(cta) * 128 + q * 32 + lane;
        col_base = 0;
        n_windows = 2;
        out_off = 0;
      } else {  // "2x2": lanes 0-63 -> columns [0,128), lanes 64-127 -> columns [128,256), same 64 rows
        row_in_tile = static_cast<int>(cta) * 64 + (q & 1) * 32 + lane;
        col_base = 0;
        n_windows = 1;
        out_off = (q >> 1) * (kBnOut / 2);
      }
      const bool valid = row_in_tile < tl.rows;
      int64_t orow_idx = tl.m0 + row_in_tile;
      bool valid_row = valid;
      if constexpr (kMode == 1 && kFuse == 1) {  // k == 1: expert row r holds token src[r] (identity if null)
        orow_idx = valid ? (fz.src ? __ldg(fz.src + orow_idx) : orow_idx) : 0;
        valid_row = valid && orow_idx >= 0 && orow_idx < fz.rows;  // a corrupt plan never writes out of bounds
      }
      __nv_bfloat16* orow = out + orow_idx * N;
      const __nv_bfloat16* rrow = (kMode == 1 && kFuse == 1 && fz.residual) ? fz.residual + orow_idx * N : nullptr;
      uint8_t* stg = s.stg[q];
      // Each 64-column output chunk: every thread puts its row's 128 B into the warp's staging tile, then
      // the warp writes 4 full rows (4 x 128 B) per store instruction (coalesced, whole L2 lines).
      for (int w = 0; w < n_windows; ++w) {
        const uint32_t wbase = tacc + static_cast<uint32_t>(col_base + w * 128);
        if (kMode == 0) {
          // window of 128 accumulator columns: gate [0,64), up [64,128) -> 64 h columns
          const int hcol0 = tl.n0 + out_off + w * 64;
#pragma unroll 1
          for (int c = 0; c < 64; c += 32) {
            uint32_t gr[32], ur[32];
            tc::tmem_ld32(wbase + c, gr);
            tc::tmem_ld32(wbase + 64 + c, ur);
            tc::tmem_wait_ld();
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = tc::silu(__uint_as_float(gr[j])) * __uint_as_float(ur[j]);
            stage_row_bf16x32(stg, lane, c / 8, v);
          }
          stage_flush(stg, lane, valid ? reinterpret_cast<uint64_t>(orow + hcol0) : 0ull, (N - hcol0) * 2,
                      false);
        } else {
#pragma unroll 1
          for (int c0 = 0; c0 < 128; c0 += 64) {
            const int col0 = tl.n0 + out_off + w * 128 + c0;
#pragma unroll 1
            for (int c = 0; c < 64; c += 32) {
              uint32_t vr[32];
              tc::tmem_ld32(wbase + c0 + c, vr);
              tc::tmem_wait_ld();
              float v[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(vr[j]);
              if (rrow && valid_row) add_bf16x32(rrow + col0 + c, v, N - (col0 + c));
              stage_row_bf16x32(stg, lane, c / 8, v);
            }
            stage_flush(stg, lane, valid_row ? reinterpret_cast<uint64_t>(orow + col0) : 0ull, (N - col0) * 2,
                        false);
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      // The MMA only needs this warp's TMEM reads finished (tcgen05.wait::ld + fence above), not its global
      // stores, so the arrive is relaxed.
      if (lane == 0) tc::mbar_arrive_cluster_relaxed(&s.tempty[acc], 0);
    }
  }

  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after();
  if (warp == 1) tc::tmem_dealloc<2>(tmem_base, kTmemCols);
}


// ===================================================================================================
// The whole expert FFN (a6 then a7, a8 fused for k == 1) in ONE persistent CTA-pair launch. The tile list
// is [every gate/up tile][every down tile], statically strided over the pairs; a down tile (g, m) starts
// once all NT1 gate/up tiles of (g, m) have stored their h rows: each epilogue warp publishes its part of
// a gate/up tile with a release add on ready[m-tile] (after a generic->async proxy fence, since the down
// tile reads h with TMA), and the down producer acquires ready[m-tile] == NT1 * 8 before loading. Down
// tiles come after every gate/up tile in every pair's sequence, so a wait only ever depends on tiles that
// are earlier in some pair's sequence. That needs every pair of the grid co-resident: the launcher sizes
// the grid with cudaOccupancyMaxActiveClusters. If co-residency still fails (an SM-holding kernel from
// another stream or process, MPS), the bounded poll gives up: the waiting thread sets
// README_DEV_SCHED_TIMEOUT in dev_status and the launch's abort word, and from then on every epilogue of
// the launch skips its stores — each output element is either its correct value or left as it was, never
// a value computed from unready rows (tests/test_gpu_parity.py::test_ffn_sm_starved_*).
struct LayerArgs {
  int H, d, E, nseg;
  const int32_t* offsets;
  __nv_bfloat16* h;          // [rows, d]
  __nv_bfloat16* y;          // [rows, H] (y_sorted) or [T, H] (scatter)
  uint32_t* ready;           // [#m-tiles] zeroed before the launch
  uint32_t* abort;           // one word of the zeroed readiness region: nonzero once a readiness wait gave up
  uint32_t* dev_status;      // nullable
  uint32_t spin_limit;       // polls before a readiness wait gives up
  Fuse fz;
  const int32_t* expert_slot;  // nullable: expert e's weights live at slot expert_slot[e] of the weight pools
  // kFuse == 2 (expert parallelism over peer memory): received row r came from rank p = v / vrows as its
  // row i = v % vrows (v = fz.src[r]); the down epilogue stores it straight into that rank's output,
  // peer_y[p] + i*H, adding peer_res[p] + i*H when non-null — the combine all-to-all fused into the GEMM.
  __nv_bfloat16* peer_y[kMaxPeers];
  const __nv_bfloat16* peer_res[kMaxPeers];
  int npeer;
  int64_t vrows;
  int pdl;  // launched as a programmatic dependent of the dispatch: 1 = griddepcontrol.wait before reading
            // x_sorted; 2 = per-row readiness flags (xready) instead, so gate/up tiles start while the
            // dispatch is still writing later experts' rows (the wait moves to the kernel's end); 3 = the
            // kernel dispatches itself (dx below), as a programmatic dependent of the route
  // pdl == 3 (a5 fused in): the epilogue warps gather x_sorted[r] = x[dsrc[r] / dk] while they wait for
  // accumulators (copy_row / wait_copying) and count each segment's copied rows in seg_rows
  const uint4* dx;
  const int32_t* dsrc;
  void* dxs;     // x_sorted (the tensor map's buffer)
  int dk, dvec;  // top-k; 16-byte vectors per row
  const uint32_t* xready;  // pdl >= 2: [rows] flags, nonzero once row r of x_sorted is written (gather dispatch)
  uint64_t* trace;         // measurement only (readme_debug_trace), normally null
  uint64_t* ttrace;        // measurement only (readme_debug_tile_trace): [pair][ttrace_max][8], normally null
  int ttrace_max;
  int askip;               // tiles of <= 64 rows: the second CTA skips its A loads (knob ffn_askip)
  int order;               // lab: 1 = gate/up tiles N-tile fastest (knob ffn_order)
  int swap_rows;           // segment tails of <= swap_rows rows run as swap-AB tiles (knob ffn_swap; 0 = none)
  int merge;               // 256-row m-tiles: segment tails ride on full m-tiles (knob ffn_merge; 0 = separate)
  int dyn;                 // dynamic tile order: tiles after each pair's first claimed from tile_ctr (knob ffn_dyn)
  uint32_t* tile_ctr;      // zeroed word of the readiness region (dyn)
  uint32_t* seg_rows;      // pdl == 3: [nseg] rows of each segment copied so far (zeroed readiness words)
  int claim_ahead;         // dyn: K steps before the end of a tile's loads at which the next tile is claimed
};

struct LTile {
  int mode, g, mt, mid, m0, rows, n0;  // mid = global m-tile id (readiness counter index)
  bool m256;  // M = 256 pair MMA (each CTA 128 A rows), else M = 128 (64 rows per CTA)
  bool swap;  // swap-AB tail tile: weights are the MMA's M side, the tile's rows its N side
  int tm0, trows;  // merged tail (256-row m-tiles): trows (<= 64) more rows from tm0, run swap-AB off this
                   // tile's weight stages; 0 = none
};

constexpr int kTailMax = 64;  // rows of a merged segment tail (swap-AB MMAs of N <= 64 per K step)
constexpr int kMaxTails = 2;  // merged tails per segment at most

// m-tiles of a segment of R rows. With merging (256-row m-tiles): floor(R / 256) full m-tiles carry the
// remainder as tails of <= 64 rows (one per full m-tile, at most kMaxTails) when it fits, else the remainder
// is an m-tile of its own, as without merging. Every m-tile streams the expert's whole weight tile through its
// SMs whatever its rows, so a separate tail tile cost as many SM cycles as a full one (~530 per K step); a
// merged tail costs its swap-AB MMAs only, ~190-250 cycles per K step whatever its rows (its MMAs re-read the
// 16 KB weight stage): worth it for one or two tails, not three (tile trace, profiles/SUMMARY.md r02).
__device__ __forceinline__ bool seg_merges(int R) {
  const int nf = R >> 8, rem = R & 255;
  return rem > 0 && rem <= kTailMax * (nf < kMaxTails ? nf : kMaxTails);
}
template <int kMT>
__device__ __forceinline__ int seg_mtiles(int R, bool merge) {
  if (kMT == 256 && merge && seg_merges(R)) return R >> 8;
  return (R + kMT - 1) / kMT;
}

constexpr int kBN1 = 128;  // h columns per gate/up tile ([gate 64 | up 64] rows per CTA)
constexpr int kBN2 = 256;  // output columns per down tile (128 W_down rows per CTA)

// Tile list of the single-launch kernel: [every gate/up tile][every down tile]; inside each phase segment ->
// N tile -> m-tile (m fastest: the 4-5 pairs working on one expert's m-tiles read the same weight tile at the
// same time, so L2 serves it once). A segment's last m-tile of <= swap_rows rows runs swap-AB in place (it
// stays next to the full m-tiles that share its weight tile: moving the cheap tails to the end of each phase
// for a longest-first schedule re-read their weights from DRAM and measured 9 % slower at config 2).
// Down tiles come after every gate/up tile, so every wait is on a tile earlier in the global order
// (deadlock-free whenever the grid is co-resident).
// A role's tiles only move forward, so a cursor walks the segments (offsets read through the read-only
// cache; no per-segment tables in shared memory, which holds one more ring stage instead).
struct Cursor {
  int phase = -1, g = 0, start = 0, mbase = 0;  // segment g's first tile index in its phase; its first m-tile id
};

template <int kMT>
__device__ __forceinline__ LTile decode_ltile(const int32_t* __restrict__ offs, int t, int nseg, int T1, int NT1,
                                             int NT2, int swap_rows, Cursor& c, bool nfast = false,
                                             bool merge = false) {
  LTile tl;
  const int phase = t < T1 ? 0 : 1;
  const int NT = phase ? NT2 : NT1;
  if (c.phase != phase) {
    c.phase = phase;
    c.g = 0;
    c.start = phase ? T1 : 0;
    c.mbase = 0;
  }
  int lo = __ldg(offs + c.g), hi = __ldg(offs + c.g + 1);
  int mt_g = seg_mtiles<kMT>(hi - lo, merge);
  while (t >= c.start + mt_g * NT && c.g + 1 < nseg) {
    c.start += mt_g * NT;
    c.mbase += mt_g;
    ++c.g;
    lo = hi;
    hi = __ldg(offs + c.g + 1);
    mt_g = seg_mtiles<kMT>(hi - lo, merge);
  }
  const int local = t - c.start;
  // m-tile fastest (default) or, for gate/up tiles with nfast (lab knob ffn_order = 1), N-tile fastest
  const bool nf = nfast && phase == 0;
  const int nt = nf ? local % NT : local / mt_g, mt = nf ? local / NT : local % mt_g;
  const int R = hi - lo;
  tl.mode = phase;
  tl.g = c.g;
  tl.mt = mt;
  tl.mid = c.mbase + mt;
  tl.m0 = lo + mt * kMT;
  tl.rows = min(kMT, R - mt * kMT);
  tl.tm0 = 0;
  tl.trows = 0;
  if (kMT == 256 && merge && seg_merges(R)) {
    const int nfull = R >> 8, rem = R & 255;
    if (mt < (rem + kTailMax - 1) / kTailMax) {
      // chunk mt of the remainder rides on full m-tile mt
      tl.tm0 = lo + (nfull << 8) + mt * kTailMax;
      tl.trows = min(kTailMax, rem - mt * kTailMax);
    }
  }
  tl.m256 = tl.rows > 128;
  tl.swap = tl.rows <= swap_rows;  // only a segment's last m-tile can be that short
  tl.n0 = nt * (phase == 0 ? kBN1 : kBN2);
  return tl;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// A readiness wait gave up (lane 0 of the waiting warp): report it and stop every later store of the launch.
__device__ __forceinline__ void sched_give_up(const LayerArgs& la) {
  if (la.dev_status) atomicOr(la.dev_status, README_DEV_SCHED_TIMEOUT);
  atomicExch(la.abort, 1u);
  __threadfence();
}

// Epilogue of a swap-AB tile (a segment tail of <= 64 rows, standalone or merged into a full m-tile): this
// CTA's TMEM lane = weight row (gate/up: 4 x [16 gate | the same 16 up] neurons, one group per epilogue warp;
// down: 128 output columns), column j = the tile's row m0 + j. Both 32-column chunks are read first; with
// hi_bar (a merged tail, which borrows the other accumulator's columns [192, 256)) the warp then releases them
// before the stores. Same fp32 values and roundings as the normal epilogue.
template <int kFuse>
__device__ __forceinline__ void swap_chunk(const LayerArgs& la, const LTile& tl, const uint32_t (&r)[32], int c,
                                           uint32_t cta, int q, int lane, bool store) {
  const int H = la.H, d = la.d;
  if (tl.mode == 0) {
    // lanes 0-15 hold gate, 16-31 up of neurons n; lanes 0-15 finish columns c..c+15, lanes 16-31 c+16..c+31
    const bool lo = lane < 16;
    const int neuron = tl.n0 + 64 * static_cast<int>(cta) + 16 * q + (lane & 15);
    const bool ok = store && neuron < d;
    __nv_bfloat16* hcol = la.h + neuron;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float send = __uint_as_float(lo ? r[16 + j] : r[j]);
      const float recv = __shfl_xor_sync(0xffffffffu, send, 16);
      const float g = lo ? __uint_as_float(r[j]) : recv, u = lo ? recv : __uint_as_float(r[16 + j]);
      const int tok = c + (lo ? j : 16 + j);
      if (ok && tok < tl.rows) hcol[static_cast<int64_t>(tl.m0 + tok) * d] = __float2bfloat16_rn(tc::silu(g) * u);
    }
  } else {
    const int col = tl.n0 + 128 * static_cast<int>(cta) + 32 * q + lane;
    const bool ok = store && col < H;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int tok = c + j;
      if (tok >= tl.rows) break;  // warp-uniform
      const int64_t rr = tl.m0 + tok;
      __nv_bfloat16* orow;
      const __nv_bfloat16* rrow = nullptr;
      bool vrow = true;
      if constexpr (kFuse == 2) {
        const int64_t v = static_cast<int64_t>(__ldg(la.fz.src + rr));
        vrow = v >= 0 && v < la.vrows * la.npeer;
        const int p = vrow ? static_cast<int>(v / la.vrows) : 0;
        const int64_t i = vrow ? v - p * la.vrows : 0;
        __nv_bfloat16* py = la.peer_y[0];
        const __nv_bfloat16* pr = la.peer_res[0];
#pragma unroll
        for (int jj = 1; jj < kMaxPeers; ++jj)
          if (p == jj) {
            py = la.peer_y[jj];
            pr = la.peer_res[jj];
          }
        orow = py + i * H;
        rrow = pr ? pr + i * H : nullptr;
      } else {
        int64_t oi = rr;
        if constexpr (kFuse == 1) {
          oi = la.fz.src ? static_cast<int64_t>(__ldg(la.fz.src + rr)) : rr;
          vrow = oi >= 0 && oi < la.fz.rows;
          if (!vrow) oi = 0;
          rrow = la.fz.residual ? la.fz.residual + oi * H : nullptr;
        }
        orow = la.y + oi * H;
      }
      float val = __uint_as_float(r[j]);
      if (ok && vrow) {
        if (rrow) val += __bfloat162float(rrow[col]);
        orow[col] = __float2bfloat16_rn(val);
      }
    }
  }
}

// Arrive (relaxed, on the leader's copy) once this warp's TMEM reads before it have completed.
__device__ __forceinline__ void release_cols(uint64_t* bar, int lane) {
  tc::fence_before();
  __syncwarp();
  if (lane == 0) tc::mbar_arrive_cluster_relaxed(bar, 0);
}

template <int kFuse>
__device__ __forceinline__ void swap_epilogue(const LayerArgs& la, const LTile& tl, uint32_t tacc, uint32_t cta,
                                              int q, int lane, bool store, uint64_t* hi_bar = nullptr) {
  uint32_t r0[32], r1[32];
  const bool two = tl.rows > 32;  // warp-uniform (rows <= 64)
  tc::tmem_ld32(tacc, r0);
  if (two) tc::tmem_ld32(tacc + 32u, r1);
  tc::tmem_wait_ld();
  if (hi_bar) release_cols(hi_bar, lane);
  swap_chunk<kFuse>(la, tl, r0, 0, cta, q, lane, store);
  if (two) swap_chunk<kFuse>(la, tl, r1, 32, cta, q, lane, store);
}

// Shared memory of the single-launch kernel: only the TMA ring, its barriers and the x-readiness cache (the
// per-segment tables live in the cursor walk, the epilogue stores straight from registers). 256-row m-tiles:
// 6 stages of 36 KB per CTA (A 16 KB + a 4 KB slot for a merged tail's rows + B 16 KB); 128-row m-tiles
// (decode): 9 stages of 24 KB.
constexpr int kTQ = 4;           // tile-id queue depth (dynamic tile order)
constexpr int kTQConsumers = 10;  // peer producer + MMA warp + 2 x 4 epilogue warps

template <int S, int SA>
struct __align__(8) SmemLT {
  uint8_t a[S][SA];
  uint8_t b[S][kStageB];
  uint64_t full[S];
  uint64_t empty[S];
  uint64_t tfull[2];
  uint64_t tempty[2];
  // hi_free[b]: accumulator b's columns [192, 256) drained by the epilogue (8 warp arrivals per use). Users
  // of those columns, in tile order: the main accumulator of a 256-row tile in b, and the merged tail of a
  // tile whose main accumulator is the other one.
  uint64_t hi_free[2];
  // dynamic tile order (la.dyn): the leader's producer claims tiles from a global counter and publishes each
  // id to both CTAs' queues; the peer's producer, the MMA warp and the epilogue warps pop them in order
  uint64_t tq_full[kTQ];   // per CTA: id written (one release arrive by the leader's producer)
  uint64_t tq_empty[kTQ];  // leader: id read by all 10 consumers
  int tq[kTQ];
  uint32_t tmem_base;
  uint32_t xok[kXokWords];  // pdl == 2: bit per m-tile, this CTA's A rows seen ready
  uint32_t segok[kMaxSeg / 32];  // pdl == 3: bit per segment, all its rows seen copied
};
constexpr int kStagesL = 6;
#ifndef README_STAGES_LD
#define README_STAGES_LD 9  // lab builds may override (README_NVCC_EXTRA=-DREADME_STAGES_LD=n)
#endif
constexpr int kStagesLD = README_STAGES_LD;
constexpr int kTailSlot = 16384;             // offset of the merged-tail rows inside a 256-row stage's A slot
constexpr int kStageAL = kStageA + 4096;     // <= 32 tail rows x 128 B per CTA
constexpr int kMaxDefer = 3;                 // K stages whose tail MMAs may wait for the borrowed columns
using SmemL = SmemLT<kStagesL, kStageAL>;
using SmemLD = SmemLT<kStagesLD, kStageAD>;
constexpr size_t kSmemBytesL = sizeof(SmemL) + 1024;
constexpr size_t kSmemBytesLD = sizeof(SmemLD) + 1024;
static_assert(kSmemBytesL <= 232448 && kSmemBytesLD <= 232448, "single-launch kernel shared memory");

// 32 fp32 values of one row -> 32 bf16 (RNE) at dst, 16 B at a time, columns at or past ncols skipped
// (ncols is a multiple of 8). Each thread writes whole 32-byte sectors of its own row.
__device__ __forceinline__ void store_row_bf16x32(__nv_bfloat16* dst, const float (&v)[32], int ncols) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (8 * j < ncols) {
      uint4 w;
      w.x = pack_bf16x2(v[8 * j + 0], v[8 * j + 1]);
      w.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
      w.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
      w.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
      st_v4(reinterpret_cast<uint4*>(dst) + j, w);
    }
  }
}

// Epilogue of one 128-lane accumulator slot of a non-swap tile (this warp's 32 rows): gate/up tiles store
// h = silu(g) * u, down tiles store y (y_sorted, the fused combine y[src[r]] + residual, or the source rank's
// row over peer memory). row_in_tile = this thread's row, ncols / acc_off = the accumulator columns it holds
// (all 256 for M = 256, half for the M = 128 "2x2" layout). valid = the row exists and nothing aborted.
// Gate/up columns: windows of 128 = [64 gate | the same 64 up] (h columns n0 + window * 64 + [0, 64)).
// hi_bar (M = 256): columns [192, 256) are read first and released on it (a merged tail of the next tile
// borrows them), then the rest.
template <int kFuse>
__device__ __forceinline__ void drain_acc(const LayerArgs& la, const LTile& tl, uint32_t tacc, int row_in_tile,
                                          int ncols, int acc_off, bool valid, uint64_t* hi_bar, int lane) {
  const int H = la.H, d = la.d;
  const int64_t r = tl.m0 + row_in_tile;
  uint32_t hi0[32], hi1[32];  // columns [192, 256) when read first
  if (hi_bar) {
    tc::tmem_ld32(tacc + 192u, hi0);
    tc::tmem_ld32(tacc + 224u, hi1);
    tc::tmem_wait_ld();
    release_cols(hi_bar, lane);
  }
  if (tl.mode == 0) {
    __nv_bfloat16* orow = la.h + r * d;
    auto gu32 = [&](int hcol, const uint32_t (&gr)[32], const uint32_t (&ur)[32]) {
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = tc::silu(__uint_as_float(gr[j])) * __uint_as_float(ur[j]);
      if (valid) store_row_bf16x32(orow + hcol, v, d - hcol);
    };
    const int nw = ncols / 128;
    if (hi_bar) {  // window 1 first: its up half is in registers
      const int hcol1 = tl.n0 + (acc_off + 128) / 2;
      uint32_t gr[32];
      tc::tmem_ld32(tacc + 128u, gr);
      tc::tmem_wait_ld();
      gu32(hcol1, gr, hi0);
      tc::tmem_ld32(tacc + 160u, gr);
      tc::tmem_wait_ld();
      gu32(hcol1 + 32, gr, hi1);
    }
#pragma unroll 1
    for (int w = 0; w < (hi_bar ? 1 : nw); ++w) {
      const uint32_t wbase = tacc + static_cast<uint32_t>(w * 128);
      const int hcol0 = tl.n0 + (acc_off + w * 128) / 2;
#pragma unroll 1
      for (int c = 0; c < 64; c += 32) {
        uint32_t gr[32], ur[32];
        tc::tmem_ld32(wbase + c, gr);
        tc::tmem_ld32(wbase + 64 + c, ur);
        tc::tmem_wait_ld();
        gu32(hcol0 + c, gr, ur);
      }
    }
    return;
  }
  __nv_bfloat16* orow;
  const __nv_bfloat16* rrow = nullptr;
  bool valid_row = valid;
  if constexpr (kFuse == 2) {
    const int64_t v = valid ? static_cast<int64_t>(__ldg(la.fz.src + r)) : -1;
    valid_row = valid && v >= 0 && v < la.vrows * la.npeer;
    const int p = valid_row ? static_cast<int>(v / la.vrows) : 0;
    const int64_t ii = valid_row ? v - p * la.vrows : 0;
    __nv_bfloat16* py = la.peer_y[0];
    const __nv_bfloat16* pr = la.peer_res[0];
#pragma unroll
    for (int j = 1; j < kMaxPeers; ++j)
      if (p == j) {
        py = la.peer_y[j];
        pr = la.peer_res[j];
      }
    orow = py + ii * H;
    rrow = pr ? pr + ii * H : nullptr;
  } else {
    int64_t orow_idx = r;
    if constexpr (kFuse == 1) {
      orow_idx = valid ? (la.fz.src ? __ldg(la.fz.src + r) : r) : 0;
      valid_row = valid && orow_idx >= 0 && orow_idx < la.fz.rows;
    }
    orow = la.y + orow_idx * H;
    rrow = (kFuse == 1 && la.fz.residual) ? la.fz.residual + orow_idx * H : nullptr;
  }
  auto chunk = [&](int c, const uint32_t (&vr)[32]) {
    const int col = tl.n0 + acc_off + c;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(vr[j]);
    if (valid_row) {
      if (rrow) add_bf16x32(rrow + col, v, H - col);
      store_row_bf16x32(orow + col, v, H - col);
    }
  };
  if (hi_bar) {
    chunk(192, hi0);
    chunk(224, hi1);
  }
  const int nlo = hi_bar ? 192 : ncols;
#pragma unroll 1
  for (int c = 0; c < nlo; c += 32) {
    uint32_t vr[32];
    tc::tmem_ld32(tacc + static_cast<uint32_t>(c), vr);
    tc::tmem_wait_ld();
    chunk(c, vr);
  }
}

// Epilogue of a merged gate/up tail. Its MMAs are two M = 128 pair MMAs (A = this CTA's 64 gate rows, then
// its 64 up rows of the tile's own weight stage; N = the tail's rows rounded up to 16), so in the "2x2"
// layout lane l < 64 holds neuron l for tail rows [0, N/2), lane 64 + l the same neuron for rows [N/2, N), with
// gate at columns [0, N/2) of the borrowed region and up at [32, 32 + N/2): both factors in the same lane.
// Warp q: neurons 32 (q & 1) + lane, tail rows (q >> 1) * N/2 + [0, N/2). Both loads first, then the columns
// are released (hi_bar) before the stores.
__device__ __forceinline__ void tail_gu_epilogue(const LayerArgs& la, const LTile& tt, uint32_t tacc, uint32_t cta,
                                                 int q, int lane, bool store, uint64_t* hi_bar) {
  const int d = la.d;
  const int half = ((tt.rows + 15) & ~15) / 2;
  uint32_t gr[32], ur[32];
  tc::tmem_ld32(tacc, gr);
  tc::tmem_ld32(tacc + 32u, ur);
  tc::tmem_wait_ld();
  release_cols(hi_bar, lane);
  const int neuron = tt.n0 + 64 * static_cast<int>(cta) + 32 * (q & 1) + lane;
  const int tok0 = (q >> 1) * half;
  if (!store || neuron >= d) return;
  __nv_bfloat16* hcol = la.h + neuron;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int tok = tok0 + j;
    if (j >= half || tok >= tt.rows) break;  // warp-uniform
    hcol[static_cast<int64_t>(tt.m0 + tok) * d] =
        __float2bfloat16_rn(tc::silu(__uint_as_float(gr[j])) * __uint_as_float(ur[j]));
  }
}

// a5 inside the expert FFN (pdl == 3): x_sorted[r] = x[src[r] / k]. Row r belongs to epilogue warp r % nw of
// the grid; a warp copies its rows in ascending order while it waits for an accumulator, but only rows up to the
// end of the segment after the one its awaited tile belongs to — so the 128 MB of row moves spread over the
// gate/up phase (a segment's rows land while the previous segment's tiles run) instead of competing for HBM
// with the first tiles' weights, and every row a running tile needs is copied by warps that are themselves
// waiting on tiles of that segment or earlier (which complete: their rows were copied first). Rows left when
// a warp runs out of tiles are copied before it exits. Per row: 8 x 16 B loads in flight per lane, then a
// generic -> async proxy fence and a release add on its segment's copied-row counter (the producers wait for
// a segment's count once per CTA); a bad index is reported and its row still counted.
struct RowCopier {
  int64_t next, step;  // this warp's next row, and the stride (epilogue warps in the grid)
  int seg;             // segment of `next` (rows ascend, so a cursor)
};
__device__ __forceinline__ void copy_row(const LayerArgs& la, int64_t r, int lane, RowCopier& rc) {
  constexpr int kU = 8;
  const int vec = la.dvec;
  const int64_t nrows = la.fz.rows;
  const int32_t sl = __ldg(la.dsrc + r);
  if (sl < 0 || sl >= nrows) {
    if (lane == 0 && la.dev_status) atomicOr(la.dev_status, README_DEV_BAD_INDEX);
  } else {
    const uint4* srow = la.dx + (sl / la.dk) * static_cast<int64_t>(vec);
    uint4* drow = reinterpret_cast<uint4*>(la.dxs) + r * vec;
    int i = lane;
    for (; i + (kU - 1) * kWarp < vec; i += kU * kWarp) {
      uint4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = ld_nc_v4(srow + i + u * kWarp);
#pragma unroll
      for (int u = 0; u < kU; ++u) st_v4(drow + i + u * kWarp, v[u]);
    }
    for (; i < vec; i += kWarp) st_v4(drow + i, ld_nc_v4(srow + i));
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncwarp();
  while (rc.seg + 1 < la.nseg && r >= __ldg(la.offsets + rc.seg + 1)) ++rc.seg;
  if (lane == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(la.seg_rows + rc.seg) : "memory");
  }
}
// Wait for an accumulator phase, copying this warp's rows below `limit` meanwhile.
__device__ __forceinline__ void wait_copying(const LayerArgs& la, uint64_t* bar, uint32_t parity, RowCopier& rc,
                                             int64_t limit, int lane) {
  while (!__all_sync(0xffffffffu, tc::mbar_test_cluster(bar, parity))) {
    if (rc.next < limit) {
      copy_row(la, rc.next, lane, rc);
      rc.next += rc.step;
    } else {
      tc::mbar_wait_cluster(bar, parity);
      break;
    }
  }
}

// Epilogue of a merged down tail (same two-M = 128 layout as tail_gu_epilogue): lane l < 64 holds output column
// n0 + 128 cta + l (first MMA, columns [0, N/2) of the region) and n0 + 128 cta + 64 + l (second, [32, 32 + N/2))
// for tail rows [0, N/2), lane 64 + l the same columns for rows [N/2, N). Each row goes where the normal down
// epilogue sends it (y_sorted, y[src[r]] + residual, or the source rank's row).
template <int kFuse>
__device__ __forceinline__ void tail_dn_epilogue(const LayerArgs& la, const LTile& tt, uint32_t tacc, uint32_t cta,
                                                 int q, int lane, bool store, uint64_t* hi_bar) {
  const int H = la.H;
  const int half = ((tt.rows + 15) & ~15) / 2;
  uint32_t ra[32], rb[32];
  tc::tmem_ld32(tacc, ra);
  tc::tmem_ld32(tacc + 32u, rb);
  tc::tmem_wait_ld();
  release_cols(hi_bar, lane);
  if (!store) return;
  const int cola = tt.n0 + 128 * static_cast<int>(cta) + 32 * (q & 1) + lane, colb = cola + 64;
  const int tok0 = (q >> 1) * half;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int tok = tok0 + j;
    if (j >= half || tok >= tt.rows) break;  // warp-uniform
    const int64_t rr = tt.m0 + tok;
    __nv_bfloat16* orow;
    const __nv_bfloat16* rrow = nullptr;
    bool vrow = true;
    if constexpr (kFuse == 2) {
      const int64_t v = static_cast<int64_t>(__ldg(la.fz.src + rr));
      vrow = v >= 0 && v < la.vrows * la.npeer;
      const int p = vrow ? static_cast<int>(v / la.vrows) : 0;
      const int64_t i = vrow ? v - p * la.vrows : 0;
      __nv_bfloat16* py = la.peer_y[0];
      const __nv_bfloat16* pr = la.peer_res[0];
#pragma unroll
      for (int jj = 1; jj < kMaxPeers; ++jj)
        if (p == jj) {
          py = la.peer_y[jj];
          pr = la.peer_res[jj];
        }
      orow = py + i * H;
      rrow = pr ? pr + i * H : nullptr;
    } else {
      int64_t oi = rr;
      if constexpr (kFuse == 1) {
        oi = la.fz.src ? static_cast<int64_t>(__ldg(la.fz.src + rr)) : rr;
        vrow = oi >= 0 && oi < la.fz.rows;
        if (!vrow) oi = 0;
        rrow = la.fz.residual ? la.fz.residual + oi * H : nullptr;
      }
      orow = la.y + oi * H;
    }
    if (!vrow) continue;
    float va = __uint_as_float(ra[j]), vb = __uint_as_float(rb[j]);
    if (cola < H) {
      if (rrow) va += __bfloat162float(rrow[cola]);
      orow[cola] = __float2bfloat16_rn(va);
    }
    if (colb < H) {
      if (rrow) vb += __bfloat162float(rrow[colb]);
      orow[colb] = __float2bfloat16_rn(vb);
    }
  }
}

// Tile-id queue of the dynamic tile order (one per CTA, kTQ slots). Consumers pop in order; the leader's
// producer pushes after every consumer released the slot. Ids >= the tile count end every role's loop.
struct TileQ {
  int slot = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next() {
    if (++slot == kTQ) {
      slot = 0;
      ph ^= 1u;
    }
  }
};
// The leader CTA's slot is a plain shared store + release arrive; the peer's is an st.async that completes
// transaction bytes on the peer's barrier, so no consumer needs a cluster-scope acquire (whose L1 invalidate
// made the read-only offsets loads of the next tile decode miss).
// The consumer's release of a slot is a relaxed arrive once the id is in a register (the shuffle needs the
// loaded value): a release arrive would first wait for all of the warp's outstanding global stores (the
// epilogue's rows) — measured as ~2K idle SM cycles per tile in the MMA pipe.
template <class SM>
__device__ __forceinline__ int tq_pop(SM& s, TileQ& q, int lane) {
  tc::mbar_wait(&s.tq_full[q.slot], q.ph);
  const int t = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile int*>(&s.tq[q.slot]), 0);
  if (lane == 0) tc::mbar_arrive_cluster_relaxed(&s.tq_empty[q.slot], 0);
  q.next();
  return t;
}
template <class SM>
__device__ __forceinline__ void tq_push(SM& s, TileQ& q, int t, int lane) {
  tc::mbar_wait(&s.tq_empty[q.slot], q.ph ^ 1u);
  if (lane == 0) {
    tc::arrive_expect_tx_cluster(&s.tq_full[q.slot], 1, 4u);
    tc::st_async_cluster_u32(&s.tq[q.slot], &s.tq_full[q.slot], 1, static_cast<uint32_t>(t));
    *reinterpret_cast<volatile int*>(&s.tq[q.slot]) = t;
    tc::mbar_arrive(&s.tq_full[q.slot]);
  }
  __syncwarp();
  q.next();
}

// Lab builds only (README_NVCC_EXTRA=-DREADME_FFN_MAXREG=n): cap the single-launch kernel's registers.
#ifdef README_FFN_MAXREG
#define README_FFN_BOUNDS __maxnreg__(README_FFN_MAXREG)
#else
#define README_FFN_BOUNDS __launch_bounds__(kThreads, 1)
#endif
template <int kFuse, int kMT>
__global__ void __cluster_dims__(2, 1, 1) README_FFN_BOUNDS
ffn_layer2_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmG,
                  const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmH,
                  const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX16,
                  const __grid_constant__ CUtensorMap tmH16, const __grid_constant__ CUtensorMap tmG16,
                  const __grid_constant__ CUtensorMap tmU16, LayerArgs la) {
  extern __shared__ uint8_t smem_raw[];
  using SM = typename std::conditional<kMT == 256, SmemL, SmemLD>::type;
  constexpr int kS = kMT == 256 ? kStagesL : kStagesLD;  // ring stages
  constexpr int kSA = kMT == 256 ? kStageAL : kStageAD;  // A bytes per stage per CTA (+ tail slot at 256)
  const bool merge = kMT == 256 && la.merge != 0;
  static_assert(kMT == 256 || kMT == 128, "kMT");
  SM& s = *reinterpret_cast<SM*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
  const uint32_t cta = tc::cluster_ctarank();
  const bool leader = cta == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int H = la.H, d = la.d, E = la.E, nseg = la.nseg;
  const int32_t* __restrict__ offs = la.offsets;
  constexpr int kN = 256;  // MMA N (both CTAs' 128-row B halves)
  const int NT1 = (d + kBN1 - 1) / kBN1, NT2 = (H + kBN2 - 1) / kBN2;
  const int KB1 = (H + kBK - 1) / kBK, KB2 = (d + kBK - 1) / kBK;
  const uint32_t ready_target = static_cast<uint32_t>(NT1) * 8u;

  for (int i = tid; i < kXokWords; i += kThreads) s.xok[i] = 0u;
  for (int i = tid; i < kMaxSeg / 32; i += kThreads) s.segok[i] = 0u;
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmX);
    tc::prefetch_tmap(&tmG);
    tc::prefetch_tmap(&tmU);
    tc::prefetch_tmap(&tmH);
    tc::prefetch_tmap(&tmD);
    if (la.swap_rows > 0 || kMT == 256) {
      tc::prefetch_tmap(&tmX16);
      tc::prefetch_tmap(&tmH16);
      tc::prefetch_tmap(&tmG16);
      tc::prefetch_tmap(&tmU16);
    }
  }
  if (warp == 1) tc::tmem_alloc<2>(&s.tmem_base, kTmemCols);
  if (la.pdl == 3) tc::pdl_wait();  // the route's offsets and src
  // total m-tiles (every thread: nseg reads of the read-only offsets, no shared table)
  int mtiles = 0;
  for (int g = 0; g < nseg; ++g) mtiles += seg_mtiles<kMT>(__ldg(offs + g + 1) - __ldg(offs + g), merge);
  if (tid == 0) {
    for (int i = 0; i < kS; ++i) {
      tc::mbar_init(&s.full[i], 1);
      tc::mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s.tfull[i], 1);
      tc::mbar_init(&s.tempty[i], 8);
      tc::mbar_init(&s.hi_free[i], 8);
    }
    for (int i = 0; i < kTQ; ++i) {
      tc::mbar_init(&s.tq_full[i], 1);
      tc::mbar_init(&s.tq_empty[i], kTQConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after();
  const int T1 = mtiles * NT1;
  const int ntiles = T1 + mtiles * NT2;
  const uint32_t tmem_base = s.tmem_base;
  // Launched with PDL behind the dispatch (la.pdl): everything above only read the routing offsets, which
  // the route kernel wrote before the dispatch began. Before waiting for the dispatch's x_sorted, start
  // pulling this pair's first gate/up weight tile into L2 — weights do not depend on the dispatch.
  if (la.pdl) {
    if (warp == 0 && lane == 0 && pair < T1) {
      Cursor c;
      const LTile tl = decode_ltile<kMT>(offs, pair, nseg, T1, NT1, NT2, la.swap_rows, c, la.order != 0, merge);
      const int e = la.expert_slot ? __ldg(la.expert_slot + tl.g % E) : tl.g % E;
      const int nr = tl.n0 + 64 * static_cast<int>(cta);
      const int kbs = KB1 < kPrefetchK ? KB1 : kPrefetchK;
      for (int kb = 0; kb < kbs; ++kb) {
        tc::tma_prefetch_3d(&tmG, kb * kBK, nr, e);
        tc::tma_prefetch_3d(&tmU, kb * kBK, nr, e);
      }
    }
    if (la.pdl == 1) tc::pdl_wait();
  }
  if (la.trace && tid == 0) trace_min(la.trace, 2);
  // Tile sequence of this pair (static): pair, pair + npairs, ...

  if (warp == 0) {
    // ===== TMA producer (both CTAs; completion counted on the leader's barrier). The whole warp walks the
    // loop so coordinates and addresses stay in uniform registers; one elected lane issues. Each tile kind
    // gets its own K loop (no per-stage branching on the tile's shape). =====
    int stage = 0;
    uint32_t phase = 0;
    Cursor cur;
    const uint32_t full0 = tc::mapa(&s.full[0], 0);  // the leader's barriers, as cluster addresses
    TileQ tq;
    const bool dyn = la.dyn != 0;
    // every pair's first tile is its index; with the dynamic order the leader's producer claims the next one
    // la.claim_ahead (knob ffn_claim, 24) K steps before the end of this tile's loads — late enough that the
    // claim order follows the pairs' finishing order, early enough to hide the atomic — and publishes it once
    // this tile's loads are issued
    for (int t = pair; t < ntiles;) {
      uint32_t claim = 0;
      const bool claimer = dyn && leader;
      bool claimed = !claimer;
      auto claim_next = [&]() {
        if (lane == 0) claim = atomicAdd(la.tile_ctr, 1u);
        claimed = true;
      };
      int t_next = t + npairs;
      const LTile tl = decode_ltile<kMT>(offs, t, nseg, T1, NT1, NT2, la.swap_rows, cur, la.order != 0, merge);
      const int e = la.expert_slot ? __ldg(la.expert_slot + tl.g % E) : tl.g % E;
      // Activation rows this CTA stages per K step: 128 (M = 256), 64 (M = 128) or, for a swap-AB tile, half
      // of its N = rows rounded up to 16 (in 16-row boxes)
      const int nsw = tl.swap ? ((tl.rows + 15) & ~15) : 0;
      const int a_rows = tl.swap ? nsw / 2 : (tl.m256 ? 128 : 64);
      const int a_row0 = tl.m0 + static_cast<int>(cta) * a_rows;
      const int nact = (a_rows + 15) / 16;  // swap tiles: 16-row activation boxes
      // merged tail: half of its N = trows rounded up to 16 per CTA, 16-row boxes into the stage's tail slot
      const int t_rows = ((tl.trows + 15) & ~15) / 2;
      const int t_row0 = tl.tm0 + static_cast<int>(cta) * t_rows;
      const int tact = (t_rows + 15) / 16;
      // A tile of ≤ 64 rows: every row the second CTA would stage is past the tile's end, so it skips its A
      // load (its MMA rows read stale shared memory; row m of the product depends on A row m only and rows
      // past tl.rows are never stored). Knob ffn_askip = 0 loads them anyway (A/B).
      const bool a_skip = la.askip && !tl.swap && !tl.m256 && tl.rows <= 64;
      const uint32_t bytes = tl.swap ? 2u * static_cast<uint32_t>(nact * 16 * 128 + 128 * 128)
                                     : 2u * static_cast<uint32_t>(a_rows * 128 + 128 * 128 + tact * 2048) -
                                           (a_skip ? static_cast<uint32_t>(a_rows * 128) : 0u);
      if (tl.mode == 0 && la.pdl == 3) {
        // a5 inside this launch: wait until every row of the tile's segment is copied (one counter per
        // segment, seen once per CTA), not per row: the per-row flag polls at every new m-tile cost the
        // producer ~1.5 us each
        const int g = tl.g;
        if (!(s.segok[g >> 5] >> (g & 31) & 1u)) {
          const uint32_t need = static_cast<uint32_t>(__ldg(offs + g + 1) - __ldg(offs + g));
          uint32_t spins = 0;
          while (ld_acquire_u32(la.seg_rows + g) < need) {
            __nanosleep(64);
            if (++spins >= la.spin_limit) {
              if (lane == 0) sched_give_up(la);
              break;
            }
          }
          if (lane == 0) s.segok[g >> 5] |= 1u << (g & 31);
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __syncwarp();
        }
      }
      if (tl.mode == 0 && la.pdl == 2) {
        // wait until the dispatch has written this CTA's A rows of the tile (rows past the segment's end are
        // padding: their products are never stored, so they are not waited for), merged tail rows included
        const int mid = tl.mid;
        const bool cached = mid < kXokWords * 32 && (s.xok[mid >> 5] >> (mid & 31) & 1u);
        if (!cached) {
          const int lo = a_row0, hi = min(a_row0 + a_rows, tl.m0 + tl.rows);
          const int tlo = t_row0, thi = min(t_row0 + t_rows, tl.tm0 + tl.trows);
          uint32_t spins = 0;
          for (;;) {
            bool ok = true;
            for (int r = lo + lane; r < hi; r += kWarp) ok = ok && ld_acquire_u32(la.xready + r) != 0u;
            for (int r = tlo + lane; r < thi; r += kWarp) ok = ok && ld_acquire_u32(la.xready + r) != 0u;
            if (__all_sync(0xffffffffu, ok)) break;
            __nanosleep(64);
            if (++spins >= la.spin_limit) {
              if (lane == 0) sched_give_up(la);
              break;
            }
          }
          if (lane == 0 && mid < kXokWords * 32) s.xok[mid >> 5] |= 1u << (mid & 31);
          if (la.trace && lane == 0) trace_min(la.trace, 3);
          // once per (m-tile, CTA): later TMA loads of these rows by this thread are ordered after it. A
          // fence per tile would also wait for this thread's in-flight TMA loads — draining the ring at
          // every tile boundary (measured: +3 us per decode step)
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __syncwarp();
        }
      }
      if (tl.mode == 1) {
        // wait until every gate/up tile of this m-tile has published its h rows
        const uint32_t* rp = la.ready + tl.mid;
        uint32_t spins = 0;
        while (ld_acquire_u32(rp) < ready_target) {
          __nanosleep(128);
          if (++spins >= la.spin_limit) {
            if (lane == 0) sched_give_up(la);
            break;
          }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
      }
      const int nrg = tl.n0 + 64 * static_cast<int>(cta), nrd = tl.n0 + 128 * static_cast<int>(cta);
      // one ring step per K block: wait for the slot, arm the leader's barrier, issue this tile kind's loads
      auto kloop = [&](int KB, auto&& issue) {
        for (int kb = 0; kb < KB; ++kb) {
          tc::mbar_wait(&s.empty[stage], phase ^ 1);
          if (tc::elect_one()) {
            const uint32_t fb = full0 + static_cast<uint32_t>(stage * 8);
            if (leader) tc::mbar_expect_tx(&s.full[stage], bytes);
            issue(s.a[stage], s.b[stage], fb, kb * kBK);
          }
          __syncwarp();
          if (++stage == kS) {
            stage = 0;
            phase ^= 1;
          }
          if (!claimed && kb == KB - la.claim_ahead) claim_next();
        }
      };
      // gate/up weight rows of a swap-AB tile as 4 x [16 gate | the same 16 up], so each epilogue warp's 32 TMEM
      // lanes hold both factors of its 16 neurons
      auto load_gu16 = [&](uint8_t* sb, uint32_t fb, int k0) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          tc::tma_load_3d_2sm(&tmG16, sb + (32 * q4) * 128, fb, k0, nrg + 16 * q4, e);
          tc::tma_load_3d_2sm(&tmU16, sb + (32 * q4 + 16) * 128, fb, k0, nrg + 16 * q4, e);
        }
      };
      if (tl.swap) {
        // swap-AB tile: the activations are the MMA's B side (nsw/2 rows here, 16-row boxes); the weights its
        // A side.
        const CUtensorMap* mA16 = tl.mode == 0 ? &tmX16 : &tmH16;
        if (tl.mode == 0) {
          kloop(KB1, [&](uint8_t* sa, uint8_t* sb, uint32_t fb, int k0) {
            for (int i = 0; i < nact; ++i) tc::tma_load_2d_2sm(mA16, sa + i * 2048, fb, k0, a_row0 + 16 * i);
            load_gu16(sb, fb, k0);
          });
        } else {
          kloop(KB2, [&](uint8_t* sa, uint8_t* sb, uint32_t fb, int k0) {
            for (int i = 0; i < nact; ++i) tc::tma_load_2d_2sm(mA16, sa + i * 2048, fb, k0, a_row0 + 16 * i);
            tc::tma_load_3d_2sm(&tmD, sb, fb, k0, nrd, e);
            tc::tma_load_3d_2sm(&tmD, sb + 64 * 128, fb, k0, nrd + 64, e);
          });
        }
      } else if (tl.trows > 0) {
        // full m-tile carrying a merged tail: A (128 rows), the tail's rows (tail slot), the weights
        if (tl.mode == 0) {
          kloop(KB1, [&](uint8_t* sa, uint8_t* sb, uint32_t fb, int k0) {
            tc::tma_load_2d_2sm(&tmX, sa, fb, k0, a_row0);
            tc::tma_load_2d_2sm(&tmX, sa + 64 * 128, fb, k0, a_row0 + 64);
            for (int i = 0; i < tact; ++i) tc::tma_load_2d_2sm(&tmX16, sa + kTailSlot + i * 2048, fb, k0, t_row0 + 16 * i);
            tc::tma_load_3d_2sm(&tmG, sb, fb, k0, nrg, e);
            tc::tma_load_3d_2sm(&tmU, sb + 64 * 128, fb, k0, nrg, e);
          });
        } else {
          kloop(KB2, [&](uint8_t* sa, uint8_t* sb, uint32_t fb, int k0) {
            tc::tma_load_2d_2sm(&tmH, sa, fb, k0, a_row0);
            tc::tma_load_2d_2sm(&tmH, sa + 64 * 128, fb, k0, a_row0 + 64);
            for (int i = 0; i < tact; ++i) tc::tma_load_2d_2sm(&tmH16, sa + kTailSlot + i * 2048, fb, k0, t_row0 + 16 * i);
            tc::tma_load_3d_2sm(&tmD, sb, fb, k0, nrd, e);
            tc::tma_load_3d_2sm(&tmD, sb + 64 * 128, fb, k0, nrd + 64, e);
          });
        }
      } else {
        const bool loadA = !(a_skip && cta == 1), A2 = tl.m256;
        if (tl.mode == 0) {
          kloop(KB1, [&](uint8_t* sa, uint8_t* sb, uint32_t fb, int k0) {
            if (loadA) tc::tma_load_2d_2sm(&tmX, sa, fb, k0, a_row0);
            if (A2) tc::tma_load_2d_2sm(&tmX, sa + 64 * 128, fb, k0, a_row0 + 64);
            // 64 rows of W_gate then the same rows of W_up
            tc::tma_load_3d_2sm(&tmG, sb, fb, k0, nrg, e);
            tc::tma_load_3d_2sm(&tmU, sb + 64 * 128, fb, k0, nrg, e);
          });
        } else {  // 128 rows of W_down in boxes of 64
          kloop(KB2, [&](uint8_t* sa, uint8_t* sb, uint32_t fb, int k0) {
            if (loadA) tc::tma_load_2d_2sm(&tmH, sa, fb, k0, a_row0);
            if (A2) tc::tma_load_2d_2sm(&tmH, sa + 64 * 128, fb, k0, a_row0 + 64);
            tc::tma_load_3d_2sm(&tmD, sb, fb, k0, nrd, e);
            tc::tma_load_3d_2sm(&tmD, sb + 64 * 128, fb, k0, nrd + 64, e);
          });
        }
      }
      if (claimer) {
        if (!claimed) claim_next();  // tiles shorter than claim_ahead K steps
        t_next = static_cast<int>(__shfl_sync(0xffffffffu, claim, 0)) + npairs;
        tq_push(s, tq, t_next, lane);  // the end marker (>= ntiles) too
      }
      t = dyn && !leader ? tq_pop(s, tq, lane) : t_next;
    }
  } else if (warp == 1) {
    if (leader) {
      // ===== MMA issuer (leader CTA): the whole warp walks the loop (descriptors in uniform registers),
      // one elected lane issues each tcgen05.mma / commit =====
      constexpr uint32_t idesc256 = tc::idesc_bf16(256, kN);
      constexpr uint32_t idesc128 = tc::idesc_bf16(128, kN);
      const uint64_t adesc0 = tc::sdesc_sw128(tc::smem_u32(s.a[0])), bdesc0 = tc::sdesc_sw128(tc::smem_u32(s.b[0]));
      int stage = 0;
      uint32_t phase = 0;
      Cursor cur;
      int i = 0;
      int huse0 = 0, huse1 = 0;  // uses of each accumulator's columns [192, 256) issued so far (hi_free phases)
      auto next_use = [&](int b) { return b ? huse1++ : huse0++; };
      TileQ tq;
      const bool dyn = la.dyn != 0;
      for (int t = pair; t < ntiles; t = dyn ? tq_pop(s, tq, lane) : t + npairs, ++i) {
        const LTile tl = decode_ltile<kMT>(offs, t, nseg, T1, NT1, NT2, la.swap_rows, cur, la.order != 0, merge);
        // swap-AB tile: M = 256 weight rows (128 per CTA, from the B slots), N = rows rounded up to 16 (from the
        // A slots): operands exchanged, accumulator lane = weight row, column = the tile's row
        const uint32_t idesc = tl.swap ? tc::idesc_bf16(256, (tl.rows + 15) & ~15) : (tl.m256 ? idesc256 : idesc128);
        const int acc = i & 1;
        const uint32_t use = static_cast<uint32_t>(i >> 1);
        uint64_t* trec = (la.ttrace && i < la.ttrace_max) ? la.ttrace + (static_cast<int64_t>(pair) * la.ttrace_max + i) * 8 : nullptr;
        const uint64_t c_wait0 = trec ? clock64() : 0;
        tc::mbar_wait_cluster(&s.tempty[acc], (use & 1u) ^ 1u);
        if (tl.m256) {  // columns [192, 256): the previous tile's merged tail may still hold them
          const int n = next_use(acc);
          tc::mbar_wait_cluster(&s.hi_free[acc], static_cast<uint32_t>(n & 1) ^ 1u);
        }
        tc::fence_after();
        uint64_t c_full = 0;
        if (trec && lane == 0) {
          const uint64_t c = clock64();
          trec[0] = globaltimer_ns();
          trec[1] = c;
          trec[7] = static_cast<uint64_t>(t) | ((c - c_wait0) << 32);
        }
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * 256);
        const int KB = tl.mode == 0 ? KB1 : KB2;
        // +1 in a descriptor's address field = +16 B: stage strides and the 32-B K steps are constants
        const uint64_t a0 = tl.swap ? bdesc0 : adesc0, b0 = tl.swap ? adesc0 : bdesc0;
        const uint32_t astep = tl.swap ? (kStageB >> 4) : (kSA >> 4), bstep = tl.swap ? (kSA >> 4) : (kStageB >> 4);
        // A merged tail (M = 256 weight rows from the B slot x N = its rows from the stage's tail slot) goes to
        // the other accumulator's columns [192, 256) once the epilogue has drained their previous user; until
        // then up to kMaxDefer stages keep their tail MMAs (and their slot) pending.
        const bool tail = tl.trows > 0;
        const int oth = acc ^ 1;
        const uint32_t t_tmem = tmem_base + static_cast<uint32_t>(oth * 256 + 192);
        // two M = 128 swap-AB pair MMAs per K step, the first 64 then the last 64 of the CTA's 128 weight rows
        // (gate/up: its 64 gate rows, then its 64 up rows, so both factors of a neuron share a lane; down: output
        // columns +0..63, +64..127), into columns +0 / +32 of the borrowed region. Per weight byte re-read they ran
        // faster than one M = 256 MMA (~25 vs ~63 cycles per MMA, tile trace, profiles/SUMMARY.md r02).
        const uint32_t tidesc = tc::idesc_bf16(128, (tl.trows + 15) & ~15);
        uint32_t tpar = 0;
        bool tok = true;
        if (tail) {
          const int n = next_use(oth);
          tpar = static_cast<uint32_t>(n & 1) ^ 1u;
          tok = false;
        }
        int pend = 0, pstage = stage, pkb = 0;
        auto issue_tails = [&]() {
          for (int p = 0; p < pend; ++p) {
            int st = pstage + p;
            if (st >= kS) st -= kS;
            const int kbp = pkb + p;
            const uint64_t wd = bdesc0 + static_cast<uint64_t>(st * (kStageB >> 4));
            const uint64_t td = adesc0 + static_cast<uint64_t>(st * (kSA >> 4) + (kTailSlot >> 4));
            if (tc::elect_one()) {
#pragma unroll
              for (int kk = 0; kk < kBK / kUK; ++kk) {
                const uint32_t acc_flag = (kbp | kk) != 0 ? 1u : 0u;
                tc::mma_f16<2>(t_tmem, wd + static_cast<uint64_t>(kk * 2), td + static_cast<uint64_t>(kk * 2), tidesc,
                               acc_flag);
                // the second 64 weight rows: 8 KB further into the stage
                tc::mma_f16<2>(t_tmem + 32u, wd + static_cast<uint64_t>((64 * 128 >> 4) + kk * 2),
                               td + static_cast<uint64_t>(kk * 2), tidesc, acc_flag);
              }
              tc::commit_2sm_mc(&s.empty[st], 0x3);
            }
            __syncwarp();
          }
          pend = 0;
        };
        for (int kb = 0; kb < KB; ++kb) {
          const uint64_t c0 = trec ? clock64() : 0;
          tc::mbar_wait_cluster(&s.full[stage], phase);
          if (trec) c_full += clock64() - c0;
          tc::fence_after();
          const uint64_t ad = a0 + static_cast<uint64_t>(stage * astep), bd = b0 + static_cast<uint64_t>(stage * bstep);
          if (tc::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kBK / kUK; ++kk)
              tc::mma_f16<2>(d_tmem, ad + static_cast<uint64_t>(kk * 2), bd + static_cast<uint64_t>(kk * 2), idesc,
                             (kb | kk) != 0 ? 1u : 0u);
            if (!tail) tc::commit_2sm_mc(&s.empty[stage], 0x3);
          }
          __syncwarp();
          if (tail) {
            if (pend == 0) {
              pstage = stage;
              pkb = kb;
            }
            ++pend;
            if (!tok) {
              bool ok = __all_sync(0xffffffffu, tc::mbar_test_cluster(&s.hi_free[oth], tpar));
              if (!ok && pend >= kMaxDefer) {
                tc::mbar_wait_cluster(&s.hi_free[oth], tpar);
                ok = true;
              }
              if (ok) tc::fence_after();
              tok = ok;
            }
            if (tok) issue_tails();
          }
          if (++stage == kS) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (tail && pend > 0) {
          if (!tok) {
            tc::mbar_wait_cluster(&s.hi_free[oth], tpar);
            tc::fence_after();
          }
          issue_tails();
        }
        if (tc::elect_one()) tc::commit_2sm_mc(&s.tfull[acc], 0x3);
        __syncwarp();
        if (trec && lane == 0) {
          trec[2] = clock64();
          trec[6] = c_full;
        }
      }
    }
  } else {
    // ===== epilogue: warps 2..5 of both CTAs =====
    const int q = warp & 3;
    RowCopier rc{static_cast<int64_t>(blockIdx.x) * 4 + (warp - 2), static_cast<int64_t>(gridDim.x) * 4, 0};
    if (la.pdl != 3) rc.next = la.fz.rows;  // nothing to copy
    Cursor cur;
    int i = 0;
    TileQ tq;
    const bool dyn = la.dyn != 0;
    for (int t = pair; t < ntiles; t = dyn ? tq_pop(s, tq, lane) : t + npairs, ++i) {
      const LTile tl = decode_ltile<kMT>(offs, t, nseg, T1, NT1, NT2, la.swap_rows, cur, la.order != 0, merge);
      const int acc = i & 1;
      const uint32_t use = static_cast<uint32_t>(i >> 1);
      if (rc.next < la.fz.rows) {
        // rows up to the end of the segment after this tile's (gate/up phase), or all of them (down phase)
        const int64_t limit = tl.mode == 0 ? static_cast<int64_t>(__ldg(offs + min(tl.g + 2, nseg))) : la.fz.rows;
        wait_copying(la, &s.tfull[acc], use & 1u, rc, limit, lane);
      } else {
        tc::mbar_wait_cluster(&s.tfull[acc], use & 1u);
      }
      tc::fence_after();
      uint64_t* trec = (la.ttrace && leader && q == 2 && lane == 0 && i < la.ttrace_max)
                           ? la.ttrace + (static_cast<int64_t>(pair) * la.ttrace_max + i) * 8 : nullptr;
      if (trec) trec[3] = clock64();
      // a readiness wait of this launch gave up: this tile may have been computed from unready rows, so it
      // (and every later tile) stores nothing
      const bool aborted = __shfl_sync(0xffffffffu, lane == 0 ? ld_volatile_u32(la.abort) : 0u, 0) != 0u;
      const uint32_t tacc = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * 256);
      // Accumulator columns of this warp's 32 rows: all kN (M=256), or half of them (M=128, "2x2" layout:
      // lanes 64-127 hold columns [kN/2, kN) at TMEM columns [0, kN/2)).
      int row_in_tile, ncols, acc_off;
      if (tl.m256) {
        row_in_tile = static_cast<int>(cta) * 128 + q * 32 + lane;
        ncols = kN;
        acc_off = 0;
      } else {
        row_in_tile = static_cast<int>(cta) * 64 + (q & 1) * 32 + lane;
        ncols = kN / 2;
        acc_off = (q >> 1) * (kN / 2);
      }
      if (tl.trows > 0) {  // merged tail first: it frees the other accumulator's columns [192, 256)
        LTile tt = tl;
        tt.m0 = tl.tm0;
        tt.rows = tl.trows;
        const uint32_t ttacc = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>((acc ^ 1) * 256 + 192);
        if (tl.mode == 0) tail_gu_epilogue(la, tt, ttacc, cta, q, lane, !aborted, &s.hi_free[acc ^ 1]);
        else tail_dn_epilogue<kFuse>(la, tt, ttacc, cta, q, lane, !aborted, &s.hi_free[acc ^ 1]);
      }
      if (tl.swap) swap_epilogue<kFuse>(la, tl, tacc, cta, q, lane, !aborted);
      else drain_acc<kFuse>(la, tl, tacc, row_in_tile, ncols, acc_off, row_in_tile < tl.rows && !aborted,
                                   tl.m256 ? &s.hi_free[acc] : nullptr, lane);
      if (trec) {
        trec[4] = clock64();
        trec[5] = globaltimer_ns();
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive_cluster_relaxed(&s.tempty[acc], 0);
        if (tl.mode == 0) {
          // publish this warp's share of the h tile to the down tiles (generic -> async proxy, then release);
          // an aborted tile still publishes, so its down tiles stop waiting (they store nothing either)
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(la.ready + tl.mid) : "memory");
        }
      }
    }
    for (; rc.next < la.fz.rows; rc.next += rc.step) copy_row(la, rc.next, lane, rc);  // rows not copied yet
  }

  if constexpr (kFuse == 2) __threadfence_system();  // remote rows performed before the ready signal
  if (la.pdl == 2) tc::pdl_wait();  // the dispatch is complete by now; keep the grid dependency explicit
  if (la.trace && tid == 0) trace_max(la.trace, 4);
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after();
  if (warp == 1) tc::tmem_dealloc<2>(tmem_base, kTmemCols);
}

// Per-device kernel attributes (max dynamic shared memory) and the co-residency limit of the single-launch
// kernels (CTA pairs that fit at once: the persistent grid never exceeds it).
struct DevInfo {
  cudaError_t err = cudaSuccess;
  int max_pairs[2] = {0, 0};  // [kMT == 128, kMT == 256]
};

const DevInfo& dev_info() {
  static std::once_flag once[64];
  static DevInfo info[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  std::call_once(once[dev], [&] {
    DevInfo& di = info[dev];
    const void* fns[3] = {reinterpret_cast<const void*>(ffn_gemm2_kernel<0, 0>),
                          reinterpret_cast<const void*>(ffn_gemm2_kernel<1, 0>),
                          reinterpret_cast<const void*>(ffn_gemm2_kernel<1, 1>)};
    for (int i = 0; i < 3 && di.err == cudaSuccess; ++i)
      di.err = cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
    const void* lfns[2][3] = {{reinterpret_cast<const void*>(ffn_layer2_kernel<0, 128>),
                               reinterpret_cast<const void*>(ffn_layer2_kernel<1, 128>),
                               reinterpret_cast<const void*>(ffn_layer2_kernel<2, 128>)},
                              {reinterpret_cast<const void*>(ffn_layer2_kernel<0, 256>),
                               reinterpret_cast<const void*>(ffn_layer2_kernel<1, 256>),
                               reinterpret_cast<const void*>(ffn_layer2_kernel<2, 256>)}};
    const size_t lsmem[2] = {kSmemBytesLD, kSmemBytesL};
    for (int v = 0; v < 2; ++v) {
      int mp = 1 << 30;
      for (int i = 0; i < 3 && di.err == cudaSuccess; ++i) {
        di.err = cudaFuncSetAttribute(lfns[v][i], cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(lsmem[v]));
        if (di.err != cudaSuccess) break;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * (num_sms() / 2));
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = lsmem[v];
        int n = 0;
        di.err = cudaOccupancyMaxActiveClusters(&n, lfns[v][i], &cfg);
        if (di.err == cudaSuccess && n < mp) mp = n;
      }
      di.max_pairs[v] = mp;
    }
  });
  return info[dev];
}

readme_status set_smem_attr() {
  const DevInfo& di = dev_info();
  if (di.err != cudaSuccess) return cuda_fail(di.err, "cudaFuncSetAttribute / cudaOccupancyMaxActiveClusters (expert FFN)");
  return README_OK;
}

}  // namespace

// One projection on CTA pairs. mode 0 (a6): A = x_sorted [rows, K=H], B0/B1 = W_gate/W_up [E][N=d][K],
// out = h [rows, d]. mode 1 (a7): A = h [rows, K=d], B0 = W_down [E][N=H][K], out = y_sorted [rows, H], or
// with src != null (k == 1 only) row r goes to out[src[r]] (+ residual): the fused combine.
readme_status launch_gemm_2cta(int mode, const __nv_bfloat16* A, int64_t rows, int32_t K, int32_t N, int32_t E,
                               int32_t nseg, const int32_t* offsets, const __nv_bfloat16* B0,
                               const __nv_bfloat16* B1, __nv_bfloat16* out, const int32_t* src,
                               const __nv_bfloat16* residual, cudaStream_t st) {
  if (rows == 0) return README_OK;
  if (nseg > kMaxSeg) {
    set_error("bf16 expert FFN supports at most %d segments (got %d)", kMaxSeg, nseg);
    return README_ERR_UNSUPPORTED;
  }
  readme_status rs = set_smem_attr();
  if (rs != README_OK) return rs;
  CUtensorMap mA, mB0, mB1;
  bool ok = tc::make_map_2d(&mA, A, K, rows, kBK, 64) && tc::make_map_3d(&mB0, B0, K, N, E, kBK, 64) &&
            (mode == 1 || tc::make_map_3d(&mB1, B1, K, N, E, kBK, 64));
  if (!ok) {
    set_error("cuTensorMapEncodeTiled failed (driver entry point missing or bad shape/alignment)");
    return README_ERR_CUDA;
  }
  if (mode == 1) mB1 = mB0;
  const int64_t mt_ub = nseg + (rows + 255) / 256;
  const int pairs = num_sms() / 2;  // no inter-CTA waits here: the grid need not be co-resident
  const int64_t tiles = mt_ub * ((N + (mode == 0 ? 127 : 255)) / (mode == 0 ? 128 : 256));
  const int grid = 2 * static_cast<int>(tiles < pairs ? tiles : pairs);
  const Fuse fz{src, static_cast<int>(rows), residual};
  if (mode == 0)
    ffn_gemm2_kernel<0, 0><<<grid, kThreads, kSmemBytes, st>>>(mA, mB0, mB1, K, N, E, nseg, offsets, out, fz);
  else if (src == nullptr && residual == nullptr)
    ffn_gemm2_kernel<1, 0><<<grid, kThreads, kSmemBytes, st>>>(mA, mB0, mB1, K, N, E, nseg, offsets, out, fz);
  else
    ffn_gemm2_kernel<1, 1><<<grid, kThreads, kSmemBytes, st>>>(mA, mB0, mB1, K, N, E, nseg, offsets, out, fz);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_gate_up_bf16(const __nv_bfloat16* xs, int64_t rows, int32_t H, int32_t E, int32_t d,
                                  int32_t nseg, const int32_t* offsets, const __nv_bfloat16* wg,
                                  const __nv_bfloat16* wu, __nv_bfloat16* h, cudaStream_t st) {
  return launch_gemm_2cta(0, xs, rows, H, d, E, nseg, offsets, wg, wu, h, nullptr, nullptr, st);
}

readme_status launch_down_bf16(const __nv_bfloat16* h, int64_t rows, int32_t H, int32_t E, int32_t d, int32_t nseg,
                               const int32_t* offsets, const __nv_bfloat16* wd, __nv_bfloat16* out,
                               const int32_t* src, const __nv_bfloat16* residual, cudaStream_t st) {
  return launch_gemm_2cta(1, h, rows, d, H, E, nseg, offsets, wd, nullptr, out, src, residual, st);
}

// Readiness region of the single-launch kernel: [down-tile counters: kMaxSeg + #128-row m-tiles][abort word]
// [pad][x_sorted row flags: rows] (the flags are used when the gather dispatch precedes the FFN, pdl == 2);
// one memset (or the route launch) zeroes all of it before every launch.
// then the tile counter, then kMaxSeg per-segment copied-row counters
int64_t ffn_layer_abort_index(int64_t rows) { return kMaxSeg + (rows + 127) / 128 + 1; }
size_t ffn_layer_xready_offset(int64_t rows) {
  return align_up(static_cast<size_t>(ffn_layer_abort_index(rows) + 2 + kMaxSeg) * sizeof(uint32_t), 256);
}
size_t ffn_layer_ready_bytes(int64_t rows, int32_t nseg) {
  (void)nseg;
  return ffn_layer_xready_offset(rows) + align_up(static_cast<size_t>(rows) * sizeof(uint32_t), 256);
}

readme_status launch_ffn_layer_2cta(const __nv_bfloat16* xs, int64_t rows, int32_t H, int32_t E, int32_t d,
                                    int32_t nseg, const int32_t* offsets, const __nv_bfloat16* wg,
                                    const __nv_bfloat16* wu, const __nv_bfloat16* wd, __nv_bfloat16* h,
                                    __nv_bfloat16* y, const int32_t* src, const __nv_bfloat16* residual,
                                    uint32_t* ready, uint32_t* dev_status, cudaStream_t st,
                                    const int32_t* expert_slot, int32_t n_slots, const PeerOut* peers,
                                    bool pdl, const uint32_t* xready, const SelfDispatch* sd) {
  if (rows == 0) return README_OK;
  if (sd && (!pdl || !xready || !sd->x || !sd->src || sd->k < 1 || (H * 2) % 16 != 0)) {
    set_error("expert FFN self-dispatch needs PDL, row flags, x, src, k >= 1 and 16-byte rows");
    return README_ERR_INVALID_ARG;
  }
  if (nseg > kMaxSeg) {
    set_error("bf16 expert FFN supports at most %d segments (got %d)", kMaxSeg, nseg);
    return README_ERR_UNSUPPORTED;
  }
  readme_status rs = set_smem_attr();
  if (rs != README_OK) return rs;
  CUtensorMap mX, mG, mU, mH, mD;
  const int32_t EW = expert_slot ? n_slots : E;  // outer extent of the weight tensors
  bool ok = tc::make_map_2d(&mX, xs, H, rows, kBK, 64) && tc::make_map_3d(&mG, wg, H, d, EW, kBK, 64) &&
            tc::make_map_3d(&mU, wu, H, d, EW, kBK, 64) && tc::make_map_2d(&mH, h, d, rows, kBK, 64) &&
            tc::make_map_3d(&mD, wd, d, H, EW, kBK, 64);
  // 128-row m-tiles with the 8-stage ring for decode-sized launches (weight streaming: more bytes in flight,
  // no B reuse to lose); knob ffn_mt = 128 | 256 overrides (A/B measurement)
  int mt = rows <= kDecodeRows ? 128 : 256;
  if (const int v = knob(Knob::kFfnMt)) mt = v == 128 ? 128 : 256;
  // Segment tails of <= swap_rows rows run as swap-AB tiles (16-row boxes for their activation rows and for the
  // [16 gate | 16 up] weight interleave). Default: tails of <= 64 rows of 256-row m-tile launches (A/B,
  // scripts/ffn_lab.py: +2.5 % at 4096 rows, +0.2..0.8 % at 8192-16384); none at decode sizes (-4 % at
  // 256-1024 rows: the tiles there are weight-bandwidth bound either way). Knob ffn_swap = n >= 0 forces it.
  const int kswap = knob(Knob::kFfnSwap);
  const int swap_rows = (kswap < 0 ? (mt == 256 ? 64 : 0) : std::min(64, kswap)) & ~15;
  CUtensorMap mX16 = mX, mH16 = mH, mG16 = mG, mU16 = mU;
  if (ok && (swap_rows > 0 || mt == 256))  // swap-AB tiles and merged tails: 16-row boxes
    ok = tc::make_map_2d(&mX16, xs, H, rows, kBK, 16) && tc::make_map_2d(&mH16, h, d, rows, kBK, 16) &&
         tc::make_map_3d(&mG16, wg, H, d, EW, kBK, 16) && tc::make_map_3d(&mU16, wu, H, d, EW, kBK, 16);
  if (!ok) {
    set_error("cuTensorMapEncodeTiled failed (driver entry point missing or bad shape/alignment)");
    return README_ERR_CUDA;
  }
  // with pdl the caller zeroed `ready` before the dispatch (a memset here would sit between the two kernels)
  if (!pdl) README_CUDA(cudaMemsetAsync(ready, 0, ffn_layer_ready_bytes(rows, nseg), st));
  const int64_t mt_ub = nseg + (rows + mt - 1) / mt;
  // Persistent grid: never more pairs than can be co-resident (down tiles wait on other pairs' gate/up
  // tiles); knob ffn_pairs = n caps it further (measurement of placement-limited grids)
  int pairs = std::min(num_sms() / 2, dev_info().max_pairs[mt == 256 ? 1 : 0]);
  if (const int v = knob(Knob::kFfnPairs)) pairs = std::max(1, std::min(pairs, v));
  if (pairs < 1) {
    set_error("expert FFN: no CTA pair of this kernel fits on the device");
    return README_ERR_UNSUPPORTED;
  }
  const int64_t tiles = mt_ub * ((d + kBN1 - 1) / kBN1 + (H + kBN2 - 1) / kBN2);
  const int grid = 2 * static_cast<int>(tiles < pairs ? tiles : pairs);
  LayerArgs la{};
  la.H = H;
  la.d = d;
  la.E = E;
  la.nseg = nseg;
  la.offsets = offsets;
  la.h = h;
  la.y = y;
  la.ready = ready;
  la.abort = ready + ffn_layer_abort_index(rows);
  la.dev_status = dev_status;
  const int spin = knob(Knob::kFfnSpin);
  la.spin_limit = spin <= 0 ? 1u : (spin >= 31 ? (1u << 31) : (1u << spin));
  la.fz = Fuse{src, static_cast<int>(rows), residual};
  la.expert_slot = expert_slot;
  la.pdl = sd ? 3 : (pdl ? (xready ? 2 : 1) : 0);
  la.xready = xready;
  if (sd) {
    la.dx = reinterpret_cast<const uint4*>(sd->x);
    la.dsrc = sd->src;
    la.dxs = const_cast<__nv_bfloat16*>(xs);
    la.dk = sd->k;
    la.dvec = H * 2 / 16;
  }
  la.trace = g_trace_buf;
  la.ttrace = g_tile_trace;
  la.ttrace_max = g_tile_trace_max;
  la.askip = knob(Knob::kFfnAskip) != 0;
  la.order = knob(Knob::kFfnOrder);
  la.swap_rows = swap_rows;
  // Dynamic tile order (greedy: a pair claims its next tile near the end of its current one) and merged
  // segment tails, together, for 256-row m-tile launches of <= kDynRows rows: there the last wave is a large
  // part of each pair's ~25-60 tiles and the tails ~1 in 5 m-tiles; merged tails make tile costs uneven, which
  // only the dynamic order balances (a static stride with merged tails left the pairs' end times ~90 us apart
  // and re-read weights from DRAM). A/B on one box (scripts/ffn_lab.py, profiles/SUMMARY.md r02): -5 % at 2048
  // rows, -6.7 % at 4096, -1.7 % at 8192, -0.8 % at 16384, but +1.4 % at 32768 and +3.4 % at 65536 (static
  // rounds keep the pairs sharing a weight tile in lockstep), so larger launches keep the static order.
  // Knobs ffn_dyn / ffn_merge = 0 | 1 force either.
  const bool big = rows > kDynRows;
  const int kdyn = knob(Knob::kFfnDyn), kmerge = knob(Knob::kFfnMerge);
  la.dyn = kdyn < 0 ? (mt == 256 && !big ? 1 : 0) : (kdyn != 0 ? 1 : 0);
  la.merge = mt == 256 && (kmerge < 0 ? la.dyn != 0 : kmerge != 0);
  la.tile_ctr = la.abort + 1;
  la.seg_rows = la.abort + 2;
  la.claim_ahead = std::max(1, knob(Knob::kFfnClaim));
  const int fuse = peers ? 2 : ((src || residual) ? 1 : 0);
  if (peers) {
    if (peers->npeer < 1 || peers->npeer > kMaxPeers || peers->vrows < 1 || !src) {
      set_error("expert FFN remote scatter: need 1..%d peers, vrows >= 1 and a row map", kMaxPeers);
      return README_ERR_INVALID_ARG;
    }
    for (int j = 0; j < peers->npeer; ++j) {
      la.peer_y[j] = peers->y[j];
      la.peer_res[j] = peers->res[j];
    }
    la.npeer = peers->npeer;
    la.vrows = peers->vrows;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = mt == 128 ? kSmemBytesLD : kSmemBytesL;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
#define README_LAYER_LAUNCH(F, MT) \
  README_CUDA(cudaLaunchKernelEx(&cfg, ffn_layer2_kernel<F, MT>, mX, mG, mU, mH, mD, mX16, mH16, mG16, mU16, la))
  if (mt == 128) {
    if (fuse == 2) README_LAYER_LAUNCH(2, 128);
    else if (fuse == 1) README_LAYER_LAUNCH(1, 128);
    else README_LAYER_LAUNCH(0, 128);
  } else {
    if (fuse == 2) README_LAYER_LAUNCH(2, 256);
    else if (fuse == 1) README_LAYER_LAUNCH(1, 256);
    else README_LAYER_LAUNCH(0, 256);
  }
#undef README_LAYER_LAUNCH
  README_CUDA(cudaGetLastError());
  return README_OK;
}

}  // namespace readme
