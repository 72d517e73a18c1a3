// ffn_sm100_2cta.cu — a6/a7 grouped expert GEMMs on CTA pairs (tcgen05.mma.cta_group::2), bf16.
//
// Same math as ffn_sm100.cu (SwiGLU reading Q4):
//     kMode 0:  h_r = silu(x_r . W_gate[e]^T) * (x_r . W_up[e]^T)      kMode 1:  y_r = h_r . W_down[e]^T
// but each tile is computed by a CLUSTER OF TWO CTAs on two SMs of a TPC: one tcgen05.mma.cta_group::2
// (issued by the even CTA) multiplies A rows held in both CTAs' shared memory by a 256-column B tile
// whose halves live in the two CTAs, accumulating into both CTAs' TMEM. Per SM this halves the B bytes
// staged per MMA (32 KB per 64-deep K stage instead of 48 KB), so a 6-deep TMA ring fits and the L2->SM
// traffic per FLOP drops by a third — the v1 profile showed the MMA warp waiting on TMA data ~13 % of
// the time with a 4-deep ring (profiles/SUMMARY.md).
//
// Tiles: 256 rows x 256 accumulator columns (M=256 MMA, each CTA 128 rows, TMEM lane = row). The last
// tile of an expert with <= 128 remaining rows runs as an M=128 MMA (each CTA 64 rows; CUTLASS's "2x2"
// TMEM layout: lanes 0-63 hold accumulator columns [0,128), lanes 64-127 columns [128,256) of the same
// rows), so padding waste stays at the 128-row granularity of v1.
// GEMM1 B operand per CTA r: 64 rows of W_gate then the same 64 rows of W_up (neurons n0+64r ..), so in
// accumulator column space gate column c pairs with up column c+64 inside every 128-column window.
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
// so the same ~192 KB ring holds 8 stages instead of 6 — a third more weight bytes in flight per SM.
constexpr int kStagesD = 8;
constexpr int kStageAD = 64 * 128;
constexpr int64_t kDecodeRows = 1024;  // launches up to this many rows use the 128-row m-tile variant

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
  int tile_start2[kMaxSeg + 1];  // merged a6+a7 kernel: the down tiles' prefix
  int mt_start[kMaxSeg + 1];     // merged kernel: first m-tile id of each segment (readiness counters)
  uint32_t xok[kXokWords];       // merged kernel, pdl == 2: bit per m-tile, this CTA's A rows seen ready
  // merged kernel, dynamic tile fetch: the leader's producer publishes each next tile id to both CTAs
  int tq[4];
  uint64_t tq_full[4];   // per CTA: the id in tq[slot] is valid (1 arrival: the leader's producer)
  uint64_t tq_empty[4];  // leader only: every consumer warp of the pair has read tq[slot] (10 arrivals)
};
using Smem = SmemT<kStages, kStageA>;
using SmemD = SmemT<kStagesD, kStageAD>;
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;
constexpr size_t kSmemBytesD = sizeof(SmemD) + 1024;
static_assert(kSmemBytesD <= 232448 && kSmemBytes <= 232448, "shared memory");
constexpr int kTQ = 4;

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
  int lab;                            // experiment knobs (README_LAB): bit0 skip output stores, bit1 N-fastest order
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
      const Tile tl = decode_tile(s, t, nseg, kBnOut, gcur, NT, (fz.lab & 2) != 0);
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
        const Tile tl = decode_tile(s, t, nseg, kBnOut, gcur, NT, (fz.lab & 2) != 0);
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
      const Tile tl = decode_tile(s, t, nseg, kBnOut, gcur, NT, (fz.lab & 2) != 0);
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
      const bool valid = row_in_tile < tl.rows && !(fz.lab & 1);
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
                      (fz.lab & 8) != 0);
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
                        (fz.lab & 8) != 0);
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      // The MMA only needs this warp's TMEM reads finished (tcgen05.wait::ld + fence above), not its global
      // stores, so the arrive is relaxed (lab bit 2 restores release semantics for A/B measurement).
      if (lane == 0) {
        if (fz.lab & 4) tc::mbar_arrive_cluster(&s.tempty[acc], 0);
        else tc::mbar_arrive_cluster_relaxed(&s.tempty[acc], 0);
      }
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
// are earlier in some pair's sequence (all pairs are co-resident: one CTA per SM, grid <= #SMs; a bounded
// poll flags README_DEV_SCHED_TIMEOUT instead of hanging if that ever fails). This removes the gate/up
// kernel's tail, the down kernel's prologue and the down kernel's last-round imbalance.
struct LayerArgs {
  int H, d, E, nseg;
  const int32_t* offsets;
  __nv_bfloat16* h;          // [rows, d]
  __nv_bfloat16* y;          // [rows, H] (y_sorted) or [T, H] (scatter)
  uint32_t* ready;           // [#m-tiles] zeroed before the launch
  uint32_t* dev_status;
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
            // dispatch is still writing later experts' rows (the wait moves to the kernel's end)
  int dyn;  // dynamic tile fetch: tiles after each pair's first come from an atomic counter (ready[sched])
  int sched;
  const uint32_t* xready;  // pdl == 2: [rows] flags, nonzero once row r of x_sorted is written (gather dispatch)
  uint64_t* trace;         // measurement only (readme_debug_trace), normally null
  int askip;               // tiles of <= 64 rows: the second CTA skips its A loads (README_FFN_ASKIP)
  int order;               // lab: 1 = gate/up tiles N-tile fastest (README_FFN_ORDER)
};

struct LTile {
  int mode, g, mt, m0, rows, n0;
  bool m256;
};

template <int kMT, class SM>
__device__ __forceinline__ LTile decode_ltile(const SM& s, int t, int nseg, int T1, int NT1, int NT2, int& gcur1,
                                             int& gcur2, int bn1, int bn2, bool nfast = false) {
  LTile tl;
  int local, g, NT;
  if (t < T1) {
    while (gcur1 + 1 < nseg && s.tile_start[gcur1 + 1] <= t) ++gcur1;
    g = gcur1;
    local = t - s.tile_start[g];
    tl.mode = 0;
    NT = NT1;
  } else {
    const int t2 = t - T1;
    while (gcur2 + 1 < nseg && s.tile_start2[gcur2 + 1] <= t2) ++gcur2;
    g = gcur2;
    local = t2 - s.tile_start2[g];
    tl.mode = 1;
    NT = NT2;
  }
  const int cnt = s.seg_off[g + 1] - s.seg_off[g];
  const int mt_g = (cnt + kMT - 1) / kMT;
  // m-tile fastest (default: consecutive pairs share a weight tile) or, for gate/up tiles with nfast (lab
  // knob README_FFN_ORDER=1), N-tile fastest (consecutive pairs share an A tile)
  const bool nf = nfast && tl.mode == 0;
  const int nt = nf ? local % NT : local / mt_g, mt = nf ? local / NT : local % mt_g;
  tl.g = g;
  tl.mt = mt;
  tl.m0 = s.seg_off[g] + mt * kMT;
  tl.rows = min(kMT, cnt - mt * kMT);
  tl.m256 = tl.rows > 128;
  tl.n0 = nt * (tl.mode == 0 ? bn1 : bn2);
  return tl;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// kNB = B rows each CTA stages per K step: 128 (default; a gate/up tile covers 128 h columns, a down tile
// 256 output columns) or 64 (small batches: twice as many, half-width tiles, so every SM streams its
// share of the touched experts' weights — decode is weight-bandwidth bound).
template <int kFuse, int kNB, int kMT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
ffn_layer2_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmG,
                  const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmH,
                  const __grid_constant__ CUtensorMap tmD, LayerArgs la) {
  extern __shared__ uint8_t smem_raw[];
  using SM = typename std::conditional<kMT == 256, Smem, SmemD>::type;
  constexpr int kS = kMT == 256 ? kStages : kStagesD;     // ring stages
  constexpr int kSA = kMT == 256 ? kStageA : kStageAD;    // A bytes per stage per CTA
  static_assert(kMT == 256 || kMT == 128, "kMT");
  SM& s = *reinterpret_cast<SM*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
  const uint32_t cta = tc::cluster_ctarank();
  const bool leader = cta == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int H = la.H, d = la.d, E = la.E, nseg = la.nseg;
  constexpr int kBN1 = kNB, kBN2 = 2 * kNB;  // h columns per gate/up tile, output columns per down tile
  constexpr int kN = 2 * kNB;               // MMA N (both CTAs' B halves)
  static_assert(kNB == 128 || kNB == 64, "kNB");
  const int NT1 = (d + kBN1 - 1) / kBN1, NT2 = (H + kBN2 - 1) / kBN2;
  const int KB1 = (H + kBK - 1) / kBK, KB2 = (d + kBK - 1) / kBK;
  const uint32_t ready_target = static_cast<uint32_t>(NT1) * 8u;

  for (int i = tid; i <= nseg; i += kThreads) s.seg_off[i] = la.offsets[i];
  for (int i = tid; i < kXokWords; i += kThreads) s.xok[i] = 0u;
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmX);
    tc::prefetch_tmap(&tmG);
    tc::prefetch_tmap(&tmU);
    tc::prefetch_tmap(&tmH);
    tc::prefetch_tmap(&tmD);
  }
  if (warp == 1) tc::tmem_alloc<2>(&s.tmem_base, kTmemCols);
  __syncthreads();
  if (tid == 0) {
    int a1 = 0, a2 = 0, am = 0;
    for (int g = 0; g < nseg; ++g) {
      const int mt_g = (s.seg_off[g + 1] - s.seg_off[g] + kMT - 1) / kMT;
      s.tile_start[g] = a1;
      s.tile_start2[g] = a2;
      s.mt_start[g] = am;
      a1 += mt_g * NT1;
      a2 += mt_g * NT2;
      am += mt_g;
    }
    s.tile_start[nseg] = a1;
    s.tile_start2[nseg] = a2;
    s.mt_start[nseg] = am;
    for (int i = 0; i < kS; ++i) {
      tc::mbar_init(&s.full[i], 1);
      tc::mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s.tfull[i], 1);
      tc::mbar_init(&s.tempty[i], 8);
    }
    for (int i = 0; i < kTQ; ++i) {
      tc::mbar_init(&s.tq_full[i], 1);
      tc::mbar_init(&s.tq_empty[i], 10);  // leader MMA warp + 4 + 4 epilogue warps + the peer's producer
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after();
  const int T1 = s.tile_start[nseg];
  const int ntiles = T1 + s.tile_start2[nseg];
  const uint32_t tmem_base = s.tmem_base;
  // Launched with PDL behind the dispatch (la.pdl): everything above only read the routing offsets, which
  // the route kernel wrote before the dispatch began. Before waiting for the dispatch's x_sorted, start
  // pulling this pair's first gate/up weight tile into L2 — weights do not depend on the dispatch.
  if (la.pdl) {
    if (warp == 0 && lane == 0 && pair < T1) {
      int g1 = 0, g2 = 0;
      const LTile tl = decode_ltile<kMT>(s, pair, nseg, T1, NT1, NT2, g1, g2, kBN1, kBN2, la.order != 0);
      const int e = la.expert_slot ? __ldg(la.expert_slot + tl.g % E) : tl.g % E;
      const int nr = tl.n0 + (kNB / 2) * static_cast<int>(cta);
      const int kbs = KB1 < kPrefetchK ? KB1 : kPrefetchK;
      for (int kb = 0; kb < kbs; ++kb) {
        tc::tma_prefetch_3d(&tmG, kb * kBK, nr, e);
        tc::tma_prefetch_3d(&tmU, kb * kBK, nr, e);
      }
    }
    if (la.pdl == 1) tc::pdl_wait();
  }
  if (la.trace && tid == 0) trace_min(la.trace, 2);
  // Tile sequence of this pair. Static: pair, pair + npairs, ... Dynamic (la.dyn): the first tile is still
  // `pair`; each later one is npairs + atomicAdd(counter), fetched by the leader's producer when it moves on
  // and published through a 4-deep queue to the pair's other warps — per-pair work evens out (tiles differ
  // in cost: M=128 tails, gate/up vs down) while the global order (and the down tiles' readiness
  // dependencies) stays the same. A consumer warp reads entry j and releases it on the leader.
  const bool dyn = la.dyn != 0;
  auto consume = [&](int j) -> int {
    if (!dyn) return pair + j * npairs;
    const int slot = j % kTQ;
    tc::mbar_wait_cluster(&s.tq_full[slot], static_cast<uint32_t>(j / kTQ) & 1u);
    const int t = *reinterpret_cast<volatile int*>(&s.tq[slot]);
    __syncwarp();
    if (lane == 0) tc::mbar_arrive_cluster(&s.tq_empty[slot], 0);
    return t;
  };
  uint32_t fetched = 0;  // lane 0 of the leader's producer: the next tile's counter ticket, fetched one tile
                         // ahead so the atomic's latency hides behind the current tile's loads
  auto produce = [&](int j) -> int {  // the leader's producer warp
    int t = pair + j * npairs;
    if (dyn) {
      if (j > 0) t = npairs + static_cast<int>(__shfl_sync(0xffffffffu, fetched, 0));
      if (lane == 0) fetched = atomicAdd(la.ready + la.sched, 1u);
      const int slot = j % kTQ;
      tc::mbar_wait_cluster(&s.tq_empty[slot], (static_cast<uint32_t>(j / kTQ) & 1u) ^ 1u);
      if (lane == 0) {
        s.tq[slot] = t;
        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(tc::mapa(&s.tq[slot], 1)), "r"(t) : "memory");
        tc::mbar_arrive_cluster(&s.tq_full[slot], 0);  // release: the id stores are visible first
        tc::mbar_arrive_cluster(&s.tq_full[slot], 1);
      }
      __syncwarp();
    }
    return t;
  };

  if (warp == 0) {
    // ===== TMA producer (both CTAs; completion counted on the leader's barrier). The whole warp walks the
    // loop so coordinates and addresses stay in uniform registers; one elected lane issues. =====
    int stage = 0;
    uint32_t phase = 0;
    int g1 = 0, g2 = 0;
    const uint32_t full0 = tc::mapa(&s.full[0], 0);  // the leader's barriers, as cluster addresses
    for (int j = 0;; ++j) {
      const int t = leader ? produce(j) : consume(j);
      if (t >= ntiles) break;
      const LTile tl = decode_ltile<kMT>(s, t, nseg, T1, NT1, NT2, g1, g2, kBN1, kBN2, la.order != 0);
      const int e = la.expert_slot ? __ldg(la.expert_slot + tl.g % E) : tl.g % E;
      const int a_rows = tl.m256 ? 128 : 64;
      const int a_row0 = tl.m0 + static_cast<int>(cta) * a_rows;
      // A tile of ≤ 64 rows: every row the second CTA would stage is past the tile's end, so it skips its A
      // load (its MMA rows read stale shared memory; row m of the product depends on A row m only and rows
      // past tl.rows are never stored). README_FFN_ASKIP=0 loads them anyway (A/B).
      const bool a_skip = la.askip && !tl.m256 && tl.rows <= 64;
      const uint32_t bytes = 2u * static_cast<uint32_t>(a_rows * 128 + kNB * 128) -
                             (a_skip ? static_cast<uint32_t>(a_rows * 128) : 0u);
      if (tl.mode == 0 && la.pdl == 2) {
        // wait until the dispatch has written this CTA's A rows of the tile (rows past the segment's end are
        // padding: their products are never stored, so they are not waited for)
        const int mid = s.mt_start[tl.g] + tl.mt;
        const bool cached = mid < kXokWords * 32 && (s.xok[mid >> 5] >> (mid & 31) & 1u);
        if (!cached) {
          const int lo = a_row0, hi = min(a_row0 + a_rows, tl.m0 + tl.rows);
          uint32_t spins = 0;
          for (;;) {
            bool ok = true;
            for (int r = lo + lane; r < hi; r += kWarp) ok = ok && ld_acquire_u32(la.xready + r) != 0u;
            if (__all_sync(0xffffffffu, ok)) break;
            __nanosleep(64);
            if (++spins == (1u << 25)) {
              if (la.dev_status && lane == 0) atomicOr(la.dev_status, README_DEV_SCHED_TIMEOUT);
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
        const uint32_t* rp = la.ready + s.mt_start[tl.g] + tl.mt;
        uint32_t spins = 0;
        while (ld_acquire_u32(rp) < ready_target) {
          __nanosleep(128);
          if (++spins == (1u << 25)) {
            if (la.dev_status && lane == 0) atomicOr(la.dev_status, README_DEV_SCHED_TIMEOUT);
            break;
          }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
      }
      const int KB = tl.mode == 0 ? KB1 : KB2;
      const CUtensorMap* mA = tl.mode == 0 ? &tmX : &tmH;
      const int nrg = tl.n0 + (kNB / 2) * static_cast<int>(cta), nrd = tl.n0 + kNB * static_cast<int>(cta);
      for (int kb = 0; kb < KB; ++kb) {
        tc::mbar_wait(&s.empty[stage], phase ^ 1);
        if (tc::elect_one()) {
          const uint32_t fb = full0 + static_cast<uint32_t>(stage * 8);
          const int k0 = kb * kBK;
          if (leader) tc::mbar_expect_tx(&s.full[stage], bytes);
          if (!(a_skip && cta == 1)) tc::tma_load_2d_2sm(mA, s.a[stage], fb, k0, a_row0);
          if (tl.m256) tc::tma_load_2d_2sm(mA, s.a[stage] + 64 * 128, fb, k0, a_row0 + 64);
          if (tl.mode == 0) {  // kNB/2 rows of W_gate then the same rows of W_up (box height kNB/2)
            tc::tma_load_3d_2sm(&tmG, s.b[stage], fb, k0, nrg, e);
            tc::tma_load_3d_2sm(&tmU, s.b[stage] + (kNB / 2) * 128, fb, k0, nrg, e);
          } else {  // kNB rows of W_down in boxes of 64
            tc::tma_load_3d_2sm(&tmD, s.b[stage], fb, k0, nrd, e);
            if constexpr (kNB == 128) tc::tma_load_3d_2sm(&tmD, s.b[stage] + 64 * 128, fb, k0, nrd + 64, e);
          }
        }
        __syncwarp();
        if (++stage == kS) {
          stage = 0;
          phase ^= 1;
        }
      }
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
      int g1 = 0, g2 = 0;
      for (int i = 0;; ++i) {
        const int t = consume(i);
        if (t >= ntiles) break;
        const LTile tl = decode_ltile<kMT>(s, t, nseg, T1, NT1, NT2, g1, g2, kBN1, kBN2, la.order != 0);
        const uint32_t idesc = tl.m256 ? idesc256 : idesc128;
        const int acc = i & 1;
        const uint32_t use = static_cast<uint32_t>(i >> 1);
        tc::mbar_wait_cluster(&s.tempty[acc], (use & 1u) ^ 1u);
        tc::fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * 256);
        const int KB = tl.mode == 0 ? KB1 : KB2;
        for (int kb = 0; kb < KB; ++kb) {
          tc::mbar_wait_cluster(&s.full[stage], phase);
          tc::fence_after();
          // +1 in a descriptor's address field = +16 B: stage strides and the 32-B K steps are constants
          const uint64_t ad = adesc0 + static_cast<uint64_t>(stage * (kSA >> 4));
          const uint64_t bd = bdesc0 + static_cast<uint64_t>(stage * (kStageB >> 4));
          if (tc::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kBK / kUK; ++kk)
              tc::mma_f16<2>(d_tmem, ad + static_cast<uint64_t>(kk * 2), bd + static_cast<uint64_t>(kk * 2), idesc,
                             (kb | kk) != 0 ? 1u : 0u);
            tc::commit_2sm_mc(&s.empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == kS) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (tc::elect_one()) tc::commit_2sm_mc(&s.tfull[acc], 0x3);
        __syncwarp();
      }
    }
  } else {
    // ===== epilogue: warps 2..5 of both CTAs =====
    const int q = warp & 3;
    uint8_t* stg = s.stg[q];
    int g1 = 0, g2 = 0;
    for (int i = 0;; ++i) {
      const int t = consume(i);
      if (t >= ntiles) break;
      const LTile tl = decode_ltile<kMT>(s, t, nseg, T1, NT1, NT2, g1, g2, kBN1, kBN2, la.order != 0);
      const int acc = i & 1;
      const uint32_t use = static_cast<uint32_t>(i >> 1);
      tc::mbar_wait_cluster(&s.tfull[acc], use & 1u);
      tc::fence_after();
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
      const bool valid = row_in_tile < tl.rows;
      const int64_t r = tl.m0 + row_in_tile;
      if (tl.mode == 0) {
        // windows of kNB columns: [gate kNB/2 | up kNB/2] of h columns n0 + (window) * kNB/2 + [0, kNB/2)
        constexpr int kHalf = kNB / 2;
        __nv_bfloat16* orow = la.h + r * d;
        for (int w = 0; w < ncols / kNB; ++w) {
          const uint32_t wbase = tacc + static_cast<uint32_t>(w * kNB);
          const int hcol0 = tl.n0 + (acc_off + w * kNB) / 2;
#pragma unroll 1
          for (int c = 0; c < kHalf; c += 32) {
            uint32_t gr[32], ur[32];
            tc::tmem_ld32(wbase + c, gr);
            tc::tmem_ld32(wbase + kHalf + c, ur);
            tc::tmem_wait_ld();
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = tc::silu(__uint_as_float(gr[j])) * __uint_as_float(ur[j]);
            stage_row_bf16x32(stg, lane, c / 8, v);
          }
          const int lim = (d - hcol0) * 2 < kHalf * 2 ? (d - hcol0) * 2 : kHalf * 2;
          stage_flush(stg, lane, valid ? reinterpret_cast<uint64_t>(orow + hcol0) : 0ull, lim, false);
        }
      } else {
        int64_t orow_idx = r;
        bool valid_row = valid;
        __nv_bfloat16* orow;
        const __nv_bfloat16* rrow = nullptr;
        if constexpr (kFuse == 2) {
          const int64_t v = valid ? static_cast<int64_t>(__ldg(la.fz.src + r)) : -1;
          valid_row = valid && v >= 0 && v < la.vrows * la.npeer;
          const int p = valid_row ? static_cast<int>(v / la.vrows) : 0;
          const int64_t i = valid_row ? v - p * la.vrows : 0;
          __nv_bfloat16* py = la.peer_y[0];
          const __nv_bfloat16* pr = la.peer_res[0];
#pragma unroll
          for (int j = 1; j < kMaxPeers; ++j)
            if (p == j) {
              py = la.peer_y[j];
              pr = la.peer_res[j];
            }
          orow = py + i * H;
          rrow = pr ? pr + i * H : nullptr;
        } else {
          if constexpr (kFuse == 1) {
            orow_idx = valid ? (la.fz.src ? __ldg(la.fz.src + r) : r) : 0;
            valid_row = valid && orow_idx >= 0 && orow_idx < la.fz.rows;
          }
          orow = la.y + orow_idx * H;
          rrow = (kFuse == 1 && la.fz.residual) ? la.fz.residual + orow_idx * H : nullptr;
        }
#pragma unroll 1
        for (int c0 = 0; c0 < ncols; c0 += 64) {
          const int col0 = tl.n0 + acc_off + c0;
#pragma unroll 1
          for (int c = 0; c < 64; c += 32) {
            uint32_t vr[32];
            tc::tmem_ld32(tacc + static_cast<uint32_t>(c0 + c), vr);
            tc::tmem_wait_ld();
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(vr[j]);
            if (rrow && valid_row) add_bf16x32(rrow + col0 + c, v, H - (col0 + c));
            stage_row_bf16x32(stg, lane, c / 8, v);
          }
          stage_flush(stg, lane, valid_row ? reinterpret_cast<uint64_t>(orow + col0) : 0ull, (H - col0) * 2, false);
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive_cluster_relaxed(&s.tempty[acc], 0);
        if (tl.mode == 0) {
          // publish this warp's share of the h tile to the down tiles (generic -> async proxy, then release)
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(la.ready + s.mt_start[tl.g] + tl.mt)
                       : "memory");
        }
      }
    }
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

// ---------------------------------------------------------------------------------------------------
// Wide-N single-launch expert FFN (README_FFN_WIDE=1; measured slower, kept for A/B). A CTA pair computes a 256-row x 2-half tile: for every
// K stage each CTA stages its 128 A rows ONCE and B rows for TWO 256-column halves, and issues two M=256
// N=256 MMAs (one per half) into two TMEM accumulators (columns [0,256) and [256,512)). Staged bytes per
// FLOP drop by a quarter against the double-buffered 256-column tile (48 KB per 1024 MMA cycles instead of
// 32 KB per 512): that kernel is bound by L2->SM throughput (~11.5 TB/s measured, the LTS cap), so the
// wide tile runs closer to the tensor-pipe bound. Gate/up half h covers h columns n0 + 128h + [0,128)
// ([gate 64 | up 64] per CTA, as in the narrow kernel); down half h covers output columns n0 + 256h +
// [0,256). A half that lies entirely past N is skipped (d = 5504 = 21.5 x 256).
// The accumulators are single-buffered across tiles; the epilogue drains accumulator 0 first and releases
// it, and the MMA issuer starts the next tile on accumulator 0 while accumulator 1 is still draining,
// catching accumulator 1 up over the stages it kept (ring depth permitting): the epilogue stays hidden.
constexpr int kWStages = 4;
constexpr int kWStageB = 2 * 128 * 128;  // two halves x 128 rows x 128 B per CTA

struct __align__(8) WSmem {
  uint8_t a[kWStages][kStageA];
  uint8_t b[kWStages][kWStageB];
  uint64_t full[kWStages];
  uint64_t empty[kWStages];
  uint64_t tfull;
  uint64_t tempty[2];
  uint32_t tmem_base;
  alignas(16) uint8_t stg[4][32 * 128];
  int seg_off[kMaxSeg + 1];
  int tile_start[kMaxSeg + 1];
  int tile_start2[kMaxSeg + 1];
  int mt_start[kMaxSeg + 1];
};
constexpr size_t kWSmemBytes = sizeof(WSmem) + 1024;
static_assert(kWSmemBytes <= 232448, "wide kernel shared memory");

__device__ __forceinline__ LTile decode_wtile(const WSmem& s, int t, int nseg, int T1, int& gcur1, int& gcur2,
                                             int bn1, int bn2) {
  LTile tl;
  int local, g;
  if (t < T1) {
    while (gcur1 + 1 < nseg && s.tile_start[gcur1 + 1] <= t) ++gcur1;
    g = gcur1;
    local = t - s.tile_start[g];
    tl.mode = 0;
  } else {
    const int t2 = t - T1;
    while (gcur2 + 1 < nseg && s.tile_start2[gcur2 + 1] <= t2) ++gcur2;
    g = gcur2;
    local = t2 - s.tile_start2[g];
    tl.mode = 1;
  }
  const int cnt = s.seg_off[g + 1] - s.seg_off[g];
  const int mt_g = (cnt + 255) / 256;
  const int nt = local / mt_g, mt = local % mt_g;
  tl.g = g;
  tl.mt = mt;
  tl.m0 = s.seg_off[g] + mt * 256;
  tl.rows = min(256, cnt - mt * 256);
  tl.m256 = tl.rows > 128;
  tl.n0 = nt * (tl.mode == 0 ? bn1 : bn2);
  return tl;
}

template <int kFuse>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
ffn_wide_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmG,
                const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmH,
                const __grid_constant__ CUtensorMap tmD, LayerArgs la) {
  extern __shared__ uint8_t smem_raw[];
  WSmem& s = *reinterpret_cast<WSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid / kWarp, lane = tid % kWarp;
  const uint32_t cta = tc::cluster_ctarank();
  const bool leader = cta == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int H = la.H, d = la.d, E = la.E, nseg = la.nseg;
  constexpr int kHW1 = 128, kHW2 = 256;            // columns per half: gate/up (h columns), down
  constexpr int kBN1 = 2 * kHW1, kBN2 = 2 * kHW2;  // columns per tile
  const int NT1 = (d + kBN1 - 1) / kBN1, NT2 = (H + kBN2 - 1) / kBN2;
  const int KB1 = (H + kBK - 1) / kBK, KB2 = (d + kBK - 1) / kBK;
  const uint32_t ready_target = static_cast<uint32_t>(NT1) * 8u;

  for (int i = tid; i <= nseg; i += kThreads) s.seg_off[i] = la.offsets[i];
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmX);
    tc::prefetch_tmap(&tmG);
    tc::prefetch_tmap(&tmU);
    tc::prefetch_tmap(&tmH);
    tc::prefetch_tmap(&tmD);
  }
  if (warp == 1) tc::tmem_alloc<2>(&s.tmem_base, kTmemCols);
  __syncthreads();
  if (tid == 0) {
    int a1 = 0, a2 = 0, am = 0;
    for (int g = 0; g < nseg; ++g) {
      const int mt_g = (s.seg_off[g + 1] - s.seg_off[g] + 255) / 256;
      s.tile_start[g] = a1;
      s.tile_start2[g] = a2;
      s.mt_start[g] = am;
      a1 += mt_g * NT1;
      a2 += mt_g * NT2;
      am += mt_g;
    }
    s.tile_start[nseg] = a1;
    s.tile_start2[nseg] = a2;
    s.mt_start[nseg] = am;
    for (int i = 0; i < kWStages; ++i) {
      tc::mbar_init(&s.full[i], 1);
      tc::mbar_init(&s.empty[i], 1);
    }
    tc::mbar_init(&s.tfull, 1);
    tc::mbar_init(&s.tempty[0], 8);
    tc::mbar_init(&s.tempty[1], 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after();
  const int T1 = s.tile_start[nseg];
  const int ntiles = T1 + s.tile_start2[nseg];
  const uint32_t tmem_base = s.tmem_base;
  if (la.pdl) {  // see ffn_layer2_kernel: warm L2 with the first weight tile, then wait for the dispatch
    if (warp == 0 && lane == 0 && pair < T1) {
      int g1 = 0, g2 = 0;
      const LTile tl = decode_wtile(s, pair, nseg, T1, g1, g2, kBN1, kBN2);
      const int e = la.expert_slot ? __ldg(la.expert_slot + tl.g % E) : tl.g % E;
      const int kbs = KB1 < kPrefetchK / 2 ? KB1 : kPrefetchK / 2;
      for (int h = 0; h < 2; ++h) {
        const int nr = tl.n0 + h * kHW1 + 64 * static_cast<int>(cta);
        if (nr >= d) break;
        for (int kb = 0; kb < kbs; ++kb) {
          tc::tma_prefetch_3d(&tmG, kb * kBK, nr, e);
          tc::tma_prefetch_3d(&tmU, kb * kBK, nr, e);
        }
      }
    }
    tc::pdl_wait();
  }

  if (warp == 0) {
    // ===== TMA producer (both CTAs; completion counted on the leader's barrier) =====
    int stage = 0;
    uint32_t phase = 0;
    int g1 = 0, g2 = 0;
    for (int t = pair; t < ntiles; t += npairs) {
      const LTile tl = decode_wtile(s, t, nseg, T1, g1, g2, kBN1, kBN2);
      const int e = la.expert_slot ? __ldg(la.expert_slot + tl.g % E) : tl.g % E;
      const bool two = tl.n0 + (tl.mode == 0 ? kHW1 : kHW2) < (tl.mode == 0 ? d : H);
      const int a_rows = tl.m256 ? 128 : 64;
      const int a_row0 = tl.m0 + static_cast<int>(cta) * a_rows;
      const uint32_t bytes = 2u * static_cast<uint32_t>(a_rows * 128 + (two ? 2 : 1) * 128 * 128);
      if (tl.mode == 1) {
        if (lane == 0) {
          const uint32_t* rp = la.ready + s.mt_start[tl.g] + tl.mt;
          uint32_t spins = 0;
          while (ld_acquire_u32(rp) < ready_target) {
            __nanosleep(128);
            if (++spins == (1u << 25)) {
              if (la.dev_status) atomicOr(la.dev_status, README_DEV_SCHED_TIMEOUT);
              break;
            }
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        __syncwarp();
      }
      const int KB = tl.mode == 0 ? KB1 : KB2;
      for (int kb = 0; kb < KB; ++kb) {
        tc::mbar_wait(&s.empty[stage], phase ^ 1);
        if (lane == 0) {
          const uint32_t fb = tc::mapa(&s.full[stage], 0);
          const int k0 = kb * kBK;
          if (leader) tc::mbar_expect_tx(&s.full[stage], bytes);
          const CUtensorMap* mA = tl.mode == 0 ? &tmX : &tmH;
          tc::tma_load_2d_2sm(mA, s.a[stage], fb, k0, a_row0);
          if (tl.m256) tc::tma_load_2d_2sm(mA, s.a[stage] + 64 * 128, fb, k0, a_row0 + 64);
          for (int h = 0; h < (two ? 2 : 1); ++h) {
            uint8_t* bh = s.b[stage] + h * (128 * 128);
            if (tl.mode == 0) {  // 64 rows of W_gate then the same 64 rows of W_up
              const int nr = tl.n0 + h * kHW1 + 64 * static_cast<int>(cta);
              tc::tma_load_3d_2sm(&tmG, bh, fb, k0, nr, e);
              tc::tma_load_3d_2sm(&tmU, bh + 64 * 128, fb, k0, nr, e);
            } else {  // 128 rows of W_down
              const int nr = tl.n0 + h * kHW2 + 128 * static_cast<int>(cta);
              tc::tma_load_3d_2sm(&tmD, bh, fb, k0, nr, e);
              tc::tma_load_3d_2sm(&tmD, bh + 64 * 128, fb, k0, nr + 64, e);
            }
          }
        }
        if (++stage == kWStages) {
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
      int g1 = 0, g2 = 0, i = 0;
      for (int t = pair; t < ntiles; t += npairs, ++i) {
        const LTile tl = decode_wtile(s, t, nseg, T1, g1, g2, kBN1, kBN2);
        const bool two = tl.n0 + (tl.mode == 0 ? kHW1 : kHW2) < (tl.mode == 0 ? d : H);
        const uint32_t idesc = tl.m256 ? idesc256 : idesc128;
        const uint32_t par = (static_cast<uint32_t>(i) & 1u) ^ 1u;  // accumulators released by tile i-1
        const int KB = tl.mode == 0 ? KB1 : KB2;
        // half-1 MMAs still owed (accumulator 1 not yet drained) for the consecutive stages
        // [pend0, pend0 + npend) of this tile, which began at k-block first_pend_kb
        int pend0 = 0, npend = 0, first_pend_kb = 0;
        bool acc1_free = !two;
        tc::mbar_wait_cluster(&s.tempty[0], par);
        tc::fence_after();
        auto issue = [&](int st, int h, bool first_k) {
          const uint64_t ad = adesc0 + static_cast<uint64_t>(st * (kStageA >> 4));
          const uint64_t bd = bdesc0 + static_cast<uint64_t>(st * (kWStageB >> 4) + h * ((128 * 128) >> 4));
          const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(h * 256);
          if (tc::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kBK / kUK; ++kk)
              tc::mma_f16<2>(d_tmem, ad + static_cast<uint64_t>(kk * 2), bd + static_cast<uint64_t>(kk * 2), idesc,
                             (!first_k || kk != 0) ? 1u : 0u);
          }
          __syncwarp();
        };
        auto release = [&](int st) {
          if (tc::elect_one()) tc::commit_2sm_mc(&s.empty[st], 0x3);
          __syncwarp();
        };
        auto catch_up = [&]() {  // accumulator 1, oldest owed stage first
          for (int j = 0; j < npend; ++j) {
            const int st = (pend0 + j) % kWStages;
            issue(st, 1, first_pend_kb + j == 0);
            release(st);
          }
          npend = 0;
        };
        for (int kb = 0; kb < KB; ++kb) {
          if (!acc1_free && npend == kWStages) {  // the ring is exhausted: wait for the drain
            tc::mbar_wait_cluster(&s.tempty[1], par);
            tc::fence_after();
            acc1_free = true;
          }
          if (!acc1_free && tc::mbar_test_cluster(&s.tempty[1], par)) {
            tc::fence_after();
            acc1_free = true;
          }
          if (acc1_free && npend) catch_up();
          tc::mbar_wait_cluster(&s.full[stage], phase);
          tc::fence_after();
          issue(stage, 0, kb == 0);
          if (!two) {
            release(stage);
          } else if (acc1_free) {
            issue(stage, 1, kb == 0);
            release(stage);
          } else {
            if (npend == 0) {
              pend0 = stage;
              first_pend_kb = kb;
            }
            ++npend;
          }
          if (++stage == kWStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (npend) {  // short tile: accumulator 1 never freed while its stages streamed
          tc::mbar_wait_cluster(&s.tempty[1], par);
          tc::fence_after();
          catch_up();
        } else if (!two) {
          tc::mbar_wait_cluster(&s.tempty[1], par);  // keep accumulator 1's phase in step with the tiles
        }
        if (tc::elect_one()) tc::commit_2sm_mc(&s.tfull, 0x3);
        __syncwarp();
      }
    }
  } else {
    // ===== epilogue: warps 2..5 of both CTAs =====
    const int q = warp & 3;
    uint8_t* stg = s.stg[q];
    int g1 = 0, g2 = 0, i = 0;
    for (int t = pair; t < ntiles; t += npairs, ++i) {
      const LTile tl = decode_wtile(s, t, nseg, T1, g1, g2, kBN1, kBN2);
      const bool two = tl.n0 + (tl.mode == 0 ? kHW1 : kHW2) < (tl.mode == 0 ? d : H);
      tc::mbar_wait_cluster(&s.tfull, static_cast<uint32_t>(i) & 1u);
      tc::fence_after();
      int row_in_tile, ncols, acc_off;
      if (tl.m256) {
        row_in_tile = static_cast<int>(cta) * 128 + q * 32 + lane;
        ncols = 256;
        acc_off = 0;
      } else {
        row_in_tile = static_cast<int>(cta) * 64 + (q & 1) * 32 + lane;
        ncols = 128;
        acc_off = (q >> 1) * 128;
      }
      const bool valid = row_in_tile < tl.rows;
      const int64_t r = tl.m0 + row_in_tile;
      // output row pointers (down tiles)
      int64_t orow_idx = r;
      bool valid_row = valid;
      __nv_bfloat16* orow = nullptr;
      const __nv_bfloat16* rrow = nullptr;
      if (tl.mode == 1) {
        if constexpr (kFuse == 2) {
          const int64_t v = valid ? static_cast<int64_t>(__ldg(la.fz.src + r)) : -1;
          valid_row = valid && v >= 0 && v < la.vrows * la.npeer;
          const int p = valid_row ? static_cast<int>(v / la.vrows) : 0;
          const int64_t iv = valid_row ? v - p * la.vrows : 0;
          __nv_bfloat16* py = la.peer_y[0];
          const __nv_bfloat16* pr = la.peer_res[0];
#pragma unroll
          for (int j = 1; j < kMaxPeers; ++j)
            if (p == j) {
              py = la.peer_y[j];
              pr = la.peer_res[j];
            }
          orow = py + iv * H;
          rrow = pr ? pr + iv * H : nullptr;
        } else {
          if constexpr (kFuse == 1) {
            orow_idx = valid ? (la.fz.src ? __ldg(la.fz.src + r) : r) : 0;
            valid_row = valid && orow_idx >= 0 && orow_idx < la.fz.rows;
          }
          orow = la.y + orow_idx * H;
          rrow = (kFuse == 1 && la.fz.residual) ? la.fz.residual + orow_idx * H : nullptr;
        }
      }
      for (int h = 0; h < 2; ++h) {
        if (h == 0 || two) {
          const uint32_t tacc = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(h * 256);
          if (tl.mode == 0) {
            __nv_bfloat16* hrow = la.h + r * d;
            for (int w = 0; w < ncols / 128; ++w) {
              const uint32_t wbase = tacc + static_cast<uint32_t>(w * 128);
              const int hcol0 = tl.n0 + h * kHW1 + (acc_off + w * 128) / 2;
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
              stage_flush(stg, lane, valid ? reinterpret_cast<uint64_t>(hrow + hcol0) : 0ull, (d - hcol0) * 2, false);
            }
          } else {
#pragma unroll 1
            for (int c0 = 0; c0 < ncols; c0 += 64) {
              const int col0 = tl.n0 + h * kHW2 + acc_off + c0;
#pragma unroll 1
              for (int c = 0; c < 64; c += 32) {
                uint32_t vr[32];
                tc::tmem_ld32(tacc + static_cast<uint32_t>(c0 + c), vr);
                tc::tmem_wait_ld();
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(vr[j]);
                if (rrow && valid_row) add_bf16x32(rrow + col0 + c, v, H - (col0 + c));
                stage_row_bf16x32(stg, lane, c / 8, v);
              }
              stage_flush(stg, lane, valid_row ? reinterpret_cast<uint64_t>(orow + col0) : 0ull, (H - col0) * 2,
                          false);
            }
          }
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster_relaxed(&s.tempty[h], 0);  // accumulator h drained
      }
      if (lane == 0 && tl.mode == 0) {
        // publish this warp's share of the h tile to the down tiles (generic -> async proxy, then release)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(la.ready + s.mt_start[tl.g] + tl.mt)
                     : "memory");
      }
    }
  }

  if constexpr (kFuse == 2) __threadfence_system();
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after();
  if (warp == 1) tc::tmem_dealloc<2>(tmem_base, kTmemCols);
}

readme_status set_smem_attr() {
  static std::once_flag once[64];
  static cudaError_t err[64];
  int dev = 0;
  README_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) dev = 0;
  std::call_once(once[dev], [&] {
    const void* fns[9] = {reinterpret_cast<const void*>(ffn_gemm2_kernel<0, 0>),
                          reinterpret_cast<const void*>(ffn_gemm2_kernel<1, 0>),
                          reinterpret_cast<const void*>(ffn_gemm2_kernel<1, 1>),
                          reinterpret_cast<const void*>(ffn_layer2_kernel<0, 128, 256>),
                          reinterpret_cast<const void*>(ffn_layer2_kernel<1, 128, 256>),
                          reinterpret_cast<const void*>(ffn_layer2_kernel<2, 128, 256>),
                          reinterpret_cast<const void*>(ffn_layer2_kernel<0, 64, 256>),
                          reinterpret_cast<const void*>(ffn_layer2_kernel<1, 64, 256>),
                          reinterpret_cast<const void*>(ffn_layer2_kernel<2, 64, 256>)};
    err[dev] = cudaSuccess;
    for (int i = 0; i < 9 && err[dev] == cudaSuccess; ++i)
      err[dev] = cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
    const void* dfns[3] = {reinterpret_cast<const void*>(ffn_layer2_kernel<0, 128, 128>),
                           reinterpret_cast<const void*>(ffn_layer2_kernel<1, 128, 128>),
                           reinterpret_cast<const void*>(ffn_layer2_kernel<2, 128, 128>)};
    for (int i = 0; i < 3 && err[dev] == cudaSuccess; ++i)
      err[dev] = cudaFuncSetAttribute(dfns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytesD));
    const void* wfns[3] = {reinterpret_cast<const void*>(ffn_wide_kernel<0>),
                           reinterpret_cast<const void*>(ffn_wide_kernel<1>),
                           reinterpret_cast<const void*>(ffn_wide_kernel<2>)};
    for (int i = 0; i < 3 && err[dev] == cudaSuccess; ++i)
      err[dev] = cudaFuncSetAttribute(wfns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kWSmemBytes));
  });
  if (err[dev] != cudaSuccess) return cuda_fail(err[dev], "cudaFuncSetAttribute(ffn_gemm2_kernel)");
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
  const int pairs = num_sms() / 2;
  const int64_t tiles = mt_ub * ((N + (mode == 0 ? 127 : 255)) / (mode == 0 ? 128 : 256));
  const int grid = 2 * static_cast<int>(tiles < pairs ? tiles : pairs);
  const char* lab = getenv("README_LAB");
  const Fuse fz{src, static_cast<int>(rows), residual, lab ? atoi(lab) : 0};
  if (mode == 0)
    ffn_gemm2_kernel<0, 0><<<grid, kThreads, kSmemBytes, st>>>(mA, mB0, mB1, K, N, E, nseg, offsets, out, fz);
  else if (src == nullptr && residual == nullptr)
    ffn_gemm2_kernel<1, 0><<<grid, kThreads, kSmemBytes, st>>>(mA, mB0, mB1, K, N, E, nseg, offsets, out, fz);
  else
    ffn_gemm2_kernel<1, 1><<<grid, kThreads, kSmemBytes, st>>>(mA, mB0, mB1, K, N, E, nseg, offsets, out, fz);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

// [readiness counters: <= kMaxSeg + #m-tiles + 1][x_sorted row flags: rows] (the flags are used when the
// gather dispatch precedes the FFN, pdl == 2); one memset zeroes both
size_t ffn_layer_xready_offset(int64_t rows) {  // counters sized for 128-row m-tiles (either kMT)
  return align_up(static_cast<size_t>(kMaxSeg + (rows + 127) / 128 + 1) * sizeof(uint32_t), 256);
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
                                    bool pdl, const uint32_t* xready) {
  if (rows == 0) return README_OK;
  if (nseg > kMaxSeg) {
    set_error("bf16 expert FFN supports at most %d segments (got %d)", kMaxSeg, nseg);
    return README_ERR_UNSUPPORTED;
  }
  readme_status rs = set_smem_attr();
  if (rs != README_OK) return rs;
  // Tile width: full width by default; README_FFN_NB=64 selects half-width tiles (twice as many tiles: more
  // SMs share a small batch's weight stream, but measured slower at decode sizes — profiles/SUMMARY.md).
  int nb = 128;
  if (const char* v = getenv("README_FFN_NB")) nb = atoi(v) == 64 ? 64 : 128;
  // README_FFN_WIDE=1 selects the wide-N tile (two 256-column halves per K stage, 25 % fewer staged bytes
  // per FLOP); measured 15 % slower than the double-buffered 256-column tile at config 2 (more DRAM
  // re-reads, single-buffered accumulators), so it is not the default (profiles/SUMMARY.md)
  bool wide = false;
  if (const char* v = getenv("README_FFN_WIDE")) wide = nb == 128 && atoi(v) != 0;
  CUtensorMap mX, mG, mU, mH, mD;
  const int32_t EW = expert_slot ? n_slots : E;  // outer extent of the weight tensors
  bool ok = tc::make_map_2d(&mX, xs, H, rows, kBK, 64) && tc::make_map_3d(&mG, wg, H, d, EW, kBK, nb / 2) &&
            tc::make_map_3d(&mU, wu, H, d, EW, kBK, nb / 2) && tc::make_map_2d(&mH, h, d, rows, kBK, 64) &&
            tc::make_map_3d(&mD, wd, d, H, EW, kBK, 64);
  if (!ok) {
    set_error("cuTensorMapEncodeTiled failed (driver entry point missing or bad shape/alignment)");
    return README_ERR_CUDA;
  }
  // with pdl the caller zeroed `ready` before the dispatch (a memset here would sit between the two kernels)
  if (!pdl) README_CUDA(cudaMemsetAsync(ready, 0, ffn_layer_ready_bytes(rows, nseg), st));
  // 128-row m-tiles with the 8-stage ring for decode-sized launches (weight streaming: more bytes in flight,
  // no B reuse to lose); README_FFN_MT=128|256 overrides (A/B measurement)
  int mt = rows <= kDecodeRows ? 128 : 256;
  if (const char* v = getenv("README_FFN_MT")) mt = atoi(v) == 128 ? 128 : 256;
  if (wide || nb == 64) mt = 256;
  const int64_t mt_ub = nseg + (rows + mt - 1) / mt;
  int pairs = num_sms() / 2;
  // README_FFN_PAIRS=n: at most n CTA pairs (measurement of placement-limited grids, e.g. 66 pairs = the
  // 132 SMs that 4-CTA clusters place on)
  if (const char* v = getenv("README_FFN_PAIRS")) pairs = std::max(1, std::min(pairs, atoi(v)));
  const int64_t tiles = wide ? mt_ub * ((d + 255) / 256 + (H + 511) / 512)
                             : mt_ub * ((d + nb - 1) / nb + (H + 2 * nb - 1) / (2 * nb));
  const int grid = 2 * static_cast<int>(tiles < pairs ? tiles : pairs);
  // README_FFN_DYNAMIC=1: dynamic tile fetch (counter = the spare readiness slot after the last m-tile).
  // Measured 1-2 % slower than the static round-robin schedule at config 2 (profiles/SUMMARY.md), so off.
  int dyn = 0;
  if (const char* v = getenv("README_FFN_DYNAMIC")) dyn = atoi(v) != 0;
  LayerArgs la{H, d, E, nseg, offsets, h, y, ready, dev_status, Fuse{src, static_cast<int>(rows), residual, 0},
               expert_slot, {}, {}, 0, 0, pdl ? (xready && !wide ? 2 : 1) : 0, dyn,
               static_cast<int>(nseg + (rows + 127) / 128), xready, g_trace_buf};
  la.askip = 1;
  if (const char* v = getenv("README_FFN_ASKIP")) la.askip = atoi(v) != 0;
  if (const char* v = getenv("README_FFN_ORDER")) la.order = atoi(v);
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
  cfg.dynamicSmemBytes = wide ? kWSmemBytes : (mt == 128 ? kSmemBytesD : kSmemBytes);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
#define README_LAYER_LAUNCH(F, NB) \
  README_CUDA(cudaLaunchKernelEx(&cfg, ffn_layer2_kernel<F, NB, 256>, mX, mG, mU, mH, mD, la))
#define README_LAYER_LAUNCH_D(F) \
  README_CUDA(cudaLaunchKernelEx(&cfg, ffn_layer2_kernel<F, 128, 128>, mX, mG, mU, mH, mD, la))
#define README_WIDE_LAUNCH(F) \
  README_CUDA(cudaLaunchKernelEx(&cfg, ffn_wide_kernel<F>, mX, mG, mU, mH, mD, la))
  if (wide) {
    if (fuse == 2) README_WIDE_LAUNCH(2);
    else if (fuse == 1) README_WIDE_LAUNCH(1);
    else README_WIDE_LAUNCH(0);
  } else if (nb == 64) {
    if (fuse == 2) README_LAYER_LAUNCH(2, 64);
    else if (fuse == 1) README_LAYER_LAUNCH(1, 64);
    else README_LAYER_LAUNCH(0, 64);
  } else if (mt == 128) {
    if (fuse == 2) README_LAYER_LAUNCH_D(2);
    else if (fuse == 1) README_LAYER_LAUNCH_D(1);
    else README_LAYER_LAUNCH_D(0);
  } else {
    if (fuse == 2) README_LAYER_LAUNCH(2, 128);
    else if (fuse == 1) README_LAYER_LAUNCH(1, 128);
    else README_LAYER_LAUNCH(0, 128);
  }
#undef README_LAYER_LAUNCH
#undef README_LAYER_LAUNCH_D
#undef README_WIDE_LAUNCH
  README_CUDA(cudaGetLastError());
  return README_OK;
}

}  // namespace readme
