// Lab microbenchmark (measurement only, not part of the library): per-SM TMA ingest rate when few SMs stream
// weight tiles, as a function of the number of streaming CTAs (one per SM), the ring depth and the copy form.
//   mode 0: 3-D tiled boxes of 64 rows x 64 bf16 (128-B swizzle) from a K-major [N][K] matrix (the FFN's
//           weight loads; rows K*2 bytes apart)
//   mode 1: 1-D cp.async.bulk of 8 KB contiguous (the first, non-cluster kernel; modes 2-4 below)
// Each CTA streams `per_cta` bytes of its own region through a ring of S stages of 16 KB (2 boxes per stage);
// a consumer thread releases each stage as soon as it lands (no compute). cold: L2 flushed before each run.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_19123_b200/csrc
//        scripts/lab_tma_rate.cu paper_2410_19123_b200/csrc/tensor_maps.cu -o /tmp/tma_rate
#include <cstdio>
#include <cstdlib>

#include "tc_common.cuh"

using namespace readme;

constexpr int kMaxS = 13;

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* base,
                                                       int K, int rows_per_cta, int S, int mode, int kb_total, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kMaxS], empty[kMaxS];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int r0 = blockIdx.x * rows_per_cta;
  // work items: (row block of 128 rows, K block of 64): K blocks fastest, like one FFN tile's loads
  const int nrb = rows_per_cta / 128;
  const int items = nrb * kb_total * reps;
  if (tid == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; it < items; ++it) {
      tc::mbar_wait(&empty[stage], phase ^ 1);
      tc::mbar_expect_tx(&full[stage], 16384);
      uint8_t* dst = smem + stage * 16384;
      const int rb = (it / kb_total) % nrb, kb = it % kb_total;
      if (mode == 0) {
        tc::tma_load_3d(&tm, dst, &full[stage], kb * 64, r0 + rb * 128, 0);
        tc::tma_load_3d(&tm, dst + 8192, &full[stage], kb * 64, r0 + rb * 128 + 64, 0);
      } else {
        const uint8_t* src = base + (static_cast<size_t>(blockIdx.x) * nrb * kb_total + it % (nrb * kb_total)) * 16384;
        for (int h = 0; h < 2; ++h)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];" ::"r"(
                  tc::smem_u32(dst + h * 8192)),
              "l"(src + h * 8192), "r"(tc::smem_u32(&full[stage]))
              : "memory");
      }
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (tid == 32) {
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; it < items; ++it) {
      tc::mbar_wait(&full[stage], phase);
      tc::mbar_arrive(&empty[stage]);
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
}

// cluster of 2: mode 2 = each CTA issues ONE of a stage's two boxes with .multicast::cluster to both CTAs (each
// CTA receives 16 KB per stage, issues 8 KB; a slot is refilled only after BOTH CTAs' consumers released it, so
// this mode measures that cross-CTA release chain more than the multicast: 13-17 GB/s, not a TMA number);
// mode 3 = same cluster, no multicast (each CTA loads both boxes);
// mode 4 = one 128-row box per stage (16 KB per instruction), no cluster use
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1)
    stream_mc_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm128, int K,
                     int rows_per_cta, int S, int mode, int kb_total, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kMaxS], empty[kMaxS];
  const int tid = threadIdx.x;
  const uint32_t cta = tc::cluster_ctarank();
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], mode == 2 ? 2 : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::cluster_sync();
  // mode 2: both CTAs of the cluster stream the SAME rows (the pair shares one operand)
  const int r0 = (mode == 2 ? (blockIdx.x >> 1) : blockIdx.x) * rows_per_cta;
  const int nrb = rows_per_cta / 128;
  const int items = nrb * kb_total * reps;
  if (tid == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; it < items; ++it) {
      tc::mbar_wait(&empty[stage], phase ^ 1);
      tc::mbar_expect_tx(&full[stage], 16384);
      uint8_t* dst = smem + stage * 16384;
      const int rb = (it / kb_total) % nrb, kb = it % kb_total;
      if (mode == 2) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], "
            "[%1, {%3, %4, %5}], [%2], %6;" ::"r"(tc::smem_u32(dst + cta * 8192)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(tc::smem_u32(&full[stage])), "r"(kb * 64),
            "r"(r0 + rb * 128 + 64 * static_cast<int>(cta)), "r"(0), "h"(static_cast<uint16_t>(3))
            : "memory");
      } else if (mode == 3) {
        tc::tma_load_3d(&tm, dst, &full[stage], kb * 64, r0 + rb * 128, 0);
        tc::tma_load_3d(&tm, dst + 8192, &full[stage], kb * 64, r0 + rb * 128 + 64, 0);
      } else {
        tc::tma_load_3d(&tm128, dst, &full[stage], kb * 64, r0 + rb * 128, 0);
      }
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (tid == 32) {
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; it < items; ++it) {
      tc::mbar_wait(&full[stage], phase);
      if (mode == 2) {
        tc::mbar_arrive_cluster(&empty[stage], 0);
        tc::mbar_arrive_cluster(&empty[stage], 1);
      } else {
        tc::mbar_arrive(&empty[stage]);
      }
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
  tc::cluster_sync();
}

int main() {
  const int K = 5504, N = 4096 * 8;  // 8 experts' W_down rows stacked: 360 MB
  const size_t bytes = static_cast<size_t>(N) * K * 2;
  uint8_t* w;
  cudaMalloc(&w, bytes);
  cudaMemset(w, 1, bytes);
  uint8_t* fl;
  const size_t flb = 512ull << 20;
  cudaMalloc(&fl, flb);
  CUtensorMap tm;
  CUtensorMap tm128;
  if (!tc::make_map_3d(&tm, w, K, N, 1, 64, 64) || !tc::make_map_3d(&tm128, w, K, N, 1, 64, 128)) {
    printf("map failed\n");
    return 1;
  }
  const int kb_total = K / 64;  // 86
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
  cudaFuncSetAttribute(stream_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("{\"runs\": [\n");
  bool first = true;
  // long streams: rows_per_cta 1024 (11 MB per CTA, cold, distinct rows) or 128 rows re-read 8x (hot in L2)
  for (int mode : {0, 2, 3, 4})
    for (int hot = 1; hot >= 0; --hot)
      for (int S : {12})
        for (int nct : {8, 16, 32, 74, 148}) {
          const int rpc = hot ? 128 : (nct <= 32 ? 1024 : 128), reps = hot ? 8 : 1;
          float best = 1e9f;
          for (int rep = 0; rep < 3; ++rep) {
            cudaMemsetAsync(fl, rep, flb);
            cudaEventRecord(a);
            if (mode == 0) stream_kernel<<<nct, 64, 200 * 1024 + 1024>>>(tm, w, K, rpc, S, mode, kb_total, reps);
            else stream_mc_kernel<<<nct, 64, 200 * 1024 + 1024>>>(tm, tm128, K, rpc, S, mode, kb_total, reps);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
          }
          const double per = static_cast<double>(rpc) * kb_total * 128 * reps;
          printf("%s{\"mode\": %d, \"hot\": %d, \"S\": %d, \"ctas\": %d, \"MB_per_cta\": %.1f, \"us\": %.1f, "
                 "\"GBps_per_sm\": %.1f, \"GBps_total\": %.0f}",
                 first ? "" : ",\n", mode, hot, S, nct, per / 1e6, best * 1e3, per / (best * 1e-3) / 1e9,
                 per * nct / (best * 1e-3) / 1e9);
          first = false;
        }
  printf("\n], \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
