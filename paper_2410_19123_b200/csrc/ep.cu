// ep.cu — expert parallelism over peer memory (stretch C4): the dispatch all-to-all is
// fused into the dispatch kernel (rows are stored straight into the owning rank's receive buffer over
// NVLink) and the combine all-to-all into the down projection's epilogue (ffn_layer2_kernel<2> stores
// each result row into its source rank's output). Ranks synchronise with release/acquire flag words in
// peer memory — no NCCL call and no host synchronisation on the per-layer path.
//
// Pre-gating makes the exchange plan a per-batch object ("expert selection can be
// determined at the outset"; :237 a token keeps its expert in every layer): every rank publishes its
// per-expert counts to every peer once per batch (readme_ep_publish_counts), and each rank derives
//   seg_offsets  its receive layout: segment (source p, local expert el) holds table[p][me*El+el] rows,
//                source-major — so each expert's rows arrive in global token order (P12);
//   row_base[e]  where its own rows for global expert e start in the owner's receive buffer
// (readme_ep_plan); every layer then reuses them.
#include "kernels.h"

namespace readme {

namespace {

constexpr int kEpThreads = 256;

__device__ __forceinline__ void st_release_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct PeerPtrs {
  void* p[kMaxPeers];
};

// The phase epoch lives in device memory (bumped here, read by the wait), so a captured CUDA graph of a
// layer stays correct on every replay.
__global__ void ep_signal_kernel(PeerPtrs flags, int G, int me, uint64_t* epoch) {
  if (threadIdx.x != 0) return;
  const uint64_t v = *epoch + 1;
  *epoch = v;
  __threadfence_system();
  for (int q = 0; q < G; ++q) st_release_sys_u64(static_cast<uint64_t*>(flags.p[q]) + me, v);
}

__global__ void ep_wait_kernel(const uint64_t* flags, int G, const uint64_t* epoch, uint32_t* dev_status) {
  const int p = threadIdx.x;
  const uint64_t value = *epoch;
  if (p < G) {
    uint32_t spins = 0;
    while (ld_acquire_sys_u64(flags + p) < value) {
      __nanosleep(256);
      if (++spins == (1u << 25)) {  // ~10 s: a peer never arrived; report instead of hanging
        if (dev_status) atomicOr(dev_status, README_DEV_EP_TIMEOUT);
        break;
      }
    }
  }
  __syncthreads();
  __threadfence_system();
}

__global__ void ep_publish_kernel(const int32_t* __restrict__ counts, int E, PeerPtrs tables, int G, int me) {
  for (int i = threadIdx.x; i < G * E; i += blockDim.x) {
    const int q = i / E, e = i % E;
    static_cast<int32_t*>(tables.p[q])[me * E + e] = counts[e];
  }
}

// table [G][E]: rows source p holds for global expert e. One thread; G*E <= 8*256.
__global__ void ep_plan_kernel(const int32_t* __restrict__ table, int G, int E, int me, int32_t* seg_offsets,
                               int32_t* row_base) {
  if (threadIdx.x != 0) return;
  const int El = E / G;
  int acc = 0;
  for (int p = 0; p < G; ++p)
    for (int el = 0; el < El; ++el) {
      seg_offsets[p * El + el] = acc;
      acc += table[p * E + me * El + el];
    }
  seg_offsets[G * El] = acc;
  for (int q = 0; q < G; ++q) {
    int base = 0;  // rows of sources p < me on q, then my rows for q's earlier local experts
    for (int p = 0; p < me; ++p)
      for (int el = 0; el < El; ++el) base += table[p * E + q * El + el];
    for (int el = 0; el < El; ++el) {
      row_base[q * El + el] = base;
      base += table[me * E + q * El + el];
    }
  }
}

// One warp per slot s = t*k + j: sorted row r = dest[s] of expert e (offsets) goes to rank q = e / El at
// row row_base[e] + r - offsets[e]; its row-map entry names where the result must return.
__global__ void __launch_bounds__(kEpThreads)
ep_dispatch_kernel(const uint4* __restrict__ x, int vec, int64_t nslots, int k, const int32_t* __restrict__ dest,
                   const int32_t* __restrict__ offsets, const int32_t* __restrict__ row_base, int E, int G, int me,
                   PeerPtrs peer_x, PeerPtrs peer_map, int64_t vrows, int to_token, uint32_t* dev_status) {
  __shared__ int32_t s_off[README_MAX_EXPERTS + 1];
  __shared__ int32_t s_base[README_MAX_EXPERTS];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) s_off[i] = offsets[i];
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_base[i] = row_base[i];
  __syncthreads();
  const int El = E / G;
  const int lane = threadIdx.x % kWarp;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kEpThreads / kWarp);
  for (int64_t s = blockIdx.x * static_cast<int64_t>(kEpThreads / kWarp) + threadIdx.x / kWarp; s < nslots;
       s += warps) {
    const int32_t r = __ldg(dest + s);
    if (r < 0 || r >= s_off[E]) {
      if (lane == 0 && dev_status) atomicOr(dev_status, README_DEV_BAD_INDEX);
      continue;
    }
    int lo = 0, hi = E - 1;  // expert e: s_off[e] <= r < s_off[e+1]
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int e = lo, q = e / El;
    const int64_t row = static_cast<int64_t>(s_base[e]) + (r - s_off[e]);
    uint4* dst = static_cast<uint4*>(peer_x.p[q]) + row * vec;
    const uint4* src = x + (s / k) * vec;
    int i = lane;  // 4 loads in flight per lane before the (possibly remote) stores
    for (; i + 3 * kWarp < vec; i += 4 * kWarp) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ld_nc_v4(src + i + u * kWarp);
#pragma unroll
      for (int u = 0; u < 4; ++u) dst[i + u * kWarp] = v[u];
    }
    for (; i < vec; i += kWarp) dst[i] = ld_nc_v4(src + i);
    if (lane == 0)
      static_cast<int32_t*>(peer_map.p[q])[row] = static_cast<int32_t>(me * vrows + (to_token ? s / k : r));
  }
  __threadfence_system();
}

PeerPtrs pack(void* const* v, int G) {
  PeerPtrs pp{};
  for (int i = 0; i < G; ++i) pp.p[i] = v[i];
  return pp;
}

}  // namespace

readme_status launch_ep_signal(uint64_t* const* peer_flags, int G, int me, uint64_t* epoch, cudaStream_t st) {
  ep_signal_kernel<<<1, 32, 0, st>>>(pack(reinterpret_cast<void* const*>(peer_flags), G), G, me, epoch);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_ep_wait(const uint64_t* flags, int G, const uint64_t* epoch, uint32_t* dev_status,
                             cudaStream_t st) {
  ep_wait_kernel<<<1, 32, 0, st>>>(flags, G, epoch, dev_status);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_ep_publish(const int32_t* counts, int E, int32_t* const* peer_tables, int G, int me,
                                cudaStream_t st) {
  ep_publish_kernel<<<1, 256, 0, st>>>(counts, E, pack(reinterpret_cast<void* const*>(peer_tables), G), G, me);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_ep_plan(const int32_t* table, int G, int E, int me, int32_t* seg_offsets, int32_t* row_base,
                             cudaStream_t st) {
  ep_plan_kernel<<<1, 32, 0, st>>>(table, G, E, me, seg_offsets, row_base);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

readme_status launch_ep_dispatch(const void* x, size_t row_bytes, int64_t T, int k, const int32_t* dest,
                                 const int32_t* offsets, const int32_t* row_base, int E, int G, int me,
                                 void* const* peer_x, int32_t* const* peer_map, int64_t vrows, int to_token,
                                 uint32_t* dev_status, cudaStream_t st) {
  const int64_t nslots = T * k;
  if (nslots == 0) return README_OK;
  const int vec = static_cast<int>(row_bytes / 16);
  const int64_t want = (nslots + (kEpThreads / kWarp) - 1) / (kEpThreads / kWarp);
  const int grid = static_cast<int>(want < 8L * num_sms() ? want : 8L * num_sms());
  ep_dispatch_kernel<<<grid, kEpThreads, 0, st>>>(static_cast<const uint4*>(x), vec, nslots, k, dest, offsets,
                                                  row_base, E, G, me, pack(peer_x, G),
                                                  pack(reinterpret_cast<void* const*>(peer_map), G), vrows,
                                                  to_token, dev_status);
  README_CUDA(cudaGetLastError());
  return README_OK;
}

}  // namespace readme
