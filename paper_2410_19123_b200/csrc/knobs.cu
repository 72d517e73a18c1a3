// knobs.cpp — the library's lab/test switches (A/B measurement of kernel variants; DESIGN.md §6 table).
//
// Every switch is read from the environment ONCE, on the first launch that consults any of them, and can be
// overridden afterwards through readme_debug_set_knob (tests and lab scripts flip variants inside one
// process that way). Defaults are the measured-best paths; no switch changes the arithmetic of the layer
// except where DESIGN.md says so (each variant is tested bitwise against the default).
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "kernels.h"

namespace readme {

namespace {

struct KnobDef {
  const char* name;  // readme_debug_set_knob name
  const char* env;   // environment variable read once at first use
  int def;           // default value
};

// Order matches enum class Knob (kernels.h).
constexpr KnobDef kDefs[static_cast<int>(Knob::kCount)] = {
    {"route", "README_ROUTE", 0},                  // 0 auto, 1 cluster (single launch), 2 lookback (multi-CTA)
    {"route_cluster", "README_ROUTE_CLUSTER", 0},  // 0 auto, else forced cluster size 1/2/4/8/16
    {"route_tile", "README_ROUTE_TILE", 0},        // 0 auto, else tokens per lookback tile
    {"dispatch", "README_DISPATCH", 0},            // 0 auto, 1 scatter, 2 gather kernel, 3 gather fused into the FFN (moe_layer)
    {"dispatch_bulk", "README_DISPATCH_BULK", -1}, // -1 auto, 0 warp-per-row, 1 bulk-copy scatter dispatch
    {"combine_bulk", "README_COMBINE_BULK", -1},   // -1 auto, 0 warp-per-row, 1 bulk-copy k=1 combine
    {"perm_unroll_d", "README_PERM_UNROLL_D", 4},  // 128-bit loads in flight per lane, scatter dispatch (4|8)
    {"perm_unroll_c", "README_PERM_UNROLL_C", 8},  // same, k = 1 gather combine (4|8)
    {"ffn_kernel", "README_FFN_KERNEL", 0},        // 0 single launch, 1 split (two CTA-pair launches), 2 unfused
    {"ffn_mt", "README_FFN_MT", 0},                // 0 auto, 128 | 256 m-tile rows of the single-launch FFN
    {"ffn_pairs", "README_FFN_PAIRS", 0},          // 0 all co-resident pairs, else at most n CTA pairs
    {"ffn_askip", "README_FFN_ASKIP", 1},          // second CTA skips A loads of tiles with <= 64 rows
    {"ffn_order", "README_FFN_ORDER", 0},          // 1: gate/up tiles N-tile fastest
    {"ffn_swap", "README_FFN_SWAP", -1},           // -1 auto, else segment tails of <= n rows run swap-AB
    {"ffn_spin", "README_FFN_SPIN", 25},           // log2 of the readiness-poll limit (timeout -> dev_status)
    {"ffn_merge", "README_FFN_MERGE", -1},         // 256-row m-tiles: segment tails ride on full m-tiles (-1: with ffn_dyn)
    {"ffn_dyn", "README_FFN_DYN", -1},             // -1 auto (dynamic order at <= 16384 rows of 256-row m-tiles), 0 static, 1 dynamic
    {"ffn_claim", "README_FFN_CLAIM", 24},         // dynamic order: claim the next tile this many K steps before a tile's loads end
};

std::atomic<int> g_val[static_cast<int>(Knob::kCount)];
std::once_flag g_once;

int parse_env(int i) {
  const char* v = getenv(kDefs[i].env);
  if (!v || !*v) return kDefs[i].def;
  switch (static_cast<Knob>(i)) {
    case Knob::kRoute:
      if (strcmp(v, "cluster") == 0) return 1;
      if (strcmp(v, "lookback") == 0) return 2;
      return 0;
    case Knob::kDispatch:
      if (strcmp(v, "scatter") == 0) return 1;
      if (strcmp(v, "gather") == 0) return 2;
      if (strcmp(v, "fused") == 0) return 3;
      return 0;
    case Knob::kFfnKernel:
      if (strcmp(v, "split") == 0) return 1;
      if (strcmp(v, "unfused") == 0) return 2;
      return 0;
    default:
      return atoi(v);
  }
}

void load_once() {
  std::call_once(g_once, [] {
    for (int i = 0; i < static_cast<int>(Knob::kCount); ++i) g_val[i].store(parse_env(i), std::memory_order_relaxed);
  });
}

int find(const char* name) {
  if (!name) return -1;
  for (int i = 0; i < static_cast<int>(Knob::kCount); ++i)
    if (strcmp(kDefs[i].name, name) == 0) return i;
  return -1;
}

}  // namespace

int knob(Knob k) {
  load_once();
  return g_val[static_cast<int>(k)].load(std::memory_order_relaxed);
}

}  // namespace readme

using namespace readme;

#pragma GCC visibility push(default)
extern "C" {

readme_status readme_debug_set_knob(const char* name, int32_t value) {
  load_once();
  const int i = find(name);
  README_CHECK_ARG(i >= 0, "unknown knob '%s'", name ? name : "(null)");
  g_val[i].store(value, std::memory_order_relaxed);
  return README_OK;
}

readme_status readme_debug_get_knob(const char* name, int32_t* value) {
  load_once();
  const int i = find(name);
  README_CHECK_ARG(i >= 0 && value != nullptr, "unknown knob '%s' or null value", name ? name : "(null)");
  *value = g_val[i].load(std::memory_order_relaxed);
  return README_OK;
}

readme_status readme_debug_reset_knob(const char* name) {
  load_once();
  const int i = find(name);
  README_CHECK_ARG(i >= 0, "unknown knob '%s'", name ? name : "(null)");
  g_val[i].store(parse_env(i), std::memory_order_relaxed);  // back to the environment's (or built-in) value
  return README_OK;
}

}  // extern "C"
#pragma GCC visibility pop
