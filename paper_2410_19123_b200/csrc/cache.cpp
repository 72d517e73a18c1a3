// cache.cpp — host runtime for READ-ME's memory-constrained mode (§4.1; NEXT-4 of SURVEY
// §8(f)): an expert cache of `capacity` device slots with LRU, Random and the Belady-inspired policy the paper
// derives from pre-gating — with routing computed at the outset, the future reference string of (layer,
// expert) accesses is known, so on a miss with a full cache the policy evicts
//     e_evict = argmax_{e in C(t-1)} F(e, t)      (F = next access time after t; never again = +inf)
// (PAPER.md:208). Ties (several +inf, equal next use) go to the lowest key (reading Q17).
// Keys are arbitrary int64 (layer * E + expert in the offload pipeline). Each resident key owns a slot index
// in [0, capacity); a miss reuses the evicted key's slot, so slot contents can be copied in place.
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <new>
#include <unordered_map>
#include <vector>

#include "../../include/readme.h"

struct readme_expert_cache {
  int32_t capacity;
  int32_t policy;
  uint64_t rng;
  int64_t clock = 0;
  std::unordered_map<int64_t, int32_t> slot_of;       // resident key -> slot
  std::unordered_map<int64_t, int64_t> last_use;      // resident key -> last access time (LRU)
  std::vector<int32_t> free_slots;
  std::unordered_map<int64_t, std::vector<int64_t>> future;  // key -> ascending access times (Belady)
  int64_t hits = 0, misses = 0;
  std::mutex mu;
};

namespace {

uint64_t splitmix64(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int64_t next_use(const readme_expert_cache* c, int64_t key, int64_t t) {
  auto it = c->future.find(key);
  if (it == c->future.end()) return INT64_MAX;
  const auto& v = it->second;
  auto j = std::upper_bound(v.begin(), v.end(), t);
  return j == v.end() ? INT64_MAX : *j;
}

}  // namespace

#pragma GCC visibility push(default)
extern "C" {

readme_expert_cache* readme_cache_create(int32_t capacity, int32_t policy, uint64_t seed) {
  if (capacity < 1 || policy < 0 || policy > 2) return nullptr;
  readme_expert_cache* c = new (std::nothrow) readme_expert_cache;
  if (!c) return nullptr;
  c->capacity = capacity;
  c->policy = policy;
  c->rng = seed;
  for (int32_t s = capacity - 1; s >= 0; --s) c->free_slots.push_back(s);
  return c;
}

void readme_cache_destroy(readme_expert_cache* c) { delete c; }

readme_status readme_cache_set_future(readme_expert_cache* c, const int64_t* keys, const int64_t* times, int64_t n) {
  if (!c || n < 0 || (n > 0 && (!keys || !times))) return README_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> g(c->mu);
  c->future.clear();
  for (int64_t i = 0; i < n; ++i) c->future[keys[i]].push_back(times[i]);
  for (auto& kv : c->future) std::sort(kv.second.begin(), kv.second.end());
  return README_OK;
}

int32_t readme_cache_access(readme_expert_cache* c, int64_t key, int64_t t, int64_t protect_since, int64_t* evicted,
                            int32_t* slot) {
  if (!c) return -1;
  std::lock_guard<std::mutex> g(c->mu);
  if (evicted) *evicted = -1;
  auto hit = c->slot_of.find(key);
  if (hit != c->slot_of.end()) {
    ++c->hits;
    c->last_use[key] = t;
    if (slot) *slot = hit->second;
    return 1;
  }
  ++c->misses;
  int32_t s;
  if (!c->free_slots.empty()) {
    s = c->free_slots.back();
    c->free_slots.pop_back();
  } else {
    // choose the victim among the residents, deterministically (ties -> lowest key)
    std::vector<int64_t> res;
    res.reserve(c->slot_of.size());
    for (const auto& kv : c->slot_of)
      if (c->last_use[kv.first] < protect_since) res.push_back(kv.first);  // keys in use are not evictable
    if (res.empty()) {
      --c->misses;
      return -2;
    }
    std::sort(res.begin(), res.end());
    int64_t victim = res[0];
    if (c->policy == 0) {  // LRU: least recently accessed
      int64_t best = INT64_MAX;
      for (int64_t k : res) {
        const int64_t lu = c->last_use[k];
        if (lu < best) {
          best = lu;
          victim = k;
        }
      }
    } else if (c->policy == 1) {  // Belady: next use farthest in the future
      int64_t best = -1;
      for (int64_t k : res) {
        const int64_t nu = next_use(c, k, t);
        if (nu > best) {
          best = nu;
          victim = k;
        }
      }
    } else {  // Random (seeded)
      victim = res[static_cast<size_t>(splitmix64(c->rng) % res.size())];
    }
    s = c->slot_of[victim];
    c->slot_of.erase(victim);
    c->last_use.erase(victim);
    if (evicted) *evicted = victim;
  }
  c->slot_of[key] = s;
  c->last_use[key] = t;
  if (slot) *slot = s;
  return 0;
}

int32_t readme_cache_lookup(readme_expert_cache* c, int64_t key) {
  if (!c) return -1;
  std::lock_guard<std::mutex> g(c->mu);
  auto it = c->slot_of.find(key);
  return it == c->slot_of.end() ? -1 : it->second;
}

void readme_cache_stats(readme_expert_cache* c, int64_t* hits, int64_t* misses) {
  if (!c) return;
  std::lock_guard<std::mutex> g(c->mu);
  if (hits) *hits = c->hits;
  if (misses) *misses = c->misses;
}

}  // extern "C"
#pragma GCC visibility pop
