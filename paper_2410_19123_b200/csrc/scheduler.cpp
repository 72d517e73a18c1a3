// scheduler.cpp — host runtime for READ-ME's expert-aware batching (Alg. 1, §4.2).
//
// Pre-gating fixes every queued token's expert before it reaches the backbone, so the
// serving loop can keep one FIFO per expert ("ReqQueueByExpert") and form each batch to
// minimise the number of unique experts (per-token latency grows linearly with them):
//   repeat: E = argmax_e len(queue_e)            (ties -> lower expert id)
//           if len(queue_E) == 0: stop            (reading Q12: the pseudocode never terminates otherwise)
//           if len(queue_E) < MaxTokenLen - len(Scheduled): take the whole queue, continue
//           elif MaxTokenLen - len(Scheduled) >= 0: take its first (MaxTokenLen - len(Scheduled)), stop
//           else stop
// (reading Q12: lines 250, 256-257 index the queue with the stale loop variable k; E is meant.)
// The batch it returns is grouped by expert already, in the order the queues were taken.
#include <stdint.h>

#include <deque>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/readme.h"

struct readme_scheduler {
  std::vector<std::deque<int64_t>> q;
  std::mutex mu;
};

#pragma GCC visibility push(default)
extern "C" {

readme_scheduler* readme_scheduler_create(int32_t E) {
  if (E < 1 || E > README_MAX_EXPERTS) return nullptr;
  readme_scheduler* s = new (std::nothrow) readme_scheduler;
  if (!s) return nullptr;
  s->q.resize(static_cast<size_t>(E));
  return s;
}

void readme_scheduler_destroy(readme_scheduler* s) { delete s; }

readme_status readme_scheduler_push(readme_scheduler* s, const int64_t* token_ids, const int32_t* experts,
                                    int64_t n) {
  if (!s || n < 0 || (n > 0 && (!token_ids || !experts))) return README_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> g(s->mu);
  const int64_t E = static_cast<int64_t>(s->q.size());
  for (int64_t i = 0; i < n; ++i)
    if (experts[i] < 0 || experts[i] >= E) return README_ERR_INVALID_ARG;  // nothing pushed on error
  for (int64_t i = 0; i < n; ++i) s->q[static_cast<size_t>(experts[i])].push_back(token_ids[i]);
  return README_OK;
}

int64_t readme_scheduler_queued(readme_scheduler* s, int32_t e) {
  if (!s) return -1;
  std::lock_guard<std::mutex> g(s->mu);
  if (e >= 0) return e < static_cast<int32_t>(s->q.size()) ? static_cast<int64_t>(s->q[e].size()) : -1;
  int64_t n = 0;
  for (const auto& d : s->q) n += static_cast<int64_t>(d.size());
  return n;
}

int64_t readme_scheduler_next_batch(readme_scheduler* s, int64_t max_tokens, int64_t* token_ids, int32_t* experts) {
  if (!s || max_tokens < 0 || (max_tokens > 0 && (!token_ids || !experts))) return -1;
  std::lock_guard<std::mutex> g(s->mu);
  const int32_t E = static_cast<int32_t>(s->q.size());
  int64_t n = 0;
  for (;;) {
    int32_t best = 0;
    for (int32_t e = 1; e < E; ++e)
      if (s->q[e].size() > s->q[best].size()) best = e;
    std::deque<int64_t>& qb = s->q[best];
    const int64_t len = static_cast<int64_t>(qb.size());
    if (len == 0) break;
    const int64_t avail = max_tokens - n;
    if (len < avail) {
      for (int64_t t : qb) {
        token_ids[n] = t;
        experts[n++] = best;
      }
      qb.clear();
    } else if (avail >= 0) {
      for (int64_t i = 0; i < avail; ++i) {
        token_ids[n] = qb.front();
        experts[n++] = best;
        qb.pop_front();
      }
      break;
    } else {
      break;
    }
  }
  return n;
}

}  // extern "C"
#pragma GCC visibility pop
