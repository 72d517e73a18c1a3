"""oracle.cache — TEST INFRASTRUCTURE ONLY. Expert-cache policies of §4.1 in plain Python:
LRU, Random (same splitmix64 stream as the native runtime), and the Belady-inspired rule the paper derives
from pre-gating: on a miss with a full cache evict e_evict = argmax_{e in C(t-1)} F(e, t), F = next access
after t (never again = +inf); ties -> lowest key (reading Q17). Plus an exhaustive optimal
oracle (branching over every eviction choice) for short traces — Belady's optimality is the pin."""
from functools import lru_cache

MASK = (1 << 64) - 1


def _splitmix64(state):
    state = (state + 0x9E3779B97F4A7C15) & MASK
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return state, z ^ (z >> 31)


def simulate(trace, capacity, policy, seed=0, protect_since=None):
    """trace: list of keys accessed at times 0..n-1. Returns (hits, misses, [(t, hit, evicted)]).
    protect_since (optional, one int per access): a resident last accessed at or after protect_since[t] is not
    a candidate for eviction at time t — the experts of the layer being assembled must all be resident when it
    runs (reading Q18). If no resident is a candidate, the access raises (the caller sized the
    cache below one layer's experts)."""
    resident, last, log = [], {}, []
    rng = seed
    hits = misses = 0
    for t, key in enumerate(trace):
        if key in resident:
            hits += 1
            last[key] = t
            log.append((t, True, -1))
            continue
        misses += 1
        ev = -1
        if len(resident) >= capacity:
            res = sorted(resident)
            if protect_since is not None:
                res = [k for k in res if last[k] < protect_since[t]]
                if not res:
                    raise ValueError("every resident expert is protected")
            if policy == "lru":
                ev = min(res, key=lambda k: (last[k], k))
            elif policy == "belady":
                def F(k):
                    for t2 in range(t + 1, len(trace)):
                        if trace[t2] == k:
                            return t2
                    return float("inf")
                ev = max(res, key=lambda k: (F(k), -k))
            else:
                rng, r = _splitmix64(rng)
                ev = res[r % len(res)]
            resident.remove(ev)
            last.pop(ev, None)
        resident.append(key)
        last[key] = t
        log.append((t, False, ev))
    return hits, misses, log


def optimal_hits(trace, capacity):
    """Maximum achievable hits over every eviction-decision sequence (exhaustive; short traces only)."""
    trace = tuple(trace)

    @lru_cache(maxsize=None)
    def best(t, res):
        if t == len(trace):
            return 0
        key = trace[t]
        if key in res:
            return 1 + best(t + 1, res)
        if len(res) < capacity:
            return best(t + 1, tuple(sorted(res + (key,))))
        return max(best(t + 1, tuple(sorted(tuple(r for r in res if r != v) + (key,)))) for v in res)

    return best(0, ())
