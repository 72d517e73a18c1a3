"""Expert cache of the memory-constrained mode (§4.1): the plain-Python oracle
(oracle/cache.py) is pinned by SPEC's worked examples, Belady's optimality against exhaustive search and
capacity monotonicity; the native policy (readme_cache_*, host C++) must reproduce it access by access."""
import json
import os

import numpy as np
import pytest

from oracle import cache

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cache_examples.json")


@pytest.mark.parametrize("case", json.load(open(GOLD))["cases"], ids=lambda c: c["cite"][:11])
def test_cache_spec_examples(case):
    if case["policy"] == "optimal":
        assert cache.optimal_hits(case["trace"], case["k"]) == case["hits"]
        return
    hits, misses, log = cache.simulate(case["trace"], case["k"], case["policy"])
    assert hits == case["hits"]
    if "evicted_at_2" in case:
        assert log[2][2] == case["evicted_at_2"]


def test_cold_misses_only_when_capacity_covers_all():
    g = np.random.default_rng(1)
    tr = g.integers(0, 5, size=60).tolist()
    for pol in ("lru", "belady", "random"):
        h, m, _ = cache.simulate(tr, 5, pol)
        assert m == len(set(tr)) and h == len(tr) - m


def test_belady_is_optimal():
    """Belady hits equal the exhaustive optimum on random short strings."""
    g = np.random.default_rng(2)
    for _ in range(300):
        n, nk, k = int(g.integers(1, 13)), int(g.integers(1, 5)), int(g.integers(1, 4))
        tr = g.integers(0, nk, size=n).tolist()
        assert cache.simulate(tr, k, "belady")[0] == cache.optimal_hits(tr, k)


def test_capacity_monotonicity():
    g = np.random.default_rng(3)
    for _ in range(50):
        tr = g.integers(0, 8, size=80).tolist()
        for pol in ("lru", "belady"):
            hs = [cache.simulate(tr, k, pol)[0] for k in range(1, 9)]
            assert all(a <= b for a, b in zip(hs, hs[1:])), (pol, hs)


@pytest.fixture(scope="module")
def rd():
    from paper_2410_19123_b200 import build, readme
    build.build()
    return readme


@pytest.mark.parametrize("policy", ["lru", "belady", "random"])
def test_native_cache_matches_oracle(rd, policy):
    g = np.random.default_rng(4)
    for trial in range(40):
        n, nk, k = int(g.integers(1, 200)), int(g.integers(1, 20)), int(g.integers(1, 8))
        keys = g.integers(0, nk, size=n).astype(np.int64) * 8 + 3  # arbitrary int64 keys
        c = rd.ExpertCache(k, policy, seed=trial)
        c.set_future(keys, np.arange(n))
        _, _, log = cache.simulate(keys.tolist(), k, policy, seed=trial)
        slots = {}
        for t, key in enumerate(keys.tolist()):
            hit, slot, ev = c.access(key, t)
            assert (hit, ev) == (log[t][1], log[t][2])
            assert 0 <= slot < k
            if ev >= 0:
                assert slots.pop(ev) == slot  # the victim's slot is reused
            slots[key] = slot
        hits, misses = c.stats()
        assert hits + misses == n


# ---- protect_since: the experts of the step being assembled are never evicted (reading Q18) -------------

def _step_trace(g, E, L, B, u):
    """Accesses of B batches x L layers; each batch touches u experts (same in every layer); the protect
    boundary of an access is the first access of its (batch, layer) step."""
    trace, prot = [], []
    for _b in range(B):
        ex = sorted(g.choice(E, u, replace=False).tolist())
        for l in range(L):
            start = len(trace)
            for e in ex:
                trace.append(l * E + e)
                prot.append(start)
    return trace, prot


def _optimal_protected(trace, cap, prot):
    """Max hits over every eviction sequence that never evicts a protected resident (exhaustive)."""
    from functools import lru_cache
    trace = tuple(trace)

    @lru_cache(maxsize=None)
    def best(t, res):  # res: sorted tuple of (key, last access)
        if t == len(trace):
            return 0
        key = trace[t]
        if key in [r[0] for r in res]:
            return 1 + best(t + 1, tuple(sorted([r for r in res if r[0] != key] + [(key, t)])))
        if len(res) < cap:
            return best(t + 1, tuple(sorted(res + ((key, t),))))
        return max(best(t + 1, tuple(sorted([r for r in res if r != v] + [(key, t)])))
                   for v in res if v[1] < prot[t])

    return best(0, ())


def test_protected_belady_is_optimal_on_step_traces():
    g = np.random.default_rng(11)
    for _ in range(150):
        u = int(g.integers(1, 3))
        tr, prot = _step_trace(g, int(g.integers(3, 6)), int(g.integers(1, 3)), int(g.integers(1, 4)), u)
        cap = int(g.integers(u, u + 3))
        assert cache.simulate(tr, cap, "belady", protect_since=prot)[0] == _optimal_protected(tr, cap, prot)


@pytest.mark.parametrize("policy", ["lru", "belady", "random"])
def test_protect_keeps_the_step_resident(policy):
    g = np.random.default_rng(12)
    for trial in range(60):
        u = int(g.integers(1, 4))
        tr, prot = _step_trace(g, 8, int(g.integers(1, 4)), int(g.integers(1, 5)), u)
        _, _, log = cache.simulate(tr, u, policy, seed=trial, protect_since=prot)  # capacity = one step
        for t, (_t, _hit, ev) in enumerate(log):
            assert ev not in tr[prot[t]:t]  # never evicts an expert this step already placed
        # with no protection boundary in force (protect_since = t + 1 protects nothing) the rule is unchanged
        free = [t + 1 for t in range(len(tr))]
        assert cache.simulate(tr, u + 1, policy, seed=trial, protect_since=free) == \
            cache.simulate(tr, u + 1, policy, seed=trial)


@pytest.mark.parametrize("policy", ["lru", "belady", "random"])
def test_native_cache_protect_matches_oracle(rd, policy):
    g = np.random.default_rng(13)
    for trial in range(40):
        u = int(g.integers(1, 4))
        tr, prot = _step_trace(g, 8, int(g.integers(1, 5)), int(g.integers(1, 6)), u)
        cap = int(g.integers(u, u + 4))
        _, _, log = cache.simulate(tr, cap, policy, seed=trial, protect_since=prot)
        c = rd.ExpertCache(cap, policy, seed=trial)
        c.set_future(np.array(tr, np.int64), np.arange(len(tr)))
        for t, key in enumerate(tr):
            hit, _slot, ev = c.access(key, t, protect_since=prot[t])
            assert (hit, ev) == (log[t][1], log[t][2])


def test_native_cache_all_protected_raises(rd):
    c = rd.ExpertCache(2, "lru")
    c.access(1, 0, protect_since=0)
    c.access(2, 1, protect_since=0)
    with pytest.raises(RuntimeError):
        c.access(3, 2, protect_since=0)


# ---- the prefetch two-resource schedule (SPEC.md:413-420 hand Gantt charts) ---------------

def test_prefetch_schedule_spec_examples():
    from oracle.prefetch import simulate_prefetch
    s, f, m = simulate_prefetch([2, 2, 2], [1, 1, 1], "prefetch")
    assert (s, f, m) == ([1, 3, 5], [3, 5, 7], 7)
    assert simulate_prefetch([2, 2, 2], [1, 1, 1], "on_demand")[2] == 9
    s, f, m = simulate_prefetch([2, 2, 2], [0, 1, 1], "prefetch")  # first layer cached
    assert (s, m) == ([0, 2, 4], 6)
    for mode in ("prefetch", "on_demand"):
        assert simulate_prefetch([2, 3, 4], [0, 0, 0], mode)[2] == 9  # all cached: sum of compute
    with pytest.raises(ValueError):
        simulate_prefetch([1], [-1], "prefetch")


def test_prefetch_schedule_bounds():
    """Prefetch never loses to on-demand, and its makespan lies between max(sum load + last compute,
    first load + sum compute) and the on-demand sum."""
    from oracle.prefetch import simulate_prefetch
    g = np.random.default_rng(21)
    for _ in range(300):
        n = int(g.integers(1, 12))
        c = g.uniform(0, 5, n).tolist()
        x = (g.uniform(0, 5, n) * (g.random(n) < 0.7)).tolist()
        pf = simulate_prefetch(c, x, "prefetch")[2]
        od = simulate_prefetch(c, x, "on_demand")[2]
        assert od == pytest.approx(sum(c) + sum(x))
        assert pf <= od + 1e-9
        assert pf >= max(sum(x) + c[-1], x[0] + sum(c)) - 1e-9
