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
