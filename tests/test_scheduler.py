"""Expert-aware batching (Alg. 1): the plain-Python oracle (oracle/alg1.py) is pinned by
SPEC's worked examples and invariants; the native scheduler (readme_scheduler_*, host C++ in
libreadme_b200.so, no GPU) must reproduce it exactly."""
import json
import os

import numpy as np
import pytest

from oracle import alg1

GOLD = os.path.join(os.path.dirname(__file__), "golden", "alg1_examples.json")


def _queues(sizes, start=0):
    out, t = [], start
    for n in sizes:
        out.append(list(range(t, t + n)))
        t += n
    return out


def _runs(scheduled):
    runs = []
    for tok, e in scheduled:
        if runs and runs[-1][0] == e:
            runs[-1][1] += 1
        else:
            runs.append([e, 1])
    return runs


@pytest.mark.parametrize("case", json.load(open(GOLD))["cases"], ids=lambda c: c["cite"][:11])
def test_alg1_spec_examples(case):
    sched, rest = alg1.schedule(_queues(case["queue_sizes"]), case["max"])
    assert _runs(sched) == case["taken"]
    assert [len(q) for q in rest] == case["remaining"]


def test_alg1_invariants():
    g = np.random.default_rng(3)
    for _ in range(300):
        E = int(g.integers(1, 9))
        sizes = g.integers(0, 12, size=E).tolist()
        mx = int(g.integers(0, 40))
        qs = _queues(sizes)
        sched, rest = alg1.schedule(qs, mx)
        assert len(sched) <= mx
        assert sum(len(q) for q in rest) + len(sched) == sum(sizes)        # conservation
        if sum(sizes) <= mx:
            assert len(sched) == sum(sizes)                                 # everything fits -> all scheduled
        else:
            assert len(sched) == mx                                         # a full batch otherwise
        for e in range(E):                                                  # FIFO per expert
            taken = [t for t, ee in sched if ee == e]
            assert taken == qs[e][:len(taken)] and rest[e] == qs[e][len(taken):]
        # whole queues are taken largest-first (ties -> lower id); at most one queue is split
        runs = _runs(sched)
        assert sum(1 for e, n in runs if n < sizes[e]) <= 1


@pytest.fixture(scope="module")
def rd():
    from paper_2410_19123_b200 import build, readme
    build.build()
    return readme


def test_native_scheduler_matches_oracle(rd):
    g = np.random.default_rng(11)
    for trial in range(200):
        E = int(g.integers(1, 17))
        sch = rd.ExpertScheduler(E)
        queues = [[] for _ in range(E)]
        tok = 0
        for rnd in range(6):
            n = int(g.integers(0, 40))
            ex = g.integers(0, E, size=n).astype(np.int32)
            ids = np.arange(tok, tok + n, dtype=np.int64)
            tok += n
            sch.push(ids, ex)
            for t, e in zip(ids.tolist(), ex.tolist()):
                queues[e].append(t)
            mx = int(g.integers(0, 48))
            ref, queues = alg1.schedule(queues, mx)
            t_ids, t_ex = sch.next_batch(mx)
            assert list(zip(t_ids.tolist(), t_ex.tolist())) == ref
            assert sch.queued() == sum(len(q) for q in queues)


def test_native_scheduler_rejects_bad_expert(rd):
    sch = rd.ExpertScheduler(4)
    with pytest.raises(rd.ReadmeError):
        sch.push([1, 2], [0, 9])
    assert sch.queued() == 0
