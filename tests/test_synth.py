"""The seeded input generators (synth/) are deterministic, shaped like the paper's workloads, and hold
no method arithmetic."""
import numpy as np

import synth


def test_deterministic_and_keyed():
    a = synth.tokens(16, 8, seed=5)
    b = synth.tokens(16, 8, seed=5)
    c = synth.tokens(16, 8, seed=6)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    # tensors are keyed independently: drawing logits first does not change x
    synth.router_logits(16, 8, seed=5)
    assert np.array_equal(synth.tokens(16, 8, seed=5), a)


def test_weight_scales():
    wg, wu, wd = synth.dense_ffn_weights(512, 256, 128, seed=1)
    assert wg.shape == (512, 256) and wd.shape == (256, 512)
    assert abs(wg.std() - 1 / 16) < 0.01 and abs(wd.std() - 1 / np.sqrt(128)) < 0.01


def test_neuron_sets():
    S = synth.neuron_sets(8, 64, 32)
    assert S.shape == (8, 32) and np.all(np.diff(S, axis=1) > 0) and S.max() < 64
    P = synth.neuron_sets(8, 64, 8, mode="partition")
    assert np.array_equal(np.sort(P.reshape(-1)), np.arange(64))


def test_assignment_recipes():
    ids = synth.assignments_markov(2, 4096, 8, 0.672)
    follow = np.mean(ids[1:4096] == ids[:4095])
    assert 0.66 < follow < 0.75  # p + (1-p)/E ~= 0.713
    z = synth.assignments_zipf(100000, 8, 1.0)
    top = np.bincount(z, minlength=8).max() / z.size
    assert abs(top - 0.368) < 0.01
    u = synth.assignments_unique(256, 3, 8)
    assert len(np.unique(u)) == 3
    lg = synth.logits_for_assignments(ids, 8, margin=0.5)
    srt = np.sort(lg, axis=1)
    assert np.array_equal(lg.argmax(axis=1), ids) and np.all(srt[:, -1] - srt[:, -2] >= 0.5)


def test_near_tie_logits_have_ties():
    lg = synth.near_tie_logits(256, 8)
    srt = np.sort(lg, axis=1)
    assert np.sum(srt[:, -1] == srt[:, -2]) > 10


def test_logits_for_assignments_finite_and_argmax():
    for E in (1, 2, 8):
        ids = synth.assignments_zipf(257, E, 2.0, seed=3)
        lg = synth.logits_for_assignments(ids, E, seed=3)
        assert np.isfinite(lg).all()
        assert np.array_equal(lg.argmax(axis=1), ids)
