"""Pins for the CPU oracle (-m "not gpu"): the oracle is checked against what the paper and the
mathematics fix, never against itself. Each test names the pin and the
passage it follows. A plausible mistake in the oracle (dropped term, wrong sign/index, transposed
operand, unstable order) fails at least one of these."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from tests.tolerances import rel_err

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---- P6: top-K rule and weights, SPEC worked examples ----------------------------------------------

@pytest.mark.parametrize("case", _gold("spec_examples.json")["topk_select"], ids=lambda c: c["cite"][:14])
def test_topk_spec_examples(case):
    lg = np.array([case["logits"]], np.float64)
    r = oracle.route(lg, case["K"])
    assert r["topk_idx"][0].tolist() == case["ids"]
    np.testing.assert_allclose(r["topk_w"][0], case["weights"], atol=case["tol"], rtol=0)
    if case["K"] == 1:
        assert r["topk_w"][0, 0] == 1.0  # bitwise 1 (Q1)


def _route_reference_numpy(lg, k):
    """Independent statement of the same rule through a library stable sort (descending logit,
    ties -> lower id) and a stable sort of slots by expert (FIFO within an expert queue)."""
    T, E = lg.shape
    order = np.argsort(-lg.astype(np.float64), axis=1, kind="stable")[:, :k]
    flat = order.reshape(-1)
    src = np.argsort(flat, kind="stable").astype(np.int32)
    dest = np.empty_like(src)
    dest[src] = np.arange(src.size, dtype=np.int32)
    counts = np.bincount(flat, minlength=E).astype(np.int32)
    return order.astype(np.int32), counts, dest, src


@pytest.mark.parametrize("T,E,k,kind", [(257, 8, 1, "normal"), (300, 8, 2, "normal"), (64, 1, 1, "normal"),
                                        (512, 8, 1, "ties"), (200, 5, 3, "ties"), (128, 256, 4, "normal"),
                                        (77, 8, 8, "normal")])
def test_route_matches_stable_sort(T, E, k, kind):
    lg = synth.router_logits(T, E) if kind == "normal" else synth.near_tie_logits(T, E)
    r = oracle.route(lg, k)
    idx, counts, dest, src = _route_reference_numpy(lg, k)
    assert np.array_equal(r["topk_idx"], idx)
    assert np.array_equal(r["counts"], counts)
    assert np.array_equal(r["dest"], dest)
    assert np.array_equal(r["src"], src)


def test_route_invariants_P3():
    T, E, k = 1000, 8, 2
    r = oracle.route(synth.router_logits(T, E), k)
    assert r["counts"].sum() == T * k
    assert r["offsets"][0] == 0 and r["offsets"][-1] == T * k
    assert np.array_equal(np.diff(r["offsets"]), r["counts"])
    assert np.array_equal(np.sort(r["dest"]), np.arange(T * k))  # bijection
    assert np.array_equal(r["src"][r["dest"]], np.arange(T * k))  # src = dest^-1
    for e in range(E):  # stability: FIFO inside each expert segment
        seg = r["src"][r["offsets"][e]:r["offsets"][e + 1]]
        assert np.all(np.diff(seg) > 0)
        assert np.all(r["topk_idx"].reshape(-1)[seg] == e)
    np.testing.assert_allclose(r["topk_w"].sum(axis=1), 1.0, atol=1e-12)
    assert np.all(np.diff(r["topk_w"], axis=1) <= 0)  # descending logit => descending weight


def test_route_k1_weight_exactly_one():
    r = oracle.route(synth.router_logits(500, 8), 1)
    assert np.all(r["topk_w"] == 1.0)


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_route_rejects_nonfinite(bad):
    lg = synth.router_logits(10, 8)
    lg[3, 2] = bad
    with pytest.raises(oracle.OracleError):
        oracle.route(lg, 1)


def test_route_T0():
    r = oracle.route(np.zeros((0, 8), np.float32), 1)
    assert r["counts"].tolist() == [0] * 8 and r["offsets"].tolist() == [0] * 9


# ---- P8: ReLU two-layer expert form, SPEC hand examples ----------------------------------------------

def _relu_expert_weights(W1, W2, mask):
    W1 = np.asarray(W1, np.float64)
    W2 = np.asarray(W2, np.float64)
    D, H = W1.shape
    return oracle.build_experts(W1, W1, W2, np.array([mask], np.int32))


@pytest.mark.parametrize("case", _gold("spec_examples.json")["relu_build_expert"], ids=lambda c: c["cite"][:10])
def test_relu_build_expert_spec(case):
    eg, eu, ed = _relu_expert_weights(case["W1"], case["W2"], case["mask"])
    x = np.array([case["x"]], np.float64)
    y = oracle.expert_ffn(x, np.array([0, 1], np.int32), eg, eu, ed, act="relu")
    assert y[0].tolist() == case["y"]


@pytest.mark.parametrize("case", _gold("spec_examples.json")["relu_dense_forward"], ids=lambda c: c["cite"][:10])
def test_relu_dense_forward_spec(case):
    W1 = np.asarray(case["W1"], np.float64)
    y = oracle.dense_ffn(np.array([case["x"]]), W1, W1, np.asarray(case["W2"], np.float64), act="relu")
    assert y[0].tolist() == case["y"]


def test_relu_pregated_combination_spec():
    case = _gold("spec_examples.json")["relu_pregated_combination"][0]
    W1 = np.asarray(case["W1"], np.float64)
    W2 = np.asarray(case["W2"], np.float64)
    eg, eu, ed = oracle.build_experts(W1, W1, W2, np.array(case["masks"], np.int32))
    y, plan = oracle.moe_layer(np.array([case["x"]]), np.array([case["logits"]]), case["K"], eg, eu, ed,
                               act="relu")
    np.testing.assert_allclose(y[0], case["y"], atol=case["tol"], rtol=0)
    yb = oracle.bruteforce(np.array([case["x"]]), np.array([case["logits"]]), case["K"], W1, W1, W2,
                           np.array(case["masks"], np.int32), act="relu")
    np.testing.assert_allclose(yb[0], case["y"], atol=case["tol"], rtol=0)


# ---- P7: SwiGLU closed forms ----------------------------------------------------------------------

def test_swiglu_closed_forms():
    g = _gold("swiglu_closed_forms.json")
    tol = g["tol_abs"]
    for c in g["cases"]:
        y = oracle.expert_ffn(np.array([c["x"]]), np.array([0, 1], np.int32),
                              np.array([c["w_gate"]], np.float64), np.array([c["w_up"]], np.float64),
                              np.array([c["w_down"]], np.float64))
        np.testing.assert_allclose(y[0], c["y"], atol=tol, rtol=0, err_msg=c["cite"])
    ex = g["experts_of_identity"]
    dn = ex["dense"]
    wg, wu, wd = (np.asarray(dn[k], np.float64) for k in ("w_gate", "w_up", "w_down"))
    eg, eu, ed = oracle.build_experts(wg, wu, wd, np.array([[0], [1]], np.int32))
    x = np.array([ex["x"]])
    for e in (0, 1):
        off = np.array([0, 1, 1] if e == 0 else [0, 0, 1], np.int32)
        y = oracle.expert_ffn(x, off, eg, eu, ed)
        np.testing.assert_allclose(y[0], ex["single"][str(e)], atol=tol, rtol=0)
    y, _ = oracle.moe_layer(x, np.array([ex["logits"]]), ex["K"], eg, eu, ed)
    np.testing.assert_allclose(y[0], ex["y"], atol=tol, rtol=0)


# ---- P1: full-FFN expert == dense FFN ---------------------------------------------------------------

@pytest.mark.parametrize("E", [1, 4])
def test_full_expert_equals_dense_P1(E):
    T, H, D = 40, 24, 48
    wg, wu, wd = synth.dense_ffn_weights(D, H, D, seed=11)
    S = synth.neuron_sets(E, D, D, mode="full")
    eg, eu, ed = oracle.build_experts(wg, wu, wd, S)
    x = synth.tokens(T, H, seed=12)
    lg = synth.router_logits(T, E, seed=13)
    y, _ = oracle.moe_layer(x, lg, 1, eg, eu, ed)
    yd = oracle.dense_ffn(x, wg, wu, wd)
    assert np.array_equal(y, yd)  # same accumulation order -> bitwise


# ---- P2: partition identity sum_e F_e(x) = F_0(x) ----------------------------------------------------

def test_partition_identity_P2():
    T, H, D, E = 16, 32, 64, 8
    d = D // E
    wg, wu, wd = synth.dense_ffn_weights(D, H, d, seed=21)
    S = synth.neuron_sets(E, D, d, mode="partition", seed=22)
    eg, eu, ed = oracle.build_experts(wg, wu, wd, S)
    x = synth.tokens(T, H, seed=23)
    acc = np.zeros((T, H))
    for e in range(E):  # force every token to expert e
        off = np.array([0] * (e + 1) + [T] * (E - e), np.int32)
        acc += oracle.expert_ffn(x, off, eg, eu, ed)
    yd = oracle.dense_ffn(x, wg, wu, wd)
    assert rel_err(acc, yd) < 1e-12


def test_build_experts_slices():
    D, H, E, d = 20, 12, 3, 7
    wg, wu, wd = synth.dense_ffn_weights(D, H, d, seed=31)
    S = synth.neuron_sets(E, D, d, seed=32)
    eg, eu, ed = oracle.build_experts(wg, wu, wd, S)
    for e in range(E):
        assert np.array_equal(eg[e], wg[S[e]].astype(np.float64))
        assert np.array_equal(eu[e], wu[S[e]].astype(np.float64))
        assert np.array_equal(ed[e], wd[:, S[e]].astype(np.float64))
    bad = S.copy()
    bad[0, 1] = bad[0, 0]  # not strictly increasing
    with pytest.raises(oracle.OracleError):
        oracle.build_experts(wg, wu, wd, bad)


# ---- P3/a5: dispatch is a bit copy through the permutation --------------------------------------------

def test_dispatch_bit_copy():
    T, H, E, k = 50, 16, 8, 2
    x = synth.to_torch(synth.tokens(T, H), "bf16")
    r = oracle.route(synth.router_logits(T, E), k)
    xs = oracle.dispatch(x, r["dest"], k)
    xf = x.double().numpy()
    for s in range(T * k):
        assert np.array_equal(xs[r["dest"][s]], xf[s // k])


# ---- P5: brute force on tiny inputs -----------------------------------------------------------------

@pytest.mark.parametrize("E,k", [(1, 1), (2, 1), (2, 2), (8, 1), (8, 2)])
def test_bruteforce_P5(E, k):
    T, H, D, d = 48, 16, 32, 16
    wg, wu, wd = synth.dense_ffn_weights(D, H, d, seed=41 + E)
    S = synth.neuron_sets(E, D, d, seed=42 + E)
    eg, eu, ed = oracle.build_experts(wg, wu, wd, S)
    x = synth.tokens(T, H, seed=43)
    lg = synth.near_tie_logits(T, E, seed=44) if E > 1 else synth.router_logits(T, E, seed=44)
    y, _ = oracle.moe_layer(x, lg, k, eg, eu, ed)
    yb = oracle.bruteforce(x, lg, k, wg, wu, wd, S)
    assert rel_err(y, yb) < 1e-12


# ---- P4: permutation equivariance -------------------------------------------------------------------

def test_permutation_equivariance_P4():
    T, H, E, d, k = 96, 16, 8, 24, 2
    eg, eu, ed = synth.expert_weights(E, d, H, seed=51)
    x = synth.tokens(T, H, seed=52)
    lg = synth.router_logits(T, E, seed=53)
    y, plan = oracle.moe_layer(x, lg, k, eg, eu, ed)
    perm = synth.rng(54, 0).permutation(T)
    yp, planp = oracle.moe_layer(x[perm], lg[perm], k, eg, eu, ed)
    assert np.array_equal(yp, y[perm])
    assert np.array_equal(planp["counts"], plan["counts"])
    assert np.array_equal(planp["offsets"], plan["offsets"])


# ---- P9: zero / edge cases ---------------------------------------------------------------------------

def test_zero_and_edges_P9():
    H, E, d = 8, 4, 6
    eg, eu, ed = synth.expert_weights(E, d, H, seed=61)
    y, _ = oracle.moe_layer(np.zeros((5, H)), synth.router_logits(5, E), 1, eg, eu, ed)
    assert np.all(y == 0.0)
    y, plan = oracle.moe_layer(np.zeros((0, H)), np.zeros((0, E)), 1, eg, eu, ed)
    assert y.shape == (0, H) and plan["offsets"].tolist() == [0] * (E + 1)
    # k = E selects every expert with softmax weights over all logits
    lg = synth.router_logits(3, E, seed=62).astype(np.float64)
    r = oracle.route(lg, E)
    sm = np.exp(lg - lg.max(axis=1, keepdims=True))
    sm /= sm.sum(axis=1, keepdims=True)
    for t in range(3):
        np.testing.assert_allclose(r["topk_w"][t], sm[t, r["topk_idx"][t]], rtol=1e-14)
        assert sorted(r["topk_idx"][t].tolist()) == list(range(E))


# ---- P10: power-of-two scaling of W_down is exact -----------------------------------------------------

def test_scaling_P10():
    T, H, E, d = 30, 16, 8, 12
    eg, eu, ed = synth.expert_weights(E, d, H, seed=71)
    x = synth.tokens(T, H, seed=72)
    lg = synth.router_logits(T, E, seed=73)
    y, _ = oracle.moe_layer(x, lg, 2, eg, eu, ed)
    y8, _ = oracle.moe_layer(x, lg, 2, eg, eu, ed.astype(np.float64) * 8.0)
    assert np.array_equal(y8, y * 8.0)


def test_residual_added():
    T, H, E, d = 10, 8, 4, 6
    eg, eu, ed = synth.expert_weights(E, d, H, seed=81)
    x = synth.tokens(T, H, seed=82)
    res = synth.residual(T, H, seed=83)
    lg = synth.router_logits(T, E, seed=84)
    y, _ = oracle.moe_layer(x, lg, 1, eg, eu, ed)
    yr, _ = oracle.moe_layer(x, lg, 1, eg, eu, ed, residual=res)
    np.testing.assert_allclose(yr - res.astype(np.float64), y, atol=1e-14, rtol=0)


# ---- P11: route once, reuse across layers ------------------------------------------------------------

def test_route_once_P11():
    T, H, E, d, L, k = 40, 16, 8, 12, 3, 1
    lg = synth.router_logits(T, E, seed=91)
    x0 = synth.tokens(T, H, seed=92)
    layers = [synth.expert_weights(E, d, H, seed=93, layer=l) for l in range(L)]
    # (a) re-route every layer from the same pre-gating logits
    xa = x0.astype(np.float64)
    plans = []
    for (eg, eu, ed) in layers:
        y, plan = oracle.moe_layer(xa, lg, k, eg, eu, ed)
        plans.append(plan)
        xa = xa + y
    # (b) route once, reuse the plan (dispatch / FFN / combine per layer)
    plan = oracle.route(lg, k)
    xb = x0.astype(np.float64)
    for (eg, eu, ed) in layers:
        xs = oracle.dispatch(xb, plan["dest"], k)
        ys = oracle.expert_ffn(xs, plan["offsets"], eg, eu, ed)
        xb = xb + oracle.combine(ys, plan["dest"], plan["topk_w"], k)
    for p in plans:
        for key in ("topk_idx", "counts", "offsets", "dest", "src"):
            assert np.array_equal(p[key], plan[key])
    assert np.array_equal(xa, xb)


# ---- P12: expert-parallel simulation == single layer ---------------------------------------------------

@pytest.mark.parametrize("G,k", [(1, 1), (2, 1), (4, 2), (8, 1)])
def test_ep_sim_equals_layer_P12(G, k):
    T, H, E, d = 64, 16, 8, 12
    eg, eu, ed = synth.expert_weights(E, d, H, seed=101)
    x = synth.to_torch(synth.tokens(T, H, seed=102), "bf16")
    lg = synth.router_logits(T, E, seed=103)
    y, _ = oracle.moe_layer(x, lg, k, eg, eu, ed)
    ye = oracle.ep_sim(G, x, lg, k, eg, eu, ed)
    assert np.array_equal(y, ye)


def test_thread_count_invariance():
    T, H, E, d = 33, 16, 8, 20
    eg, eu, ed = synth.expert_weights(E, d, H, seed=111)
    x = synth.tokens(T, H, seed=112)
    lg = synth.router_logits(T, E, seed=113)
    y1, _ = oracle.moe_layer(x, lg, 2, eg, eu, ed, nthreads=1)
    y8, _ = oracle.moe_layer(x, lg, 2, eg, eu, ed, nthreads=8)
    assert np.array_equal(y1, y8)


# ---- a6 / a7 separately: composition equals the whole expert FFN; P7(i) hidden value -----------------

def test_hidden_then_down_equals_expert_ffn():
    rows, H, E, d = 70, 24, 4, 40
    eg, eu, ed = synth.expert_weights(E, d, H, seed=121)
    x = synth.tokens(rows, H, seed=122)
    off = np.array([0, 10, 10, 45, 70], np.int32)
    h = oracle.expert_hidden(x, off, eg, eu)
    assert np.array_equal(oracle.expert_down(h, off, ed), oracle.expert_ffn(x, off, eg, eu, ed))


def test_hidden_closed_form():
    c = _gold("swiglu_closed_forms.json")["cases"][0]  # h = silu(2) * 3 (W_down = [[1],[0]] copies it to y0)
    h = oracle.expert_hidden(np.array([c["x"]]), np.array([0, 1], np.int32), np.array([c["w_gate"]], np.float64),
                             np.array([c["w_up"]], np.float64))
    np.testing.assert_allclose(h[0, 0], c["y"][0], atol=1e-6, rtol=0)


# ---- RMSNorm and the route-once stack (config 4, reading Q10) ---------------------------------------

def test_rmsnorm_closed_form():
    # x = (3, 4): mean square 12.5, rms = 3.5355339 -> (0.8485281, 1.1313708); eps = 0
    y = oracle.rmsnorm(np.array([[3.0, 4.0]]), eps=0.0)
    np.testing.assert_allclose(y[0], [0.8485281374238571, 1.131370849898476], rtol=1e-15)
    x = synth.tokens(5, 16, seed=131).astype(np.float64)
    np.testing.assert_allclose(oracle.rmsnorm(7.0 * x, eps=0.0), oracle.rmsnorm(x, eps=0.0), rtol=1e-14)
    np.testing.assert_allclose(np.mean(oracle.rmsnorm(x, eps=0.0) ** 2, axis=1), 1.0, rtol=1e-14)


def test_stack_zero_down_is_identity_and_routes_once():
    T, H, E, d, L = 20, 16, 4, 8, 3
    x = synth.tokens(T, H, seed=141)
    lg = synth.router_logits(T, E, seed=142)
    layers = []
    for l in range(L):
        eg, eu, ed = synth.expert_weights(E, d, H, seed=143, layer=l)
        layers.append((eg, eu, np.zeros_like(ed)))
    y, plan = oracle.moe_stack(x, lg, 1, layers)
    assert np.array_equal(y, x.astype(np.float64))  # W_down = 0 -> every layer adds exactly 0
    ref = oracle.route(lg, 1)
    assert np.array_equal(plan["dest"], ref["dest"])


# ---- NEXT-3: permanent expert ----------------------------------------------------------

def test_permanent_expert_folds_into_every_expert_Q6():
    """k=1: an expert whose neuron set is S_e plus the permanent set P (disjoint) equals expert S_e plus the
    always-on expert P — outputs sum over neurons (linearity of W_2 M^T in PAPER.md:159)."""
    T, H, D, E, d, p = 24, 16, 64, 4, 10, 6
    wg, wu, wd = synth.dense_ffn_weights(D, H, d, seed=151)
    g = synth.rng(152, 0)
    perm = g.permutation(D)
    P = np.sort(perm[:p]).astype(np.int32)
    rest = perm[p:]
    S = np.stack([np.sort(g.choice(rest, size=d, replace=False)) for _ in range(E)]).astype(np.int32)
    SP = np.sort(np.concatenate([S, np.tile(P, (E, 1))], axis=1), axis=1).astype(np.int32)
    x = synth.tokens(T, H, seed=153)
    lg = synth.router_logits(T, E, seed=154)
    folded, _ = oracle.moe_layer(x, lg, 1, *oracle.build_experts(wg, wu, wd, SP))
    base, _ = oracle.moe_layer(x, lg, 1, *oracle.build_experts(wg, wu, wd, S))
    pg, pu, pd = oracle.build_experts(wg, wu, wd, P[None, :])
    perm_y = oracle.expert_ffn(x, np.array([0, T], np.int32), pg, pu, pd)
    assert rel_err(base + perm_y, folded) < 1e-12


# ---- NEXT-1: the pre-gating router G (oracle.router) ----------------------------------------------------

def _small_router(vocab=300, N=8, seed=161):
    import torch
    W = synth.router_weights(vocab=vocab, n_experts=N, seed=seed)
    return {k: torch.from_numpy(v).to(torch.bfloat16) for k, v in W.items()}


def test_router_param_count_matches_paper():
    """table:router_details: 18.0 M parameters at vocab 32000, dim 512, MLP 512."""
    from oracle import router
    W = synth.router_weights(vocab=32000, n_experts=8)
    n = router.param_count(W)
    assert abs(n - 18.0e6) / 18.0e6 < 0.02, n


def test_router_masked_equals_incremental():
    """The masked full-sequence evaluation equals a token-by-token evaluation with a growing KV cache
    (no mask): pins the causal mask, RoPE positions (restart per sequence) and the block wiring."""
    from oracle import router
    W = _small_router()
    ids = synth.token_ids(23, vocab=300, seed=162)
    starts = np.array([0, 9, 9, 23])  # includes an empty sequence
    a = router.forward(ids, starts, W)
    b = router.forward_incremental(ids, starts, W)
    assert np.max(np.abs(a - b)) < 1e-10


def test_router_causal_prefix_invariance():
    """Appending tokens never changes earlier decisions (causality)."""
    from oracle import router
    W = _small_router()
    ids = synth.token_ids(40, vocab=300, seed=163)
    full = router.forward(ids, np.array([0, 40]), W)
    pre = router.forward(ids[:17], np.array([0, 17]), W)
    assert np.max(np.abs(full[:17] - pre)) < 1e-10


def test_rope_invariants():
    """RoPE: identity at position 0, norm-preserving, and <R(p)q, R(p')k> depends only on p - p'."""
    from oracle import router
    g = np.random.default_rng(5)
    q, k = g.standard_normal((1, 128)), g.standard_normal((1, 128))
    assert np.array_equal(router.rope(q, np.array([0])), q)
    r = router.rope(q, np.array([37]))
    assert abs(np.linalg.norm(r) - np.linalg.norm(q)) < 1e-12
    d1 = router.rope(q, np.array([10])) @ router.rope(k, np.array([3])).T
    d2 = router.rope(q, np.array([107])) @ router.rope(k, np.array([100])).T
    assert abs(d1 - d2).max() < 1e-10


def test_router_zero_head_gives_zero_logits():
    from oracle import router
    import torch
    W = _small_router()
    W["w_head"] = torch.zeros_like(W["w_head"])
    out = router.forward(synth.token_ids(12, vocab=300, seed=164), np.array([0, 12]), W)
    assert np.all(out == 0.0)


# ---- closed forms for the router block (Q15) and the pre-norm stack (Q10) ---------------------------------
# tests/golden/router_and_stack_closed_forms.json holds the hand derivations; the recipes below build the
# weights those derivations describe (eps = 0 so every RMSNorm of a one-hot row is sqrt(512) times it).

def _zero_router(vocab, n_heads_out):
    D = 512
    z = lambda *s: np.zeros(s, np.float64)
    return {"emb": np.eye(vocab, D), "norm1": np.ones(D), "w_qkv": z(3 * D, D), "w_o": z(D, D),
            "norm2": np.ones(D), "w_gate": z(D, D), "w_up": z(D, D), "w_down": z(D, D), "norm_f": np.ones(D),
            "w_head": z(n_heads_out, D)}


def _attention_case():
    r = math.sqrt(512.0)
    W = _zero_router(2, 3)
    a = math.sqrt(math.sqrt(128.0) * math.log(3.0)) / r
    W["w_qkv"][0, 1] = a            # W_q, head 0 dim 0 <- model dim 1 (token 1 only)
    W["w_qkv"][512 + 0, 1] = a      # W_k, head 0 dim 0 <- model dim 1 (k_0 = 0)
    W["w_qkv"][1024 + 0, 1] = 1.0 / r  # W_v, head 0 dim 0: v_1 = 1, v_0 = 0
    W["w_o"][2, 0] = 1.0            # attention head-0 dim 0 -> model dim 2
    W["w_head"][0, 2] = W["w_head"][1, 1] = W["w_head"][2, 0] = 1.0
    return W


def _mlp_case():
    r = math.sqrt(512.0)
    W = _zero_router(1, 2)
    W["w_gate"][0, 0] = 2.0 / r
    W["w_up"][0, 0] = 3.0 / r
    W["w_down"][3, 0] = 1.0
    W["norm_f"][:] = 2.0
    W["w_head"][0, 3] = W["w_head"][1, 0] = 1.0
    return W


@pytest.mark.parametrize("evaluate", ["forward", "forward_incremental"])
def test_router_attention_closed_form(evaluate):
    """Q15 attention pinned by hand: the 1/sqrt(128) score scale (weights (1/4, 3/4) from scores (0, ln 3)),
    the causal mask (token 0 sees only itself), RoPE's position invariance of q.k at equal positions, the
    residual around attention and the final RMSNorm + head. Dropping the scale gives r(0.7071, 0.7071, 0)."""
    from oracle import router
    g = _gold("router_and_stack_closed_forms.json")["attention"]
    out = getattr(router, evaluate)(np.array(g["ids"]), np.array([0, 2]), _attention_case(), eps=0.0)
    np.testing.assert_allclose(out, np.array(g["logits"]), atol=g["tol_abs"], rtol=0)


@pytest.mark.parametrize("evaluate", ["forward", "forward_incremental"])
def test_router_mlp_head_closed_form(evaluate):
    """Q15 MLP and gating head pinned by hand: silu(W_g m) * (W_u m) (P7(i)'s silu(2)*3), W_down, the residual
    around the MLP, the final RMSNorm with its weight g_f = 2, and W_head's rows. ReLU for silu, gate and up
    exchanged, or g_f dropped each move the logits by far more than the tolerance."""
    from oracle import router
    g = _gold("router_and_stack_closed_forms.json")["mlp_head"]
    out = getattr(router, evaluate)(np.array(g["ids"]), np.array([0, 1]), _mlp_case(), eps=0.0)
    np.testing.assert_allclose(out, np.array(g["logits"]), atol=g["tol_abs"], rtol=0)


def test_moe_stack_prenorm_closed_form():
    """Q10 pinned by hand: one pre-norm layer on P7(ii)'s identity expert maps x = (3, 5) to
    x + F(x / sqrt(17)) = (3.356972, 6.133489); without the RMSNorm it would be (11.573167, 29.832679),
    without the residual (0.356972, 1.133489)."""
    g = _gold("router_and_stack_closed_forms.json")["prenorm_stack"]
    I = np.eye(2)
    wg, wu, wd = oracle.build_experts(I, I, I, np.array([[0, 1]], np.int32))
    y, plan = oracle.moe_stack(np.array([g["x"]]), np.zeros((1, 1), np.float32), 1, [(wg, wu, wd)], eps=0.0)
    np.testing.assert_allclose(y[0], g["y"], atol=g["tol_abs"], rtol=0)
    assert plan["counts"].tolist() == [1]
