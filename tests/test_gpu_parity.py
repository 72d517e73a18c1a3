"""GPU parity (-m gpu): the CUDA path, called through the C ABI, against the CPU oracle on the same
seeded inputs. Rules (BASELINE.json north_star):
  routing integers (topk_idx, counts, offsets, dest, src): bit-exact;
  dispatch and k=1 combine: bit copies;
  FP outputs: per-token inf-norm relative error <= 2e-2 (bf16) / <= 1e-4 (fp32); topk_w fp32 rule,
  and exactly 1.0f for k=1.
Sizes span several tiles and ragged tails; full-size config 2 is checked on sampled tokens."""
import time

import numpy as np
import pytest
import torch

import oracle
import synth
from tests.tolerances import BF16_TOL, F32_TOL, rel_err

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def rd():
    from paper_2410_19123_b200 import build, readme
    build.build()
    readme.lib()
    return readme


@pytest.fixture
def knob(rd):
    """knob(name, value): set a library lab switch (readme_debug_set_knob) for this test only."""
    touched = []

    def set_(name, value):
        touched.append(name)
        rd.set_knob(name, int(value))

    yield set_
    for n in touched:
        rd.reset_knob(n)


ROUTE_IMPL = {"cluster": 1, "lookback": 2}


def _np(t):
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        t = t.float()
    return t.numpy()


def _check_plan(plan, ref, k):
    torch.cuda.synchronize()
    assert np.array_equal(_np(plan.topk_idx), ref["topk_idx"])
    assert np.array_equal(_np(plan.counts), ref["counts"])
    assert np.array_equal(_np(plan.offsets), ref["offsets"])
    assert np.array_equal(_np(plan.dest), ref["dest"])
    assert np.array_equal(_np(plan.src), ref["src"])
    w = _np(plan.topk_w).astype(np.float64)
    if k == 1:
        assert np.all(w == 1.0)
    else:
        assert np.max(np.abs(w - ref["topk_w"])) <= F32_TOL


# ---- a1-a4 route -----------------------------------------------------------------------------------

ROUTE_CASES = [
    (8192, 8, 1, "normal", "f32"),
    (8192, 8, 1, "ties", "f32"),
    (1000, 8, 2, "normal", "f32"),   # T not a multiple of the tile
    (1, 8, 1, "normal", "f32"),
    (4097, 1, 1, "normal", "f32"),   # E = 1
    (3000, 256, 4, "normal", "f32"),  # max experts
    (777, 5, 5, "ties", "f32"),      # k = E
    (5000, 8, 1, "normal", "bf16"),
    (65536, 8, 1, "normal", "f32"),
    (2000, 33, 3, "ties", "bf16"),
]


@pytest.mark.parametrize("impl", ["cluster", "lookback"])
@pytest.mark.parametrize("T,E,k,kind,ldt", ROUTE_CASES)
def test_route_bit_exact(rd, knob, impl, T, E, k, kind, ldt):
    # both route implementations: the single-launch cluster route (default up to 256K slots) and the
    # multi-CTA decoupled-lookback route (larger batches)
    knob("route", ROUTE_IMPL[impl])
    lg = synth.router_logits(T, E, seed=T + E) if kind == "normal" else synth.near_tie_logits(T, E, seed=T + E)
    lg_t = synth.to_torch(lg, ldt)
    ref = oracle.route(lg_t, k)  # the oracle sees exactly the bits the GPU sees
    plan = rd.route(lg_t.to(DEV), k)
    _check_plan(plan, ref, k)
    assert int(plan.dev_status.item()) == 0


@pytest.mark.parametrize("impl", [None, "cluster"])
def test_route_large_batch(rd, knob, impl):
    # 300K slots: past the cluster route's default range (lookback), and forced through the cluster route
    # (each of the 16 CTAs walks ~19 sub-tiles, carrying its running per-expert counts)
    if impl:
        knob("route", ROUTE_IMPL[impl])
    lg = synth.router_logits(150001, 8, seed=5)
    ref = oracle.route(lg, 2)
    plan = rd.route(torch.from_numpy(lg).to(DEV), 2)
    _check_plan(plan, ref, 2)


def test_route_locality_runs(rd):
    ids = synth.assignments_markov(4, 4096, 8, 0.672)
    lg = synth.logits_for_assignments(ids, 8)
    plan = rd.route(torch.from_numpy(lg).to(DEV), 1)
    _check_plan(plan, oracle.route(lg, 1), 1)
    assert np.array_equal(_np(plan.topk_idx)[:, 0], ids)


def test_route_single_expert_all_tokens(rd):
    lg = np.zeros((3000, 8), np.float32)
    lg[:, 5] = 1.0
    plan = rd.route(torch.from_numpy(lg).to(DEV), 1)
    _check_plan(plan, oracle.route(lg, 1), 1)


def test_route_T0(rd):
    plan = rd.new_plan(0, 8, 1, DEV)
    plan.counts.fill_(7)
    plan.offsets.fill_(7)
    rd.route(torch.zeros((0, 8), device=DEV), 1, plan=plan)
    torch.cuda.synchronize()
    assert plan.counts.tolist() == [0] * 8 and plan.offsets.tolist() == [0] * 9


@pytest.mark.parametrize("E,impl", [(8, "cluster"), (8, "lookback"), (40, "cluster"), (40, "lookback")])
def test_route_nonfinite_flag(rd, knob, E, impl):
    """Q3: non-finite logits are flagged; ids stay in range and the k > 1 weights stay finite and sum to 1 even
    for a +inf maximum (uniform over the tied +inf entries) or an all -inf row (uniform over the selection)."""
    knob("route", ROUTE_IMPL[impl])
    lg = synth.router_logits(600, E)
    lg[17, 3] = np.nan
    lg[400, 0] = np.inf
    lg[401, 1] = lg[401, 5] = np.inf
    lg[402, :] = -np.inf
    plan = rd.route(torch.from_numpy(lg).to(DEV), 2)
    torch.cuda.synchronize()
    assert int(plan.dev_status.item()) & rd.README_DEV_NONFINITE_LOGIT
    w = _np(plan.topk_w)
    idx = _np(plan.topk_idx)
    assert np.all(np.isfinite(w)) and np.allclose(w.sum(axis=1), 1.0, atol=1e-6)
    assert idx.min() >= 0 and idx.max() < E
    assert idx[400, 0] == 0 and w[400].tolist() == [1.0, 0.0]
    assert idx[401].tolist() == [1, 5] and w[401].tolist() == [0.5, 0.5]
    assert w[402].tolist() == [0.5, 0.5]
    # permutation still valid
    assert np.array_equal(np.sort(_np(plan.dest)), np.arange(1200))


def test_route_deterministic(rd):
    lg = torch.from_numpy(synth.router_logits(20000, 8)).to(DEV)
    a = rd.route(lg, 2)
    b = rd.route(lg, 2)
    torch.cuda.synchronize()
    assert torch.equal(a.dest, b.dest) and torch.equal(a.topk_w, b.topk_w)


# ---- a5 dispatch / a8 combine -----------------------------------------------------------------------

# >= 4096 slots take the bulk-copy kernel (rows of <= 12 KiB), the rest the warp-per-row kernel
@pytest.mark.parametrize("T,H,k,dt", [(1000, 4096, 1, "bf16"), (333, 264, 2, "bf16"), (256, 64, 1, "f32"),
                                      (100, 72, 3, "f32"), (5000, 4096, 1, "bf16"), (2100, 264, 2, "bf16"),
                                      (4500, 72, 1, "f32"), (1500, 1032, 3, "f32"), (4100, 4096, 1, "f32")])
def test_dispatch_bit_exact(rd, T, H, k, dt):
    x = synth.to_torch(synth.tokens(T, H, seed=T), dt)
    ref_plan = oracle.route(synth.router_logits(T, 8, seed=T + 1), k)
    dest = torch.from_numpy(ref_plan["dest"]).to(DEV)
    xs = rd.dispatch(x.to(DEV), dest, k)
    ref = oracle.dispatch(x, ref_plan["dest"], k)
    assert np.array_equal(_np(xs).astype(np.float64), ref)


@pytest.mark.parametrize("bulk", ["0", "1"])
def test_dispatch_bad_index_flagged(rd, knob, bulk):
    """An out-of-range dest entry is flagged in dev_status and skipped; every other row still lands."""
    knob("dispatch_bulk", bulk)
    T, H = 6000, 256
    x = synth.to_torch(synth.tokens(T, H, seed=5), "bf16").to(DEV)
    dest = torch.from_numpy(np.random.default_rng(6).permutation(T).astype(np.int32)).to(DEV)
    bad = 1234
    lost = int(dest[bad].item())
    dest[bad] = T + 7
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    out = torch.zeros((T, H), dtype=torch.bfloat16, device=DEV)
    rd.dispatch(x, dest, 1, out=out, dev_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & rd.README_DEV_BAD_INDEX
    keep = torch.ones(T, dtype=torch.bool, device=DEV)
    keep[bad] = False
    assert torch.equal(out[dest[keep].long()], x[keep])
    assert torch.count_nonzero(out[lost]) == 0


@pytest.mark.parametrize("bulk", ["0", "1"])
def test_combine_k1_bad_index_flagged(rd, knob, bulk):
    """k = 1 gather combine: an out-of-range dest entry is flagged and its output row left untouched."""
    knob("combine_bulk", bulk)
    T, H = 6000, 256
    ys = synth.to_torch(synth.tokens(T, H, seed=7), "bf16").to(DEV)
    dest = torch.from_numpy(np.random.default_rng(8).permutation(T).astype(np.int32)).to(DEV)
    dest[77] = -3
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    y = torch.zeros((T, H), dtype=torch.bfloat16, device=DEV)
    rd.combine(ys, dest, None, 1, out=y, dev_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & rd.README_DEV_BAD_INDEX
    keep = torch.ones(T, dtype=torch.bool, device=DEV)
    keep[77] = False
    assert torch.equal(y[keep], ys[dest[keep].long()])
    assert torch.count_nonzero(y[77]) == 0


@pytest.mark.parametrize("T,H,dt", [(2000, 4096, "bf16"), (5000, 4096, "bf16"), (4200, 264, "bf16"),
                                    (4500, 1032, "f32"), (4100, 4096, "f32")])
def test_combine_k1_is_bit_gather(rd, T, H, dt):
    """>= 4096 rows take the bulk-copy kernel (rows of <= 12 KiB), the rest the warp-per-row kernel."""
    ys = synth.to_torch(synth.tokens(T, H, seed=3), dt).to(DEV)
    plan = oracle.route(synth.router_logits(T, 8, seed=4), 1)
    y = rd.combine(ys, torch.from_numpy(plan["dest"]).to(DEV), None, 1)
    ys_np = _np(ys)
    assert np.array_equal(_np(y), ys_np[plan["dest"]])


@pytest.mark.parametrize("dt,k", [("bf16", 2), ("f32", 2), ("bf16", 1), ("f32", 4)])
def test_combine_weighted_residual(rd, dt, k):
    T, H, E = 700, 256, 8
    ys = synth.to_torch(synth.tokens(T * k, H, seed=5), dt)
    res = synth.to_torch(synth.residual(T, H, seed=6), dt)
    plan = oracle.route(synth.router_logits(T, E, seed=7), k)
    gplan = rd.route(torch.from_numpy(synth.router_logits(T, E, seed=7)).to(DEV), k)
    y = rd.combine(ys.to(DEV), gplan.dest, gplan.topk_w, k, residual=res.to(DEV))
    # teacher-forced: the oracle combines the same y_sorted with its own (bit-identical) plan
    ref = oracle.combine(ys.double().numpy(), plan["dest"], plan["topk_w"], k, residual=res)
    assert rel_err(_np(y), ref) <= (BF16_TOL if dt == "bf16" else F32_TOL)


# ---- a6-a7 expert FFN --------------------------------------------------------------------------------

def _ffn_case(T, H, d, E, k, dt, seed, skew=None):
    x = synth.to_torch(synth.tokens(T, H, seed=seed), dt)
    if skew == "empty":
        ids = synth.assignments_unique(T, max(1, E // 2), E, seed=seed)
        lg = synth.logits_for_assignments(ids, E, seed=seed)
    elif skew == "zipf":
        lg = synth.logits_for_assignments(synth.assignments_zipf(T, E, 2.0, seed=seed), E, seed=seed)
    else:
        lg = synth.router_logits(T, E, seed=seed)
    wg, wu, wd = (synth.to_torch(w, dt) for w in synth.expert_weights(E, d, H, seed=seed))
    return x, lg, wg, wu, wd


FFN_KERNEL = {"merged": 0, "split": 1, "unfused": 2}


def _set_kernel(knob, kernel):
    """merged (single launch, 256-row m-tiles above 1024 rows, segment tails riding on full m-tiles) /
    merged-mt128 / merged-mt256 / merged-swap (tails of <= 64 rows as their own swap-AB tiles) /
    merged-noswap (tails as M = 128 tiles) / split (two launches)."""
    if kernel == "merged-mt128":
        knob("ffn_mt", 128)
    elif kernel == "merged-mt256":
        knob("ffn_mt", 256)
    elif kernel == "merged-swap":
        knob("ffn_merge", 0)
        knob("ffn_swap", 64)
    elif kernel == "merged-noswap":
        knob("ffn_merge", 0)
        knob("ffn_swap", 0)
    knob("ffn_kernel", FFN_KERNEL["split" if kernel == "split" else "merged"])


KERNELS = ["merged", "merged-mt128", "merged-mt256", "merged-swap", "merged-noswap", "split"]


@pytest.mark.parametrize("T,H,d,E,k,skew", [
    (1000, 256, 384, 8, 1, None),      # several M/N tiles, ragged segments
    (700, 512, 264, 8, 2, "empty"),    # empty experts, N tails (264 = 2*128 + 8), k = 2
    (300, 128, 136, 3, 1, "zipf"),     # H < BN, K = 2 x 64
    (2048, 4096, 512, 8, 1, None),     # Llama-2 H, K = 64 x 64
    (129, 72, 40, 2, 1, None),         # K tail (72 = 64 + 8), d tiny
    (4000, 512, 256, 8, 1, "zipf"),    # many 256-row tiles, 128-row and 256-row tails
    (1024, 256, 128, 4, 1, None),      # counts ~256 -> exact and near-exact tiles
])
@pytest.mark.parametrize("kernel", KERNELS)
def test_expert_ffn_bf16_teacher_forced(rd, knob, kernel, T, H, d, E, k, skew):
    _set_kernel(knob, kernel)
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, k, "bf16", seed=T + H, skew=skew)
    plan = rd.route(torch.from_numpy(lg).to(DEV), k)
    xs = rd.dispatch(x.to(DEV), plan.dest, k)
    ys = rd.expert_ffn(xs, plan.offsets, wg.to(DEV), wu.to(DEV), wd.to(DEV))
    torch.cuda.synchronize()
    ref = oracle.expert_ffn(xs.cpu(), plan.offsets.cpu().numpy(), wg, wu, wd)
    assert rel_err(_np(ys), ref) <= BF16_TOL


def test_expert_ffn_f32_config1(rd):
    c = synth.CONFIGS[1]
    T, H, d, E, k = c["T"], c["H"], c["d"], c["E"], c["k"]
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, k, "f32", seed=synth.MASTER_SEED + 1)
    plan = rd.route(torch.from_numpy(lg).to(DEV), k)
    xs = rd.dispatch(x.to(DEV), plan.dest, k)
    ys = rd.expert_ffn(xs, plan.offsets, wg.to(DEV), wu.to(DEV), wd.to(DEV))
    ref = oracle.expert_ffn(xs.cpu(), plan.offsets.cpu().numpy(), wg, wu, wd)
    assert rel_err(_np(ys), ref) <= F32_TOL


@pytest.mark.parametrize("T,H,d,E", [(256, 64, 128, 8), (777, 128, 96, 5), (40, 32, 8, 3)])
def test_f32_one_launch_ffn_bitwise(rd, T, H, d, E):
    """Small fp32 layers (H, d <= 128) run a6 + a7 in one launch (h in shared memory) and, inside
    readme_moe_layer with logits, gather their rows straight from x through src: bitwise equal to the two
    separate launches (readme_expert_gate_up + readme_expert_down, the same fmaf order), to plan-in mode, and
    within the fp32 rule of the oracle."""
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, "f32", seed=T + H + d)
    res = synth.to_torch(synth.residual(T, H, seed=T + 5), "f32").to(DEV)
    x, wg, wu, wd = x.to(DEV), wg.to(DEV), wu.to(DEV), wd.to(DEV)
    lgt = torch.from_numpy(lg).to(DEV)
    plan = rd.route(lgt, 1)
    xs = rd.dispatch(x, plan.dest, 1)
    ys = rd.expert_ffn(xs, plan.offsets, wg, wu, wd)
    h = rd.expert_gate_up(xs, plan.offsets, wg, wu)
    assert torch.equal(ys, rd.expert_down(h, plan.offsets, wd))
    y, p2 = rd.moe_layer(x, wg, wu, wd, k=1, logits=lgt, residual=res)
    assert torch.equal(p2.src, plan.src) and torch.equal(p2.offsets, plan.offsets)
    assert torch.equal(y, rd.expert_down(h, plan.offsets, wd, src=plan.src, residual=res))
    y_in, _ = rd.moe_layer(x, wg, wu, wd, k=1, plan=plan, residual=res)
    assert torch.equal(y, y_in)
    ref = oracle.combine(oracle.expert_ffn(xs.cpu(), plan.offsets.cpu().numpy(), wg.cpu(), wu.cpu(), wd.cpu()),
                         plan.dest.cpu().numpy(), np.ones((T, 1)), 1, residual=res.cpu())
    assert rel_err(_np(y), ref) <= F32_TOL


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_gate_up_and_down_separately(rd, dt):
    """a6 and a7 each teacher-forced against the oracle; a7 with src scatters rows (fused combine)."""
    T, H, d, E = 1500, 512, 264, 8
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, dt, seed=91)
    res = synth.to_torch(synth.residual(T, H, seed=92), dt)
    plan = rd.route(torch.from_numpy(lg).to(DEV), 1)
    xs = rd.dispatch(x.to(DEV), plan.dest, 1)
    off = plan.offsets.cpu().numpy()
    h = rd.expert_gate_up(xs, plan.offsets, wg.to(DEV), wu.to(DEV))
    tol = BF16_TOL if dt == "bf16" else F32_TOL
    assert rel_err(_np(h), oracle.expert_hidden(xs.cpu(), off, wg, wu)) <= tol
    ys = rd.expert_down(h, plan.offsets, wd.to(DEV))
    assert rel_err(_np(ys), oracle.expert_down(h.cpu(), off, wd)) <= tol
    y = rd.expert_down(h, plan.offsets, wd.to(DEV), src=plan.src, residual=res.to(DEV))
    ref = oracle.combine(oracle.expert_down(h.cpu(), off, wd), plan.dest.cpu().numpy(), np.ones((T, 1)), 1,
                         residual=res)
    assert rel_err(_np(y), ref) <= tol


@pytest.mark.parametrize("kernel", KERNELS)
def test_expert_ffn_tile_edges(rd, knob, kernel):
    """Segment sizes on every tile boundary: empty, 1 row, 64/128/256 +- 1 (M=128 vs M=256 tails)."""
    _set_kernel(knob, kernel)
    counts = [0, 1, 63, 64, 65, 127, 128, 129, 255, 256, 257, 383, 384, 385, 511, 512]
    E, H, d = len(counts), 128, 136
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    rows = int(off[-1])
    xs = synth.to_torch(synth.tokens(rows, H, seed=13), "bf16")
    wg, wu, wd = (synth.to_torch(w, "bf16") for w in synth.expert_weights(E, d, H, seed=14))
    ys = rd.expert_ffn(xs.to(DEV), torch.from_numpy(off).to(DEV), wg.to(DEV), wu.to(DEV), wd.to(DEV))
    ref = oracle.expert_ffn(xs, off, wg, wu, wd)
    assert rel_err(_np(ys), ref) <= BF16_TOL


# variants of the single-launch FFN that compute every output element from the same K-ordered MMAs:
# (m-tile rows, second CTA skips A loads of <= 64-row tiles, max CTA pairs, gate/up N-tile-fastest order,
# segment tails of <= n rows as swap-AB tiles, 256-row m-tiles carry merged tails, tile order: -1 auto /
# 0 static / 1 dynamic)
FFN_VARIANTS = [(256, 1, 0, 0, 0, 1, -1), (128, 1, 0, 0, 0, 1, -1), (128, 0, 0, 0, 0, 1, 1), (256, 0, 0, 0, 0, 0, 0),
                (256, 1, 3, 0, 0, 1, -1), (128, 1, 1, 0, 0, 1, 1), (256, 1, 0, 1, 0, 1, 0), (128, 1, 0, 1, 0, 1, -1),
                (256, 1, 0, 0, 64, 0, 1), (128, 1, 0, 0, 64, 1, -1), (256, 1, 0, 0, 32, 0, -1),
                (256, 1, 3, 0, 64, 0, 0), (128, 1, 1, 0, 48, 1, -1), (256, 0, 0, 1, 16, 0, 1), (256, 1, 1, 0, 64, 1, -1),
                (256, 1, 0, 1, 64, 1, 1), (256, 1, 2, 0, 64, 1, 0)]


@pytest.mark.parametrize("T,d,skew", [(256, 5504, "zipf"), (2000, 264, None), (40, 136, "empty")])
def test_ffn_variants_bitwise_equal(rd, knob, T, d, skew):
    """128-row vs 256-row m-tiles, with and without the A-load skip, on 3 and 1 CTA pairs (every pair walks
    a long tile list; the down tiles wait on gate/up tiles of the same few pairs), in N-tile-fastest order,
    and with segment tails as swap-AB tiles (operands exchanged: weights on the MMA's M side): bitwise equal
    results, with and without the fused residual scatter."""
    H, E = 4096 if d == 5504 else 256, 8
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, "bf16", seed=T + d, skew=skew)
    x, lg = x.to(DEV), torch.from_numpy(lg).to(DEV)
    wg, wu, wd = wg.to(DEV), wu.to(DEV), wd.to(DEV)
    outs = []
    for mt, askip, pairs, order, swap, merge, dyn in FFN_VARIANTS:
        knob("ffn_dyn", dyn)
        knob("ffn_merge", merge)
        knob("ffn_swap", swap)
        knob("ffn_mt", mt)
        knob("ffn_askip", askip)
        knob("ffn_pairs", pairs)
        knob("ffn_order", order)
        y, _ = rd.moe_layer(x, wg, wu, wd, logits=lg, residual=x)
        plan = rd.route(lg, 1)
        ys = rd.expert_ffn(rd.dispatch(x, plan.dest, 1), plan.offsets, wg, wu, wd)
        outs.append((y, ys))
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(outs[0][0], o[0]) and torch.equal(outs[0][1], o[1])


# segment sizes around the tail merge: full 256-row m-tiles carrying remainders of 1..64 rows (one or two
# tails), remainders past what is merged (three or more 64-row chunks, or more than the full m-tiles can carry:
# their own M = 128 / M = 256 tile), exact multiples, empty and tiny segments
MERGE_COUNTS = [257, 272, 273, 320, 512 + 65, 512 + 128, 768 + 192, 768 + 193, 1024 + 200, 256 + 65, 0, 5, 512,
                256 + 63, 64, 1024 + 255]


@pytest.mark.parametrize("H,d", [(256, 264), (4096, 384)])
def test_ffn_merged_tails(rd, knob, H, d):
    """256-row m-tiles with merged segment tails (the tail's swap-AB MMAs read the full m-tile's weight stages
    and accumulate into the other accumulator's columns [192, 256)): vs the fp64 oracle, and bitwise equal to
    tails as their own swap-AB tiles and as M = 128 tiles, through expert_ffn and the whole layer (gather
    dispatch + row flags, fused residual scatter), on all pairs and on 1 and 3 CTA pairs."""
    counts = MERGE_COUNTS
    E = len(counts)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    rows = int(off[-1])
    xs = synth.to_torch(synth.tokens(rows, H, seed=21), "bf16").to(DEV)
    wg, wu, wd = (synth.to_torch(w, "bf16") for w in synth.expert_weights(E, d, H, seed=22))
    W = [w.to(DEV) for w in (wg, wu, wd)]
    offd = torch.from_numpy(off).to(DEV)
    # logits that send exactly counts[e] tokens to expert e (the layer path routes them itself)
    lg = np.full((rows, E), -5.0, dtype=np.float32)
    lg[np.arange(rows), np.repeat(np.arange(E), counts)] = 5.0
    perm = synth.rng(23, 0).permutation(rows)
    lg = torch.from_numpy(lg[perm]).to(DEV)
    x = xs  # token t goes to expert argmax(lg[t])
    knob("ffn_mt", 256)
    outs = []
    for merge, swap, pairs, dyn in [(1, -1, 0, -1), (0, 64, 0, 0), (0, 0, 0, 1), (1, -1, 1, -1), (1, -1, 3, 0),
                                    (1, -1, 0, 0), (1, -1, 2, 1)]:
        knob("ffn_dyn", dyn)
        knob("ffn_merge", merge)
        knob("ffn_swap", swap)
        knob("ffn_pairs", pairs)
        st = torch.zeros(1, dtype=torch.int32, device=DEV)
        ys = rd.expert_ffn(xs, offd, *W, dev_status=st)
        y, plan = rd.moe_layer(x, *W, logits=lg, residual=x)
        torch.cuda.synchronize()
        assert int(st.item()) == 0 and int(plan.dev_status.item()) == 0
        outs.append((ys, y))
    ref = oracle.expert_ffn(xs.cpu(), off, wg, wu, wd)
    assert rel_err(_np(outs[0][0]), ref) <= BF16_TOL
    for o in outs[1:]:
        assert torch.equal(outs[0][0], o[0]) and torch.equal(outs[0][1], o[1])


# ---- co-residency of the single-launch FFN (its down tiles wait on other CTA pairs' gate/up tiles) ------

def _starve_setup(rd, T=8192, H=1024, d=1024, E=8):
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, "bf16", seed=601)
    W = [w.to(DEV) for w in (wg, wu, wd)]
    plan = rd.route(torch.from_numpy(lg).to(DEV), 1)
    xs = rd.dispatch(x.to(DEV), plan.dest, 1)
    ref = rd.expert_ffn(xs, plan.offsets, *W)  # uncontended launch
    torch.cuda.synchronize()
    n_hold = torch.cuda.get_device_properties(0).multi_processor_count - 8
    return x.to(DEV), lg, plan, xs, W, ref, n_hold


def test_ffn_sm_starved_recovers(rd, knob):
    """140 of 148 SMs held by another stream's kernel for 0.3 s while the FFN launches: the few pairs that
    fit wait for the rest (bounded polls, far below the give-up limit) and the result is bitwise the
    uncontended one, dev_status clean."""
    x, lg, plan, xs, W, ref, n_hold = _starve_setup(rd)
    hold, work = torch.cuda.Stream(), torch.cuda.Stream()
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    out = torch.full_like(ref, 7.0)
    torch.cuda.synchronize()
    rd.debug_hold_sms(n_hold, 300_000_000, hold)
    time.sleep(0.05)
    with torch.cuda.stream(work):
        rd.expert_ffn(xs, plan.offsets, *W, out=out, dev_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert torch.equal(out, ref)
    # the whole layer (dispatch, FFN behind it with PDL) under the same starvation: the default scatter
    # dispatch, and the gather run by the FFN's own epilogue warps (row flags waited on per tile)
    y0, _ = rd.moe_layer(x, *W, logits=torch.from_numpy(lg).to(DEV), residual=x)
    torch.cuda.synchronize()
    for form in (0, 3):
        knob("dispatch", form)
        y1 = torch.full_like(y0, 7.0)
        plan1 = rd.new_plan(x.shape[0], 8, 1, DEV)
        torch.cuda.synchronize()
        rd.debug_hold_sms(n_hold, 300_000_000, hold)
        time.sleep(0.05)
        with torch.cuda.stream(work):
            rd.moe_layer(x, *W, logits=torch.from_numpy(lg).to(DEV), residual=x, plan=plan1, out=y1)
        torch.cuda.synchronize()
        assert int(plan1.dev_status.item()) == 0
        assert torch.equal(y1, y0)


def test_ffn_sm_starved_gives_up_without_wrong_values(rd, knob):
    """The same starvation held for 2 s with the poll limit cut to 2^12: a readiness wait gives up, the
    launch reports README_DEV_SCHED_TIMEOUT, and every output element is either untouched (the sentinel)
    or exactly the uncontended value — never one computed from unready rows."""
    x, lg, plan, xs, W, ref, n_hold = _starve_setup(rd)
    knob("ffn_spin", 12)
    hold, work = torch.cuda.Stream(), torch.cuda.Stream()
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    out = torch.full_like(ref, 7.0)
    torch.cuda.synchronize()
    rd.debug_hold_sms(n_hold, 2_000_000_000, hold)
    time.sleep(0.05)
    with torch.cuda.stream(work):
        rd.expert_ffn(xs, plan.offsets, *W, out=out, dev_status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & rd.README_DEV_SCHED_TIMEOUT
    touched = out != 7.0
    assert torch.equal(out[touched], ref[touched])
    assert int(touched.sum().item()) < out.numel()  # the give-up really stopped stores


def test_expert_ffn_segments_n_src(rd):
    """EP receive layout: n_src groups of E segments, expert = segment % E."""
    H, d, E, G = 256, 128, 4, 3
    rows = 900
    xs = synth.to_torch(synth.tokens(rows, H, seed=9), "bf16")
    wg, wu, wd = (synth.to_torch(w, "bf16") for w in synth.expert_weights(E, d, H, seed=10))
    cuts = np.sort(synth.rng(11, 0).integers(0, rows, size=G * E - 1))
    off = np.concatenate([[0], cuts, [rows]]).astype(np.int32)
    ys = rd.expert_ffn(xs.to(DEV), torch.from_numpy(off).to(DEV), wg.to(DEV), wu.to(DEV), wd.to(DEV), n_src=G)
    ref = oracle.expert_ffn(xs, off, wg, wu, wd, n_src=G)
    assert rel_err(_np(ys), ref) <= BF16_TOL


# ---- whole layer -------------------------------------------------------------------------------------

@pytest.mark.parametrize("path", ["fused", "gather-fused", "gather", "scatter", "lookback", "split", "unfused"])
@pytest.mark.parametrize("dt,T,H,d,E,k", [("f32", 256, 64, 128, 8, 1), ("f32", 256, 64, 128, 8, 2),
                                           ("bf16", 1500, 512, 640, 8, 1), ("bf16", 600, 256, 256, 8, 2),
                                           ("bf16", 3000, 1024, 1376, 8, 1)])
def test_moe_layer_end_to_end(rd, knob, path, dt, T, H, d, E, k):
    # fused: cluster route -> gather dispatch with per-row flags -> single-launch FFN waiting per tile;
    # lookback: multi-CTA route -> finalize fused into the dispatch -> FFN behind a whole-grid PDL wait
    # gather-fused / gather / scatter force the dispatch form (default: scatter, the FFN behind it as a PDL
    # dependent; "gather" = the gather kernel publishing row flags, "gather-fused" = the same gather run by
    # the FFN launch's own epilogue warps)
    if path == "lookback":
        knob("route", 2)
    elif path in ("gather-fused", "gather", "scatter"):
        knob("dispatch", {"gather-fused": 3, "gather": 2, "scatter": 1}[path])
    elif path != "fused":
        knob("ffn_kernel", FFN_KERNEL[path])
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, k, dt, seed=T * 3 + 1)
    res = synth.to_torch(synth.residual(T, H, seed=12), dt)
    y, plan = rd.moe_layer(x.to(DEV), wg.to(DEV), wu.to(DEV), wd.to(DEV), k=k,
                           logits=torch.from_numpy(lg).to(DEV), residual=res.to(DEV))
    yref, pref = oracle.moe_layer(x, lg, k, wg, wu, wd, residual=res)
    _check_plan(plan, pref, k)
    assert rel_err(_np(y), yref) <= (BF16_TOL if dt == "bf16" else F32_TOL)


@pytest.mark.parametrize("T,k,d", [(2500, 1, 512), (1300, 2, 264), (700, 1, 5504)])
def test_moe_layer_dispatch_forms_bitwise(rd, knob, T, k, d):
    """a5 as a scatter kernel, as a gather kernel with per-row flags, and inside the FFN launch (its epilogue
    warps gather the rows before their first tile): the same x_sorted, so the same layer output bit for bit,
    clean dev_status."""
    H, E = 4096 if d == 5504 else 512, 8
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, k, "bf16", seed=T + k)
    x, lg, W = x.to(DEV), torch.from_numpy(lg).to(DEV), [w.to(DEV) for w in (wg, wu, wd)]
    outs = []
    for form in (1, 2, 3):
        knob("dispatch", form)
        y, plan = rd.moe_layer(x, *W, k=k, logits=lg, residual=x)
        torch.cuda.synchronize()
        assert int(plan.dev_status.item()) == 0
        outs.append(y)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])


def _fuzz_cases(n=24, seed=2410):
    g = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        E = int(g.integers(1, 17))
        k = int(g.integers(1, min(E, 4) + 1))
        T = int(g.choice([1, 7, 64, 129, 511, 700, 1025, 2100, 3000]))
        H = int(8 * g.integers(4, 97))     # 32..768, any multiple of 8
        d = int(8 * g.integers(2, 81))     # 16..640
        out.append((T, E, k, H, d))
    return out


@pytest.mark.parametrize("T,E,k,H,d", _fuzz_cases())
def test_moe_layer_fuzz_bf16(rd, T, E, k, H, d):
    # seeded random shapes through the default path (cluster route; scatter or gather dispatch by size; the
    # single-launch FFN with 128- or 256-row m-tiles by size; fused combine for k = 1, combine launch
    # otherwise) against the oracle: routing bit-exact, outputs within the bf16 rule
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, k, "bf16", seed=T * 7 + E + H + d)
    res = synth.to_torch(synth.residual(T, H, seed=T + 3), "bf16")
    y, plan = rd.moe_layer(x.to(DEV), wg.to(DEV), wu.to(DEV), wd.to(DEV), k=k,
                           logits=torch.from_numpy(lg).to(DEV), residual=res.to(DEV))
    yref, pref = oracle.moe_layer(x, lg, k, wg, wu, wd, residual=res)
    _check_plan(plan, pref, k)
    assert int(plan.dev_status.item()) == 0
    assert rel_err(_np(y), yref) <= BF16_TOL


def _tail_fuzz_cases(n=12, seed=4103):
    g = synth.rng(seed, 0)
    out = []
    for i in range(n):
        E = int(g.integers(1, 13))
        # segment sizes around multiples of 256 (remainders 0..255, some empty segments)
        counts = [0 if g.random() < 0.1 else int(256 * g.integers(0, 6) + g.integers(0, 256)) for _ in range(E)]
        if sum(counts) < 1100:  # above the decode size, so 256-row m-tiles (where tails merge) are used
            counts[0] += 1100
        out.append((i, counts, int(64 * g.integers(2, 9)), int(8 * g.integers(8, 49))))
    return out


@pytest.mark.parametrize("case,counts,H,d", _tail_fuzz_cases())
def test_ffn_tail_fuzz_bitwise(rd, knob, case, counts, H, d):
    """Seeded random segment sizes through the single-launch FFN: merged tails under the dynamic order (the
    default below 16384 rows), merged tails under the static order, and separate tails under the static order
    give the same bits; the default also vs the fp64 oracle."""
    E = len(counts)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    rows = int(off[-1])
    xs = synth.to_torch(synth.tokens(rows, H, seed=300 + case), "bf16").to(DEV)
    wg, wu, wd = (synth.to_torch(w, "bf16") for w in synth.expert_weights(E, d, H, seed=400 + case))
    W = [w.to(DEV) for w in (wg, wu, wd)]
    offd = torch.from_numpy(off).to(DEV)
    outs = []
    for merge, dyn in [(-1, -1), (1, 0), (0, 0), (1, 1)]:
        knob("ffn_merge", merge)
        knob("ffn_dyn", dyn)
        st = torch.zeros(1, dtype=torch.int32, device=DEV)
        outs.append(rd.expert_ffn(xs, offd, *W, dev_status=st))
        torch.cuda.synchronize()
        assert int(st.item()) == 0
    for o in outs[1:]:
        assert torch.equal(outs[0], o)
    ref = oracle.expert_ffn(xs.cpu(), off, wg, wu, wd)
    assert rel_err(_np(outs[0]), ref) <= BF16_TOL


@pytest.mark.parametrize("T,E,k,H,d", _fuzz_cases(8, seed=19123))
def test_moe_layer_fuzz_f32(rd, T, E, k, H, d):
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, k, "f32", seed=T * 5 + E + H + d)
    y, plan = rd.moe_layer(x.to(DEV), wg.to(DEV), wu.to(DEV), wd.to(DEV), k=k, logits=torch.from_numpy(lg).to(DEV))
    yref, pref = oracle.moe_layer(x, lg, k, wg, wu, wd)
    _check_plan(plan, pref, k)
    assert rel_err(_np(y), yref) <= F32_TOL


@pytest.mark.parametrize("T,E,k,H,d", [(8192, 64, 1, 512, 256), (4096, 128, 2, 256, 128), (3000, 256, 1, 128, 64)])
def test_moe_layer_many_experts(rd, T, E, k, H, d):
    # fine-grained expert counts (up to README_MAX_EXPERTS = 256 segments): many empty and one-row experts,
    # 128-row tails everywhere
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, k, "bf16", seed=E + T)
    y, plan = rd.moe_layer(x.to(DEV), wg.to(DEV), wu.to(DEV), wd.to(DEV), k=k, logits=torch.from_numpy(lg).to(DEV))
    yref, pref = oracle.moe_layer(x, lg, k, wg, wu, wd)
    _check_plan(plan, pref, k)
    assert int(plan.dev_status.item()) == 0
    assert rel_err(_np(y), yref) <= BF16_TOL


@pytest.mark.parametrize("T,sub", [(1500, 700), (4096, 512), (3000, 2100)])
def test_batch_invariance_bitwise(rd, T, sub):
    """P13: a token's output does not depend on the other tokens of its batch — bitwise, across batch sizes
    that take different paths (128- vs 256-row m-tiles at <= / > 1024 rows, scatter vs gather dispatch at
    < / >= 2048 rows): no split-K, the K order of every output element is fixed."""
    H, d, E = 512, 384, 8
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, "bf16", seed=T + sub)
    W = tuple(w.to(DEV) for w in (wg, wu, wd))
    xd, lgd = x.to(DEV), torch.from_numpy(lg).to(DEV)
    y_all, _ = rd.moe_layer(xd, *W, logits=lgd, residual=xd)
    idx = torch.from_numpy(synth.rng(T, 95).choice(T, size=sub, replace=False).astype(np.int64)).to(DEV)
    xs_, lgs_ = xd[idx].contiguous(), lgd[idx].contiguous()
    y_sub, _ = rd.moe_layer(xs_, *W, logits=lgs_, residual=xs_)
    torch.cuda.synchronize()
    assert torch.equal(y_all[idx], y_sub)


def test_moe_layer_plan_in_equals_route(rd):
    T, H, d, E = 800, 256, 256, 8
    x, lg, wg, wu, wd = (t.to(DEV) if isinstance(t, torch.Tensor) else t
                         for t in _ffn_case(T, H, d, E, 1, "bf16", seed=21))
    y1, plan = rd.moe_layer(x, wg, wu, wd, logits=torch.from_numpy(lg).to(DEV))
    y2, _ = rd.moe_layer(x, wg, wu, wd, plan=plan)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)


def test_full_expert_equals_dense_gpu(rd):
    """P1 on the GPU: experts whose neuron set is the whole dense FFN reproduce the dense FFN."""
    T, H, D, E = 512, 256, 384, 4
    wg, wu, wd = synth.dense_ffn_weights(D, H, D, seed=31)
    S = synth.neuron_sets(E, D, D, mode="full")
    g = [synth.to_torch(w, "bf16").to(DEV) for w in (wg, wu, wd)]
    eg, eu, ed = rd.build_experts(*g, torch.from_numpy(S).to(DEV))
    x = synth.to_torch(synth.tokens(T, H, seed=32), "bf16")
    y, _ = rd.moe_layer(x.to(DEV), eg, eu, ed, logits=torch.from_numpy(synth.router_logits(T, E, seed=33)).to(DEV))
    yd = oracle.dense_ffn(x, *(t.cpu() for t in g))
    assert rel_err(_np(y), yd) <= BF16_TOL


def test_build_experts_bit_exact(rd):
    D, H, E, d = 1000, 264, 8, 504
    wg, wu, wd = (synth.to_torch(w, "bf16") for w in synth.dense_ffn_weights(D, H, d, seed=41))
    S = synth.neuron_sets(E, D, d, seed=42)
    eg, eu, ed = rd.build_experts(wg.to(DEV), wu.to(DEV), wd.to(DEV), torch.from_numpy(S).to(DEV))
    ref = oracle.build_experts(wg, wu, wd, S)
    for got, want in zip((eg, eu, ed), ref):
        assert np.array_equal(_np(got).astype(np.float64), want)


@pytest.mark.parametrize("with_residual", [False, True])
def test_fused_scatter_vs_unfused(rd, knob, with_residual):
    """k=1: the combine fused into GEMM2's epilogue (y[src[r]] = res + acc, one rounding) equals the unfused
    sequence bit for bit without a residual; with one, the unfused path rounds twice (y_sorted, then
    res + y_sorted), so both are checked against the oracle instead."""
    T, H, d, E = 2000, 512, 384, 8
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, "bf16", seed=41)
    res = synth.to_torch(synth.residual(T, H, seed=42), "bf16") if with_residual else None
    W = [w.to(DEV) for w in (wg, wu, wd)]
    lgt = torch.from_numpy(lg).to(DEV)
    r_dev = res.to(DEV) if res is not None else None
    y1, _ = rd.moe_layer(x.to(DEV), *W, logits=lgt, residual=r_dev)
    knob("ffn_kernel", 2)
    y2, _ = rd.moe_layer(x.to(DEV), *W, logits=lgt, residual=r_dev)
    torch.cuda.synchronize()
    if not with_residual:
        assert torch.equal(y1, y2)
    else:
        yref, _ = oracle.moe_layer(x, lg, 1, wg, wu, wd, residual=res)
        assert rel_err(_np(y1), yref) <= BF16_TOL and rel_err(_np(y2), yref) <= BF16_TOL


def test_fused_plan_in_with_corrupt_src_is_safe(rd):
    """A plan whose src holds out-of-range rows must not write out of bounds (rows are skipped)."""
    T, H, d, E = 512, 256, 128, 8
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, "bf16", seed=44)
    W = [w.to(DEV) for w in (wg, wu, wd)]
    y, plan = rd.moe_layer(x.to(DEV), *W, logits=torch.from_numpy(lg).to(DEV))
    plan.src[5] = 10 ** 6
    plan.src[6] = -3
    y2, _ = rd.moe_layer(x.to(DEV), *W, plan=plan)
    torch.cuda.synchronize()
    assert y2.shape == y.shape


def test_permutation_equivariance_bitwise_gpu(rd):
    """P4/P13: permuting tokens permutes outputs bitwise (fixed K order, no split-K)."""
    T, H, d, E = 1200, 512, 384, 8
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, "bf16", seed=51)
    W = [w.to(DEV) for w in (wg, wu, wd)]
    y, plan = rd.moe_layer(x.to(DEV), *W, logits=torch.from_numpy(lg).to(DEV))
    perm = torch.from_numpy(synth.rng(52, 0).permutation(T))
    yp, planp = rd.moe_layer(x[perm].to(DEV), *W, logits=torch.from_numpy(lg[perm.numpy()]).to(DEV))
    torch.cuda.synchronize()
    assert torch.equal(yp.cpu(), y.cpu()[perm])
    assert torch.equal(plan.counts, planp.counts)


def test_scaling_exact_gpu(rd):
    """P10: W_down * 2 -> y * 2 exactly."""
    T, H, d, E = 500, 256, 256, 8
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, "bf16", seed=61)
    lgt = torch.from_numpy(lg).to(DEV)
    y, _ = rd.moe_layer(x.to(DEV), wg.to(DEV), wu.to(DEV), wd.to(DEV), logits=lgt)
    y2, _ = rd.moe_layer(x.to(DEV), wg.to(DEV), wu.to(DEV), (wd * 2).to(DEV), logits=lgt)
    torch.cuda.synchronize()
    assert torch.equal(y2, y * 2)


def test_zero_input_gpu(rd):
    T, H, d, E = 300, 256, 128, 8
    _, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, "bf16", seed=71)
    y, _ = rd.moe_layer(torch.zeros((T, H), dtype=torch.bfloat16, device=DEV), wg.to(DEV), wu.to(DEV), wd.to(DEV),
                        logits=torch.from_numpy(lg).to(DEV))
    torch.cuda.synchronize()
    assert torch.count_nonzero(y).item() == 0


def test_cuda_graph_capture(rd):
    T, H, d, E = 1024, 512, 256, 8
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, "bf16", seed=81)
    x, wg, wu, wd = (t.to(DEV) for t in (x, wg, wu, wd))
    lgt = torch.from_numpy(lg).to(DEV)
    plan = rd.new_plan(T, E, 1, DEV)
    out = torch.empty_like(x)
    ws = torch.empty(rd.moe_layer_workspace_bytes(T, H, E, d, 1, x.dtype), dtype=torch.uint8, device=DEV)
    y_eager, _ = rd.moe_layer(x, wg, wu, wd, logits=lgt)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        rd.moe_layer(x, wg, wu, wd, logits=lgt, plan=plan, out=out, ws=ws)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        rd.moe_layer(x, wg, wu, wd, logits=lgt, plan=plan, out=out, ws=ws)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, y_eager)


# ---- full size: every token of configs 2 and 3, 8192 of config 5, against the fp64 oracle ------------------
# The oracle's experts are sliced by the oracle itself from the dense weights (oracle.build_experts), never
# taken from the GPU; a brute-force sample straight from the dense weights (no sort, scan or buffers) is
# checked beside it.

def _dense_and_oracle_experts(seed):
    c = synth.CONFIGS[2]
    H, D, d, E = c["H"], c["D"], c["d"], c["E"]
    wg, wu, wd = synth.dense_ffn_weights(D, H, d, seed=seed)
    S = synth.neuron_sets(E, D, d, seed=seed)
    dense = [synth.to_torch(w, "bf16") for w in (wg, wu, wd)]
    del wg, wu, wd
    return dense, S, oracle.build_experts(*dense, S)


def _gpu_experts(rd, dense, S):
    return rd.build_experts(*(t.to(DEV) for t in dense), torch.from_numpy(S).to(DEV))


def test_config2_full_population(rd):
    """Config 2 as the bench runs it (T = 8192, Llama-2-7B expert shape, bf16): the routing plan bit-exact
    and EVERY token's output within the bf16 rule of the fp64 oracle (Eq. 2)."""
    c = synth.CONFIGS[2]
    T, H, E = c["T"], c["H"], c["E"]
    seed = synth.MASTER_SEED + 2
    dense, S, (og, ou, od) = _dense_and_oracle_experts(seed)
    eg, eu, ed = _gpu_experts(rd, dense, S)
    x = synth.to_torch(synth.tokens(T, H, seed=seed), "bf16")
    lg = synth.router_logits(T, E, seed=seed)
    y, plan = rd.moe_layer(x.to(DEV), eg, eu, ed, logits=torch.from_numpy(lg).to(DEV))
    torch.cuda.synchronize()
    yref, pref = oracle.moe_layer(x, lg, 1, og, ou, od)
    _check_plan(plan, pref, 1)
    yg = _np(y)
    assert rel_err(yg, yref) <= BF16_TOL
    # 8 tokens per expert by brute force from the dense weights
    idx = pref["topk_idx"][:, 0]
    g = synth.rng(seed, 99)
    sample = np.concatenate([g.choice(np.nonzero(idx == e)[0], size=8, replace=False) for e in range(E)])
    yb = oracle.bruteforce(x[sample], lg[sample], 1, *dense, S)
    assert rel_err(yg[sample], yb) <= BF16_TOL


@pytest.mark.parametrize("B,s", [(512, 1.0), (256, 1.0), (64, 2.0)])
def test_config3_decode_full_shape(rd, B, s):
    """Config 3 as bench.py runs it: Zipf-skewed pre-gated assignments, Llama-2-7B expert shape, the whole layer
    captured in a CUDA graph and replayed; routing bit-exact and EVERY token within the bf16 rule of the fp64
    oracle, plus brute force from the dense weights on 4 tokens per touched expert."""
    c = synth.CONFIGS[3]
    H, E = c["H"], c["E"]
    seed = synth.MASTER_SEED + 2
    dense, S, (og, ou, od) = _dense_and_oracle_experts(seed)
    eg, eu, ed = _gpu_experts(rd, dense, S)
    ids = synth.assignments_zipf(B, E, s, seed=seed + B)
    lg = synth.logits_for_assignments(ids, E, seed=B)
    x = synth.to_torch(synth.tokens(B, H, seed=B), "bf16")
    xd, lgd = x.to(DEV), torch.from_numpy(lg).to(DEV)
    plan = rd.new_plan(B, E, 1, DEV)
    y = torch.empty_like(xd)
    ws = torch.empty(rd.moe_layer_workspace_bytes(B, H, E, c["d"], 1, torch.bfloat16), dtype=torch.uint8,
                     device=DEV)
    fn = lambda: rd.moe_layer(xd, eg, eu, ed, k=1, logits=lgd, plan=plan, out=y, ws=ws)
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    y.zero_()
    g.replay()
    torch.cuda.synchronize()
    yref, pref = oracle.moe_layer(x, lg, 1, og, ou, od)
    _check_plan(plan, pref, 1)
    assert int(plan.dev_status.item()) == 0
    yg = _np(y)
    assert rel_err(yg, yref) <= BF16_TOL
    gs = synth.rng(seed, 98)
    sample = np.concatenate([gs.choice(np.nonzero(ids == e)[0], size=min(4, int((ids == e).sum())), replace=False)
                             for e in range(E) if (ids == e).any()])
    yb = oracle.bruteforce(x[sample], lg[sample], 1, *dense, S)
    assert rel_err(yg[sample], yb) <= BF16_TOL


def test_config5_full_size_sampled(rd):
    """Config 5 at G = 1 (T = 65536 on one GPU): routing bit-exact on all tokens; 1024 tokens of every expert
    (8192 in all, drawn at random from each expert's rows) within the bf16 rule of the fp64 oracle."""
    c = synth.CONFIGS[5]
    T, H, E = c["T"], c["H"], c["E"]
    seed = synth.MASTER_SEED + 2
    dense, S, (og, ou, od) = _dense_and_oracle_experts(seed)
    eg, eu, ed = _gpu_experts(rd, dense, S)
    x = synth.to_torch(synth.tokens(T, H, seed=seed + 5), "bf16")
    lg = synth.router_logits(T, E, seed=seed + 5)
    y, plan = rd.moe_layer(x.to(DEV), eg, eu, ed, logits=torch.from_numpy(lg).to(DEV))
    torch.cuda.synchronize()
    pref = oracle.route(lg, 1)
    _check_plan(plan, pref, 1)
    idx = pref["topk_idx"][:, 0]
    gs = synth.rng(seed, 97)
    sample = np.sort(np.concatenate([gs.choice(np.nonzero(idx == e)[0], size=1024, replace=False)
                                     for e in range(E)]))
    yref, _ = oracle.moe_layer(x[sample], lg[sample], 1, og, ou, od)
    yg = _np(y)[sample]
    assert rel_err(yg, yref) <= BF16_TOL
    yb = oracle.bruteforce(x[sample[:16]], lg[sample[:16]], 1, *dense, S)
    assert rel_err(yg[:16], yb) <= BF16_TOL


def test_config4_full_size_sampled(rd):
    # config 4 as bench.py runs it (T = 16384, 32 layers, Markov routing, ONE readme_moe_stack call), then
    # (i) the same stack as 32 plan-in calls of one layer each is bitwise identical, and (ii) each layer is
    # teacher-forced against the oracle on sampled tokens: tokens are independent in the MoE-only stack,
    # so the oracle runs a layer on 8 tokens of every expert with only that expert's weights (~2000
    # token-layers over the 32 layers)
    c = synth.CONFIGS[4]
    T, H, d, E, L = c["T"], c["H"], c["d"], c["E"], c["L"]
    seed = synth.MASTER_SEED + 4
    layers = [synth.expert_weights_device(E, d, H, DEV, seed=seed, layer=l) for l in range(L)]
    ids = synth.assignments_markov(T // 4096, 4096, E, 0.672, seed=seed)
    lg = synth.logits_for_assignments(ids, E, seed=seed)
    x0 = synth.to_torch(synth.tokens(T, H, seed=seed), "bf16").to(DEV)
    x = x0.clone()
    _, plan = rd.moe_stack(x, layers, logits=torch.from_numpy(lg).to(DEV))
    torch.cuda.synchronize()
    _check_plan(plan, oracle.route(lg, 1), 1)
    gs = synth.rng(seed, 96)
    toks = {e: gs.choice(np.nonzero(ids == e)[0], size=8, replace=False) for e in range(E) if (ids == e).sum() >= 8}
    assert len(toks) >= 6
    xl = x0.clone()
    worst = 0.0
    for l in range(L):
        xin = xl[np.concatenate(list(toks.values()))].cpu()
        rd.moe_stack(xl, [layers[l]], plan=plan)
        torch.cuda.synchronize()
        out = _np(xl)
        off = 0
        for e, tk in toks.items():
            w1 = tuple(w[e:e + 1].cpu() for w in layers[l])
            lg1 = np.zeros((tk.size, 1), np.float32)
            yref, _ = oracle.moe_stack(xin[off:off + tk.size], lg1, 1, [w1])
            err = rel_err(out[tk], yref)
            worst = max(worst, err)
            assert err <= BF16_TOL, (l, e, err)
            off += tk.size
    assert torch.equal(xl, x)  # one L=32 call == 32 plan-in calls of one layer, bit for bit
    assert worst > 0.0


# ---- config 4: pre-norm dispatch and the route-once stack ----------------------------------------------

@pytest.mark.parametrize("dt,k,H", [("bf16", 1, 4096), ("bf16", 2, 4096), ("bf16", 1, 768), ("bf16", 2, 1000),
                                    ("f32", 1, 256)])
def test_dispatch_rmsnorm(rd, dt, k, H):
    """Pre-norm dispatch (the row-in-registers kernel for bf16 rows of 256 * n <= 4096, the two-pass kernel
    otherwise): within the tolerance of the fp64 oracle, and per element within one final rounding of it."""
    T = 700
    x = synth.to_torch(synth.tokens(T, H, seed=151) * 3.0, dt)
    plan = oracle.route(synth.router_logits(T, 8, seed=152), k)
    xs = rd.dispatch_rmsnorm(x.to(DEV), torch.from_numpy(plan["dest"]).to(DEV), k, eps=1e-5)
    ref = oracle.dispatch(oracle.rmsnorm(x, 1e-5), plan["dest"], k)
    assert rel_err(_np(xs), ref) <= (BF16_TOL if dt == "bf16" else F32_TOL)
    if dt == "bf16":  # one bf16 rounding of an fp32 product: <= 2^-8 relative (+ fp32 statistics slack)
        got = _np(xs).astype(np.float64)
        assert np.all(np.abs(got - ref) <= 2.0 ** -8 * 1.01 * np.abs(ref) + 1e-30)


@pytest.mark.parametrize("path", ["fused", "gather", "split"])
@pytest.mark.parametrize("dt,k,L", [("bf16", 1, 4), ("bf16", 2, 3), ("f32", 1, 3)])
def test_moe_stack_end_to_end(rd, knob, path, dt, k, L):
    # fused: gather-form pre-norm dispatch with row flags + single-launch FFN (k = 1, bf16); split: the
    # scatter dispatch + two-launch FFN
    if path == "split":
        knob("ffn_kernel", 1)
    elif path == "gather":
        knob("dispatch", 2)
    T, H, d, E = 600, 256, 256, 8
    x = synth.to_torch(synth.tokens(T, H, seed=161), dt)
    ids = synth.assignments_markov(2, T // 2, E, 0.672, seed=162)
    lg = synth.logits_for_assignments(ids, E, seed=163) if k == 1 else synth.router_logits(T, E, seed=163)
    layers = [tuple(synth.to_torch(w, dt) for w in synth.expert_weights(E, d, H, seed=164, layer=l))
              for l in range(L)]
    xg = x.to(DEV).clone()
    yg, plan = rd.moe_stack(xg, [tuple(w.to(DEV) for w in ly) for ly in layers], k=k,
                            logits=torch.from_numpy(lg).to(DEV))
    yref, pref = oracle.moe_stack(x, lg, k, layers)
    _check_plan(plan, pref, k)
    assert rel_err(_np(yg), yref) <= (BF16_TOL if dt == "bf16" else F32_TOL)


def test_moe_stack_plan_in_equals_routed(rd):
    T, H, d, E, L = 700, 256, 384, 8, 3
    x = synth.to_torch(synth.tokens(T, H, seed=181), "bf16").to(DEV)
    lg = torch.from_numpy(synth.router_logits(T, E, seed=182)).to(DEV)
    layers = [tuple(synth.to_torch(w, "bf16").to(DEV) for w in synth.expert_weights(E, d, H, seed=183, layer=l))
              for l in range(L)]
    y1, plan = rd.moe_stack(x.clone(), layers, logits=lg)
    y2, _ = rd.moe_stack(x.clone(), layers, plan=plan)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)


# ---- NEXT-2: expert-aware batching on the GPU serving loop ---------------------------------------------

def test_serving_expert_aware_touches_fewer_experts(rd):
    from paper_2410_19123_b200 import serving
    E, d, H = 8, 256, 512
    W = [synth.to_torch(w, "bf16").to(DEV) for w in synth.expert_weights(E, d, H, seed=171)]
    a = serving.simulate("expert_aware", *W, n_requests=256, max_tokens=64, steps=20, device=DEV)
    b = serving.simulate("fifo", *W, n_requests=256, max_tokens=64, steps=20, device=DEV)
    assert a["tokens"] == b["tokens"] == 20 * 64
    assert a["mean_unique_experts"] < b["mean_unique_experts"]


# ---- NEXT-3: permanent expert ---------------------------------------------------------------------------

@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_permanent_expert(rd, dt):
    T, H, d, E, dp = 900, 256, 256, 8, 136
    x, lg, wg, wu, wd = _ffn_case(T, H, d, E, 1, dt, seed=181)
    pg, pu, pd = (synth.to_torch(w, dt) for w in synth.expert_weights(1, dp, H, seed=182))
    y, _ = rd.moe_layer(x.to(DEV), wg.to(DEV), wu.to(DEV), wd.to(DEV), logits=torch.from_numpy(lg).to(DEV))
    rd.permanent_expert(x.to(DEV), pg[0].to(DEV), pu[0].to(DEV), pd[0].to(DEV), y)
    yref, _ = oracle.moe_layer(x, lg, 1, wg, wu, wd)
    yref = yref + oracle.expert_ffn(x, np.array([0, T], np.int32), pg, pu, pd)
    assert rel_err(_np(y), yref) <= (BF16_TOL if dt == "bf16" else F32_TOL)


# ---- NEXT-1: the pre-gating router G ---------------------------------------------------------------------

def test_router_forward_parity(rd):
    """readme_router_forward vs the fp64 oracle on ragged sequences (1 token, exact 32-multiples, several
    query tiles). Logits: bf16 rule. Decisions: identical where the oracle's top-two margin exceeds twice the
    bf16 rule's band; inside it any expert within that band of the oracle's max is accepted (the north star's
    near-tie consistency rule, widened to the bf16 error of a router computed on the GPU, reading Q16). The
    routing plan built from the GPU's own logits is then bit-exact (as in every route test)."""
    from oracle import router
    vocab, N = 32000, 8
    W = {k: synth.to_torch(v, "bf16") for k, v in synth.router_weights(vocab=vocab, n_experts=N, seed=191).items()}
    lens = [1, 64, 100, 37, 300]
    starts = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(starts[-1])
    ids = synth.token_ids(T, vocab=vocab, seed=192)
    lg = rd.router_forward(torch.from_numpy(ids).to(DEV), torch.from_numpy(starts).to(DEV),
                           {k: v.to(DEV) for k, v in W.items()})
    torch.cuda.synchronize()
    ref = router.forward(ids, starts, W)
    got = _np(lg).astype(np.float64)
    assert rel_err(got, ref) <= BF16_TOL
    # decisions, with a FIXED band from the bf16 rule (not from the observed error): every logit of row t is
    # within tol_t = 2e-2 * ||ref_t||_inf of the oracle, so the argmax can only move where the oracle's top-two
    # margin is below 2 tol_t; there it must land on an expert within 2 tol_t of the oracle's max
    tol = BF16_TOL * np.abs(ref).max(axis=1)
    top = np.sort(ref, axis=1)
    gpu_ids = got.argmax(axis=1)
    clear = (top[:, -1] - top[:, -2]) > 2.0 * tol
    assert clear.mean() > 0.5  # the rule is not vacuous on these logits
    assert np.array_equal(gpu_ids[clear], ref.argmax(axis=1)[clear])
    assert np.all(ref[np.arange(T), gpu_ids] >= top[:, -1] - 2.0 * tol)
    plan = rd.route(lg, 1)
    _check_plan(plan, oracle.route(lg.cpu(), 1), 1)


@pytest.mark.parametrize("k,impl", [(1, None), (2, None), (1, "lookback")])
def test_router_forward_route_fused(rd, knob, k, impl):
    """NEXT-1 fusion: readme_router_forward_route computes the final RMSNorm + gating head + a1-a4 in ONE route
    launch from the block's hidden state. Its logits are bit-identical to readme_router_forward's, its plan is
    bit-identical to readme_route on those logits (and to the fp64 oracle's route of them), and its decisions
    follow the fixed bf16 band vs the fp64 router oracle. impl = lookback forces the fallback (head kernel,
    then the multi-CTA route): same results."""
    from oracle import router
    if impl:
        knob("route", ROUTE_IMPL[impl])
    vocab, N = 32000, 8
    W = {kk: synth.to_torch(v, "bf16") for kk, v in synth.router_weights(vocab=vocab, n_experts=N, seed=195).items()}
    Wd = {kk: v.to(DEV) for kk, v in W.items()}
    lens = [1, 64, 100, 37, 300, 1500]
    starts = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(starts[-1])
    ids = synth.token_ids(T, vocab=vocab, seed=196)
    ids_d, st_d = torch.from_numpy(ids).to(DEV), torch.from_numpy(starts).to(DEV)
    lg_sep = rd.router_forward(ids_d, st_d, Wd)
    lg, plan = rd.router_forward_route(ids_d, st_d, Wd, k=k)
    plan2 = rd.route(lg_sep, k)
    torch.cuda.synchronize()
    assert torch.equal(lg, lg_sep)
    for name in ("topk_idx", "topk_w", "counts", "offsets", "dest", "src"):
        assert torch.equal(getattr(plan, name), getattr(plan2, name)), name
    assert int(plan.dev_status.item()) == 0
    _check_plan(plan, oracle.route(lg.cpu(), k), k)
    ref = router.forward(ids, starts, W)
    got = _np(lg).astype(np.float64)
    assert rel_err(got, ref) <= BF16_TOL
    tol = BF16_TOL * np.abs(ref).max(axis=1)
    top = np.sort(ref, axis=1)
    gpu_ids = _np(plan.topk_idx)[:, 0]
    clear = (top[:, -1] - top[:, -2]) > 2.0 * tol
    assert np.array_equal(gpu_ids[clear], ref.argmax(axis=1)[clear])
    assert np.all(ref[np.arange(T), gpu_ids] >= top[:, -1] - 2.0 * tol)


def test_router_long_sequence_tcgen05_attention(rd):
    """The prefill attention on tcgen05/TMEM (128-query tiles, 128-key blocks, O accumulated in TMEM with the
    base moved only by > 2^8): a 4096-token request (32 key blocks, the paper's sequence length) beside ragged
    ones, every logit within the bf16 rule of the fp64 router oracle."""
    from oracle import router
    vocab, N = 32000, 8
    W = {kk: synth.to_torch(v, "bf16") for kk, v in synth.router_weights(vocab=vocab, n_experts=N, seed=197).items()}
    lens = [4096, 129, 1, 255]
    starts = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(starts[-1])
    ids = synth.token_ids(T, vocab=vocab, seed=198)
    lg = rd.router_forward(torch.from_numpy(ids).to(DEV), torch.from_numpy(starts).to(DEV),
                           {kk: v.to(DEV) for kk, v in W.items()})
    torch.cuda.synchronize()
    ref = router.forward(ids, starts, W)
    assert rel_err(_np(lg).astype(np.float64), ref) <= BF16_TOL


def test_router_causal_on_gpu(rd):
    """Appending tokens to a sequence never changes the GPU logits of its prefix (bitwise: the kernels
    process each query row against keys <= it in a fixed order)."""
    vocab, N = 32000, 8
    W = {k: synth.to_torch(v, "bf16").to(DEV) for k, v in synth.router_weights(vocab=vocab, n_experts=N, seed=193).items()}
    ids = torch.from_numpy(synth.token_ids(200, vocab=vocab, seed=194)).to(DEV)
    full = rd.router_forward(ids, torch.tensor([0, 200], dtype=torch.int32, device=DEV), W)
    pre = rd.router_forward(ids[:70].contiguous(), torch.tensor([0, 70], dtype=torch.int32, device=DEV), W)
    torch.cuda.synchronize()
    assert rel_err(_np(pre), _np(full[:70])) <= 1e-6


# ---- NEXT-4: memory-constrained mode (expert cache + prefetch) ----------------------------------------

@pytest.mark.parametrize("policy,prefetch,cap", [("belady", True, 3), ("lru", False, 3), ("belady", True, 8),
                                                  ("random", True, 4)])
def test_offloaded_stack_equals_resident_stack(rd, policy, prefetch, cap):
    """Experts streamed from pinned host memory through a small device cache give exactly the same result
    as the all-resident route-once stack (readme_moe_stack): the cache only moves weights."""
    from paper_2410_19123_b200.offload import OffloadedStack
    T, H, d, E, L = 512, 256, 256, 8, 4
    x = synth.to_torch(synth.tokens(T, H, seed=201), "bf16").to(DEV)
    ids = synth.assignments_unique(T, 3, E, seed=202)
    lg = torch.from_numpy(synth.logits_for_assignments(ids, E, seed=203)).to(DEV)
    layers = [tuple(synth.to_torch(w, "bf16") for w in synth.expert_weights(E, d, H, seed=204, layer=l))
              for l in range(L)]
    ref, _ = rd.moe_stack(x.clone(), [tuple(w.to(DEV) for w in ly) for ly in layers], logits=lg)
    host = [tuple(w.pin_memory() for w in ly) for ly in layers]
    st = OffloadedStack(host, cap, policy, DEV)
    y, stats = st.forward(x.clone(), lg, prefetch=prefetch)
    torch.cuda.synchronize()
    assert torch.equal(y, ref)
    assert stats["hits"] + stats["misses"] == L * 3


@pytest.mark.parametrize("policy,prefetch", [("belady", True), ("lru", True), ("belady", False)])
def test_offloaded_queue_matches_resident_and_cache_oracle(rd, policy, prefetch):
    """A queue of pre-gated batches through the offloaded stack: every batch's output equals the resident
    stack's, and the hit/miss count equals the oracle cache simulation of the same reference string with the
    protection boundary (oracle/cache.py, reading Q18): the current step, plus the previous one with prefetch."""
    from oracle import cache as ocache
    from paper_2410_19123_b200.offload import OffloadedStack
    T, H, d, E, L, B, cap = 384, 256, 256, 8, 3, 4, 6
    layers = [tuple(synth.to_torch(w, "bf16") for w in synth.expert_weights(E, d, H, seed=214, layer=l))
              for l in range(L)]
    dev_layers = [tuple(w.to(DEV) for w in ly) for ly in layers]
    batches, refs, trace, prot = [], [], [], []
    prev = 0
    for b in range(B):
        x = synth.to_torch(synth.tokens(T, H, seed=220 + b), "bf16").to(DEV)
        ids = synth.assignments_unique(T, 2 + b % 2, E, seed=230 + b)
        lg = torch.from_numpy(synth.logits_for_assignments(ids, E, seed=240 + b)).to(DEV)
        refs.append(rd.moe_stack(x.clone(), dev_layers, logits=lg)[0])
        batches.append((x.clone(), lg))
        ex = sorted(set(ids.reshape(-1).tolist()))
        for l in range(L):
            start = len(trace)
            for e in ex:  # prefetch also protects the step still computing (cap 6 >= two steps of <= 3 experts)
                trace.append(l * E + e)
                prot.append(prev if prefetch else start)
            prev = start
    st = OffloadedStack([tuple(w.pin_memory() for w in ly) for ly in layers], cap, policy, DEV)
    outs, stats = st.run(batches, prefetch=prefetch)
    torch.cuda.synchronize()
    for y, r in zip(outs, refs):
        assert torch.equal(y, r)
    hits, misses, _ = ocache.simulate(trace, cap, policy, protect_since=prot)
    assert (stats["hits"], stats["misses"]) == (hits, misses)


# ---- NEXT-1, incremental: the router over a key/value cache (decode) ----------------------------------

def test_router_step_token_by_token_matches_oracle(rd):
    """Requests advance one token per call (interleaved, ragged lengths) through readme_router_step; every
    logit row matches the fp64 oracle (bf16 rule) and the prefill path within the same bound, and decisions
    follow the near-tie rule of test_router_forward_parity (reading Q16)."""
    from oracle import router
    vocab, N = 32000, 8
    W = {k: synth.to_torch(v, "bf16") for k, v in synth.router_weights(vocab=vocab, n_experts=N, seed=195).items()}
    Wd = {k: v.to(DEV) for k, v in W.items()}
    lens = [1, 70, 33, 129]
    starts = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids = synth.token_ids(int(starts[-1]), vocab=vocab, seed=196)
    cache = rd.new_router_cache(len(lens), 256, DEV)
    got = np.zeros((int(starts[-1]), N))
    status = torch.zeros(1, dtype=torch.int32, device=DEV)
    for step in range(max(lens)):
        live = [r for r in range(len(lens)) if step < lens[r]]
        tok = torch.tensor([ids[starts[r] + step] for r in live], dtype=torch.int32, device=DEV)
        sl = torch.tensor(live, dtype=torch.int32, device=DEV)
        ps = torch.full((len(live),), step, dtype=torch.int32, device=DEV)
        lg = rd.router_step(tok, sl, ps, cache, Wd, dev_status=status)
        got[[starts[r] + step for r in live]] = _np(lg)
    assert int(status.item()) == 0
    ref = router.forward(ids, starts, W)
    assert rel_err(got, ref) <= BF16_TOL
    pre = _np(rd.router_forward(torch.from_numpy(ids).to(DEV), torch.from_numpy(starts).to(DEV), Wd))
    assert rel_err(got, pre) <= BF16_TOL
    band = 4.0 * np.max(np.abs(got - ref))
    top = np.sort(ref, axis=1)
    clear = (top[:, -1] - top[:, -2]) > band
    assert np.array_equal(got.argmax(axis=1)[clear], ref.argmax(axis=1)[clear])


def test_router_step_chunk_equals_token_by_token(rd):
    """Several tokens of one request in one call (a prefill chunk, any order) == one token per call, bitwise:
    all appends of a call precede its attention, and no kernel mixes rows."""
    vocab, N = 32000, 8
    Wd = {k: synth.to_torch(v, "bf16").to(DEV) for k, v in synth.router_weights(vocab=vocab, n_experts=N, seed=197).items()}
    n = 50
    ids = torch.from_numpy(synth.token_ids(n, vocab=vocab, seed=198)).to(DEV)
    c1, c2 = rd.new_router_cache(2, 64, DEV), rd.new_router_cache(2, 64, DEV)
    one = torch.cat([rd.router_step(ids[i:i + 1], torch.tensor([1], dtype=torch.int32, device=DEV),
                                    torch.tensor([i], dtype=torch.int32, device=DEV), c1, Wd) for i in range(n)])
    perm = torch.from_numpy(np.random.default_rng(5).permutation(n)).to(DEV)
    chunk = rd.router_step(ids[perm].contiguous(), torch.ones(n, dtype=torch.int32, device=DEV),
                           perm.to(torch.int32).contiguous(), c2, Wd)
    torch.cuda.synchronize()
    assert torch.equal(chunk, one[perm]) and torch.equal(c1, c2)


def test_router_step_bad_slot_flagged(rd):
    vocab, N = 1000, 4
    Wd = {k: synth.to_torch(v, "bf16").to(DEV) for k, v in synth.router_weights(vocab=vocab, n_experts=N, seed=199).items()}
    cache = rd.new_router_cache(2, 8, DEV)
    status = torch.zeros(1, dtype=torch.int32, device=DEV)
    rd.router_step(torch.tensor([1, 2], dtype=torch.int32, device=DEV), torch.tensor([0, 5], dtype=torch.int32, device=DEV),
                   torch.tensor([0, 0], dtype=torch.int32, device=DEV), cache, Wd, dev_status=status)
    torch.cuda.synchronize()
    assert int(status.item()) & rd.README_DEV_BAD_INDEX


def test_host_pipeline_equals_layer(rd):
    """Batches streamed from pinned host memory with overlapped H2D / layer / D2H give exactly the layer's
    output for every batch (double-buffered device buffers, event-ordered reuse)."""
    from paper_2410_19123_b200.pipeline import HostPipeline
    T, H, d, E, k = 700, 256, 256, 8, 1
    W = [synth.to_torch(w, "bf16").to(DEV) for w in synth.expert_weights(E, d, H, seed=301)]
    xs = [synth.to_torch(synth.tokens(T, H, seed=310 + i), "bf16").pin_memory() for i in range(5)]
    lgs = [torch.from_numpy(synth.router_logits(T, E, seed=320 + i)).pin_memory() for i in range(5)]
    ys = [torch.empty_like(x).pin_memory() for x in xs]
    HostPipeline(T, H, E, k, *W, device=DEV).run(xs, lgs, ys)
    torch.cuda.synchronize()
    for x, lg, y in zip(xs, lgs, ys):
        ref, _ = rd.moe_layer(x.to(DEV), *W, logits=lg.to(DEV))
        assert torch.equal(y, ref.cpu())
