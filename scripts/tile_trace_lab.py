"""Per-tile timeline of the single-launch expert FFN (readme_debug_tile_trace), measurement only.

Runs config-2-shaped moe_layer steps (graph replays, L2 flushed between them), records for every CTA pair
when each tile's MMAs were issued and when its accumulator was full / stored, and reports where the SM
cycles go: per tile kind the cycles between consecutive accumulator completions against the ideal MMA
cycles (8192 bf16 FLOP per SM cycle), the MMA warp's waits on loaded stages, and the spread of the pairs'
end times (the last wave). Env: TT_T (rows, 8192), TT_K (top-k, 1), TT_REPS (5).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_19123_b200 import readme as rd  # noqa: E402

T, H, E, d = int(os.environ.get("TT_T", "8192")), int(os.environ.get("TT_H", "4096")), 8, int(os.environ.get("TT_D", "5504"))
K = int(os.environ.get("TT_K", "1"))
REPS = int(os.environ.get("TT_REPS", "5"))
MAXT = 64
NREC = int(os.environ.get("TT_NREC", MAXT))  # per-tile records read (lab builds may use the rest of a pair's rows)
g = torch.Generator(device="cuda").manual_seed(1)
wg = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wu = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wd = (torch.randn(E, H, d, device="cuda", generator=g) / (d ** 0.5)).bfloat16()
x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
U = int(os.environ.get("TT_U", "0"))  # > 0: tokens spread evenly over experts 0..U-1 (decode studies)
if U > 0:
    lgn = np.full((T, E), -4.0, dtype=np.float32)
    lgn[np.arange(T), np.arange(T) % U] = 4.0
    lg = torch.from_numpy(lgn).cuda()
else:
    lg = torch.from_numpy(synth.router_logits(T, E)).cuda()
plan = rd.new_plan(T, E, K, "cuda")
ws = torch.empty(rd.moe_layer_workspace_bytes(T, H, E, d, K, torch.bfloat16), dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
NP = torch.cuda.get_device_properties(0).multi_processor_count // 2
tt = torch.zeros(NP * MAXT * 8, dtype=torch.int64, device="cuda")


def run():
    rd.moe_layer(x, wg, wu, wd, k=K, logits=lg, plan=plan, out=y, ws=ws)


flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd.lib().readme_debug_tile_trace(tt.data_ptr(), MAXT)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        run()
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=s):
    run()
offs = plan.offsets.cpu().numpy().astype(np.int64)

# tile list (python restatement of decode_ltile's order: 256-row m-tiles, tails of <= 64 rows merged into full
# m-tiles when the remainder fits, else their own tile; MERGE=0 restates the separate swap-AB tails)
MERGE = int(os.environ.get("README_FFN_MERGE", "1"))
NT1, NT2 = (d + 127) // 128, (H + 255) // 256
KB1, KB2 = (H + 63) // 64, (d + 63) // 64


def seg_tiles(R):
    if not MERGE or R < 256:
        return [(min(256, R - 256 * m), 0) for m in range((R + 255) // 256)]
    nf, rem = R >> 8, R & 255
    if rem == 0 or rem > 64 * min(nf, 2):
        return [(min(256, R - 256 * m), 0) for m in range(nf + (1 if rem else 0))]
    return [(256, min(64, rem - 64 * m) if m * 64 < rem else 0) for m in range(nf)]


def mma_cyc(rows, trows):
    if rows <= 64:
        c, kind = 128 * ((rows + 15) // 16 * 16) / 256, "swap"
    elif rows > 128:
        c, kind = 128, "m256"
    else:
        c, kind = 64, "m128"
    if trows:
        c, kind = c + 128 * ((trows + 15) // 16 * 16) / 256, "m256+tail"
    return c, kind


kinds = []
for ph in (0, 1):
    NT, KB = (NT1, KB1) if ph == 0 else (NT2, KB2)
    for gi in range(len(offs) - 1):
        tiles = seg_tiles(int(offs[gi + 1] - offs[gi]))
        for n in range(NT):
            for rows, trows in tiles:
                c, kind = mma_cyc(rows, trows)
                kinds.append((ph, kind, KB * 4 * c))

res = []
for it in range(REPS):
    tt.zero_()
    flush.fill_(it)
    flush.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    gr.replay()
    b.record()
    torch.cuda.synchronize()
    rec = tt.view(NP, MAXT, 8).cpu().numpy().astype(np.uint64).astype(np.float64)
    per_kind = {}
    ends, starts, busy_ideal, full_wait, acc_wait, span_cyc, ideal_pair = [], [], 0.0, 0.0, 0.0, [], []
    for p in range(NP):
        r = rec[p]
        n = int((r[:NREC, 1] > 0).sum())
        if n == 0:
            continue
        prev = None
        for i in range(n):
            t = int(r[i, 7]) & 0xFFFFFFFF
            ph, kind, ideal = kinds[t]
            c1, c3 = r[i, 1], r[i, 3]
            start = c1 if prev is None else max(prev, c1)
            ex = c3 - start
            key = f"{'gu' if ph == 0 else 'dn'}_{kind}"
            e = per_kind.setdefault(key, [0, 0.0, 0.0, 0.0])
            e[0] += 1
            e[1] += ex
            e[2] += ideal
            e[3] += r[i, 6]
            busy_ideal += ideal
            full_wait += r[i, 6]
            acc_wait += (int(r[i, 7]) >> 32)
            prev = c3
        ideal_pair.append(sum(kinds[int(r[i, 7]) & 0xFFFFFFFF][2] for i in range(n)))
        starts.append(r[0, 0])
        ends.append(r[n - 1, 5])
        span_cyc.append(r[n - 1, 4] - r[0, 1])
    t0 = min(starts)
    ends_us = (np.array(ends) - t0) / 1e3
    res.append({
        "event_us": a.elapsed_time(b) * 1e3,
        "pairs": len(ends),
        "end_us": {"min": float(ends_us.min()), "mean": float(ends_us.mean()), "max": float(ends_us.max())},
        "span_cycles_mean": float(np.mean(span_cyc)), "span_cycles_max": float(np.max(span_cyc)),
        "ideal_cycles_per_pair": busy_ideal / len(ends),
        "ideal_pair_max": float(np.max(ideal_pair)), "ideal_pair_min": float(np.min(ideal_pair)),
        "ntiles_pair": [int((rec[p][:NREC, 1] > 0).sum()) for p in range(NP)],
        "ideal_over_max_span": busy_ideal / len(ends) / float(np.max(span_cyc)),
        "clock_ghz_est": float(np.mean(span_cyc)) / (float(np.mean(np.array(ends) - np.array(starts)))),
        "kinds": {k: {"n": v[0], "exec_cyc": v[1] / v[0], "ideal_cyc": v[2] / v[0], "eff": v[2] / v[1],
                      "full_wait_cyc": v[3] / v[0]} for k, v in sorted(per_kind.items())},
    })
rd.lib().readme_debug_tile_trace(None, 0)
out = {"T": T, "H": H, "d": d, "k": K, "counts": np.diff(offs).tolist(), "runs": res}
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/tile_trace_last.npy", tt.view(NP, MAXT, 8).cpu().numpy())
print(json.dumps(out, indent=1))
