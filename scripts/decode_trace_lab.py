"""Per-tile timeline of a decode-sized expert FFN launch (readme_expert_ffn) at B tokens over U experts, from
the kernel's tile trace (readme_debug_tile_trace). Measurement only.
Usage: python scripts/decode_trace_lab.py B U [knob=v:knob=v]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_19123_b200 import readme as rd  # noqa: E402

B, U = int(sys.argv[1]), int(sys.argv[2])
for kv in (sys.argv[3].split(":") if len(sys.argv) > 3 and sys.argv[3] else []):
    rd.set_knob(kv.split("=")[0], int(kv.split("=")[1]))
H, E, d = 4096, 8, 5504
MAXT = 64
g = torch.Generator(device="cuda").manual_seed(1)
wg = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wu = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wd = (torch.randn(E, H, d, device="cuda", generator=g) / 74).bfloat16()
x = torch.randn(B, H, device="cuda", generator=g).bfloat16()
lg = np.full((B, E), -4.0, dtype=np.float32)
lg[np.arange(B), np.arange(B) % U] = 4.0
plan = rd.route(torch.from_numpy(lg).cuda(), 1)
xs = rd.dispatch(x, plan.dest, 1)
ys = torch.empty_like(xs)
ws = torch.empty(rd.expert_ffn_workspace_bytes(B, H, E, d, torch.bfloat16), dtype=torch.uint8, device="cuda")
NP = torch.cuda.get_device_properties(0).multi_processor_count // 2
tt = torch.zeros(NP * MAXT * 8, dtype=torch.int64, device="cuda")
rd.lib().readme_debug_tile_trace(tt.data_ptr(), MAXT)
fn = lambda: rd.expert_ffn(xs, plan.offsets, wg, wu, wd, out=ys, ws=ws)
for _ in range(3):
    fn()
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
counts = plan.counts.cpu().tolist()
mt = 128 if B <= 1024 else 256
n_m = sum((c + mt - 1) // mt for c in counts)
n_gu = n_m * ((d + 127) // 128)
out = []
for it in range(3):
    tt.zero_()
    flush.fill_(it)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    rec = tt.view(NP, MAXT, 8).cpu().numpy().astype(np.uint64)
    rows = []
    for p in range(NP):
        for i in range(MAXT):
            r = rec[p, i]
            if r[1] == 0:
                break
            t = int(r[7]) & 0xFFFFFFFF
            rows.append((p, t, int(r[0]), int(r[5]), int(r[6]), int(r[3] - r[1]), int(r[4] - r[3])))
    t0 = min(r[2] for r in rows)
    gu = [r for r in rows if r[1] < n_gu]
    dn = [r for r in rows if r[1] >= n_gu]
    f = lambda v: round(v / 1e3, 2)
    out.append({
        "event_us": round(a.elapsed_time(b) * 1e3, 1),
        "pairs_used": len({r[0] for r in rows}), "gu_tiles": len(gu), "dn_tiles": len(dn),
        "gu_start_us_min_max": [f(min(r[2] for r in gu) - t0), f(max(r[2] for r in gu) - t0)],
        "gu_end_us_min_max": [f(min(r[3] for r in gu) - t0), f(max(r[3] for r in gu) - t0)],
        "dn_start_us_min_max": [f(min(r[2] for r in dn) - t0), f(max(r[2] for r in dn) - t0)] if dn else None,
        "dn_end_us_min_max": [f(min(r[3] for r in dn) - t0), f(max(r[3] for r in dn) - t0)] if dn else None,
        "gu_tile_us_mean": f(np.mean([r[3] - r[2] for r in gu])),
        "dn_tile_us_mean": f(np.mean([r[3] - r[2] for r in dn])) if dn else None,
        "gu_fullwait_frac": round(float(np.mean([r[4] / max(1, r[5]) for r in gu])), 3),
        "dn_fullwait_frac": round(float(np.mean([r[4] / max(1, r[5]) for r in dn])), 3) if dn else None,
        "dn_tiles_per_pair_max": max(np.bincount([r[0] for r in dn])) if dn else 0,
        "gu_tiles_per_pair_max": int(max(np.bincount([r[0] for r in gu]))),
    })
print(json.dumps({"B": B, "U": U, "counts": counts, "mt": mt, "runs": out}, default=int))
