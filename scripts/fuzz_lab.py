"""Extended shape fuzz of readme_moe_layer against the oracle (many seeded random (T, E, k, H, d, dtype)
cases through the default paths). Measurement/validation only; prints failures."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2410_19123_b200 import readme as rd  # noqa: E402
from tests.tolerances import BF16_TOL, F32_TOL, rel_err  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 777)
fails = 0
for c in range(n):
    dt = "bf16" if g.random() < 0.8 else "f32"
    E = int(g.integers(1, 33))
    k = int(g.integers(1, min(E, 4) + 1))
    T = int(g.integers(1, 4097))
    H = int(8 * g.integers(4, 129))
    d = int(8 * g.integers(2, 97))
    res_on = bool(g.random() < 0.5)
    x = synth.to_torch(synth.tokens(T, H, seed=c), dt)
    lg = synth.router_logits(T, E, seed=c) if g.random() < 0.7 else synth.logits_for_assignments(
        synth.assignments_zipf(T, E, 2.0, seed=c), E, seed=c)
    wg, wu, wd = (synth.to_torch(w, dt) for w in synth.expert_weights(E, d, H, seed=c))
    res = synth.to_torch(synth.residual(T, H, seed=c + 1), dt) if res_on else None
    try:
        y, plan = rd.moe_layer(x.cuda(), wg.cuda(), wu.cuda(), wd.cuda(), k=k, logits=torch.from_numpy(lg).cuda(),
                               residual=res.cuda() if res is not None else None)
        torch.cuda.synchronize()
        yref, pref = oracle.moe_layer(x, lg, k, wg, wu, wd, residual=res)
        ok_plan = all(np.array_equal(getattr(plan, nm).cpu().numpy(), pref[nm])
                      for nm in ("topk_idx", "counts", "offsets", "dest", "src"))
        yy = y.float().cpu().numpy() if dt == "bf16" else y.cpu().numpy()
        err = rel_err(yy, yref)
        tol = BF16_TOL if dt == "bf16" else F32_TOL
        st = int(plan.dev_status.item())
        if not ok_plan or err > tol or st != 0:
            fails += 1
            print(f"FAIL case {c}: dt={dt} T={T} E={E} k={k} H={H} d={d} res={res_on} plan_ok={ok_plan} err={err:.3e} "
                  f"status={st}")
    except Exception as ex:  # noqa: BLE001
        fails += 1
        print(f"ERROR case {c}: dt={dt} T={T} E={E} k={k} H={H} d={d}: {type(ex).__name__}: {ex}")
print(f"{n - fails}/{n} cases passed")
