import json
import sys

d = json.loads(open(sys.argv[1]).readline())
print(round(d["value"]), round(d["roofline"]["frac"], 3), d["stage_ms_mean"], d["clocks"])
print("router_step", d["router_step"])
print([(p["B"], round(p["ms"] * 1000, 1), round(p["hbm_frac"], 3)) for p in d["decode_sweep"]])
