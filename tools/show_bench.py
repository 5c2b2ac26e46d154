"""Compact view of a bench.py JSON line (headline, roofline, e2e, ntt, per-config values)."""
import json, sys
for line in open(sys.argv[1]):
    if not line.startswith("{"): continue
    d = json.loads(line)
    print("value", round(d["value"], 1), d["unit"], "ms/step", round(d["ms_per_step"], 4))
    if "roofline" in d: print("roofline", {k: d["roofline"][k] for k in ("achieved", "frac", "launch_us")})
    if "e2e" in d: print("e2e", round(d["e2e"]["value"], 1))
    if "ntt" in d: print("ntt", d["ntt"]["us_per_limb"], d["ntt"]["int_roofline"]["frac"])
    for k, v in d.get("configs", {}).items():
        print(" ", k, round(v["value"], 2), {kk: vv for kk, vv in v.items() if kk.startswith("e2e_images")})
