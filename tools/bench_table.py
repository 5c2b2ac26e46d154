"""One-screen summary of bench.py JSON lines: headline, e2e, roofline, CPU legs, every config."""
import json, sys
for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if d.get("impl") == "reference":
            print(f"{path}: reference arm {d['value']:.1f} {d['unit']} ({d['cpu_baseline']['cores']} cores); "
                  f"simulator {d['reference_simulator']['value']:.0f}/s")
            continue
        rf = d.get("roofline", {})
        print(f"{path}: value {d['value']:.0f} ({d['ms_per_step'] * 1e3:.1f} us/step, steps {d['steps']}) e2e {d['e2e']['value']:.0f} "
              f"launches/step {d.get('gpu_launches_per_step')} clocks {d.get('clocks', {}).get('sm_mhz')}")
        if rf:
            st = rf.get("step", {})
            print(f"  dominant kernel {rf['kernel']}: {rf['achieved']:.0f} GB/s frac {rf['frac']:.3f} ({rf['launch_us']:.1f} us); "
                  f"step frac {st.get('frac', 0):.3f} (hbm {st.get('hbm_frac', 0):.3f} int {st.get('int_frac', 0):.3f})")
        cb = d.get("cpu_baseline") or {}
        print(f"  cpu_baseline {cb.get('value')} ({cb.get('cores')} cores)")
        for k, v in d.get("configs", {}).items():
            r = v.get("roofline") or {}
            c = v.get("cpu_baseline") or {}
            sim = v.get("reference_simulator") or {}
            e2e = v.get("e2e") or {}
            print(f"  {k:11s} {v['value']:10.1f}  roofline {r.get('bound', '-'):3s} {r.get('frac', 0):.3f} (hbm {r.get('hbm_frac', 0):.3f} "
                  f"int {r.get('int_frac', 0):.3f})  cpu {c.get('value') or 0:.2f}  sim {sim.get('value') or 0:.1f}  e2e {e2e.get('value') or 0:.1f}")
        if "ntt" in d:
            n = d["ntt"]
            print(f"  ntt {n['us_per_limb']:.3f} us/limb, {n['gbs']:.0f} GB/s, int frac {n['int_roofline']['frac']:.3f}")
