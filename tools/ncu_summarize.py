"""Summarise the k_tensor_sum ncu --set full capture (gpurun_out/prof_ts.ncu-rep) into
profiles/ncu_summary.json (bench.py reads the per-launch DRAM traffic from it)."""
import csv, io, json, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
rep = sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "gpurun_out" / "prof_ts.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]


def f(d, k):
    try:
        return float(d[k])
    except (KeyError, ValueError):
        return None


out = {"round": 1, "source": "ncu --set full --clock-control none -k regex:k_tensor_sum; python tools/step_profile.py --cfg 2 --steps 2",
       "units": "bytes per launch", "kernels": {}}
N, nl, n = 16384, 5, 64
for row in rows[2:]:
    d = dict(zip(hdr, row))
    name = d["Kernel Name"]
    mode = 2 if "1, 2>" in name or ", 2>" in name.split("k_tensor_sum")[-1] else 1
    key = "k_tensor_sum_d01" if mode == 2 else "k_tensor_sum_d2"
    if key in out["kernels"]:
        continue
    rd, wr = f(d, "dram__bytes_read.sum"), f(d, "dram__bytes_write.sum")
    alg = (4 if mode == 2 else 2) * n * nl * N * 8 + (2 if mode == 2 else 1) * nl * N * 8
    out["kernels"][key] = {
        "kernel": name[:120], "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
        "duration_us_under_ncu": f(d, "gpu__time_duration.sum") / 1e3,  # base unit: ns
        "dram_pct_of_peak": f(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_active_pct": f(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers_per_thread": f(d, "launch__registers_per_thread"), "algorithmic_bytes_per_launch": alg}
out_path = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "profiles" / "ncu_summary.json"
out_path.write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
