"""Summarise the ncu --set full captures of tools/prof_all.sh (gpurun_out/ncu_<tag>.ncu-rep) into
profiles/ncu_summary.json: per kernel the duration, DRAM bytes against the algorithmic bytes, DRAM /
SM throughput, achieved occupancy, registers, issue-slot use, pipe utilisation (FP64, FMA/IMAD, ALU,
LSU ...), L2 hit rate, top warp-stall reasons and the instruction count.  bench.py reads the per-launch
DRAM traffic of the dominant kernel from it.

    python tools/ncu_summarize.py [gpurun_out] [profiles/ncu_summary.json]
"""

import csv
import io
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

# algorithmic bytes per launch (8-byte residues): what the kernel must read + write at minimum
N14, N15 = 1 << 14, 1 << 15
ALG = {
    "ts_onepass": 4 * 64 * 5 * N14 * 8 + 3 * 5 * N14 * 8,  # 128 cts both polys + (d0, d1, d2)
    "ts_d01": 4 * 64 * 5 * N14 * 8 + 2 * 5 * N14 * 8,
    "ts_d2": 2 * 64 * 5 * N14 * 8 + 1 * 5 * N14 * 8,
    "ts_cfg5a": (4 * 256 + 256) * 2 * 8 * N15 * 8 + 4 * 3 * 8 * N15 * 8,
    "ntt_cl8_fwd": 2 * 256 * 5 * N14 * 8,  # in place: read + write every limb
    "ts_many_cfg1": 32 * (4 * 8 * 2 * (1 << 13) * 8 + 3 * 2 * (1 << 13) * 8),  # 32 products of 16 cts + their (d0, d1, d2)
}
NOTES = {
    "ts_onepass": "config 2 one-pass (d0, d1, d2) tensor sum, the dominant kernel of the asynchronous step (multicipher.py:88-103)",
    "ts_d01": "config 2 (d0, d1) tensor sum of the synchronous schedule (VR_ASYNC=0)",
    "ts_d2": "config 2 d2 tensor sum of the synchronous schedule",
    "ts_cfg5a": "config 5a four-row-block tensor sum, row blocks interleaved so CTAs sharing R tiles run together (L2 reuse)",
    "modup_ntt": "relinearisation ModUp lift + NTT (cluster kernel, 8 CTAs per transform), config 2 (engine.py:215-220)",
    "modup_intt": "relinearisation ModUp INTT of the d2 digits (cluster kernel), config 2",
    "ks_inner_cfg2": "key-switch inner product with the relinearisation key, config 2",
    "moddown_store": "ModDown + rescale fused store pass (StRelinRescale), config 2",
    "ntt_cl8_fwd": "forward NTT, N = 2^14, 1280 limbs (4 of 5 primes on the FP64 body): the bench NTT line",
    "ntt_pass_fwd_n15": "forward NTT N = 2^15 column pass (two-pass path), 2048 limbs",
    "ntt_pass_rows_n15": "forward NTT N = 2^15 row pass",
    "conv_mac": "conv_columns tap MAC over channels x taps x filters (multicipher.py:150-161), config 4",
    "ks_inner_cfg4": "hoisted-rotation key-switch inner product, config 4 (l = 8)",
    "lift_ntt_cfg4": "rotation ModUp lift + NTT column pass, config 4",
    "pt_matvec": "plaintext dense layer 845 -> 64 (config 3)",
    "enc_ntt": "fused secret-key encryption through the cluster NTT (sampler + NTT(m+e) - a s), config 2 encode_left (engine.py:193-202)",
    "encode": "slot FFT encode + Gaussian noise, 64 ciphertexts (config 2)",
    "decode": "slot FFT decode (engine.py:204-206)",
    "ts_many_cfg1": "matmul_outer_many tensor sum: 32 independent config-1 products in one launch (a right operand per product)",
}
WANT = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_of_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers_per_thread": "launch__registers_per_thread",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warp_instructions": "smsp__inst_executed.sum",
    "l2_hit_rate_pct": "lts__t_sector_hit_rate.pct",
    "l1_hit_rate_pct": "l1tex__t_sector_hit_rate.pct",
    "lsu_data_pipe_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
    "cluster_size": "launch__cluster_dim_x",
}


def num(v):
    try:
        return float(v.replace(",", ""))
    except (AttributeError, ValueError):
        return None


def summarize(rep: Path) -> dict:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    d = dict(zip(hdr, rows[2]))  # first profiled launch (row 1 holds units)
    out = {"kernel": d.get("Kernel Name", "")[:160]}
    for k, m in WANT.items():
        out[k] = num(d.get(m))
    if out["duration_ns"]:
        out["duration_us_under_ncu"] = out.pop("duration_ns") / 1e3
    rd, wr = out.get("dram_read_bytes") or 0.0, out.get("dram_write_bytes") or 0.0
    out["dram_bytes_per_launch"] = rd + wr
    pipes = {}
    for k, v in d.items():
        m = re.fullmatch(r"sm__(?:pipe_(\w+?)_cycles_active|inst_executed_pipe_(\w+?))\.avg\.pct_of_peak_sustained_active", k)
        if m and num(v) is not None and num(v) > 0.5:
            name = ("cycles_" + m.group(1)) if m.group(1) else ("inst_" + m.group(2))
            pipes[name] = round(num(v), 2)
    out["pipe_utilisation_pct"] = dict(sorted(pipes.items(), key=lambda kv: -kv[1])[:10])
    stalls = {}
    for k, v in d.items():
        m = re.fullmatch(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", k)
        if m and num(v):
            stalls[m.group(1)] = round(num(v), 3)
    out["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
    return out


def main():
    src = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "gpurun_out"
    dst = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "profiles" / "ncu_summary.json"
    res = {"round": 2, "source": "tools/prof_all.sh: ncu --set full --clock-control none, one launch per kernel after a "
                                 "warm-up launch (cold-cache, serialised; durations are ncu's, not bench values)",
           "units": "bytes per launch, percent of peak", "kernels": {}}
    for rep in sorted(src.glob("ncu_*.ncu-rep")):
        tag = rep.stem[len("ncu_"):]
        try:
            s = summarize(rep)
        except (subprocess.CalledProcessError, IndexError) as exc:
            print(f"skip {rep}: {exc}", file=sys.stderr)
            continue
        s["what"] = NOTES.get(tag, "")
        if tag in ALG:
            s["algorithmic_bytes_per_launch"] = ALG[tag]
            s["dram_over_algorithmic"] = round(s["dram_bytes_per_launch"] / ALG[tag], 3)
            if s.get("duration_us_under_ncu"):
                s["algorithmic_gbs_under_ncu"] = round(ALG[tag] / s["duration_us_under_ncu"] / 1e3, 1)
        res["kernels"][tag] = s
    # bench.py keys
    for tag, key in (("ts_onepass", "k_tensor_sum_d012"), ("ts_d01", "k_tensor_sum_d01"), ("ts_d2", "k_tensor_sum_d2")):
        if tag in res["kernels"]:
            res["kernels"][key] = {"alias_of": tag, "dram_bytes_per_launch": res["kernels"][tag]["dram_bytes_per_launch"]}
    dst.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1)[:4000])


if __name__ == "__main__":
    main()
