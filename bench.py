#!/usr/bin/env python
"""Benchmark: HE matmul/s of the column-ciphertext matmul (BASELINE.json config 2)
on B200, plus NTT GB/s and the CPU baselines.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one HE matmul A(64x64)*B(64x64): matmul_outer over n = 64 resident
column-ciphertext pairs (N = 2^14, 5 ciphertext primes + 60-bit special prime,
scale 2^40, seed 1) = fused tensor-sum + one relinearisation + one rescale.
Under torchrun every rank runs independent HE matmuls (weak scaling) and
`value` is the whole-job throughput, timed on the device as the max over ranks.

`e2e` is the same metric through the public API with host buffers: every step
uploads A and B from pinned host memory, encrypts the 128 column ciphertexts
(encode_left/encode_right), runs matmul_outer and downloads the decoded result.

`--impl reference` times the CPU restatement of the same path (oracle/, real
RNS-CKKS in C + OpenMP) on rank 0 only; the reference package itself is a
float64 simulator with no cryptography and is reported as
`reference_simulator` beside it.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "HE matmul/s (column-ciphertext matmul_outer, BASELINE config 2: A,B 64x64, n=64 cts/operand, N=2^14)"
UNIT = "HE matmul/s"
CFG = 2
DIM = 64


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-extra", action="store_true", help="skip the NTT/config-1 side measurements")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def inputs(cfg=CFG, dim=DIM):
    rng = np.random.default_rng(cfg - 1)  # BASELINE.json: config c uses seed c-1
    a = rng.uniform(-1, 1, (dim, dim))
    b = rng.uniform(-1, 1, (dim, dim))
    return a, b


# ---------------------------------------------------------------------------
# clocks sampled DURING the timed region
class ClockSampler:
    """NVML sampling thread (no subprocess fork inside the timed region): SM clock and throttle reasons."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index: int, period: float = 0.01):
        self.index = index
        self.period = period
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
            self.max_mhz = None

    def _sample(self):
        nv = self._nv
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        self.samples.append((sm, reasons))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self._nv is not None and not os.environ.get("VR_BENCH_NO_NVML"):
            self._sample()  # first sample before the timed region starts
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        reasons = sorted({nm for _, r in self.samples for nm, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str):
    """dram bytes per launch from the committed ncu --set full summary, if present."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    v = d.get("kernels", {}).get(kernel, {})
    return v.get("dram_bytes_per_launch")


# ---------------------------------------------------------------------------
def cpu_port_matmul(cfg=CFG, dim=DIM, reps=1):
    """Time the CPU residue oracle (C + OpenMP) on HE matmuls of the same workload."""
    from oracle.engine import OracleEngine
    from paper_2512_18646_b200.params import config_params

    p = config_params(cfg)
    e = OracleEngine.from_params(p)
    a, b = inputs(cfg, dim)
    L = [e.enc(np.repeat(a[:, k], dim)) for k in range(dim)]
    R = [e.enc(np.tile(b[k, :], dim)) for k in range(dim)]
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = e.matmul_outer_blocks([L], R)[0]
        times.append(time.perf_counter() - t0)
    got = e.dec(out)[: dim * dim].reshape(dim, dim)
    err = float(np.max(np.abs(got - a @ b)))
    return times, err


def simulator_matmul(cfg=CFG, dim=DIM, reps=20):
    """Time the reference algorithm (float64 slot simulator, numpy restatement)."""
    from oracle import sim

    a, b = inputs(cfg, dim)
    slots = {1: 4096, 2: 8192}[cfg]
    eng = sim.SimEngine(slots)
    L, R = sim.encode_left(eng, a, dim), sim.encode_right(eng, b, dim)
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        sim.matmul_outer(eng, L, R, dim, dim)
        t.append(time.perf_counter() - t0)
    return min(t)


def run_reference(args, ws, rank):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_port_matmul(reps=1)
    times, err = cpu_port_matmul(reps=args.steps)
    per = statistics.mean(times)
    v = 1.0 / per
    sim_t = simulator_matmul()
    line = {
        "impl": "reference",
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seed 1, U[-1,1])",
        "config": {"workload": "cfg2 HE matmul 64x64 (n=64 column ciphertexts), N=2^14, 5 primes + P"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{args.steps} cfg-2 HE matmuls (matmul_outer on resident ciphertexts) in the C RNS-CKKS oracle, OpenMP over (limb, coefficient chunk) work items and key-switch target primes",
                         "max_abs_err": err},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_simulator": {"value": 1.0 / sim_t, "unit": UNIT, "cores": 1,
                                "note": "reference algorithm as an exact float64 slot simulator (no cryptography)"},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_ours(args, ws, rank, local):
    import torch

    from paper_2512_18646_b200 import _lib
    from paper_2512_18646_b200 import CkksEngine, encode_left, encode_right, matmul_outer
    from paper_2512_18646_b200.params import config_params

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    eng = CkksEngine(config_params(CFG), device=local)
    lib = eng._lib
    stream = eng._stream
    a, b = inputs()
    left = encode_left(eng, a, DIM)
    right = encode_right(eng, b, DIM)
    # correctness gate before timing
    first = matmul_outer(eng, left, right)
    err = float(np.max(np.abs(first.decode(eng) - a @ b)))
    assert err < 1e-3, f"HE matmul error {err}"

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # setup: let clocks, allocator pools and pointer-table caches settle (untimed)
    # the warm-up loops hold the previous result exactly like the timed loop, so the allocator has
    # both output buffers before timing starts (the first second buffer cost one cudaMalloc: ~90 ms)
    t_settle = time.perf_counter()
    out = None
    while time.perf_counter() - t_settle < 0.25:
        out = matmul_outer(eng, left, right)
        torch.cuda.synchronize()
    for _ in range(args.warmup):
        out = matmul_outer(eng, left, right)
    barrier()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = lib.vr_launch_count()
    chunks = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if os.environ.get("VR_BENCH_CHUNKS") else None
    # no Python garbage-collection pauses inside the timed regions (as timeit does): a gen-2
    # collection stalled the host for up to ~25 ms and starved the device in some runs
    gc.collect()
    gc.disable()
    with ClockSampler(local) as clk:
        st.record(stream)
        slow = []
        for i in range(args.steps):
            if chunks is not None and i % max(1, args.steps // 4) == 0 and i // max(1, args.steps // 4) < 4:
                chunks[i // max(1, args.steps // 4)].record(stream)
            hc = time.perf_counter()
            out = matmul_outer(eng, left, right)
            if chunks is not None and time.perf_counter() - hc > 1e-3:
                slow.append((i, round((time.perf_counter() - hc) * 1e3, 2)))
        en.record(stream)
        torch.cuda.synchronize()
    if chunks is not None:
        chunks[4] = en
        print("chunk ms:", [round(chunks[j].elapsed_time(chunks[j + 1]), 3) for j in range(4)], "slow host calls:", slow,
              file=sys.stderr)
    launches = lib.vr_launch_count() - l0
    gc.enable()
    barrier()
    step_s = max_over_ranks(st.elapsed_time(en) / 1e3 / args.steps)
    value = ws / step_s

    # dominant kernel: the (d0, d1) tensor-sum the step runs beside the d2 key switch, timed alone
    # on the same stream (mode 2 reads all 2n column ciphertexts; mode 1 reads only their c1 halves)
    nl = eng.L + 1
    ptrsL = _lib.ptr_array([c.ptr() for c in left.cts])
    ptrsR = _lib.ptr_array([c.ptr() for c in right.cts])
    d3 = torch.empty((3, nl, eng.N), dtype=torch.int64, device="cuda")
    for _ in range(3):
        _lib.check(lib.vr_tensor_sum_mode(eng.handle, ptrsL, ptrsR, DIM, eng.L, d3.data_ptr(), 2))
    reps = max(args.steps, 20)
    torch.cuda.synchronize()
    st.record(stream)
    for _ in range(reps):
        _lib.check(lib.vr_tensor_sum_mode(eng.handle, ptrsL, ptrsR, DIM, eng.L, d3.data_ptr(), 2))
    en.record(stream)
    torch.cuda.synchronize()
    ts_s = st.elapsed_time(en) / 1e3 / reps
    alg_bytes = DIM * 4 * nl * eng.N * 8 + 2 * nl * eng.N * 8
    peak, peak_src = peaks()
    achieved = alg_bytes / ts_s / 1e9

    # e2e through the public API with host buffers
    pin_a = torch.from_numpy(a).pin_memory()
    pin_b = torch.from_numpy(b).pin_memory()
    e2e_steps = max(3, min(50, args.steps // 4))
    res = None
    t_settle = time.perf_counter()
    while time.perf_counter() - t_settle < 0.25:  # same statement as the timed loop
        res = matmul_outer(eng, encode_left(eng, pin_a.numpy(), DIM), encode_right(eng, pin_b.numpy(), DIM)).decode(eng)
    barrier()
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()
    t0 = time.perf_counter()
    st.record(stream)
    for _ in range(e2e_steps):
        res = matmul_outer(eng, encode_left(eng, pin_a.numpy(), DIM), encode_right(eng, pin_b.numpy(), DIM)).decode(eng)
    en.record(stream)
    torch.cuda.synchronize()
    gc.enable()
    e2e_s = max_over_ranks(max(st.elapsed_time(en) / 1e3, time.perf_counter() - t0) / e2e_steps)
    h2d = 2 * DIM * DIM * 8  # the raw A and B (broadcast/tiling happens in the encode kernel)
    d2h = eng.slots * 8

    extra = {}
    cfg5 = {}
    if not args.no_extra:
        del left, right, first, out
        cfg5["cfg5a"] = bench_cfg5a(ws, rank, local, max_over_ranks, barrier)
        cfg5["cfg5b"] = bench_cfg5b(ws, rank, local, max_over_ranks, barrier)
    if not args.no_extra and rank == 0:
        extra["ntt"] = bench_ntt(eng, peak)
        extra["configs"] = {"cfg1": bench_cfg1(), "cfg2_alg3": bench_cfg2_alg3(), "table1_cnn": bench_table1(), "cfg3": bench_cfg3(), "cfg4": bench_cfg4(steps=3), **cfg5}
    line = None
    if rank == 0:
        cpu = None
        try:
            times, cerr = cpu_port_matmul(reps=2)
            cv = 1.0 / statistics.median(times)
            cpu = {"value": cv, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
                   "sample": "2 cfg-2 HE matmuls (matmul_outer on resident ciphertexts) in the C RNS-CKKS oracle, OpenMP over (limb, coefficient chunk) work items and key-switch target primes",
                   "max_abs_err": cerr}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port", "sample": f"failed: {exc}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64", "data": "synthetic (seed 1, U[-1,1]); inputs larger than L2 (128 cts = 168 MB)",
            "config": {"workload": "cfg2 HE matmul 64x64 (n=64 column ciphertexts/operand), N=2^14, q0 60b + 4x40b + P 60b, scale 2^40",
                       "parallelism": f"replicas x{ws}", "l2": "inputs larger than L2"},
            "max_abs_err": err,
            "roofline": {"bound": "hbm", "kernel": "k_tensor_sum<MODE=2> (d0,d1)", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic("k_tensor_sum_d01"),
                         "alg_bytes_per_launch": alg_bytes, "launch_us": ts_s * 1e6, "step_share": ts_s / step_s,
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": {"value": ws / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": "encode_left+encode_right (encrypt 128 cts) -> matmul_outer -> decode"},
            "gpu_launches": int(launches),
            "gpu_launches_per_step": launches / args.steps,
            "clocks": clk.summary(),
            **extra,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def bench_cfg1(steps=50):
    """Config 1: HE matmul 8x8 (n = 8 column ciphertexts, N = 2^13), device time per matmul."""
    import torch

    from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer
    from tools.workloads import cfg_matmul

    a, b = cfg_matmul(1)
    eng = CkksEngine(config_params(1))
    left, right = encode_left(eng, a, 8), encode_right(eng, b, 8)
    err = float(np.max(np.abs(matmul_outer(eng, left, right).decode(eng) - a @ b)))
    for _ in range(3):
        matmul_outer(eng, left, right)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    st.record(eng._stream)
    for _ in range(steps):
        matmul_outer(eng, left, right)
    en.record(eng._stream)
    torch.cuda.synchronize()
    t = st.elapsed_time(en) / 1e3 / steps
    return {"metric": "HE matmul/s (cfg1 8x8, N=2^13)", "value": 1.0 / t, "ms_per_matmul": t * 1e3, "max_abs_err": err}


def bench_cfg2_alg3(steps=5):
    """Config 2, Algorithm 3 (revolver matmul, the rotation-heavy single-ciphertext product):
    A, B 64x64 padded to row width 128 so the 64x128 layout fills 8192 slots (fast path,
    depth 3).  64 hoisted rotations of B, 64 products, 64 x 14 cascade rotations, 128 cmuls."""
    import torch

    from paper_2512_18646_b200 import CkksEngine, config_params, encode_revolver, encode_row_major, matmul
    from tools.workloads import cfg_matmul

    a, b = cfg_matmul(2)
    eng = CkksEngine(config_params(2))
    ap = np.zeros((64, 128))
    ap[:, :64] = a
    bp = np.zeros((128, 64))
    bp[:64] = b
    ca, cb = encode_row_major(eng, ap), encode_revolver(eng, bp, target_m=64)
    err = float(np.max(np.abs(matmul(eng, ca, cb).decode(eng)[:, :64] - a @ b)))
    for _ in range(2):
        matmul(eng, ca, cb)
    before = eng.meter_snapshot()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    st.record(eng._stream)
    for _ in range(steps):
        matmul(eng, ca, cb)
    en.record(eng._stream)
    torch.cuda.synchronize()
    t = st.elapsed_time(en) / 1e3 / steps
    d = eng.meter_snapshot().delta_since(before)
    return {"metric": "HE matmul/s (cfg2 Algorithm 3 revolver, 64x64 at width 128, N=2^14)", "value": 1.0 / t,
            "ms_per_matmul": t * 1e3, "max_abs_err": err,
            "ops_per_matmul": {"rot": d.rot_count // steps, "mul": d.mul_count // steps, "cmul": d.cmul_count // steps,
                               "add": d.add_count // steps}}


def bench_table1(steps=3):
    """The paper's Table-1 encrypted CNN (pipeline.forward_encoded): 32 MNIST-sized images per
    32768-slot ciphertext, conv 4x3x3 -> act -> ReForm -> FC 2704->64 -> act -> FC 64->10, depth 13,
    N = 2^16 on q0 60b + 13 x 45b + P 60b.  Model encoded once; per batch: encrypt the images,
    forward, decode the scores.  Synthetic seeded images/weights in the reference suite's ranges."""
    import torch

    sys.path.insert(0, str(ROOT))
    from oracle.sim import table1_weights
    from paper_2512_18646_b200 import EngineParams, Kernel, ModelWeights, SlotEngine, encode_model, forward_encoded, pack_batch

    act1 = (-0.00015120704, 0.4610149, 2.0225089, -1.4511951)
    act2 = (-1.5650465, -0.9943767, 1.6794522, 0.5350255)
    kw, kb, f1w, f1b, f2w, f2b = table1_weights(7)
    weights = ModelWeights([Kernel(kw[i], bias=float(kb[i])) for i in range(4)], f1w, f1b, f2w, f2b, act1, act2)
    imgs = np.random.default_rng(8).uniform(0, 1, size=(32, 28, 28))
    eng = SlotEngine(EngineParams(slots=32768, prime_bits=(60,) + (45,) * 13))
    model = encode_model(eng, weights)
    scores = forward_encoded(eng, pack_batch(eng, imgs), model).decode(eng)[:, :10]
    want = np.stack([weights.fc2_weight @ _t1_hidden(weights, im) + weights.fc2_bias for im in imgs])
    err = float(np.max(np.abs(scores - want)))
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    st.record(eng._stream)
    for _ in range(steps):
        forward_encoded(eng, pack_batch(eng, imgs), model).decode(eng)
    en.record(eng._stream)
    torch.cuda.synchronize()
    t = st.elapsed_time(en) / 1e3 / steps
    return {"metric": "encrypted-CNN images/s (paper Table 1: 32 images x 28x28 per ciphertext, depth 13, N=2^16)",
            "value": 32.0 / t, "s_per_batch": t, "max_abs_err": err,
            "note": "per batch: encrypt images, forward (36 conv products, ~5.8k rotations), decode; model encoded once"}


def _t1_hidden(weights, img):
    def poly(x, c):
        return c[0] + c[1] * x + c[2] * x * x + c[3] * x * x * x

    maps = []
    for kern in weights.conv_kernels:
        k = kern.k
        out = np.full((28 - k + 1, 28 - k + 1), float(kern.bias))
        for p in range(k):
            for q in range(k):
                out += kern.weights[p, q] * img[p:p + 28 - k + 1, q:q + 28 - k + 1]
        maps.append(poly(out, weights.act1).reshape(-1))
    return poly(weights.fc1_weight @ np.concatenate(maps) + weights.fc1_bias, weights.act2)


def bench_cfg4(steps=2):
    """Config 4: 16 images 3x224x224, 16-filter 3x3 conv (padding 1) + 0.125x^2+0.5x+0.25, N = 2^15."""
    import torch

    from paper_2512_18646_b200 import CkksEngine, config_params
    from paper_2512_18646_b200.cnn import conv_layer, decode_layer, encode_images
    from tools.workloads import ACT4, cfg4, conv_plain, poly_plain

    imgs, w, b = cfg4(16)
    eng = CkksEngine(config_params(4))
    chans = encode_images(eng, imgs, padding=1)
    ys = conv_layer(eng, chans, w, b, activation=ACT4)  # warm-up + correctness
    got = decode_layer(eng, ys)
    err = float(np.max(np.abs(got - poly_plain(conv_plain(imgs, w, b, padding=1), ACT4))))
    del ys
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    l0 = eng._lib.vr_launch_count()
    st.record(eng._stream)
    for _ in range(steps):
        ys = conv_layer(eng, chans, w, b, activation=ACT4)
        del ys
    en.record(eng._stream)
    torch.cuda.synchronize()
    t = st.elapsed_time(en) / 1e3 / steps
    launches = (eng._lib.vr_launch_count() - l0) / steps
    # e2e: encrypt from host, layer, decrypt to host
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ys = conv_layer(eng, encode_images(eng, imgs, padding=1), w, b, activation=ACT4)
    decode_layer(eng, ys)
    torch.cuda.synchronize()
    te = time.perf_counter() - t0
    return {"metric": "encrypted-CNN images/s (cfg4 conv 16x3x3x3 + degree-2 activation, 16 images/batch, N=2^15)",
            "value": 16 / t, "s_per_batch": t, "max_abs_err": err, "launches_per_batch": launches,
            "e2e_images_per_s": 16 / te, "e2e_h2d_bytes": 3 * 226 * 16 * 226 * 8, "e2e_d2h_bytes": 16 * 224 * 16 * 224 * 8}


def bench_cfg3(steps=3):
    """Config 3: 64 images 28x28 -> conv 5x4x4 stride 2 -> square -> dense 845->64 -> square -> dense 64->10
    (N = 2^14, depth 5), images/s of the encrypted inference (inputs resident, dense plaintexts included)."""
    import torch

    from paper_2512_18646_b200 import CkksEngine, config_params
    from paper_2512_18646_b200.cnn import cnn_cfg3, decode_logits, encode_cfg3_model
    from tools.workloads import cfg3, cfg3_plain

    imgs, w, w1, w2 = cfg3()
    eng = CkksEngine(config_params(3))
    t0 = time.perf_counter()
    model = encode_cfg3_model(eng, w, w1, w2)  # one-time model encoding (provider side)
    torch.cuda.synchronize()
    t_model = time.perf_counter() - t0
    logits = cnn_cfg3(eng, imgs, w, model=model)
    err = float(np.max(np.abs(decode_logits(eng, logits, 64, 28) - cfg3_plain(imgs, w, w1, w2))))
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    st.record(eng._stream)
    for _ in range(steps):
        logits = cnn_cfg3(eng, imgs, w, model=model)
    en.record(eng._stream)
    torch.cuda.synchronize()
    t = st.elapsed_time(en) / 1e3 / steps
    return {"metric": "encrypted-CNN images/s (cfg3 small CNN, 64 images per pass, N=2^14, depth 5)",
            "value": 64 / t, "s_per_pass": t, "max_abs_err": err, "model_encode_s": t_model,
            "note": "each pass encrypts the 28 image columns; the 4160+640 dense-layer plaintexts are encoded once"}


def bench_cfg5a(ws, rank, local, max_over_ranks, barrier, steps=5):
    """Config 5a: HE matmul 256x256 (4 row blocks of 64 x 256 column cts), k sharded over ranks,
    degree-2 partials summed in int64 with one NCCL reduce per row block onto the block's owner rank,
    which alone relinearises + rescales it (strong scaling; at N=1 one rank finishes all four)."""
    import torch

    from paper_2512_18646_b200 import CkksEngine, config_params
    from paper_2512_18646_b200.dist import encode_operands_sharded, matmul_outer_sharded_owned, shard_range
    from tools.workloads import cfg_matmul

    a, b = cfg_matmul(5)
    blocks = [a[64 * i: 64 * (i + 1)] for i in range(4)]
    eng = CkksEngine(config_params(5), device=local)
    lo, hi = shard_range(256, rank, ws)
    lefts, right = encode_operands_sharded(eng, blocks, b, lo, hi)
    outs = matmul_outer_sharded_owned(eng, lefts, right)
    errs = [float(np.max(np.abs(eng.dec(o)[: 64 * 256].reshape(64, 256) - blocks[bi] @ b))) for bi, o in outs.items()]
    err = max_over_ranks(max(errs) if errs else 0.0)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    st.record(eng._stream)
    for _ in range(steps):
        outs = matmul_outer_sharded_owned(eng, lefts, right)
    en.record(eng._stream)
    torch.cuda.synchronize()
    t = max_over_ranks(st.elapsed_time(en) / 1e3 / steps)
    return {"metric": "HE matmul/s (cfg5a 256x256, 4 row blocks x 256 column cts, k sharded, NCCL int64 reduce per block)",
            "value": 1.0 / t, "ms_per_matmul": t * 1e3, "n_gpus": ws, "scaling": "strong", "max_abs_err": err,
            "k_per_rank": hi - lo}


def bench_cfg5b(ws, rank, local, max_over_ranks, barrier, images=512, group=64):
    """Config 5b: the config-4 layer on 512 images, 64 images per column ciphertext (8 groups),
    groups sharded over ranks, no collective (strong scaling)."""
    import torch

    from paper_2512_18646_b200 import CkksEngine, config_params
    from paper_2512_18646_b200.cnn import conv_layer, decode_layer, encode_images
    from paper_2512_18646_b200.dist import image_groups
    from tools.workloads import ACT4, cfg5b, conv_plain, poly_plain

    imgs, w, b = cfg5b(images)
    eng = CkksEngine(config_params(5), device=local)
    mine = image_groups(images, group, rank, ws)
    chans = [encode_images(eng, imgs[lo:hi], padding=1) for lo, hi in mine]
    err = 0.0
    if mine:  # correctness on the first local group
        lo, hi = mine[0]
        got = decode_layer(eng, conv_layer(eng, chans[0], w, b, activation=ACT4))
        err = float(np.max(np.abs(got - poly_plain(conv_plain(imgs[lo:hi], w, b, padding=1), ACT4))))
    err = max_over_ranks(err)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    st.record(eng._stream)
    for ch in chans:
        ys = conv_layer(eng, ch, w, b, activation=ACT4)
        del ys
    en.record(eng._stream)
    torch.cuda.synchronize()
    t = max_over_ranks(st.elapsed_time(en) / 1e3)
    return {"metric": "encrypted-CNN images/s (cfg5b: cfg4 layer on 512 images, 64 images/ct, groups sharded)",
            "value": images / t, "s_per_512_images": t, "n_gpus": ws, "scaling": "strong", "max_abs_err": err,
            "groups_per_rank": len(mine)}


def bench_ntt(eng, peak):
    """Forward NTT throughput on a batch larger than L2 (N=2^14 limbs, in place)."""
    import torch

    from paper_2512_18646_b200 import _lib

    nl = eng.L + 1
    polys = 256
    data = torch.randint(0, 2 ** 39, (polys, nl, eng.N), dtype=torch.int64, device="cuda")
    lib = eng._lib
    for _ in range(3):
        _lib.check(lib.vr_ntt(eng.handle, data.data_ptr(), polys, nl, 0, 0))
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    torch.cuda.synchronize()
    st.record(eng._stream)
    for _ in range(reps):
        _lib.check(lib.vr_ntt(eng.handle, data.data_ptr(), polys, nl, 0, 0))
    en.record(eng._stream)
    torch.cuda.synchronize()
    t = st.elapsed_time(en) / 1e3 / reps
    nbytes = polys * nl * eng.N * 8
    gbs = 2 * nbytes / t / 1e9  # read + write of every limb
    butterflies = polys * nl * (eng.N // 2) * eng.params.log_n
    # integer-pipe peak: the same butterfly on registers only (k_bfly_peak)
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    blocks, iters = 148 * 16, 256
    _lib.check(lib.vr_bench_butterflies(eng.handle, blocks, 16, sink.data_ptr()))
    torch.cuda.synchronize()
    st.record(eng._stream)
    _lib.check(lib.vr_bench_butterflies(eng.handle, blocks, iters, sink.data_ptr()))
    en.record(eng._stream)
    torch.cuda.synchronize()
    tp = st.elapsed_time(en) / 1e3
    peak_int = blocks * 256 * iters * 8 / tp / 1e9
    # FP64-pipe peak: the FP64 NTT butterfly on registers only (primes < 2^46 run the FP64 body)
    f_iters = 32
    _lib.check(lib.vr_bench_butterflies_f64(eng.handle, blocks, 4, sink.data_ptr()))
    torch.cuda.synchronize()
    st.record(eng._stream)
    _lib.check(lib.vr_bench_butterflies_f64(eng.handle, blocks, f_iters, sink.data_ptr()))
    en.record(eng._stream)
    torch.cuda.synchronize()
    peak_f64 = blocks * 256 * f_iters * 64 / (st.elapsed_time(en) / 1e3) / 1e9
    n_f64 = sum(1 for q in eng.q[:nl] if q < (1 << 46))
    # limb-weighted roofline: time per butterfly = share_int / peak_int + share_f64 / peak_f64
    peak_mix = 1.0 / ((nl - n_f64) / nl / peak_int + n_f64 / nl / peak_f64)
    achieved = butterflies / t / 1e9
    return {"metric": "NTT HBM GB/s (forward, in place)", "N": eng.N, "limbs": polys * nl,
            "gbs": gbs, "peak": peak, "frac": gbs / peak, "us_per_limb": t / (polys * nl) * 1e6,
            "gbutterfly_s": achieved,
            "int_roofline": {"bound": "IMAD pipe (60-bit limbs) + FP64 pipe (limbs < 2^46)", "achieved_gbutterfly_s": achieved,
                             "peak_gbutterfly_s": peak_mix, "frac": achieved / peak_mix,
                             "peak_int_gbutterfly_s": peak_int, "peak_f64_gbutterfly_s": peak_f64,
                             "limbs_f64": f"{n_f64}/{nl}",
                             "peak_source": "measured live: k_bfly_peak (Harvey/Shoup) and k_bfly_peak_f64 (FP64 Shoup), "
                                            "register-only, weighted by the limb mix"}}


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
