"""Device time of the config-2 matmul_outer loop in short timed regions.

    python tools/step_probe.py [steps] [rounds]

Per round: events only around the loop (like bench.py), with and without the NVML clock
sampler, then per-step events between consecutive calls (shows first-step latency)."""
import sys, time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from bench import ClockSampler
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
eng = CkksEngine(config_params(2))
rng = np.random.default_rng(1)
a, b = rng.uniform(-1, 1, (2, 64, 64))
L, R = encode_left(eng, a, 64), encode_right(eng, b, 64)
out = None
for _ in range(10):
    out = matmul_outer(eng, L, R)
torch.cuda.synchronize()


def loop(k, sampler):
    global out
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with ClockSampler(0) if sampler else open("/dev/null") as _:
        st.record()
        for _ in range(k):
            out = matmul_outer(eng, L, R)
        eng.join()
        en.record()
        th = time.perf_counter() - t0
        torch.cuda.synchronize()
    return st.elapsed_time(en) * 1e3 / k, th / k * 1e6


for r in range(rounds):
    for k in (steps, 10 * steps):
        for smp in (False, True):
            d, h = loop(k, smp)
            print(f"round {r} steps {k:4d} sampler {int(smp)}: {d:6.1f} us/step device, host {h:5.1f} us/call")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
torch.cuda.synchronize()
ev[0].record()
for i in range(steps):
    out = matmul_outer(eng, L, R)
    ev[i + 1].record()
torch.cuda.synchronize()
print("per-step (events between calls):", " ".join(f"{ev[i].elapsed_time(ev[i + 1]) * 1e3:.0f}" for i in range(steps)))
