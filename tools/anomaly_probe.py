"""Repeat the bench's headline loop (cfg-2 matmul_outer, async slots) and report device time plus the
slowest host calls, to catch occasional slow runs."""
import gc, sys, time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from bench import ClockSampler
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer

eng = CkksEngine(config_params(2))
a, b = np.random.default_rng(1).uniform(-1, 1, (2, 64, 64))
L, R = encode_left(eng, a, 64), encode_right(eng, b, 64)
t0 = time.perf_counter()
while time.perf_counter() - t0 < 0.25:
    for _ in range(8):
        out = matmul_outer(eng, L, R)
    torch.cuda.synchronize()
for rnd in range(4):
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    gc.disable()
    hs = []
    use = len(sys.argv) > 1 and sys.argv[1] == "nvml"
    with ClockSampler(0) if use else open("/dev/null") as clk:
        st.record()
        for _ in range(200):
            h0 = time.perf_counter()
            out = matmul_outer(eng, L, R)
            hs.append(time.perf_counter() - h0)
        eng.join()
        en.record()
        torch.cuda.synchronize()
    if use:
        print(clk.summary())
    gc.enable()
    hs = np.array(hs) * 1e6
    print(f"round {rnd}: {st.elapsed_time(en) / 200 * 1e3:.1f} us/step; host mean {hs.mean():.1f} us, max {hs.max():.0f} us, "
          f">200us: {(hs > 200).sum()}", flush=True)
