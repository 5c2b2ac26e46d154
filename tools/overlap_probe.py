"""Upper bound of cross-call overlap for config-2 matmul_outer: two engines (own arenas, streams,
graphs), each driven on its own torch stream, calls interleaved.  Device time per matmul.
    VR_GRAPH_MAX_MB=1000 python tools/overlap_probe.py   (graph replay for both)"""
import sys, time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer

rng = np.random.default_rng(1)
a, b = rng.uniform(-1, 1, (2, 64, 64))
NE = int(sys.argv[1]) if len(sys.argv) > 1 else 2
streams = [torch.cuda.Stream() for _ in range(NE)]
engs, ops = [], []
for s in streams:
    with torch.cuda.stream(s):
        e = CkksEngine(config_params(2))
        engs.append(e)
        ops.append((encode_left(e, a, 64), encode_right(e, b, 64)))
torch.cuda.synchronize()
outs = [None] * NE


def run(k, both):
    for i in range(k):
        for j in range(NE) if both else (0,):
            with torch.cuda.stream(streams[j]):
                outs[j] = matmul_outer(engs[j], *ops[j])


for both in (False, True):
    run(10, both)
    torch.cuda.synchronize()
    for k in (20, 200):
        main = torch.cuda.current_stream()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record(main)
        for s in streams:
            s.wait_stream(main)
        t0 = time.perf_counter()
        run(k, both)
        th = time.perf_counter() - t0
        for j, s in enumerate(streams):
            with torch.cuda.stream(s):
                engs[j].join()
            main.wait_stream(s)
        en.record(main)
        torch.cuda.synchronize()
        n = k * (NE if both else 1)
        print(f"{str(NE) + ' engines' if both else 'one engine'} {k:4d} calls each: {st.elapsed_time(en) * 1e3 / n:6.1f} us/matmul "
              f"device, host {th / n * 1e6:5.1f} us/matmul")
