"""Host time per public call of the pipelined e2e cfg-2 step (is the e2e loop host- or device-bound?)."""
import sys, time, os; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch, gc
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer
from tools.workloads import cfg_matmul
a, b = cfg_matmul(2)
eng = CkksEngine(config_params(2))
pa, pb = torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory()
pc = time.perf_counter
for depth in (2, 3, 4):
    acc = {k: 0.0 for k in ("encL", "encR", "matmul", "decode_async", "result")}
    def run(k, rec):
        futs = []
        for _ in range(k):
            t0 = pc(); L = encode_left(eng, pa.numpy(), 64)
            t1 = pc(); R = encode_right(eng, pb.numpy(), 64)
            t2 = pc(); P = matmul_outer(eng, L, R)
            t3 = pc(); futs.append(P.decode_async(eng))
            t4 = pc()
            if len(futs) >= depth:
                futs.pop(0).result()
            t5 = pc()
            if rec:
                for key, d in zip(acc, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
                    acc[key] += d
        while futs:
            futs.pop(0).result()
    run(30, False); torch.cuda.synchronize(); gc.collect(); gc.disable()
    t0 = pc(); run(200, True); torch.cuda.synchronize(); dt = (pc() - t0) / 200
    gc.enable()
    print(f"depth {depth}: {dt * 1e6:.1f} us/step ({1 / dt:.0f}/s); host us/step:", {k: round(v / 200 * 1e6, 1) for k, v in acc.items()}, flush=True)
