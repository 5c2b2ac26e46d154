"""Host submission time vs device time of the config-4 layer, with clocks."""
import subprocess, sys, time, threading
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18646_b200 import CkksEngine, config_params
from paper_2512_18646_b200.cnn import conv_layer, encode_images
from tools.workloads import ACT4, cfg4
from bench import ClockSampler

imgs, w, b = cfg4(16)
eng = CkksEngine(config_params(4))
chans = encode_images(eng, imgs, padding=1)
ys = conv_layer(eng, chans, w, b, activation=ACT4); del ys
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import gc, os
if os.environ.get("NOGC"):
    gc.collect(); gc.freeze(); gc.disable()
with ClockSampler(0) as clk:
    for it in range(6):
        st.record(eng._stream)
        t0 = time.perf_counter()
        ys = conv_layer(eng, chans, w, b, activation=ACT4)
        t1 = time.perf_counter()
        en.record(eng._stream)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        free, total = torch.cuda.mem_get_info()
        print(f"iter {it}: host submit {t1-t0:.3f}s, wall {t2-t0:.3f}s, device {st.elapsed_time(en)/1e3:.3f}s, "
              f"free {free/2**30:.1f} GiB, torch reserved {torch.cuda.memory_reserved()/2**30:.1f} GiB", flush=True)
        del ys
print(clk.summary())
