import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18646_b200 import CkksEngine, config_params, multicipher, pipeline
from paper_2512_18646_b200.cnn import conv_layer, encode_images
from tools.workloads import ACT4, cfg4
import paper_2512_18646_b200._lib as L
imgs, w, b = cfg4(16)
eng = CkksEngine(config_params(4))
chans = encode_images(eng, imgs, padding=1)
lib = eng._lib
orig_conv, orig_poly, orig_enc = lib.vr_conv_columns, lib.vr_poly_activation, lib.vr_encode
T = {}
def wrap(name, fn):
    def f(*a):
        t = time.perf_counter(); r = fn(*a); T[name] = T.get(name, 0) + time.perf_counter() - t; return r
    return f
lib.vr_conv_columns = wrap("conv", orig_conv); lib.vr_poly_activation = wrap("poly", orig_poly); lib.vr_encode = wrap("encode", orig_enc)
for it in range(8):
    T.clear(); torch.cuda.synchronize(); t0 = time.perf_counter()
    ys = conv_layer(eng, chans, w, b, activation=ACT4)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"iter {it}: submit {t1-t0:.3f} total {t2-t0:.3f}  " + " ".join(f"{k}={v:.3f}" for k, v in T.items()), flush=True)
    del ys
