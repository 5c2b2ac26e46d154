"""Config 4 end to end on one GPU: encrypt 16 padded 3x224x224 images (3 x 226 column
ciphertexts), 16-filter 3x3 conv + 0.125x^2+0.5x+0.25 activation, decrypt, compare."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18646_b200 import CkksEngine, config_params
from paper_2512_18646_b200.cnn import conv_layer, decode_layer, encode_images
from tools.workloads import ACT4, cfg4, conv_plain, poly_plain

images = int(sys.argv[1]) if len(sys.argv) > 1 else 16
filters = int(sys.argv[2]) if len(sys.argv) > 2 else 16
imgs, w, b = cfg4(images)
w, b = w[:filters], b[:filters]
eng = CkksEngine(config_params(4))
torch.cuda.synchronize(); t0 = time.perf_counter()
chans = encode_images(eng, imgs, padding=1)
torch.cuda.synchronize(); t1 = time.perf_counter()
ys = conv_layer(eng, chans, w, b, activation=ACT4)
torch.cuda.synchronize(); t2 = time.perf_counter()
ys = conv_layer(eng, chans, w, b, activation=ACT4)
torch.cuda.synchronize(); t3 = time.perf_counter()
got = decode_layer(eng, ys)
t4 = time.perf_counter()
want = poly_plain(conv_plain(imgs, w, b, padding=1), ACT4)
err = float(np.max(np.abs(got - want)))
print(f"cfg4 images={images} filters={filters}: encrypt {t1-t0:.3f}s, layer(first) {t2-t1:.3f}s, layer {t3-t2:.3f}s, "
      f"decrypt {t4-t3:.3f}s, max|err|={err:.2e}, images/s(layer)={images/(t3-t2):.1f}, "
      f"peak mem {torch.cuda.max_memory_allocated()/2**30:.1f} GiB")
