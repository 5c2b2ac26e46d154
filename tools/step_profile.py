"""Run a few bench steps of one workload for ncu launch lists / --set full captures.

    python tools/step_profile.py [--cfg 2|4] [--steps 3]

Prints the number of library kernel launches before the profiled steps so ncu
can skip setup with `-s <that number>`.
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18646_b200 import (  # noqa: E402
    CkksEngine, conv_columns_multi, config_params, encode_image_columns, encode_left, encode_right, matmul_outer,
    pad_images, poly_activation_batch)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--images", type=int, default=16)
    ap.add_argument("--filters", type=int, default=16)
    args = ap.parse_args()
    eng = CkksEngine(config_params(args.cfg))
    lib = eng._lib
    if args.cfg == 2:
        rng = np.random.default_rng(1)
        a, b = rng.uniform(-1, 1, (64, 64)), rng.uniform(-1, 1, (64, 64))
        left, right = encode_left(eng, a, 64), encode_right(eng, b, 64)
        step = lambda: matmul_outer(eng, left, right)  # noqa: E731
    else:
        rng = np.random.default_rng(3)
        imgs = rng.uniform(0, 1, (args.images, 3, 224, 224))
        W = rng.normal(0, 0.05, (args.filters, 3, 3, 3))
        padded = pad_images(imgs, 1)
        chans = [encode_image_columns(eng, padded[:, c]) for c in range(3)]

        def step():
            ys = conv_columns_multi(eng, chans, W, np.zeros(args.filters))
            return [poly_activation_batch(eng, y.cts, (0.25, 0.5, 0.125, 0.0)) for y in ys]
    step()
    torch.cuda.synchronize()
    print(f"launches_before_steps={lib.vr_launch_count()}", flush=True)
    l0 = lib.vr_launch_count()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    print(f"launches_per_step={(lib.vr_launch_count() - l0) / args.steps}", flush=True)


if __name__ == "__main__":
    main()
