"""Forward / inverse NTT time per limb, split by arithmetic body: the 60-bit limb (IMAD pipe) alone,
the < 2^46 limbs (FP64 pipe) alone, and the full chain, at cfg 2 (N=2^14, cluster kernel) and cfg 4
(N=2^15, two passes); plus the 128-ciphertext cfg-2 encryption (slot FFT + fused NTT)."""
import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2512_18646_b200 import CkksEngine, config_params, _lib, encode_left, encode_right


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(reps):
        fn()
    en.record()
    torch.cuda.synchronize()
    return st.elapsed_time(en) / reps * 1e3  # us


cfgs = [int(x) for x in sys.argv[1:]] or [2, 4]
for cfg in cfgs:
    eng = CkksEngine(config_params(cfg)); torch.cuda.set_stream(eng._stream)
    nl = eng.L + 1
    total = 1280 if cfg == 2 else 2048
    for name, p0, limbs in (("int60", 0, 1), ("f64", 1, nl - 1), ("all", 0, nl)):
        polys = total // limbs
        data = torch.randint(0, 2 ** 39, (polys, limbs, eng.N), dtype=torch.int64, device="cuda")
        for inv in (0, 1):
            us = timeit(lambda: _lib.check(eng._lib.vr_ntt(eng.handle, data.data_ptr(), polys, limbs, p0, inv)))
            bf = (eng.N // 2) * eng.params.log_n
            print(f"cfg{cfg} N=2^{eng.params.log_n} {name:5s} inv={inv}: {us / (polys * limbs):.4f} us/limb  "
                  f"{polys * limbs * bf / us / 1e3:.0f} Gbfly/s  ({polys * limbs} limbs, {us:.1f} us)", flush=True)
        del data
    if cfg == 2:
        from tools.workloads import cfg_matmul
        a, b = cfg_matmul(2)
        def enc():
            L = encode_left(eng, a, 64); R = encode_right(eng, b, 64); eng.handle
        print(f"cfg2 encrypt 128 cts (h2d + slot FFT + fused NTT): {timeit(enc, 20):.1f} us", flush=True)
