"""cfg-2 batch of B independent products: matmul_outer_many (one launch sequence) against B asynchronous
matmul_outer calls over the slot graphs.  us per product, CUDA events, operands larger than L2."""
import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer, matmul_outer_many
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dim = {1: 8, 2: 64}[cfg]
eng = CkksEngine(config_params(cfg))
rng = np.random.default_rng(1)
mats = [tuple(rng.uniform(-1, 1, (2, dim, dim))) for _ in range(B)]
pairs = [(encode_left(eng, a, dim), encode_right(eng, b, dim)) for a, b in mats]
def timed(fn, reps):
    for _ in range(5): fn()
    eng.join(); torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(reps): fn()
    eng.join(); en.record(); torch.cuda.synchronize()
    return st.elapsed_time(en) * 1e3 / reps / B
def many(): matmul_outer_many(eng, pairs)
def sep():
    for l, r in pairs: matmul_outer(eng, l, r)
outs = matmul_outer_many(eng, pairs)
ref = [matmul_outer(eng, l, r) for l, r in pairs]
assert all(np.array_equal(x.ct.residues(), y.ct.residues()) for x, y in zip(outs, ref))
for _ in range(2):
    print(f"cfg {cfg} B={B}: many {timed(many, 50):.2f} us/product, separate async {timed(sep, 50):.2f} us/product")
# two alternating streams: the chain of batch i overlaps the tensor sum of batch i + 1
for ns in (2, 3):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    state = {"i": 0}
    def many_alt():
        s = streams[state["i"] % ns]; state["i"] += 1
        with torch.cuda.stream(s):
            matmul_outer_many(eng, pairs)
    def timed_alt(reps):
        for _ in range(6): many_alt()
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        st.record()
        for s in streams: s.wait_stream(cur)
        for _ in range(reps): many_alt()
        for s in streams: cur.wait_stream(s)
        en.record(); torch.cuda.synchronize()
        return st.elapsed_time(en) * 1e3 / reps / B
    print(f"cfg {cfg} B={B}: many on {ns} alternating streams {timed_alt(60):.2f} us/product")
