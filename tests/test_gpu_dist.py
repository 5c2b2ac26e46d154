"""Config 5a's sharded HE matmul on one GPU with virtual ranks: per-shard
partials (product code) summed like the NCCL all-reduce, then finished, must be
bit-identical to the unsharded 4-block matmul_outer, for 1, 2, 4 and 8 shards,
and decode to A*B (256x256) within 1e-3."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2512_18646_b200 import CkksEngine, config_params, encode_left, encode_right, matmul_outer_blocks  # noqa: E402
from paper_2512_18646_b200.dist import encode_operands_sharded, matmul_finish, matmul_partials, shard_range  # noqa: E402
from tools.workloads import cfg_matmul  # noqa: E402


def test_cfg5a_sharded_equals_unsharded():
    a, b = cfg_matmul(5)
    blocks = [a[64 * i: 64 * (i + 1)] for i in range(4)]
    eng = CkksEngine(config_params(5))
    lefts = [encode_left(eng, blk, 256) for blk in blocks]
    right = encode_right(eng, b, 64)
    want = matmul_outer_blocks(eng, lefts, right)
    ref = [w.residues() for w in want]
    got_c = np.concatenate([eng.dec(w)[: 64 * 256].reshape(64, 256) for w in want])
    assert float(np.max(np.abs(got_c - a @ b))) < 1e-3
    del lefts, right, want
    for world in (2, 4, 8):
        total = None
        lv = None
        for rank in range(world):
            lo, hi = shard_range(256, rank, world)
            ls, rs = encode_operands_sharded(eng, blocks, b, lo, hi)
            part, lv = matmul_partials(eng, ls, rs)
            total = part if total is None else total + part  # the int64 all-reduce
            del ls, rs
        outs = matmul_finish(eng, total, lv, 64, 256)
        for o, r in zip(outs, ref):
            np.testing.assert_array_equal(o.residues(), r)


def test_cfg5a_owned_world1_equals_unsharded():
    """matmul_outer_sharded_owned on one rank finishes every block, bit-identical to matmul_outer_blocks."""
    from paper_2512_18646_b200.dist import matmul_outer_sharded_owned

    a, b = cfg_matmul(5)
    blocks = [a[64 * i: 64 * (i + 1)] for i in range(4)]
    eng = CkksEngine(config_params(5))
    lefts = [encode_left(eng, blk, 256) for blk in blocks]
    right = encode_right(eng, b, 64)
    ref = [w.residues() for w in matmul_outer_blocks(eng, lefts, right)]
    del lefts, right
    ls, rs = encode_operands_sharded(eng, blocks, b, 0, 256)
    outs = matmul_outer_sharded_owned(eng, ls, rs)
    assert sorted(outs) == [0, 1, 2, 3]
    for bi, r in enumerate(ref):
        np.testing.assert_array_equal(outs[bi].residues(), r)
