"""The parity suite rerun under the library's alternative code paths (each is selected once per
process from the environment, so every variant runs in its own interpreter):

* VR_NTT_CL=1  -- every NTT through the one-kernel 8-CTA cluster transform (default: batches >= 256)
* VR_PDL=0     -- plain stream ordering instead of programmatic dependent launch
* VR_MM_ORDER=2 -- matmul_outer's key-switch chain on the high-priority stream
* VR_MM_ORDER=0, VR_NTT_F64=0 -- both tensor sums forked together on normal-priority streams, and
  every NTT on the integer (IMAD-pipe) body
* VR_GRAPH=0   -- every driver call eager (no CUDA-graph replay)
* VR_ASYNC=0   -- matmul_outer synchronous (no slot streams)
* VR_ROT_BATCH=1, VR_NTT_ST_ASYNC=0, VR_TS_LD=0 -- hoisted rotations in one launch sequence, the
  cluster NTT exchanging through scatter + cluster barriers, the TMA-ring tensor sum
* VR_ENC_ON_SLOT=1, VR_CHAIN_PRIO=1, VR_TS_LD=12 -- deferred operand encryptions on the product's slot
  stream, prioritised chain kernels, the cp.async-ring tensor sum at every n
* VR_DEFER_ENC=0, VR_DECODE_TICKETS=0, VR_TS_LD=4 -- eager encryptions, torch-tensor decode futures,
  the split-K register tensor sum
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("env", [{"VR_NTT_CL": "1"}, {"VR_PDL": "0"}, {"VR_MM_ORDER": "2", "VR_NTT_CL": "1"}, {"VR_MM_ORDER": "0", "VR_NTT_F64": "0"},
                                 {"VR_GRAPH": "0"}, {"VR_ASYNC": "0"},
                                 {"VR_ROT_BATCH": "1", "VR_NTT_ST_ASYNC": "0", "VR_TS_LD": "0"},
                                 {"VR_ENC_ON_SLOT": "1", "VR_CHAIN_PRIO": "1", "VR_TS_LD": "12"},
                                 {"VR_DEFER_ENC": "0", "VR_DECODE_TICKETS": "0", "VR_TS_LD": "4"}],
                         ids=["cluster-ntt", "no-pdl", "hi-prio-chain", "order0-int-ntt", "no-graph", "sync", "alt-kernels",
                              "enc-on-slot", "eager-host-path"])
def test_parity_suite_under_variant(env):
    pytest.importorskip("torch").cuda.is_available() or pytest.skip("no CUDA device")
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_gpu_configs.py", "tests/test_gpu_alg3.py",
                        "tests/test_gpu_hostpath.py"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
