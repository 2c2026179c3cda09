"""Sharded stem across 2+ GPUs: amplitudes vs the oracle with fp16 and int8
(group-quantised, Eq. 1) mode swaps.  Tolerances: rel-L2 <= 2e-2 (fp16 comm), <= 5e-2 (int8 comm)."""
import json
import os
import subprocess
import sys
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_stem_vs_oracle(world):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    with tempfile.NamedTemporaryFile(suffix=".json", delete=False) as f:
        out = f.name
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(ROOT, "tests", "mgpu_worker.py"), out]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    v = json.load(open(out))
    assert v["swaps"] >= 1
    assert v["rel_fp16_oracle"] <= 2e-2
    assert v["rel_int8_oracle"] <= 5e-2
    assert v["rel_fp16_vs_1gpu"] == 0.0          # fp16 swaps: bit-identical to one GPU
    assert v["rel_int8_all_c2_oracle"] <= 5e-2
