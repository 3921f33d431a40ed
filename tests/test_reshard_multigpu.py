"""Multi-GPU reshard over NVLink (needs >= 2 GPUs; skipped on 1-GPU boxes)."""

import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
def test_reshard_across_gpus_byte_identical():
    n = 4 if torch.cuda.device_count() >= 4 else 2
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                          "--master-port", "29533", str(ROOT / "tools" / "reshard_check.py")],
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "mismatched words 0" in res.stdout
