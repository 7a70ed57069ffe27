"""Multi-GPU parity through NCCL (runs only where >= N GPUs are visible)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("layout,n", [("dp2", 2), ("pp2", 2), ("cfg1_tiny", 3), ("pp1+3", 4), ("dp4z3", 4),
                                      ("pp2x2", 4), ("llama1f1b2x2", 4), ("xl1+3", 4)])
def test_multi_gpu_layout(layout, n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29531",
           os.path.join(ROOT, "scripts", "mgpu_check.py"), layout]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
