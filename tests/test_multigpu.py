"""Multi-process (torchrun, one process per GPU) parity: runs
tests/mp_gpu_worker.py on 2 GPUs when the box has them."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif(_ngpu() < 2 if __import__("torch").cuda.is_available() else True,
                    reason="needs >= 2 GPUs")
def test_two_gpu_processes_match_reference():
    n = min(_ngpu(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29617",
           os.path.join(ROOT, "tests", "mp_gpu_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
