"""Multi-process (torchrun, one process per GPU) parity: runs
tests/mp_gpu_worker.py with 2 and 4 processes against the reference's golden
vectors.

On a box with fewer GPUs than processes, World.init maps LOCAL_RANK onto
LOCAL_RANK % device_count, so several processes share one device.  CUDA IPC
works between processes on the same device, so the multi-process data path
(IPC-mapped halos and parity double-buffering, the device barrier across the
side and main streams, the split own-block / halo SpMM with beta=1, the
cross-process GroupReducer / RowGroupReducer, the sharded builder) runs
unchanged on a 1-GPU box -- only the transport is HBM instead of NVLink."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nproc,rank_map", [(2, "block"), (4, "block"), (2, "cyclic"),
                                            (4, "cyclic")])
def test_multiprocess_matches_reference(nproc, rank_map):
    """block: replicas of a row group share a process; cyclic: they sit on
    different processes, so 1.5D runs the cross-process reduce-scatter +
    all-gather (engine.DevicePlan._reduce_scatter_all_gather)."""
    import torch
    ngpu = torch.cuda.device_count()
    env = dict(os.environ, OMP_NUM_THREADS="2", DG_RANK_MAP=rank_map)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
           "--master-port", str(29617 + nproc + (10 if rank_map == "cyclic" else 0)),
           os.path.join(ROOT, "tests", "mp_gpu_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, env=env)
    out = r.stdout[-6000:] + r.stderr[-6000:]
    print(f"[{nproc} processes on {min(ngpu, nproc)} GPU(s), {rank_map} rank map]\n"
          + r.stdout[-3000:])
    assert r.returncode == 0, out
    assert out.count("0 failures") == nproc, out
