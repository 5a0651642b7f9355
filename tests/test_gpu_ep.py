"""Expert-parallel parity on >= 2 GPUs: launches tools/ep_check.py under
torchrun (one process per GPU, NCCL).  Skipped on single-GPU boxes; the host
logic of the same path is covered on CPU by tests/test_ep_gloo.py."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_ep_matches_single_gpu_per_rank():
    n = min(torch.cuda.device_count(), 8)
    n = 8 if n >= 8 else (4 if n >= 4 else 2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29561", os.path.join(ROOT, "tools", "ep_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
    # (6 vs 1-GPU + 2 vs oracle) x {p2p, nccl} + recompute / pull + drop_h + graph + guards
    assert r.stdout.count("PASS") == 20 * n


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_model_step_ep_dp_matches_single_gpu():
    """Model step with EP MoE layers + overlapped DP gradient all-reduce vs the
    single-GPU model on every rank's batch (tools/model_ep_check.py)."""
    n = 4 if torch.cuda.device_count() >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29562", os.path.join(ROOT, "tools", "model_ep_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
    assert r.stdout.count("PASS") == 2 + n   # rank 0 checks both transports; every rank the ZeRO-1 step
