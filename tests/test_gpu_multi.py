"""Multi-GPU parity as a test: when >= 2 GPUs are visible, launch
tools/mgpu_check.py under torchrun (NCCL, one process per GPU) at G = 2 (and
G = 4 when 4 GPUs are visible).  It checks the sharded engine -- the routed
projection into the owners' symmetric buffers (against projection +
all_to_all), host rows streamed through the API, refinement passes, sparse /
mixed pipelines and the benchmark's law at 1M -- against the golden
reference outputs."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _launch(nproc: int):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--local-addr", "127.0.0.1",
           f"--nproc-per-node={nproc}", os.path.join(ROOT, "tools", "mgpu_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    print(r.stdout[-6000:])
    print(r.stderr[-3000:], file=sys.stderr)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "MISMATCH" not in r.stdout and "OK" in r.stdout


@pytest.mark.parametrize("nproc", [2, 4])
def test_multi_gpu_engine_parity(nproc):
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs ({torch.cuda.device_count()} visible)")
    _launch(nproc)
