"""Multi-GPU parity through NCCL (needs >= 2 GPUs on one box; skipped otherwise).
Launches tests/mp_gpu_parity.py under torchrun, one process per GPU."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_two_rank_parity_nccl(mode):
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=%d" % (29600 + os.getpid() % 300),
           os.path.join(HERE, "mp_gpu_parity.py"), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert r.stdout.count("replicas identical") == 2
