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


@pytest.mark.parametrize("world,mode", [(2, "fp32"), (2, "bf16"), (2, "bf16-nccl"), (2, "bf16-fp32x"), (4, "bf16"),
                                        (4, "bf16-fp32x"), (2, "fp32-fifo"), (2, "fp32-firo")])
def test_multi_rank_parity(world, mode):
    """fp32: NCCL all-reduce; bf16: the in-kernel NVLink exchange (dW tiles reduce-added
    into their owner's buffer, fused Adam at the owner, shadow rows pushed to every rank);
    bf16-nccl: reduce-scatter / sharded Adam / all-gather through NCCL; bf16-fp32x: the
    in-kernel exchange with fp32 contributions (default: bf16); fp32-fifo / fp32-firo: the
    comparison buffers on every rank."""
    if _ngpu() < world:
        pytest.skip("needs %d GPUs" % world)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % world,
           "--master-addr=127.0.0.1", "--master-port=%d" % (29600 + os.getpid() % 300),
           os.path.join(HERE, "mp_gpu_parity.py"), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert r.stdout.count("replicas identical") == world


@pytest.mark.parametrize("world", [2])
def test_multi_rank_ingest(world):
    """Client processes -> per-rank shared-memory rings (round robin from the client id)
    -> reservoir_ingest on every rank -> collective training (tests/mp_gpu_ingest.py)."""
    if _ngpu() < world:
        pytest.skip("needs %d GPUs" % world)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % world,
           "--master-addr=127.0.0.1", "--master-port=%d" % (29300 + os.getpid() % 300),
           os.path.join(HERE, "mp_gpu_ingest.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert r.stdout.count("replicas identical") == world
