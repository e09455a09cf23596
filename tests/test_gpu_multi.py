"""Multi-GPU parity: N worker processes (one per GPU) over NCCL against the
N-worker CPU oracle.  Skipped when fewer than 2 GPUs are visible."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("policy,s,frac", [(0, 10, 0.1), (1, 3, 0.05), (0, 0, 0.1), (0, 0xFFFFFFFF, 0.2)])
@pytest.mark.parametrize("p2p", ["1", "0"])
def test_multi_gpu_parity(policy, s, frac, p2p):
    """p2p=1: device-initiated exchange over NVLink peer memory (default);
    p2p=0: the NCCL send/recv exchange with host-read counts."""
    n = min(ngpu(), 4)
    env = dict(os.environ, HET_P2P=p2p)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + policy * 7 + (s % 97) + 200 * int(p2p)}",
           os.path.join(ROOT, "tests", "mgpu_worker.py"), str(policy), str(s), str(frac), "60"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "MGPU_OK" in r.stdout


@pytest.mark.skipif(ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("shape,policy,s,frac,T", [("reddit", 0, 10, 0.1, 12), ("wide", 0, 3, 0.1, 30),
                                                   ("wide", 1, 100, 0.05, 30), ("toy", 2, 10, 0.1, 60)])
@pytest.mark.parametrize("p2p", ["1", "0"])
def test_multi_gpu_parity_shapes(shape, policy, s, frac, T, p2p):
    """BASELINE configs[2]-shaped batches (14,208 distinct ids per worker: the
    large-n dedup and the non-fused exchange round) and 4 KB rows."""
    n = min(ngpu(), 4)
    env = dict(os.environ, HET_P2P=p2p)
    port = 31000 + 10 * policy + (s % 7) + 100 * int(p2p) + (0 if shape == "reddit" else 50)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tests", "mgpu_worker.py"), str(policy), str(s), str(frac), str(T), shape, "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "MGPU_OK" in r.stdout
