"""NEXT-4 smoke: the end-to-end training examples (dense towers in PyTorch,
embeddings through the HET C-ABI) learn the synthetic teacher."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("model,auc", [("wdl", 0.6), ("dcn", 0.6), ("graphsage", 0.6)])
def test_train_learns(model, auc):
    """NEXT-4: the WDL-, DCN- and GraphSAGE-shaped towers learn the synthetic
    teacher through the C-ABI (PAPER.md:719-740 workloads; pattern only)."""
    cmd = [sys.executable, os.path.join(ROOT, "examples", "train.py"), "--model", model, "--staleness", "10",
           "--steps", "300", "--rows", "200000"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["model"] == model and res["progressive_auc"] > auc, res
