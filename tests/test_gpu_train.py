"""NEXT-4 smoke: the end-to-end WDL-shaped training example (dense tower in
PyTorch, embeddings through the HET C-ABI) learns the synthetic teacher."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_train_wdl_learns():
    cmd = [sys.executable, os.path.join(ROOT, "examples", "train_wdl.py"), "--staleness", "10", "--steps", "300",
           "--rows", "200000"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["progressive_auc"] > 0.6, res
