"""Vocabulary-sharded verification on >= 2 GPUs of one box: the
collective call through the C ABI must give, on every rank, the outputs of the unsharded call
on the full rows and of the oracle (tools/shard_check.py does the comparisons)."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(world: int, tmp_path):
    out = tmp_path / f"shard_{world}.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29531", os.path.join(ROOT, "tools", "shard_check.py"),
           "--out", str(out), "--c5"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-4000:]
    res = json.loads(out.read_text())
    assert res["ok"], res
    for r in res["results"]:
        assert "error" not in r, r
        assert r["replicated"], r
    return res


@pytest.mark.gpu
def test_vocab_sharded_two_gpus(tmp_path):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    _run(2, tmp_path)


@pytest.mark.gpu
def test_vocab_sharded_four_gpus(tmp_path):
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs (gpurun --gpus 4)")
    _run(4, tmp_path)
