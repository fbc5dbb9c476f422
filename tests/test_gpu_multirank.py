"""Multi-GPU parity (P14, decomposition invariance): launches tests/mr_parity.py
under torchrun on 2, 3 and 4 GPUs of this box (when available; 3 = an odd ring)."""
import json
import os
import subprocess
import sys
import tempfile

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("nproc", [2, 3, 4])
def test_multirank_parity(nproc):
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "rep.json")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(29500 + nproc * 7),
               os.path.join(HERE, "mr_parity.py"), "--out", out]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
        rep = json.load(open(out))
        assert rep["ok"], rep
        assert any(x.get("sent", 0) > 0 for x in rep["reports"])
        assert any("sources_ok" in x for x in rep["reports"])


@pytest.mark.parametrize("config", ["c4"])
def test_multirank_fullsize_sampled(config):
    """C4 at full size (4.29e9 particles, open faces, absorbing planet,
    count-balanced slabs) on 4 GPUs, sampled against the oracle (mr_fullsize.py)."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "rep.json")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
               "--master-addr", "127.0.0.1", "--master-port", "29571",
               os.path.join(HERE, "mr_fullsize.py"), "--config", config, "--out", out]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
        assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
        rep = json.load(open(out))
        assert rep["ok"], rep


def test_multirank_long_graph_run():
    """C1r for 40 cycles replayed from CUDA graphs over the peer transport on
    2 GPUs (every replay advances the device-side barrier epochs and reuses the
    receive buffers), checked against the oracle by id."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "rep.json")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr", "127.0.0.1", "--master-port", "29583",
               os.path.join(HERE, "mr_parity.py"), "--long", "40", "--out", out]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
        rep = json.load(open(out))
        assert rep["ok"], rep
        assert any(x.get("sent", 0) > 0 for x in rep["reports"])
