"""The z-slab decomposition across GPUs: one rank per
GPU under torchrun, NCCL ghost exchange (stream-ordered, overlapped by the interior sweeps) or
the CUDA-IPC fused ghost stores, bit for bit against the single-domain run.  Needs >= 2 visible
GPUs and skips otherwise (every gpurun box of this build has one; the driver's multi-GPU node
runs it).  Marked gpu."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("cfg,n,extra", [(0, (48, 40, 36), []), (2, (40, 36, 44), []), (0, (48, 40, 36), ["--fused"]),
                                         (0, (40, 32, 36), ["--divb", "2"]), (4, (48, 35, 36), ["--divb", "2"])])
def test_slabs_across_gpus_bitwise(tmp_path, cfg, n, extra):
    from paper_1810_04597_b200 import build

    build.build()
    world = min(_ngpu(), 4)
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "multi_gpu_slab_check.py"),
           "--config", str(cfg), "--n", *map(str, n), "--steps", "2", "--out", str(out), *extra]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["world"] == world and res["dt_equal"] and res["U_bitwise"] and res["P_bitwise"], res
    assert res.get("b_bitwise", True), res
