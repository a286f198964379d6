"""The C-ABI from plain C on the GPU: examples/echo_c_demo.c (ordering and unphysical-state
errors, a uniform state kept bit for bit, mass and energy conserved to 1e-12 over 5 echo_advance
steps of a periodic wave, no floors) must exit 0."""
import subprocess

import pytest

from tests.test_lib_cpu import build_c_demo

pytestmark = pytest.mark.gpu


def test_c_demo_runs(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1810_04597_b200 import build

    exe = build_c_demo(build.build(), str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c demo ok" in r.stdout
