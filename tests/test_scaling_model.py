"""the analytic strong-scaling model of the z-slab decomposition
(paper_1810_04597_b200/scaling_model.py), CPU only: SPEC.md's worked examples for
Amdahl and the sweet spot, the compute-only limit, and the calibration reproducing the
measured one-GPU runs it was fitted to (profiles/)."""
import importlib.util
import json
import math
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _S():
    spec = importlib.util.spec_from_file_location("scaling_model",
                                                  os.path.join(ROOT, "paper_1810_04597_b200", "scaling_model.py"))
    m = importlib.util.module_from_spec(spec)
    import sys

    sys.modules["scaling_model"] = m  # dataclasses resolve the module by name
    spec.loader.exec_module(m)
    return m


def test_amdahl_spec_examples():
    S = _S()
    assert S.amdahl(0.15, 28) == pytest.approx(5.5446, abs=1e-4)  # SPEC.md: "parallel speed-up of 5.5x"
    assert S.amdahl(0.0, 17) == 17
    assert S.amdahl(0.4, 1) == 1
    assert all(S.amdahl(0.1, n + 1) > S.amdahl(0.1, n) for n in range(1, 50))
    assert S.amdahl(0.1, 10 ** 9) < 10.0  # bounded by 1/f


def test_sweet_spot_examples():
    S = _S()
    assert S.sweet_spot([{"nslabs": 32, "sec_per_step": 1.0}, {"nslabs": 64, "sec_per_step": 0.9},
                         {"nslabs": 128, "sec_per_step": 1.1}]) == 64
    assert S.sweet_spot([{"nslabs": r, "sec_per_step": 1.0 / r} for r in (1, 2, 4, 8)]) == 8
    assert S.sweet_spot([{"nslabs": 2, "sec_per_step": 1.0}, {"nslabs": 4, "sec_per_step": 1.0}]) == 2
    with pytest.raises(ValueError):
        S.sweet_spot([])


def test_compute_only_limit():
    S = _S()
    m = S.Model(t_plane=2e-4, g=0.0, t_launch=0.0, fused_exposed=0.0)
    c = m.curve((512, 512, 512), [1, 2, 4, 8], mode="fused")
    for p in c:
        assert p["sec_per_step"] == pytest.approx(c[0]["sec_per_step"] / p["nslabs"], rel=1e-12)
    assert S.sweet_spot(c) == 8


def test_exchange_volume():
    S = _S()
    # 3 stages x 2 sides x 6 planes x 2 records x (8 x 512 + 8) doubles x 512 rows x 8 B
    assert S.exchange_bytes(512, 512) == 3 * 2 * 6 * 2 * (8 * 512 + 8) * 512 * 8
    # round 2's messages: 8 doubles per cell (echo_halo_doubles), about half
    assert S.exchange_bytes(512, 512, "r02") == 3 * 2 * 6 * 512 * 8 * 512 * 8


def test_calibration_reproduces_measurements():
    S = _S()
    prof = os.path.join(ROOT, "profiles")
    m = S.calibrate(prof)
    t1 = json.load(open(os.path.join(prof, "r01_bench_default.json")))["ms_per_step"] * 1e-3
    assert m.step_time((512, 512, 512), 1)["sec_per_step"] == pytest.approx(t1, rel=0.01)
    # S slabs on one GPU run serially: S x the per-slab step of an S-slab decomposition
    for name, s, mode in (("r01_bench_decomp_slabs2.json", 2, "copy"), ("r01_bench_decomp_slabs4.json", 4, "copy"),
                          ("r01_bench_decomp_slabs2_fused.json", 2, "fused"),
                          ("r01_bench_decomp_slabs4_fused.json", 4, "fused")):
        meas = json.load(open(os.path.join(prof, name)))["ms_per_step"] * 1e-3
        pred = s * m.step_time((512, 512, 512), s, mode=mode, link="local")["sec_per_step"]
        if mode == "fused":  # one GPU: the fused stores are part of the measured updates
            pred -= s * m.step_time((512, 512, 512), s, mode="fused", link="local")["exchange"]
        assert pred == pytest.approx(meas, rel=0.03), (name, pred, meas)
    # strong scaling on 8 GPUs over NVLink: better than 75% (the model's explanation of f1)
    c = m.curve((512, 512, 512), [1, 8], mode="fused")
    assert c[0]["sec_per_step"] / (8 * c[1]["sec_per_step"]) > 0.75
    # round 2's overlapped NCCL exchange: the 8-GPU messages (2 x 12.6 MB per stage) hide behind the
    # interior sweeps entirely, so only the ghost-plane work and the launches separate it from ideal
    o = m.curve((512, 512, 512), [1, 2, 4, 8], mode="overlap")
    assert all(p["exchange"] <= 12 * m.t_launch + 1e-12 for p in o[1:])
    assert o[0]["sec_per_step"] / (8 * o[3]["sec_per_step"]) > c[0]["sec_per_step"] / (8 * c[1]["sec_per_step"])
