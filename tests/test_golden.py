"""The golden fixtures (tests/golden/): every value carries its citation, and SPEC.md's worked
examples that hold for this scheme are checked against the oracle here (the SURVEY App. A
values are used by test_oracle_pointwise / test_oracle_scheme).  CPU only."""
import glob
import json
import math
import os

import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_every_fixture_is_cited():
    files = sorted(glob.glob(os.path.join(GOLDEN, "*.json")))
    assert len(files) >= 5
    for f in files:
        d = json.load(open(f))
        assert d.get("cite"), f
        assert "SPEC.md" in d["cite"] or "SURVEY.md" in d["cite"], f


def test_spec_worked_values(orc):
    d = json.load(open(os.path.join(GOLDEN, "spec_worked_values.json")))
    for case in d["weno5"]:
        for rec in (0, 1):  # A2's point form and SPEC's finite-volume form agree on these
            assert orc.weno5_left(case["stencil"], rec) == pytest.approx(case["value"], rel=1e-15), case["cite"]
    fr = d["flux_rest_state"]
    W = 1.0 / math.sqrt(1.0 - sum(v * v for v in fr["v"]))
    pr = [fr["rho"], *(W * v for v in fr["v"]), fr["p"], *fr["B"]]
    f = orc.flux_pt(orc.Cfg(), [0.5, 0.5, 0.5], pr, fr["axis"])
    assert list(f) == fr["flux"], fr["cite"]
    for a in range(3):  # the induction flux's own component is 0 for every state and axis
        pr2 = [0.7, 0.2, -0.1, 0.3, 0.4, 0.3, -0.5, 0.8]
        f2 = orc.flux_pt(orc.Cfg(), [0.5, 0.5, 0.5], pr2, a)
        # slots 5..7 hold the fluxes of B^1..3; the a-th is the normal one
        assert f2[5 + a] == 0.0
