"""P6: the oracle's L(U) on 4^3 grids against a 50-digit mpmath transcription
(tests/bruteforce_mp.py) that shares no code with oracle/*.c and takes its
metric derivatives by numerical differentiation.  CPU only."""
import math

import numpy as np
import pytest

import echo_inputs as I
from tests import bruteforce_mp as B
from tests.util import CONS_GROUPS, group_errors


def _compare(orc, c, G, P8, tol=1e-13):
    U, P = orc.set_prims(c, np.ascontiguousarray(P8))
    L = orc.rhs(c, U, P)
    S = B.Scheme(G, U, P)
    n = c.n
    Lmp = np.zeros_like(L)
    for k in range(n[2]):
        for j in range(n[1]):
            for i in range(n[0]):
                Lmp[:, k, j, i] = [float(v) for v in S.rhs_cell([i, j, k])]
    errs = group_errors(L, Lmp, CONS_GROUPS)
    assert all(e <= tol for e in errs.values()), errs
    return errs


def test_bruteforce_periodic_turbulence(orc):
    p = I.problem(0, n=(4, 4, 4), seed=11)
    p.params.update(amp=0.2, vmax=0.5)
    P8 = I.initial_prims(p)
    c = orc.Cfg(**p.grid_kwargs())
    G = B.Grid(p.n, p.lo, p.hi, p.bc)
    _compare(orc, c, G, P8)


@pytest.mark.parametrize("divb,der,rec", [(1, 4, 0), (0, 6, 1), (0, 6, 2), (1, 6, 2), (0, 6, 3), (0, 2, 4), (0, 4, 5),
                                          (0, 6, 6), (1, 6, 6)])
def test_bruteforce_switches(orc, divb, der, rec):
    p = I.problem(0, n=(4, 4, 4), seed=12)
    p.params.update(amp=0.2, vmax=0.5)
    P8 = I.initial_prims(p)
    c = orc.Cfg(**{**p.grid_kwargs(), "divb": divb, "der": der, "rec": rec})
    G = B.Grid(p.n, p.lo, p.hi, p.bc, divb=divb, der=der, rec=rec)
    _compare(orc, c, G, P8)


@pytest.mark.parametrize("rec", [0, 2, 3, 4, 5, 6])
def test_bruteforce_outflow_blast(orc, rec):
    # outflow in x and y, periodic z; a pressure jump exercises the positivity fallback
    # (and, rec=2, the MP5 limiter)
    n = (4, 4, 4)
    bc = ((1, 1), (1, 1), (0, 0))
    P8 = I.uniform_prims(n, 0.01, (0, 0, 0), 1e-3, (0.1, 0.05, 0.0))
    P8[4, :, :2, :2] = 1.0
    P8[0] *= 1 + 0.1 * I.white_noise(5, 64).reshape(4, 4, 4)
    P8[1, 1, 2, 1] = 0.3
    c = orc.Cfg(n=n, bc=bc, rec=rec)
    G = B.Grid(n, (0, 0, 0), (1, 1, 1), bc, rec=rec)
    _compare(orc, c, G, P8)


def test_bruteforce_kerr_schild_patch(orc):
    # a 4^3 patch of the torus on Kerr-Schild (a = 0.9), with a magnetic field
    n = (4, 4, 4)
    lo = (math.log(9.0), 1.3, 0.0)
    hi = (math.log(11.0), 1.8, 0.4)
    bc = ((1, 1), (1, 1), (0, 0))
    p = I.problem(4, n=n)
    p.lo, p.hi = lo, hi
    P8 = I.initial_prims(p)
    P8[5] = 1e-3 * (1 + 0.3 * I.white_noise(7, 64).reshape(4, 4, 4))
    P8[6] = 2e-3 * (1 + 0.3 * I.white_noise(8, 64).reshape(4, 4, 4))
    P8[7] = 1e-3
    c = orc.Cfg(**{**p.grid_kwargs(), "lo": lo, "hi": hi, "bc": bc})
    G = B.Grid(n, lo, hi, bc, metric=1, M=1, a=0.9)
    _compare(orc, c, G, P8, tol=1e-12)


def _compare_uct(orc, c, G, P8, b3, tol=1e-13):
    U, P, b = orc.set_prims_uct(c, np.ascontiguousarray(P8), np.ascontiguousarray(b3))
    L = orc.rhs_uct(c, U, P, b)
    S = B.SchemeUCT(G, U, P, b)
    n = c.n
    Lmp = np.zeros_like(L)
    for k in range(n[2]):
        for j in range(n[1]):
            for i in range(n[0]):
                Lmp[:, k, j, i] = [float(v) for v in S.rhs_cell([i, j, k])]
    errs = group_errors(L, Lmp, {"D": [0], "S": [1, 2, 3], "tau": [4], "b": [5, 6, 7]})
    assert all(e <= tol for e in errs.values()), errs
    return errs


@pytest.mark.parametrize("rec", [0, 2])
def test_bruteforce_uct_periodic(orc, rec):
    # f2 / A37-A41: the oracle's UCT rhs (hydro with staggered normal fields + L(b) from the
    # edge EMFs) against the independent mpmath transcription in bruteforce_mp.SchemeUCT
    p = I.problem(0, n=(4, 4, 4), seed=13)
    p.params.update(amp=0.2, vmax=0.5)
    p.divb, p.rec = 2, rec
    c = orc.Cfg(**p.grid_kwargs())
    G = B.Grid(p.n, p.lo, p.hi, p.bc, divb=2, rec=rec)
    _compare_uct(orc, c, G, I.initial_prims(p), I.face_field(p))


def test_bruteforce_uct_outflow_and_kerr_schild(orc):
    # A42 ghost rule on outflow sides, A43 transport velocity and face metric (a = 0.9 patch)
    n = (4, 4, 4)
    lo = (math.log(9.0), 1.3, 0.0)
    hi = (math.log(11.0), 1.8, 0.4)
    bc = ((1, 1), (1, 1), (0, 0))
    p = I.problem(4, n=n)
    p.lo, p.hi = lo, hi
    P8 = I.initial_prims(p)
    b3 = np.ascontiguousarray(np.stack([2e-1 * (1 + 0.3 * I.white_noise(17, 64).reshape(4, 4, 4)),
                                        3e-1 * (1 + 0.3 * I.white_noise(18, 64).reshape(4, 4, 4)),
                                        np.full((4, 4, 4), 0.1)]))
    c = orc.Cfg(**{**p.grid_kwargs(), "lo": lo, "hi": hi, "bc": bc, "divb": 2})
    G = B.Grid(n, lo, hi, bc, metric=1, M=1, a=0.9, divb=2)
    _compare_uct(orc, c, G, P8, b3, tol=1e-12)
