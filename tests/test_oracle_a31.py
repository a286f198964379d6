"""Reading A31, the DER shock switch, pinned from both sides.

PAPER.md:19 fixes only "high-order reconstruction algorithms" on a finite-difference
grid; BASELINE.json's north star asks for "the high-order flux derivative" (DER, A5)
AND for a blast wave that "stresses con2prim floors and shocks" (configs[2]) and a
torus with an atmosphere (configs[4]).  A31 drops the DER correction (H = F) at faces
whose 5-face stencil touches a relative rho or p jump above der_jump = 0.5.  Two
claims make it a reading rather than a tuning knob, and both are checked here on
the oracle alone (CPU):

1. inert on smooth data: on the config 0 / 1 / 3 recipes the rhs and a full SSP-RK3
   step are bit-for-bit the same with the switch on (0.5) and off (<= 0);
2. necessary at discontinuities: with the switch off, the config-2 blast and the
   config-4 torus fire floors / Newton failures and run away within a few steps,
   while with it on the blast stays floor-free and the torus fails no Newton solve.
"""
import numpy as np
import pytest

import echo_inputs as I


def _state(orc, cfg, n, der_jump):
    p = I.problem(cfg, n=n)
    p.der_jump = der_jump
    oc = orc.Cfg(**p.grid_kwargs())
    U, P = orc.set_prims(oc, I.initial_prims(p))
    return p, oc, U, P


@pytest.mark.parametrize("cfg,n", [(0, (32, 32, 32)), (1, (128, 128, 128)), (3, (64, 64, 64))])
def test_a31_bitwise_inert_on_smooth_configs(orc, cfg, n):
    """Config 0 at its full size, config 1 at its full size, config 3's recipe (32 modes,
    k <= 8) at 64^3, where its cell-to-cell jumps are 8x those at 512^3."""
    outs = []
    for dj in (0.5, 0.0):
        p, oc, U, P = _state(orc, cfg, n, dj)
        L = orc.rhs(oc, U, P)
        dt = orc.max_dt(oc, U, P, p.cfl)
        U1, P1, cnt = orc.step(oc, dt, U, P)
        outs.append((L, U1, P1, cnt))
    (La, Ua, Pa, ca), (Lb, Ub, Pb, cb) = outs
    assert np.array_equal(La, Lb) and np.array_equal(Ua, Ub) and np.array_equal(Pa, Pb)
    assert tuple(ca) == tuple(cb) == (0, 0)


def _run(orc, cfg, n, dj, steps):
    p, oc, U, P = _state(orc, cfg, n, dj)
    cnt = [0, 0]
    for _ in range(steps):
        dt = orc.max_dt(oc, U, P, p.cfl)
        U, P, c = orc.step(oc, dt, U, P)
        cnt[0] += c[0]
        cnt[1] += c[1]
    return cnt, float(P[4].max())


def test_a31_needed_for_the_blast(orc):
    """Config 2's recipe (p jump 1000x at r = 0.1) on 64^3, 3 steps: without the switch the
    DER correction's overshoot at the jump drives p <= 0 (floors on the first step) and the
    pressure runs away; with it, no floor fires and max p stays at the initial 1."""
    on, pmax_on = _run(orc, 2, (64, 64, 64), 0.5, 3)
    off, pmax_off = _run(orc, 2, (64, 64, 64), 0.0, 3)
    assert on == [0, 0] and pmax_on < 1.001
    assert off[0] > 1000 and pmax_off > 100.0


def test_a31_needed_for_the_torus(orc):
    """Config 4's torus (Kerr-Schild a = 0.9) on 64 x 32 x 16, 10 steps: the atmosphere
    floors fire either way (rho = 1e-6 meets the torus edge, counted, A9), but only without
    the switch do Newton solves fail and the pressure run away (the torus has p <= 1e-3)."""
    on, pmax_on = _run(orc, 4, (64, 32, 16), 0.5, 10)
    off, pmax_off = _run(orc, 4, (64, 32, 16), 0.0, 10)
    assert on[1] == 0 and pmax_on < 2e-3
    assert off[1] > 1000 and pmax_off > 1.0
