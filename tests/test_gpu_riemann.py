"""The GPU path on the relativistic shock tubes of tests/test_oracle_riemann.py, along each of the
three axes (the x, y and z sweeps are different kernels): it converges to the exact Riemann
solution in L1 as the oracle does, and its errors agree with the oracle's.  Marked gpu."""
from dataclasses import replace

import numpy as np
import pytest

import echo_inputs as I
from tests.test_oracle_riemann import TUBES, l1_errors, run_oracle, tube_prims

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1810_04597_b200 import build

    build.build()
    from paper_1810_04597_b200 import echo

    return echo


def run_gpu(E, N, L, R, tend, axis, cfl=0.4):
    n = [1, 1, 1]
    n[axis] = N
    hi = [1.0 / N] * 3
    hi[axis] = 1.0
    bc = [(I.PERIODIC, I.PERIODIC)] * 3
    bc[axis] = (I.OUTFLOW, I.OUTFLOW)
    p = replace(I.problem(0, n=tuple(n)), hi=tuple(hi), bc=tuple(bc), cfl=cfl)
    P8 = tube_prims(N, L, R)  # [8][1][1][N] along x
    if axis:
        P8 = np.moveaxis(P8, 3, 3 - axis).copy()
        vel = P8[1].copy()
        P8[1] = 0.0
        P8[1 + axis] = vel
    g = E.Echo(p)
    g.set_prims(P8)
    t = 0.0
    while t < tend * (1 - 1e-14):
        dt = min(g.max_dt(cfl), tend - t)
        g.step(dt)
        t += dt
    out = g.get_prims().reshape(8, -1)
    st = g.stats()
    g.close()
    return out[0], out[4], out[1 + axis], [st["floor_events"], st["c2p_failures"]]


@pytest.mark.parametrize("name", list(TUBES))
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_gpu_converges_to_the_exact_riemann_solution(E, orc, name, axis):
    L, R, tend = TUBES[name]
    errs = []
    for N in (100, 200, 400):
        rho, p, v, events = run_gpu(E, N, L, R, tend, axis)
        assert events == [0, 0]
        errs.append(l1_errors(rho, p, v, N, L, R, tend))
    errs = np.array(errs)
    overall = np.log2(errs[0] / errs[-1]) / 2
    assert np.all(overall > 0.7) and np.all(np.log2(errs[:-1] / errs[1:]) > 0.3), (name, axis, errs)
    # the oracle's errors at N = 400 (same scheme, same dt sequence up to rounding)
    ro, po, vo, _ = run_oracle(orc, 400, L, R, tend)
    eo = np.array(l1_errors(ro, po, vo, 400, L, R, tend))
    assert np.allclose(errs[-1], eo, rtol=1e-3, atol=0.0), (name, axis, errs[-1], eo)
