"""The fused update + x sweep (fused.cu): the update of stage s also sweeps x for
the state it produces, into the second accumulator.  It must give bit-for-bit the results of
the separate kernels (the default; ECHO_FUSED_UPDATE=1 at echo_create turns the fusion on) on every path that interleaves
it with other calls: host stages, echo_step, echo_advance (two step graphs, one per
accumulator parity), echo_rhs after a step, state setters in between.  Marked gpu."""
import os

import numpy as np
import pytest

import echo_inputs as I

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


def make(E, p, fused):
    old = os.environ.pop("ECHO_FUSED_UPDATE", None)
    if fused:
        os.environ["ECHO_FUSED_UPDATE"] = "1"
    try:
        return E.Echo(p)
    finally:
        os.environ.pop("ECHO_FUSED_UPDATE", None)
        if old is not None:
            os.environ["ECHO_FUSED_UPDATE"] = old


def script(E, g, p, P8):
    """Every call pattern: stages one by one, rhs, steps, a device loop of odd length (the
    accumulator parity flips), a state setter in the middle, another loop."""
    out = []
    g.set_prims(P8)
    dt = g.max_dt(p.cfl)
    for s in (1, 2, 3):
        g.stage(s, dt)
        out.append(g.get_state())
    out.append(g.rhs())
    g.step(g.max_dt(p.cfl))
    out.append(g.rhs())
    out.append(g.advance(3, p.cfl))
    out.append(g.get_state())
    g.step(g.max_dt(p.cfl))
    out.append(g.get_state())
    E.set_cons(g.ctx, np.ascontiguousarray(g.get_cons()))
    out.append(g.advance(2, p.cfl))
    out.append(g.get_state())
    out.append(g.get_prims())
    st = g.stats()
    out.append(np.array([st["floor_events"], st["c2p_failures"]], dtype=np.float64))
    return out


def flat(xs):
    for x in xs:
        if isinstance(x, tuple):
            yield from flat(x)
        else:
            yield np.asarray(x)


@pytest.mark.parametrize("cfg,n,kw", [(0, (32, 32, 32), {}), (2, (40, 36, 34), {}), (0, (70, 13, 9), {"rec": 2}),
                                      (0, (33, 9, 10), {"divb": 1, "der": 4}), (2, (45, 38, 41), {"rec": 5})])
def test_fused_update_bitwise(E, cfg, n, kw):
    p = I.problem(cfg, n=n)
    for k, v in kw.items():
        setattr(p, k, v)
    P8 = I.initial_prims(p)
    ref = script(E, make(E, p, False), p, P8)
    got = script(E, make(E, p, True), p, P8)
    for a, b in zip(flat(got), flat(ref)):
        assert a.shape == b.shape and np.array_equal(a, b)


def test_fused_kernel_is_the_one_launched(E):
    """The fused context launches update_sweep_x and no separate update; the unfused none."""
    p = I.problem(0, n=(32, 32, 32))
    P8 = I.initial_prims(p)
    for fused in (True, False):
        g = make(E, p, fused)
        g.set_prims(P8)
        E.profile(g.ctx, True)
        g.step(g.max_dt(p.cfl))
        g.step(g.max_dt(p.cfl))
        prof = E.profile_read(g.ctx)
        E.profile(g.ctx, False)
        if fused:
            assert prof["update_sweep_x"][1] == 6 and prof["update_stage"][1] == 0
            assert prof["sweep_x"][1] == 1  # only the very first stage sweeps x on its own
        else:
            assert prof["update_sweep_x"][1] == 0 and prof["update_stage"][1] == 6 and prof["sweep_x"][1] == 6
        g.close()
