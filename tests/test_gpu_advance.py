"""echo_advance (include/echo.h): K steps with the time step computed on the device and
each step replayed from one captured CUDA graph.  The dt kernel divides cfl by the
same reduction echo_max_dt reads back (IEEE division on both sides), and the captured
kernels are the ones echo_step launches, so K x (echo_max_dt + echo_step) and
echo_advance(K) must agree BIT FOR BIT in dt sequence and state.  Marked gpu."""
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


@pytest.mark.parametrize("cfg,n,steps", [
    (0, (32, 32, 32), 4),     # periodic turbulence
    (1, (24, 16, 20), 3),     # CP Alfven, ragged grid
    (2, (32, 32, 32), 3),     # outflow blast (floors may fire)
    (4, (32, 16, 32), 2),     # Kerr-Schild torus
])
def test_advance_matches_host_loop_bitwise(E, cfg, n, steps):
    p = I.problem(cfg, n=n)
    P8 = I.initial_prims(p)
    a, b = E.Echo(p), E.Echo(p)
    a.set_prims(P8)
    b.set_prims(P8)
    dts = []
    for _ in range(steps):
        dt = a.max_dt(p.cfl)
        dts.append(dt)
        a.step(dt)
    # split over two calls: the second replays the graph captured by the first
    d1 = b.advance(steps - 1, p.cfl)
    d2 = b.advance(1, p.cfl)
    got = np.concatenate([d1, d2])
    assert got.tolist() == dts
    ua, _, pa = a.get_state()
    ub, _, pb = b.get_state()
    assert np.array_equal(ua, ub) and np.array_equal(pa, pb)
    sa, sb = a.stats(), b.stats()
    assert sa == sb
    # after advance the CFL reduction of the final state is valid for the host path too
    assert b.max_dt(p.cfl) == a.max_dt(p.cfl)


def test_advance_cfl_change_recaptures_and_arguments(E):
    p = I.problem(0, n=(16, 16, 16))
    P8 = I.initial_prims(p)
    a, b = E.Echo(p), E.Echo(p)
    a.set_prims(P8)
    b.set_prims(P8)
    for cfl in (0.4, 0.2, 0.4):
        dt = a.max_dt(cfl)
        a.step(dt)
        assert b.advance(1, cfl).tolist() == [dt]
    assert np.array_equal(a.get_state()[0], b.get_state()[0])
    assert b.advance(0, 0.4).tolist() == []
    assert b.advance(2, 0.4, log=False) is None
    with pytest.raises(E.EchoError):
        b.advance(1, 0.0)
    with pytest.raises(E.EchoError):
        b.advance(-1, 0.4)
    b.stage(1, 1e-4)  # a step in progress
    with pytest.raises(E.EchoError):
        b.advance(1, 0.4)


def test_advance_profiled_path_matches(E):
    """with per-kernel profiling on, the loop is issued without the graph: same bits"""
    p = I.problem(0, n=(16, 16, 16))
    P8 = I.initial_prims(p)
    a, b = E.Echo(p), E.Echo(p)
    a.set_prims(P8)
    b.set_prims(P8)
    E.profile(b.ctx, True)
    da = a.advance(3, p.cfl)
    db = b.advance(3, p.cfl)
    assert da.tolist() == db.tolist()
    assert np.array_equal(a.get_state()[0], b.get_state()[0])
