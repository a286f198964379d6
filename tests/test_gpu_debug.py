"""Failure detection (SURVEY.md §8(b) "Errors": ECHO_E_NONFINITE comes from a debug-mode
NaN scan naming the first bad cell; §5 "Failure detection"): echo_check_finite and the
ECHO_DEBUG_NANSCAN mode of echo_step / echo_advance.  Marked gpu."""
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


def test_check_finite_names_the_first_bad_cell(E):
    p = I.problem(0, n=(12, 10, 8))
    g = E.Echo(p)
    g.set_prims(I.initial_prims(p))
    g.check_finite()  # a clean state passes
    g.step(g.max_dt(p.cfl))
    g.check_finite()
    # poison one magnetic-field value (floors never rewrite U_B, A9) through the C-ABI's state
    # setter, and a later cell in linear order, which must not be the one reported
    U = g.get_cons()
    U[6, 5, 4, 7] = np.nan
    U[5, 6, 0, 0] = np.inf
    E.set_cons(g.ctx, np.ascontiguousarray(U))
    with pytest.raises(E.EchoError) as ei:
        g.check_finite()
    assert ei.value.code == E.E_NONFINITE
    assert "(7,4,5)" in str(ei.value), str(ei.value)
    g.close()


def test_debug_scan_stops_step_and_advance(E):
    p = I.problem(0, n=(16, 12, 10))
    P8 = I.initial_prims(p)
    # an absurd dt overflows the RK combine: the scan must catch it at stage 1
    g = E.Echo(p)
    g.set_prims(P8)
    g.set_debug()
    with pytest.raises(E.EchoError) as ei:
        g.step(1e300)
    assert ei.value.code == E.E_NONFINITE and "stage 1" in str(ei.value), str(ei.value)
    g.close()
    # echo_advance: halts on the device and reports at its end
    g = E.Echo(p)
    g.set_prims(P8)
    g.set_debug()
    with pytest.raises(E.EchoError) as ei:
        g.advance(3, 1e300)
    assert ei.value.code == E.E_NONFINITE and "debug scan" in str(ei.value), str(ei.value)
    g.close()


def test_debug_scan_is_transparent(E):
    """On a healthy run the scan changes nothing: bitwise the same state, host and device loop."""
    p = I.problem(2, n=(24, 20, 18))
    P8 = I.initial_prims(p)
    outs = []
    for dbg in (0, 1):
        g = E.Echo(p)
        g.set_prims(P8)
        if dbg:
            g.set_debug()
        for _ in range(2):
            g.step(g.max_dt(p.cfl))
        g.advance(2, p.cfl)
        outs.append(g.get_state())
        g.close()
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
