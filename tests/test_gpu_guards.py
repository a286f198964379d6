"""Out-of-bounds write detection on every kernel path (SURVEY §4 "Sanitizers", §5 race /
memory checks).  compute-sanitizer is closed on this build's GPU pool
(profiles/r02_sanitizer_closed.txt), so the library's own guard bands stand in for memcheck's
write checks: with ECHO_GUARD_BANDS=1 every state array sits between two 32 KB bands of 0xA5
bytes, and echo_check_guards verifies them after each call.  Grids are chosen ragged and small
(lines shorter than a chunk, odd sizes, single-cell axes) so that the march's tail and ghost
index maps are at their limits.  Marked gpu."""
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


def guarded(E, p):
    os.environ["ECHO_GUARD_BANDS"] = "1"
    try:
        return E.Echo(p)
    finally:
        os.environ.pop("ECHO_GUARD_BANDS", None)


CASES = [
    (0, (33, 9, 10), {}),                    # one cell past a chunk along x, short y/z lines
    (0, (1, 16, 1), {}),                     # single-cell x and z axes
    (2, (5, 3, 7), {}),                      # outflow everywhere, below one chunk
    (4, (36, 35, 8), {}),                    # Kerr-Schild (metric tables, sources)
    (0, (20, 12, 9), {"rec": 6}),            # characteristic-wise reconstruction
    (0, (20, 12, 9), {"rec": 5, "der": 4}),  # PPM, DER4
    (2, (17, 11, 13), {"divb": 2}),          # UCT: face data, edge EMFs, induction, centring
    (0, (18, 14, 12), {"divb": 1, "rec": 2}),
]


@pytest.mark.parametrize("cfg,n,kw", CASES)
def test_no_out_of_bounds_writes(E, cfg, n, kw):
    p = I.problem(cfg, n=n)
    for k, v in kw.items():
        setattr(p, k, v)
    g = guarded(E, p)
    g.set_prims(I.initial_prims(p))
    if p.divb == 2:
        g.set_face_field(I.face_field(p))
    g.check_guards()
    dt = g.max_dt(p.cfl)
    for s in (1, 2, 3):
        g.stage(s, dt)
        g.check_guards()
    g.rhs()
    g.check_guards()
    g.step(g.max_dt(p.cfl))
    g.advance(2, p.cfl)
    g.check_guards()
    if p.divb != 2:  # (UCT keeps its field staggered: no cons setter)
        E.set_cons(g.ctx, np.ascontiguousarray(g.get_cons()))
    else:
        g.set_face_field(g.get_face_field())
    g.get_prims()
    g.get_state()
    g.check_guards()
    g.close()


def test_fused_update_no_out_of_bounds_writes(E):
    p = I.problem(0, n=(33, 13, 9))
    os.environ["ECHO_FUSED_UPDATE"] = "1"
    try:
        g = guarded(E, p)
    finally:
        os.environ.pop("ECHO_FUSED_UPDATE", None)
    g.set_prims(I.initial_prims(p))
    for _ in range(2):
        g.step(g.max_dt(p.cfl))
    g.advance(3, p.cfl)
    g.check_guards()
    g.close()


def test_guards_off_is_an_order_error(E):
    g = E.Echo(I.problem(0, n=(8, 8, 8)))
    with pytest.raises(E.EchoError) as ei:
        g.check_guards()
    assert ei.value.code == E.E_ORDER
    g.close()
