"""Checkpoint / restart (SURVEY.md §5 "Checkpoint/resume", include/echo.h echo_checkpoint_*):
a run stopped after k steps, saved, loaded into a NEW context and continued must equal the
uninterrupted run bit for bit — every U^n and P value, the staggered field with UCT, and the
CFL dt sequence — on periodic, outflow, Kerr-Schild and UCT configurations."""
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


CASES = [
    (0, (32, 32, 32), {}),
    (2, (40, 36, 30), {}),              # outflow blast (A31 switch and floors in play)
    (4, (64, 32, 16), {}),              # Kerr-Schild torus (B in the P record, curved con2prim)
    (2, (40, 24, 20), {"divb": 2}),     # UCT: the staggered field is part of the state
    (3, (48, 40, 36), {"rec": 6}),      # characteristic-wise WENO5
]


def start(E, cfg, n, kw):
    p = I.problem(cfg, n=n)
    for k, v in kw.items():
        setattr(p, k, v)
    g = E.Echo(p)
    g.set_prims(I.initial_prims(p))
    if p.divb == 2:
        g.set_face_field(I.face_field(p))
    return p, g


def final(g, p):
    un, _, p5 = g.get_state()
    b = g.get_face_field() if p.divb == 2 else None
    return un, p5, b


@pytest.mark.parametrize("cfg,n,kw", CASES)
def test_checkpoint_restart_is_bitwise(E, cfg, n, kw):
    p, a = start(E, cfg, n, kw)
    dts_a = np.asarray(a.advance(4, p.cfl))
    ref = final(a, p)
    a.close()

    p, b = start(E, cfg, n, kw)
    dts_b1 = np.asarray(b.advance(2, p.cfl))
    ck = b.checkpoint()
    assert ck.size == E.checkpoint_doubles(b.ctx) > 0
    b.close()
    p, c = start(E, cfg, n, kw)          # a fresh context, its own (initial) state overwritten
    c.restore(ck)
    dts_b2 = np.asarray(c.advance(2, p.cfl))
    got = final(c, p)
    c.close()

    assert np.array_equal(np.concatenate([dts_b1, dts_b2]), dts_a)
    assert np.array_equal(got[0], ref[0]), "U^n differs after the restart"
    assert np.array_equal(got[1], ref[1]), "P differs after the restart"
    if p.divb == 2:
        assert np.array_equal(got[2], ref[2]), "b differs after the restart"


def test_checkpoint_host_loop_and_device_buffer(E):
    """the host loop (echo_max_dt + echo_step) across a checkpoint held in device memory"""
    import torch

    p, a = start(E, 0, (40, 24, 20), {})
    for _ in range(3):
        a.step(a.max_dt(p.cfl))
    ref = final(a, p)
    a.close()
    p, b = start(E, 0, (40, 24, 20), {})
    b.step(b.max_dt(p.cfl))
    buf = torch.empty(E.checkpoint_doubles(b.ctx), dtype=torch.float64, device="cuda")
    E.checkpoint_save(b.ctx, buf)
    p, c = start(E, 0, (40, 24, 20), {})
    E.checkpoint_load(c.ctx, buf)
    for _ in range(2):
        c.step(c.max_dt(p.cfl))
    got = final(c, p)
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])


def test_checkpoint_refused_inside_a_step(E):
    p, g = start(E, 0, (16, 16, 16), {})
    dt = g.max_dt(p.cfl)
    g.stage(1, dt)
    with pytest.raises(E.EchoError) as ei:
        g.checkpoint()
    assert ei.value.code == E.E_ORDER and "inside a step" in str(ei.value)
    g.stage(2, dt)
    g.stage(3, dt)
    g.checkpoint()  # at the step boundary again


def test_checkpoint_refused_on_slabs_and_without_state(E):
    p = I.problem(0, n=(16, 12, 8))
    g = E.Echo(p, bc=((0, 0), (0, 0), (E.BC_HALO, E.BC_HALO)))
    assert E.checkpoint_doubles(g.ctx) == 0
    with pytest.raises(E.EchoError) as ei:
        E.checkpoint_save(g.ctx, np.zeros(16))
    assert ei.value.code == E.E_ORDER and "slab" in str(ei.value)
    g.close()
    h = E.Echo(p)  # a state is needed before a save
    with pytest.raises(E.EchoError) as ei:
        h.checkpoint()
    assert ei.value.code == E.E_ORDER
