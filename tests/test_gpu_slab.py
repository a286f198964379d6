"""z-slab domain decomposition on one GPU: the grid
split into 2-3 slabs held by one process, ghost planes exchanged by device copies
between the contexts before every stage (paper_1810_04597_b200/slab.py LocalSlabs).
Every face flux is computed by one thread from the same inputs in both runs, so the
decomposed step must reproduce the single-domain step BIT FOR BIT; it is also
checked against the oracle.  Marked gpu."""
import numpy as np
import pytest

import echo_inputs as I
from tests.util import CONS_GROUPS, PRIM5_GROUPS, assert_groups

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


@pytest.mark.parametrize("fused", [False, True, "split"])
@pytest.mark.parametrize("cfg,n,nslabs,steps", [
    (0, (32, 24, 32), 2, 3),     # periodic turbulence: a ring of 2 (both neighbours the same slab)
    (0, (20, 16, 40), 3, 3),     # periodic, 3 unequal slabs (14/13/13 planes)
    (0, (16, 16, 16), 1, 2),     # one periodic slab: its own neighbour on both sides
    (2, (16, 16, 20), 1, 2),     # one outflow slab: no halo side at all (nothing to exchange)
    (2, (24, 20, 36), 3, 3),     # outflow blast: physical ends filled locally, shocks crossing slab edges
    (4, (48, 24, 24), 2, 2),     # Kerr-Schild torus, slabs in phi
])
def test_slabs_match_single_domain_bitwise(E, orc, cfg, n, nslabs, steps, fused):
    """fused=False: export/copy/import before every stage; fused=True: the updates store
    their edge planes into the neighbours' ghost planes (echo_halo_link); "split": the copy
    exchange between each stage's interior sweeps and its boundary sweeps (DistSlab.step's
    overlap, echo_stage_sweeps_interior / _boundary)."""
    from paper_1810_04597_b200.slab import LocalSlabs

    p = I.problem(cfg, n=n)
    P8 = I.initial_prims(p)
    one = E.Echo(p)
    one.set_prims(P8)
    sl = LocalSlabs(p, nslabs, fused=fused is True)
    sl.set_prims(P8)
    for _ in range(steps):
        dt1 = one.max_dt(p.cfl)
        dts = sl.max_dt(p.cfl)
        assert dts == dt1  # max over cells is order independent
        one.step(dt1)
        sl.step(dts, split=fused == "split")
    un1, _, p1 = one.get_state()
    uns = sl.gather(lambda g: g.get_state()[0])
    ps = sl.gather(lambda g: g.get_state()[2])
    assert np.array_equal(uns, un1) and np.array_equal(ps, p1)
    # and the oracle agrees with both at the multi-step tolerance
    oc = orc.Cfg(**p.grid_kwargs())
    U, P = orc.set_prims(oc, P8)
    for _ in range(steps):
        U, P, _ = orc.step(oc, orc.max_dt(oc, U, P, p.cfl), U, P)
    assert_groups(uns, U, CONS_GROUPS, 1e-10, what="slabs U")
    assert_groups(ps, P, PRIM5_GROUPS, 1e-10, what="slabs P")
    st = [g.stats() for g, _, _ in sl.parts]
    assert sum(s["floor_events"] for s in st) == one.stats()["floor_events"]
    sl.close()
    one.close()


def test_slab_api_errors(E):
    p = I.problem(0, n=(8, 8, 12))
    g = E.Echo(p, bc=((0, 0), (0, 0), (E.BC_HALO, E.BC_HALO)))
    g.set_prims(I.initial_prims(p))
    with pytest.raises(E.EchoError) as ei:
        g.step(1e-3)  # a slab needs an exchange before every stage
    assert ei.value.code == E.E_ORDER
    with pytest.raises(E.EchoError):
        g.advance(1, 0.4)  # so does the device-driven loop
    with pytest.raises(E.EchoError):
        E.halo_fill(g.ctx, 0)  # a halo side is imported, not filled
    with pytest.raises(E.EchoError) as ei:
        E.stage_sweeps_boundary(g.ctx, 1)  # the interior half comes first
    assert ei.value.code == E.E_ORDER
    E.stage_sweeps_interior(g.ctx, 1)
    with pytest.raises(E.EchoError):
        g.stage(1, 1e-3)  # a half-swept stage is finished by its boundary half only
    with pytest.raises(E.EchoError):
        E.create(n=(8, 8, 4), lo=(0, 0, 0), hi=(1, 1, 1), bc=((0, 0), (0, 0), (2, 2)))  # thinner than the halo
    with pytest.raises(E.EchoError):
        E.create(n=(8, 8, 8), lo=(0, 0, 0), hi=(1, 1, 1), bc=((2, 2), (0, 0), (0, 0)))  # halo only along z
    g.close()


@pytest.mark.parametrize("cfg,n,nslabs,steps", [
    (0, (24, 20, 32), 2, 2),     # periodic turbulence, a ring of 2
    (0, (20, 16, 27), 3, 2),     # 3 unequal periodic slabs (9 planes each)
    (2, (20, 18, 36), 3, 2),     # outflow blast: physical ends filled locally (b included, A42)
    (4, (48, 35, 24), 2, 2),     # Kerr-Schild torus, slabs in phi
])
def test_uct_slabs_match_single_domain_bitwise(E, orc, cfg, n, nslabs, steps):
    """UCT (divb = 2) on z slabs with the copy exchange: ECHO_HALO_PLANES_UCT = 8 ghost planes,
    the messages carry the staggered field too; the x/y sweeps and the z sweep cover 5 ghost
    planes, the edge EMFs 3.  Bit for bit the single-domain UCT run, b included."""
    from paper_1810_04597_b200.slab import LocalSlabs

    p = I.problem(cfg, n=n)
    p.divb = 2
    P8, b3 = I.initial_prims(p), I.face_field(p)
    one = E.Echo(p)
    one.set_prims(P8)
    one.set_face_field(b3)
    sl = LocalSlabs(p, nslabs)
    sl.set_prims(P8)
    sl.set_face_field(b3)
    assert np.array_equal(sl.gather(lambda g: g.get_state()[0]), one.get_state()[0])  # the centring, edges included
    for _ in range(steps):
        dt1 = one.max_dt(p.cfl)
        assert sl.max_dt(p.cfl) == dt1
        one.step(dt1)
        sl.step(dt1)
    assert np.array_equal(sl.gather(lambda g: g.get_state()[0]), one.get_state()[0])
    assert np.array_equal(sl.gather(lambda g: g.get_state()[2]), one.get_state()[2])
    assert np.array_equal(sl.gather(lambda g: g.get_face_field()), one.get_face_field())
    st = [g.stats() for g, _, _ in sl.parts]
    assert sum(s["floor_events"] for s in st) == one.stats()["floor_events"]
    sl.close()
    one.close()


def test_uct_slab_refusals(E):
    """UCT slabs: thinner than 8 planes, or the fused links, are refused."""
    with pytest.raises(E.EchoError):
        E.create(n=(8, 8, 7), lo=(0, 0, 0), hi=(1, 1, 1), bc=((0, 0), (0, 0), (2, 2)), divb=2)
    p = I.problem(0, n=(8, 8, 16))
    p.divb = 2
    g = E.Echo(p, bc=((0, 0), (0, 0), (E.BC_HALO, E.BC_HALO)))
    with pytest.raises(E.EchoError):
        E.halo_link(g.ctx, 0, g.ctx)
    g.close()


def test_destroy_unlinks_the_peers(E):
    """A context linked to a peer (echo_halo_link) forgets the link when the peer is destroyed:
    its updates can no longer store into freed ghost planes (echo_halo_pull then reports the
    side as unlinked)."""
    p = I.problem(0, n=(8, 8, 24))
    bc = ((0, 0), (0, 0), (E.BC_HALO, E.BC_HALO))
    a = E.Echo(p, n=(8, 8, 12), bc=bc)
    b = E.Echo(p, n=(8, 8, 12), bc=bc)
    E.halo_link(a.ctx, 1, b.ctx)
    E.halo_link(b.ctx, 0, a.ctx)
    P8 = I.initial_prims(I.problem(0, n=(8, 8, 12)))
    a.set_prims(P8)
    b.set_prims(P8)
    E.halo_pull(a.ctx, 1)  # linked: fine
    b.close()
    with pytest.raises(E.EchoError) as ei:
        E.halo_pull(a.ctx, 1)
    assert "not linked" in str(ei.value)
    a.close()
