"""GPU parity of the UCT mode (divb = 2: staggered field + upwind constrained transport;
SURVEY.md §8(f) f2, readings A37-A41) against the oracle's UCT path, same
seeded inputs, element by element, normwise per variable group (A16): 1e-12 per stage
(rhs incl. L(b) at the faces, stage outputs incl. the staggered field), 1e-10 after 10
steps; plus the invariant the scheme exists for (div_H b preserved to roundoff on the
GPU) and the API rules.  Marked gpu."""
import numpy as np
import pytest

import echo_inputs as I
from tests.util import CONS_GROUPS, PRIM5_GROUPS, assert_groups, assert_rhs_groups, flux_scale

pytestmark = pytest.mark.gpu

TOL_STAGE = 1e-12
TOL_10 = 1e-10
HYDRO = {"D": [0], "S": [1, 2, 3], "tau": [4]}
FACE = {"b": [0, 1, 2]}


@pytest.fixture(scope="module")
def E():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1810_04597_b200 import build

    build.build()
    from paper_1810_04597_b200 import echo

    return echo


def uct_problem(cfg, n, rec=0):
    p = I.problem(cfg, n=n)
    p.divb = 2
    p.rec = rec
    return p


def start(E, orc, p):
    P8 = I.initial_prims(p)
    b = I.face_field(p)
    oc = orc.Cfg(**p.grid_kwargs())
    U, P, ob = orc.set_prims_uct(oc, P8, b)
    g = E.Echo(p)
    g.set_prims(P8)
    g.set_face_field(b)
    return oc, g, U, P, ob


CASES = [(0, (32, 32, 32)), (0, (70, 13, 36)), (1, (24, 20, 28)), (2, (45, 38, 41)), (3, (40, 40, 40)),
         (4, (72, 35, 24))]


@pytest.mark.parametrize("cfg,n", CASES)
def test_uct_rhs_and_stage_parity(E, orc, cfg, n):
    p = uct_problem(cfg, n)
    oc, g, U, P, ob = start(E, orc, p)
    gun, _, gp = g.get_state()
    assert_groups(gun, U, CONS_GROUPS, TOL_STAGE, what="set: U (B = I6(b))")
    assert np.array_equal(g.get_face_field(), ob)
    dt = orc.max_dt(oc, gun, gp, p.cfl)
    assert g.max_dt(p.cfl) == pytest.approx(dt, rel=1e-14)
    L = orc.rhs_uct(oc, gun, gp, ob)
    Lg = g.rhs()
    fs = flux_scale(orc, oc, gun, gp)
    assert_rhs_groups(Lg[:5], L[:5], gun[:5], dt, HYDRO, TOL_STAGE, what=f"uct rhs hydro cfg{cfg}", fscale=fs)
    assert_rhs_groups(Lg[5:], L[5:], ob, dt, FACE, TOL_STAGE, what=f"uct rhs L(b) cfg{cfg}", fscale={"b": fs["B"]})
    # stage-chained: each oracle stage starts from the GPU's own input state
    bn = g.get_face_field()
    bs = bn
    for s in (1, 2, 3):
        un, us, pp = g.get_state()
        g.stage(s, dt)
        Uo, Po, bo, _ = orc.stage_uct(oc, s, dt, un, un if s == 1 else us, pp, bn, bs)
        gn, gs, gP = g.get_state()
        assert_groups(gs if s < 3 else gn, Uo, CONS_GROUPS, TOL_STAGE, what=f"stage {s} U cfg{cfg}")
        assert_groups(gP, Po, PRIM5_GROUPS, TOL_STAGE, what=f"stage {s} P cfg{cfg}")
        bg = g.get_face_field()
        assert_groups(bg, bo, FACE, TOL_STAGE, what=f"stage {s} b cfg{cfg}")
        bs = bg
        if s == 3:
            bn = bg


@pytest.mark.parametrize("cfg,n,steps,rec", [(0, (32, 32, 32), 10, 0), (1, (32, 32, 32), 10, 0),
                                              (0, (24, 28, 20), 10, 2), (0, (24, 28, 20), 6, 5),
                                              (2, (40, 36, 34), 10, 0), (2, (40, 36, 34), 10, 2),
                                              (4, (64, 32, 16), 10, 0)])
def test_uct_multistep_parity(E, orc, cfg, n, steps, rec):
    p = uct_problem(cfg, n, rec)
    oc, g, U, P, ob = start(E, orc, p)
    ocnt = [0, 0]
    for _ in range(steps):
        dt = orc.max_dt(oc, U, P, p.cfl)
        U, P, ob, cnt = orc.step_uct(oc, dt, U, P, ob)
        ocnt = [ocnt[0] + cnt[0], ocnt[1] + cnt[1]]
        g.step(dt)
    gn, _, gp = g.get_state()
    assert_groups(gn, U, CONS_GROUPS, TOL_10, what=f"{steps} steps U")
    assert_groups(gp, P, PRIM5_GROUPS, TOL_10, what=f"{steps} steps P")
    assert_groups(g.get_face_field(), ob, FACE, TOL_10, what=f"{steps} steps b")
    st = g.stats()
    assert [st["floor_events"], st["c2p_failures"]] == ocnt  # counted, identical (A9)
    if cfg not in (2, 4):  # blast / torus atmosphere floors may fire; the smooth configs' never
        assert ocnt == [0, 0]


def test_uct_divh_preserved_on_gpu_and_advance_bitwise(E, orc):
    p = uct_problem(0, (48, 40, 36))
    oc, g, U, P, ob = start(E, orc, p)
    d0 = orc.uct_divh(oc, ob)
    b0 = g.get_face_field()
    h = E.Echo(p)
    h.set_prims(I.initial_prims(p))
    h.set_face_field(b0)
    dts = []
    for _ in range(5):
        dt = g.max_dt(p.cfl)
        dts.append(dt)
        g.step(dt)
    b = g.get_face_field()
    scale = np.max(np.abs(b)) / min(oc.dx(a) for a in range(3))
    assert np.max(np.abs(orc.uct_divh(oc, b) - d0)) < 200 * np.finfo(float).eps * scale
    # the device-driven loop gives the same bits
    assert h.advance(5, p.cfl).tolist() == dts
    assert np.array_equal(h.get_face_field(), b)
    assert np.array_equal(h.get_state()[0], g.get_state()[0])


def test_uct_api_rules(E):
    p = uct_problem(0, (16, 16, 16))
    g = E.Echo(p)
    P8 = I.initial_prims(p)
    g.set_prims(P8)
    with pytest.raises(E.EchoError):
        g.step(1e-3)                  # no staggered field yet
    with pytest.raises(E.EchoError):
        g.get_face_field()
    g.set_face_field(I.face_field(p))
    with pytest.raises(E.EchoError):
        E.set_cons(g.ctx, g.get_cons())  # U_B must stay I6(b)
    q = I.problem(0, n=(16, 16, 16))  # field-CD context: no face field
    h = E.Echo(q)
    h.set_prims(P8)
    with pytest.raises(E.EchoError):
        h.set_face_field(I.face_field(p))
    r = I.problem(0, n=(16, 16, 7))  # UCT slabs need >= ECHO_HALO_PLANES_UCT = 8 planes
    r.divb = 2
    r.bc = ((0, 0), (0, 0), (2, 2))
    with pytest.raises(E.EchoError):
        E.Echo(r)
    with pytest.raises(E.EchoError):  # and no echo_step on a slab (an exchange precedes every stage)
        r.n = (16, 16, 16)
        s = E.Echo(r)
        s.set_prims(I.initial_prims(I.problem(0, n=(16, 16, 16))))
        s.set_face_field(I.face_field(I.problem(0, n=(16, 16, 16))))
        s.step(1e-3)


def test_uct_full_size_conservation_and_divh(E):
    """Properties that hold at any size, at BASELINE.json's 512^3 (config 3) with UCT:
    the sums of sqrt(g) U (hydro) and of every staggered component are conserved to
    roundoff over 2 steps, and div_H b (A41: sum_a delta_a Dh_a b^a) changes only by
    roundoff.  The reductions and the DER6 divergence are test-side torch ops."""
    import torch

    p = uct_problem(3, None)
    g = E.Echo(p)
    g.set_prims(I.initial_prims(p, device="cuda"))
    g.set_face_field(I.face_field(p, device="cuda"))
    N = p.ncells
    U = torch.empty((8, N), dtype=torch.float64, device="cuda")
    b = torch.empty((3, p.n[2], p.n[1], p.n[0]), dtype=torch.float64, device="cuda")
    c0, c1, c2 = 1067.0 / 960.0, -29.0 / 480.0, 3.0 / 640.0

    def divh():
        out = torch.zeros_like(b[0])
        for a in range(3):
            ax = 2 - a
            f = b[a]
            D = c0 * f + c1 * (torch.roll(f, 1, ax) + torch.roll(f, -1, ax)) + c2 * (torch.roll(f, 2, ax) + torch.roll(f, -2, ax))
            out += (D - torch.roll(D, 1, ax)) * p.n[a]
            del D
        return out

    def state():
        E.get_cons(g.ctx, U)
        E.get_face_field(g.ctx, b)
        torch.cuda.synchronize()
        s = [float(U[q].sum()) for q in range(5)] + [float(b[a].sum()) for a in range(3)]
        m = [float(U[q].abs().sum()) for q in range(5)] + [float(b[a].abs().sum()) for a in range(3)]
        return s, m

    s0, m0 = state()
    d0 = divh()
    bmax = float(b.abs().max())
    for _ in range(2):
        g.step(g.max_dt(p.cfl))
    s1, _ = state()
    d1 = divh()
    change = float((d1 - d0).abs().max())
    assert change < 200 * 2.2e-16 * bmax * p.n[0], (change, bmax)
    for q in range(8):
        assert abs(s1[q] - s0[q]) <= 1e-12 * m0[q], (q, s0[q], s1[q], m0[q])
    st = g.stats()
    assert st["floor_events"] == 0 and st["c2p_failures"] == 0
    g.close()


@pytest.mark.parametrize("n,bc", [((33, 1, 1), ((0, 0), (0, 0), (0, 0))), ((1, 24, 7), ((0, 0), (0, 0), (0, 0))),
                                  ((5, 3, 9), ((1, 1), (0, 0), (1, 1))), ((1, 1, 1), ((0, 0), (0, 0), (0, 0)))])
def test_uct_degenerate_grids_parity(E, orc, n, bc):
    """UCT edge cases: single-cell axes (edges whose transverse stencils wrap onto one
    cell), lines shorter than a chunk or the halo, outflow sides on short axes; rhs and
    3 steps against the oracle."""
    p = uct_problem(0, n)
    p.bc = bc
    oc, g, U, P, ob = start(E, orc, p)
    dt = orc.max_dt(oc, U, P, p.cfl)
    L = orc.rhs_uct(oc, U, P, ob)
    Lg = g.rhs()
    fs = flux_scale(orc, oc, U, P)
    assert_rhs_groups(Lg[:5], L[:5], U[:5], dt, HYDRO, TOL_STAGE, what=f"uct rhs {n}", fscale=fs)
    assert_rhs_groups(Lg[5:], L[5:], ob, dt, FACE, TOL_STAGE, what=f"uct L(b) {n}", fscale={"b": fs["B"]})
    for _ in range(3):
        dt = orc.max_dt(oc, U, P, p.cfl)
        U, P, ob, _ = orc.step_uct(oc, dt, U, P, ob)
        g.step(dt)
    gn, _, gp = g.get_state()
    assert_groups(gn, U, CONS_GROUPS, TOL_10, what=f"3 steps U {n}")
    assert_groups(gp, P, PRIM5_GROUPS, TOL_10, what=f"3 steps P {n}")
    assert_groups(g.get_face_field(), ob, FACE, TOL_10, what=f"3 steps b {n}")
