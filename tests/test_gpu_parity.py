"""GPU parity: the C-ABI library (sm_100a kernels) against the oracle on the
same seeded inputs, element by element, normwise per variable group (A16):
1e-12 per RK stage, 1e-10 after 10 steps (BASELINE.json north_star).
Marked gpu: run on a B200 with `pytest -m gpu`."""
import math

import numpy as np
import pytest

import echo_inputs as I
from tests.util import CONS_GROUPS, PRIM5_GROUPS, PRIM8_GROUPS, assert_groups, assert_rhs_groups, flux_scale

pytestmark = pytest.mark.gpu

TOL_STAGE = 1e-12
TOL_10 = 1e-10


@pytest.fixture(scope="module")
def E():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1810_04597_b200 import build

    build.build()
    from paper_1810_04597_b200 import echo

    return echo


def small_problem(cfg, n):
    p = I.problem(cfg, n=n)
    return p


def ocfg(orc, p):
    return orc.Cfg(**p.grid_kwargs())


# ------------------------------------------------------------ invariants
def test_uniform_state_gpu(E):
    n = (70, 9, 6)
    P8 = I.uniform_prims(n, 0.7, (0.3, -0.2, 0.1), 1.3, (0.4, -0.6, 0.2))
    g = E.Echo(n=n, lo=(0, 0, 0), hi=(1, 1, 1), bc=((0, 0), (1, 1), (0, 0)))
    g.set_prims(P8)
    L = g.rhs()
    assert not np.any(L)
    g.step(0.01)
    U = g.get_cons()
    for q in range(8):
        assert np.all(U[q] == U[q].flat[0])


# --------------------------------------------------------- stage parity
CASES = [
    # (config, grid) — grids span several tiles (64 along the sweep, 4 across) and ragged tails
    (0, (32, 32, 32)),            # config 0 at its full size
    (0, (150, 13, 70)),           # multi-tile + ragged in every direction
    (1, (40, 36, 34)),            # CP Alfven recipe, reduced grid
    (2, (45, 38, 41)),            # outflow blast, reduced grid
    (3, (48, 48, 48)),            # config-3 recipe (32 modes, k<=8), reduced grid
    (4, (72, 35, 24)),            # Kerr-Schild torus, reduced grid (36 theta cells would put a ghost face on the pole)
]


@pytest.mark.parametrize("cfg,n", CASES)
def test_rhs_and_stage_parity(E, orc, cfg, n):
    p = small_problem(cfg, n)
    P8 = I.initial_prims(p)
    oc = ocfg(orc, p)
    Un, P5 = orc.set_prims(oc, P8)
    g = E.Echo(p)
    g.set_prims(P8)
    gun, _, gp = g.get_state()
    assert_groups(gun, Un, CONS_GROUPS, TOL_STAGE, what="prim2cons")
    assert_groups(gp, P5, PRIM5_GROUPS, TOL_STAGE, what="prim2cons P5")
    # CFL
    dt_o = orc.max_dt(oc, gun, gp, p.cfl)
    # rhs on identical inputs
    L = orc.rhs(oc, gun, gp)
    assert_rhs_groups(g.rhs(), L, gun, dt_o, CONS_GROUPS, TOL_STAGE, what=f"rhs cfg{cfg} {n}",
                      fscale=flux_scale(orc, oc, gun, gp))
    dt_g = g.max_dt(p.cfl)
    assert dt_g == pytest.approx(dt_o, rel=1e-14)
    # stage-chained parity: each oracle stage starts from the GPU's own input state
    for s in (1, 2, 3):
        un, us, pp = g.get_state()
        g.stage(s, dt_o)
        Uo, Po, cnt = orc.stage(oc, s, dt_o, un, un if s == 1 else us, pp)
        gn, gs, gP = g.get_state()
        Ug = gs if s < 3 else gn
        assert_groups(Ug, Uo, CONS_GROUPS, TOL_STAGE, what=f"stage {s} U cfg{cfg}")
        assert_groups(gP, Po, PRIM5_GROUPS, TOL_STAGE, what=f"stage {s} P cfg{cfg}")


@pytest.mark.parametrize("cfg,n,steps", [(0, (32, 32, 32), 10), (1, (32, 32, 32), 10), (2, (40, 40, 40), 10),
                                         (3, (40, 40, 40), 5), (4, (64, 32, 16), 10)])
def test_multistep_parity(E, orc, cfg, n, steps):
    p = small_problem(cfg, n)
    P8 = I.initial_prims(p)
    oc = ocfg(orc, p)
    U, P = orc.set_prims(oc, P8)
    g = E.Echo(p)
    g.set_prims(P8)
    ocnt = [0, 0]
    for _ in range(steps):
        dt = orc.max_dt(oc, U, P, p.cfl)
        U, P, cnt = orc.step(oc, dt, U, P)
        ocnt[0] += cnt[0]
        ocnt[1] += cnt[1]
        g.step(dt)
    gn, _, gp = g.get_state()
    assert_groups(gn, U, CONS_GROUPS, TOL_10, what=f"{steps} steps U cfg{cfg}")
    assert_groups(gp, P, PRIM5_GROUPS, TOL_10, what=f"{steps} steps P cfg{cfg}")
    st = g.stats()
    assert (st["floor_events"], st["c2p_failures"]) == tuple(ocnt)
    if cfg in (0, 1, 3):
        assert ocnt == [0, 0]
    # the user-facing prims agree too
    assert_groups(g.get_prims(), orc.get_prims(oc, U, P), PRIM8_GROUPS, TOL_10, what="get_prims")


@pytest.mark.parametrize("cfg,n,steps,rec", [(0, (32, 32, 32), 10, 2), (2, (40, 40, 40), 10, 2),
                                              (4, (64, 32, 16), 5, 2), (0, (32, 32, 32), 10, 3),
                                              (2, (40, 40, 40), 10, 3), (2, (40, 40, 40), 10, 4),
                                              (0, (32, 32, 32), 10, 5), (2, (40, 40, 40), 10, 5),
                                              (0, (32, 32, 32), 10, 6), (2, (40, 40, 40), 10, 6),
                                              (1, (36, 20, 28), 10, 6), (3, (70, 13, 33), 5, 6)])
def test_multistep_parity_mp5(E, orc, cfg, n, steps, rec):
    """MP5 (rec=2, A33), WENO-Z (rec=3, A34), MC2 (4), PPM (5) and characteristic-wise WENO5
    (rec=6, A44) reconstruction: multi-step parity, incl. the blast (limiter
    active at the shock) and the Kerr-Schild torus (not for rec 6: flat only); the rec-6
    cases include a ragged multi-tile grid (70 x 13 x 33)."""
    p = small_problem(cfg, n)
    p.rec = rec
    P8 = I.initial_prims(p)
    oc = ocfg(orc, p)
    U, P = orc.set_prims(oc, P8)
    g = E.Echo(p)
    g.set_prims(P8)
    ocnt = [0, 0]
    for _ in range(steps):
        dt = orc.max_dt(oc, U, P, p.cfl)
        U, P, cnt = orc.step(oc, dt, U, P)
        ocnt[0] += cnt[0]
        ocnt[1] += cnt[1]
        g.step(dt)
    gn, _, gp = g.get_state()
    assert_groups(gn, U, CONS_GROUPS, TOL_10, what=f"rec{rec} {steps} steps U cfg{cfg}")
    assert_groups(gp, P, PRIM5_GROUPS, TOL_10, what=f"rec{rec} {steps} steps P cfg{cfg}")
    st = g.stats()
    assert (st["floor_events"], st["c2p_failures"]) == tuple(ocnt)


def test_con2prim_parity(E, orc):
    p = small_problem(2, (20, 18, 16))
    P8 = I.initial_prims(p)
    oc = ocfg(orc, p)
    U, P = orc.set_prims(oc, P8)
    # perturb the conserved state so the Newton solve has work to do, incl. floors
    rng = np.random.default_rng(3)
    U2 = U * (1 + 1e-3 * rng.standard_normal(U.shape))
    U2[4, 0, 0, :5] = -1e-3  # tau < 0: pressure floor
    g = E.Echo(p)
    g.set_prims(P8)
    E.set_cons(g.ctx, np.ascontiguousarray(U2))
    Uo, Po, cnt = orc.con2prim(oc, U2, P)
    gn, _, gp = g.get_state()
    assert_groups(gn, Uo, CONS_GROUPS, TOL_STAGE, what="con2prim U")
    assert_groups(gp, Po, PRIM5_GROUPS, TOL_STAGE, what="con2prim P")
    st = g.stats()
    assert (st["floor_events"], st["c2p_failures"]) == cnt
    assert cnt[0] + cnt[1] >= 5


def test_switches_parity(E, orc):
    # rec=FV, der=4, divb=none on a multi-tile grid
    p = small_problem(0, (70, 9, 10))
    for kw in ({"rec": 1}, {"der": 4}, {"divb": 1}, {"der": 2}, {"rec": 2}, {"rec": 2, "divb": 1}, {"rec": 3}, {"rec": 4, "der": 2}, {"rec": 5, "der": 4},
               {"rec": 6}, {"rec": 6, "divb": 1, "der": 4}):
        for k, v in kw.items():
            setattr(p, k, v)
        P8 = I.initial_prims(p)
        oc = ocfg(orc, p)
        U, P = orc.set_prims(oc, P8)
        g = E.Echo(p)
        g.set_prims(P8)
        dt = orc.max_dt(oc, U, P, 0.4)
        assert_rhs_groups(g.rhs(), orc.rhs(oc, U, P), U, dt, CONS_GROUPS, TOL_STAGE, what=f"rhs {kw}",
                          fscale=flux_scale(orc, oc, U, P))
        p = small_problem(0, (70, 9, 10))


# ------------------------------------------------ full-size sampled parity
# (config, reconstruction): the default WENO5 on every config, plus the characteristic-wise
# (rec 6, A44) sweeps at 512^3 and at the blast
FULL = [(1, None), (2, None), (4, None), (3, None), (3, 6), (2, 6)]


def _full_state(E, p, device_ic):
    import torch

    g = E.Echo(p)
    if device_ic:
        P8 = I.initial_prims(p, device="cuda")
        g.set_prims(P8)
        del P8
    else:
        g.set_prims(I.initial_prims(p))
    return g


@pytest.mark.parametrize("cfg,rec", FULL)
def test_full_size_sampled_stage_parity(E, orc, cfg, rec):
    """At BASELINE.json's full sizes, in the bench launch configuration: each RK
    stage's output at 2000 sampled cells (incl. the 8 corners) against the
    oracle's per-cell path on the GPU's own input state."""
    import torch

    p = I.problem(cfg)
    if rec is not None:
        p.rec = rec
    g = _full_state(E, p, device_ic=(cfg == 3))
    oc = ocfg(orc, p)
    cells = I.sample_cells(p.n, 2000, seed=100 + cfg)
    lin = (cells[:, 2] * p.n[1] + cells[:, 1]) * p.n[0] + cells[:, 0]
    lin_t = torch.as_tensor(lin, device="cuda")
    N = p.ncells
    un = torch.empty((8, N), dtype=torch.float64, device="cuda")
    us = torch.empty((8, N), dtype=torch.float64, device="cuda")
    pp = torch.empty((5, N), dtype=torch.float64, device="cuda")
    E.get_state(g.ctx, un, None, pp)
    un_h = un.cpu().numpy().reshape(8, *p.n[::-1])
    pp_h = pp.cpu().numpy().reshape(5, *p.n[::-1])
    dt = g.max_dt(p.cfl)
    assert dt == pytest.approx(orc.max_dt(oc, un_h, pp_h, p.cfl), rel=1e-14)
    us_h = un_h
    for s in (1, 2, 3):
        g.stage(s, dt)
        Uo, Po, _ = orc.stage_cells(oc, s, dt, un_h, us_h, pp_h, cells)
        E.get_state(g.ctx, un, us, pp)
        torch.cuda.synchronize()
        Ug = (us if s < 3 else un)[:, lin_t].cpu().numpy().T
        Pg = pp[:, lin_t].cpu().numpy().T
        assert_groups(Ug, Uo, CONS_GROUPS, TOL_STAGE, axis=1, what=f"full cfg{cfg} stage {s} U")
        assert_groups(Pg, Po, PRIM5_GROUPS, TOL_STAGE, axis=1, what=f"full cfg{cfg} stage {s} P")
        if s < 3:
            un_h = un.cpu().numpy().reshape(8, *p.n[::-1])
            us_h = us.cpu().numpy().reshape(8, *p.n[::-1])
            pp_h = pp.cpu().numpy().reshape(5, *p.n[::-1])
    g.close()


# ------------------------------------------------------------ robustness
def test_determinism_bitwise(E):
    p = small_problem(2, (70, 33, 20))
    P8 = I.initial_prims(p)
    outs = []
    for _ in range(2):
        g = E.Echo(p)
        g.set_prims(P8)
        for _ in range(3):
            g.step(g.max_dt(0.4))
        outs.append(g.get_state())
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_errors_are_loud(E):
    p = small_problem(0, (8, 8, 8))
    g = E.Echo(p)
    with pytest.raises(E.EchoError) as ei:
        g.step(0.01)
    assert ei.value.code == E.E_ORDER
    P8 = I.initial_prims(p)
    P8[4, 3, 2, 1] = -1.0
    with pytest.raises(E.EchoError) as ei:
        g.set_prims(P8)
    assert ei.value.code == E.E_UNPHYSICAL and "(1,2,3)" in str(ei.value)
    P8[4, 3, 2, 1] = 1.0
    g.set_prims(P8)
    with pytest.raises(E.EchoError) as ei:
        g.stage(2, 0.01)
    assert ei.value.code == E.E_ORDER
    with pytest.raises(E.EchoError):
        E.create(n=(0, 4, 4), lo=(0, 0, 0), hi=(1, 1, 1), bc=((0, 0),) * 3)


# ------------------------------------------------------------ degenerate grids
@pytest.mark.parametrize("n,bc", [
    ((16, 1, 1), ((0, 0), (0, 0), (0, 0))),   # 1-D along x (the y/z sweeps see single-cell lines)
    ((1, 16, 1), ((0, 0), (0, 0), (0, 0))),   # 1-D along y
    ((1, 1, 16), ((0, 0), (0, 0), (0, 0))),   # 1-D along z
    ((4, 4, 4), ((0, 0), (0, 0), (0, 0))),    # every axis shorter than the 5-cell halo (wrap mod n, A12)
    ((5, 3, 7), ((1, 1), (1, 1), (1, 1))),    # outflow everywhere, odd sizes below one chunk
    ((33, 2, 9), ((0, 0), (1, 1), (0, 0))),   # one cell past a 32-cell chunk, 2-cell outflow axis
])
def test_degenerate_grids_parity(E, orc, n, bc):
    """Edge cases of the march: lines shorter than a chunk or the halo, single-cell axes,
    ragged chunk tails; stage-chained parity and 3 steps."""
    p = I.problem(0, n=n)
    p.bc = bc
    P8 = I.initial_prims(p)
    oc = ocfg(orc, p)
    U, P = orc.set_prims(oc, P8)
    g = E.Echo(p)
    g.set_prims(P8)
    dt = orc.max_dt(oc, U, P, p.cfl)
    assert g.max_dt(p.cfl) == pytest.approx(dt, rel=1e-14)
    assert_rhs_groups(g.rhs(), orc.rhs(oc, U, P), U, dt, CONS_GROUPS, TOL_STAGE, what=f"rhs {n}",
                      fscale=flux_scale(orc, oc, U, P))
    for _ in range(3):
        dt = orc.max_dt(oc, U, P, p.cfl)
        U, P, _ = orc.step(oc, dt, U, P)
        g.step(dt)
    gn, _, gp = g.get_state()
    assert_groups(gn, U, CONS_GROUPS, TOL_10, what=f"3 steps U {n}")
    assert_groups(gp, P, PRIM5_GROUPS, TOL_10, what=f"3 steps P {n}")


def test_full_size_conservation_and_divb(E):
    """Properties that hold at any size, checked at BASELINE.json's 512^3 (config 3, the
    bench workload and launch configuration): periodic Minkowski -> the sums of
    sqrt(g) U are conserved to roundoff over 2 steps (P2), and the field-CD scheme keeps
    the D2 divergence of B at roundoff (P3).  The reductions are test-side torch ops."""
    import math

    import torch

    p = I.problem(3)
    g = E.Echo(p)
    P8 = I.initial_prims(p, device="cuda")
    g.set_prims(P8)
    del P8
    N = p.ncells
    U = torch.empty((8, N), dtype=torch.float64, device="cuda")

    def sums_and_div():
        E.get_cons(g.ctx, U)
        torch.cuda.synchronize()
        s = [float(U[q].sum()) for q in range(8)]
        a = [float(U[q].abs().sum()) for q in range(8)]
        B = U[5:8].view(3, p.n[2], p.n[1], p.n[0])
        dx = 1.0 / p.n[0]
        div = ((torch.roll(B[0], -1, 2) - torch.roll(B[0], 1, 2)) + (torch.roll(B[1], -1, 1) - torch.roll(B[1], 1, 1)) +
               (torch.roll(B[2], -1, 0) - torch.roll(B[2], 1, 0))) / (2 * dx)
        return s, a, float(div.abs().max()), float(B.abs().max())

    s0, a0, d0, bmax = sums_and_div()
    dx = 1.0 / p.n[0]
    assert d0 < 100 * 2.2e-16 * bmax / dx
    for _ in range(2):
        g.step(g.max_dt(p.cfl))
    s1, _, d1, _ = sums_and_div()
    assert d1 < 100 * 2.2e-16 * bmax / dx, (d0, d1)
    for q in range(8):
        # summation error of the test's own float64 reductions (~sqrt(N) eps) dominates the bound
        assert abs(s1[q] - s0[q]) <= 1e-12 * a0[q], (q, s0[q], s1[q], a0[q])
    st = g.stats()
    assert st["floor_events"] == 0 and st["c2p_failures"] == 0
    g.close()


@pytest.mark.parametrize("n,bc", [((4, 4, 4), ((0, 0), (0, 0), (0, 0))), ((5, 3, 7), ((1, 1), (1, 1), (1, 1))),
                                  ((33, 2, 9), ((0, 0), (1, 1), (0, 0)))])
def test_characteristic_degenerate_grids_parity(E, orc, n, bc):
    """rec = 6 (A44) on grids shorter than the halo / a chunk, outflow on short axes: rhs and 3 steps."""
    p = I.problem(0, n=n)
    p.bc, p.rec = bc, 6
    P8 = I.initial_prims(p)
    oc = ocfg(orc, p)
    U, P = orc.set_prims(oc, P8)
    g = E.Echo(p)
    g.set_prims(P8)
    dt = orc.max_dt(oc, U, P, p.cfl)
    assert_rhs_groups(g.rhs(), orc.rhs(oc, U, P), U, dt, CONS_GROUPS, TOL_STAGE, what=f"rec6 rhs {n}",
                      fscale=flux_scale(orc, oc, U, P))
    for _ in range(3):
        dt = orc.max_dt(oc, U, P, p.cfl)
        U, P, _ = orc.step(oc, dt, U, P)
        g.step(dt)
    gn, _, gp = g.get_state()
    assert_groups(gn, U, CONS_GROUPS, TOL_10, what=f"rec6 3 steps U {n}")
    assert_groups(gp, P, PRIM5_GROUPS, TOL_10, what=f"rec6 3 steps P {n}")


def test_characteristic_scope_refused(E):
    """A44 is flat-metric and field-CD / none only: Kerr-Schild or UCT with rec = 6 fail at create."""
    for cfg, kw in ((4, {}), (0, {"divb": 2})):
        p = I.problem(cfg, n=(8, 8, 8))
        p.rec = 6
        for k, v in kw.items():
            setattr(p, k, v)
        with pytest.raises(E.EchoError) as ei:
            E.Echo(p)
        assert ei.value.code == E.E_ARG and "rec = 6" in str(ei.value)
