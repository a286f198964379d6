"""Pins of the oracle's grid-level algorithm (SURVEY.md §8(c)
P1-P3, P12, P15-P17): invariants, symmetries, conservation, div B, CFL worked
values, convergence orders.  CPU only."""
import math

import numpy as np
import pytest

import echo_inputs as I


def cfg_of(orc, p, **kw):
    d = p.grid_kwargs()
    d.update(kw)
    return orc.Cfg(**d)


def state(orc, c, P8):
    return orc.set_prims(c, np.ascontiguousarray(P8))


def random_smooth(n, seed=0, amp=0.05):
    p = I.problem(0, n=n, seed=seed)
    p.params.update(modes=4, kmax=2, amp=amp)
    return I.initial_prims(p)


# --------------------------------------------------------- uniform state
@pytest.mark.parametrize("bc", [0, 1])
def test_uniform_state_exact(orc, bc):
    # P1: every face sees identical inputs -> L = 0 exactly; the
    # step keeps all cells bitwise equal to each other.
    n = (6, 5, 4)
    c = orc.Cfg(n=n, bc=((bc, bc),) * 3)
    P8 = I.uniform_prims(n, 0.7, (0.3, -0.2, 0.1), 1.3, (0.4, -0.6, 0.2))
    U, P = state(orc, c, P8)
    L = orc.rhs(c, U, P)
    assert not np.any(L)
    U2, P2, cnt = orc.step(c, 0.01, U, P)
    assert cnt == (0, 0)
    for q in range(8):
        assert np.all(U2[q] == U2[q].flat[0])
        assert U2[q].flat[0] == pytest.approx(U[q].flat[0], rel=1e-15, abs=1e-300)


# ------------------------------------------------------- symmetries
def test_periodic_translation_invariance(orc):
    # periodic ghost fill (A12): shifting the input shifts L bitwise, also for n < g = 5
    for n in ((4, 4, 4), (8, 6, 5)):
        c = orc.Cfg(n=n)
        P8 = random_smooth(n, seed=3, amp=0.1)
        U, P = state(orc, c, P8)
        L = orc.rhs(c, U, P)
        s = (1, 2, 3)
        P8s = np.roll(P8, s, axis=(3, 2, 1))
        Us, Ps = state(orc, c, P8s)
        Ls = orc.rhs(c, Us, Ps)
        assert np.array_equal(Ls, np.roll(L, s, axis=(3, 2, 1)))


def test_outflow_mirror_symmetry(orc):
    # outflow ghost fill + mirrored reconstruction: a state symmetric under
    # x -> 1-x (v^x, S_x odd) gives a mirror-symmetric L
    n = (10, 4, 4)
    c = orc.Cfg(n=n, bc=((1, 1), (0, 0), (0, 0)), divb=1)
    x = (np.arange(n[0]) + 0.5) / n[0]
    f = np.exp(-((x - 0.5) / 0.2) ** 2)
    P8 = I.uniform_prims(n, 1.0, (0, 0, 0), 1.0, (0.3, 0.0, 0.0))
    P8[0] += 0.3 * f[None, None, :]
    P8[4] += 0.5 * f[None, None, :]
    P8[1] += 0.2 * (x - 0.5)[None, None, :]
    P8[2] += 0.1 * f[None, None, :]
    U, P = state(orc, c, P8)
    L = orc.rhs(c, U, P)
    Lm = L[:, :, :, ::-1]
    odd = [1, 6, 7]  # S_x flips sign; B is axial: B^y, B^z flip, B^x does not
    for q in range(8):
        sgn = -1.0 if q in odd else 1.0
        np.testing.assert_allclose(L[q], sgn * Lm[q], rtol=0, atol=1e-13 * max(1.0, np.abs(L[q]).max()))


# ------------------------------------------------ path equivalences
@pytest.mark.parametrize("kind", ["periodic", "outflow", "ks"])
def test_cell_path_matches_grid_path(orc, kind):
    if kind == "periodic":
        p = I.problem(0, n=(8, 7, 6))
        c = cfg_of(orc, p)
        P8 = I.initial_prims(p)
    elif kind == "outflow":
        p = I.problem(2, n=(9, 8, 7))
        c = cfg_of(orc, p)
        P8 = I.initial_prims(p)
    else:
        p = I.problem(4, n=(12, 8, 3))
        c = cfg_of(orc, p)
        P8 = I.initial_prims(p)
    U, P = state(orc, c, P8)
    L = orc.rhs(c, U, P)
    n = p.n
    cells = [(i, j, k) for k in range(n[2]) for j in range(n[1]) for i in range(n[0])]
    Lc = orc.rhs_cells(c, U, P, cells)
    assert np.array_equal(Lc.T.reshape(8, n[2], n[1], n[0]), L)
    dt = 0.3 * orc.max_dt(c, U, P, 0.4)
    Uo, Po, cnt = orc.stage(c, 1, dt, U, U, P)
    Uc, Pc, cntc = orc.stage_cells(c, 1, dt, U, U, P, cells)
    assert np.array_equal(Uc.T.reshape(8, n[2], n[1], n[0]), Uo)
    assert np.array_equal(Pc.T.reshape(5, n[2], n[1], n[0]), Po)
    assert cnt == cntc


def test_thread_count_invariance(orc):
    # P17: the oracle is bitwise independent of its thread count
    p = I.problem(0, n=(16, 12, 10))
    P8 = I.initial_prims(p)
    res = []
    for nt in (1, 3, 8):
        c = cfg_of(orc, p, nthreads=nt)
        U, P = state(orc, c, P8)
        res.append(orc.step(c, 0.005, U, P)[:2])
    for r in res[1:]:
        assert np.array_equal(r[0], res[0][0]) and np.array_equal(r[1], res[0][1])


# --------------------------------------------- conservation and div B
def test_conservation_and_divb(orc):
    # P2 / P3: periodic Minkowski grid, config-0 recipe at 16^3, 4 steps
    p = I.problem(0, n=(16, 16, 16))
    c = cfg_of(orc, p)
    U, P = state(orc, c, I.initial_prims(p))
    U0 = U.copy()
    dx = 1.0 / 16
    bmax = np.abs(U[5:8]).max()
    assert orc.divb(c, U) < 100 * 2.2e-16 * bmax / dx
    for _ in range(4):
        dt = orc.max_dt(c, U, P, 0.4)
        U, P, cnt = orc.step(c, dt, U, P)
        assert cnt == (0, 0)
        assert orc.divb(c, U) < 100 * 2.2e-16 * bmax / dx
    for q in range(8):
        s0 = math.fsum(U0[q].ravel())
        s1 = math.fsum(U[q].ravel())
        assert abs(s1 - s0) <= 1e-14 * 4 * math.fsum(np.abs(U0[q]).ravel()), q


def test_divb_diagnostic_spec_examples(orc):
    # SPEC.md:175-177
    n = (32, 8, 8)
    c = orc.Cfg(n=n)
    x = (np.arange(32) + 0.5) / 32
    P8 = I.uniform_prims(n, 1, (0, 0, 0), 1, (0.3, 0.2, 0.1))
    U, _ = state(orc, c, P8)
    assert orc.divb(c, U) == 0
    P8[6] = np.sin(2 * np.pi * x)[None, None, :]
    U, _ = state(orc, c, P8)
    assert orc.divb(c, U) <= 1e-12
    errs = []
    for N in (32, 64):
        xs = (np.arange(N) + 0.5) / N
        cN = orc.Cfg(n=(N, 4, 4))
        P8 = I.uniform_prims((N, 4, 4), 1, (0, 0, 0), 1, (0, 0, 0))
        P8[5] = np.sin(2 * np.pi * xs)[None, None, :]
        U, _ = state(orc, cN, P8)
        errs.append(abs(orc.divb(cN, U) - 2 * np.pi))
    assert math.log2(errs[0] / errs[1]) == pytest.approx(2.0, abs=0.05)


# ----------------------------------------------------------------- CFL
def test_cfl_worked_values(orc):
    # P16 (tests/golden/cfl_worked.json: SURVEY §8(c) P16), unit box, CFL 0.4
    import json
    import os

    gold = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfl_worked.json")))
    dt_rest, dt_b, dt_blast = (c["dt"] for c in gold["cases"])
    c = orc.Cfg(n=(32, 32, 32))
    U, P = state(orc, c, I.uniform_prims((32, 32, 32), 1, (0, 0, 0), 1, (0, 0, 0)))
    assert orc.max_dt(c, U, P, 0.4) == pytest.approx(dt_rest, rel=1e-13)
    U, P = state(orc, c, I.uniform_prims((32, 32, 32), 1, (0, 0, 0), 1, (0.5, 0, 0)))
    assert orc.max_dt(c, U, P, 0.4) == pytest.approx(dt_b, rel=1e-13)
    c2 = orc.Cfg(n=(32, 32, 32), hi=(2.0, 2.0, 2.0))  # doubling Delta doubles dt
    assert orc.max_dt(c2, U, P, 0.4) == pytest.approx(2 * dt_b, rel=1e-13)
    # blast ambient, n = 256 (one line is enough: uniform)
    cb = orc.Cfg(n=(256, 1, 1), hi=(1.0, 1 / 256, 1 / 256))
    U, P = state(orc, cb, I.uniform_prims((256, 1, 1), 0.01, (0, 0, 0), 0.001, (0.1, 0, 0)))
    assert orc.max_dt(cb, U, P, 0.4) == pytest.approx(dt_blast, rel=1e-13)


# ------------------------------------------------------- convergence
def _alfven_x(N, t, eta=0.1, divb=0, rec=0, der=6):
    """1-D CP Alfven wave along x on an (N,1,1) periodic grid, exact at time t."""
    va = I.cp_alfven_speed(eta)
    x = (np.arange(N) + 0.5) / N
    ph = 2 * np.pi * (x - va * t)
    P8 = I.uniform_prims((N, 1, 1), 1.0, (0, 0, 0), 1.0, (1.0, 0, 0))
    P8[6] = eta * np.cos(ph)[None, None, :]
    P8[7] = eta * np.sin(ph)[None, None, :]
    P8[2] = -va * eta * np.cos(ph)[None, None, :]
    P8[3] = -va * eta * np.sin(ph)[None, None, :]
    return P8


def _run_alfven(orc, N, divb, tend=0.25, der=6, rec=0):
    c = orc.Cfg(n=(N, 1, 1), hi=(1.0, 1.0 / N, 1.0 / N), divb=divb, der=der, rec=rec)
    U, P = state(orc, c, _alfven_x(N, 0.0))
    nsteps = int(math.ceil(tend / (0.5 * (1.0 / N) ** (5.0 / 3.0))))
    dt = tend / nsteps
    for _ in range(nsteps):
        U, P, _ = orc.step(c, dt, U, P)
    ex = _alfven_x(N, tend)
    P8 = orc.get_prims(c, U, P)
    return np.mean(np.abs(P8[6] - ex[6])) + np.mean(np.abs(P8[2] - ex[2]))


def test_alfven_convergence(orc):
    # P4: exact nonlinear CP Alfven wave; divb=none -> nominal 5th order;
    # field-CD updates B with a 2nd-order central curl -> nominal 2nd order
    e = [_run_alfven(orc, N, 1) for N in (16, 32)]
    assert math.log2(e[0] / e[1]) > 4.5, e
    e = [_run_alfven(orc, N, 0) for N in (16, 32)]
    assert math.log2(e[0] / e[1]) > 1.8, e


def test_alfven_convergence_mp5(orc):
    # f3 / A33: the whole scheme with MP5 reconstruction is 5th order on the exact CP
    # Alfven wave (divb=none; the limiter must stay inactive on this smooth solution)
    e = [_run_alfven(orc, N, 1, rec=2) for N in (16, 32)]
    assert math.log2(e[0] / e[1]) > 4.5, e


def _sound(N, amp=1e-2):
    x = (np.arange(N) + 0.5) / N
    P8 = I.uniform_prims((N, 1, 1), 1.0, (0, 0, 0), 1.0, (0, 0, 0))
    P8[0] *= 1 + amp * np.sin(2 * np.pi * x)[None, None, :]
    P8[4] *= 1 + (4.0 / 3.0) * amp * np.sin(2 * np.pi * x)[None, None, :]
    return P8


def test_sound_wave_self_convergence(orc):
    # P5 (B = 0): nonlinear smooth sound wave; self-convergence over N = 24/48/96
    # measured on the first Fourier coefficient of rho (sampling-offset free)
    c1 = []
    tend = 0.2
    for N in (24, 48, 96):
        c = orc.Cfg(n=(N, 1, 1), hi=(1.0, 1.0 / N, 1.0 / N))
        U, P = state(orc, c, _sound(N))
        nsteps = int(math.ceil(tend / (0.5 * (1.0 / N) ** (5.0 / 3.0))))
        for _ in range(nsteps):
            U, P, _ = orc.step(c, tend / nsteps, U, P)
        rho = orc.get_prims(c, U, P)[0, 0, 0]
        x = (np.arange(N) + 0.5) / N
        c1.append(np.mean(rho * np.exp(-2j * np.pi * x)))
    e1, e2 = abs(c1[0] - c1[1]), abs(c1[1] - c1[2])
    assert math.log2(e1 / e2) > 4.5, (e1, e2)


def test_rk3_temporal_order(orc):
    # P15: SSP-RK3 is 3rd order in time: errors against a fine-dt run shrink by 8x per dt halving
    N = 16
    c = orc.Cfg(n=(N, 1, 1), hi=(1.0, 1.0 / N, 1.0 / N))
    U0, P0 = state(orc, c, _sound(N, 0.05))
    tend = 0.4

    def run(nsteps):
        U, P = U0.copy(), P0.copy()
        for _ in range(nsteps):
            U, P, _ = orc.step(c, tend / nsteps, U, P)
        return U

    ref = run(320)
    e = [np.max(np.abs(run(m) - ref)) for m in (10, 20, 40)]
    assert math.log2(e[0] / e[1]) == pytest.approx(3.0, abs=0.35)
    assert math.log2(e[1] / e[2]) == pytest.approx(3.0, abs=0.35)


# ------------------------------------------------------ GR equilibria
def _torus_2d(orc, n1, n2):
    p = I.problem(4, n=(n1, n2, 1))
    p.params.update(beta=1e300, pert=0.0)  # B -> 0, no perturbation
    P8 = I.initial_prims(p)
    P8[5:8] = 0.0
    c = cfg_of(orc, p)
    return p, c, P8


def test_torus_equilibrium_convergence(orc):
    # P12: the constant-ell torus is stationary; interior L(U) -> 0 with resolution
    errs = []
    for n1, n2 in ((48, 24), (96, 48), (192, 96)):
        p, c, P8 = _torus_2d(orc, n1, n2)
        U, P = state(orc, c, P8)
        L = orc.rhs(c, U, P)
        rho = P8[0]
        mask = rho >= 0.5 * rho.max()
        errs.append(np.mean(np.abs(L[1][mask] / U[0][mask])) + np.mean(np.abs(L[4][mask] / U[0][mask])))
    assert math.log2(errs[0] / errs[1]) > 2.0, errs
    assert math.log2(errs[1] / errs[2]) > 2.0, errs


def test_static_gas_flat_spherical_convergence(orc):
    # P12: M = 0, uniform gas at rest in (ln r, theta, phi): sources balance the flux divergence
    errs = []
    for n1, n2 in ((16, 16), (32, 32), (64, 64)):
        c = orc.Cfg(n=(n1, n2, 1), lo=(math.log(2.0), 0.6, 0.0), hi=(math.log(4.0), 2.4, 0.5),
                    bc=((1, 1), (1, 1), (0, 0)), metric=1, M=0.0, a=0.0)
        U, P = state(orc, c, I.uniform_prims((n1, n2, 1), 1.0, (0, 0, 0), 0.7, (0, 0, 0)))
        L = orc.rhs(c, U, P)
        inner = (slice(None), slice(6, -6), slice(6, -6))
        errs.append(np.max(np.abs(L[1][inner] / U[4][inner])))
    assert math.log2(errs[0] / errs[1]) > 4.0, errs
    assert math.log2(errs[1] / errs[2]) > 4.0, errs


# ------------------------------------------------------------ floors
def test_floors_counted_and_consistent(orc):
    # A9: floors fire, are counted, and U is recomputed from the floored prims
    n = (4, 4, 4)
    c = orc.Cfg(n=n, rho_floor=1e-3, p_floor=1e-5)
    P8 = I.uniform_prims(n, 1.0, (0, 0, 0), 1.0, (0, 0, 0))
    U, P = state(orc, c, P8)
    U[4, 0, 0, 0] = -0.5  # tau < 0 at one cell: p would be negative
    U[0, 1, 1, 1] = 1e-5  # D below the density floor
    U2, P2, (nfl, nfa) = orc.con2prim(c, U, P)
    assert nfl + nfa == 2
    assert P2[4, 0, 0, 0] >= 1e-5 and P2[0, 1, 1, 1] >= 1e-3
    Ur, _ = state(orc, c, orc.get_prims(c, U2, P2))
    np.testing.assert_allclose(U2[:5], Ur[:5], rtol=1e-14, atol=1e-16)
