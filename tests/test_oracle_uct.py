"""Pins of the oracle's UCT mode (divb = 2: staggered field + upwind constrained
transport, readings A37-A41).  CPU only.

What pins what:
  * the centring I6 (A37): exact on constants, 6th-order on a sine (a wrong weight
    drops the order or breaks the constant);
  * the preserved divergence (A41): div_H b changes only by roundoff over steps on a
    random 3-D state (a wrong sign, index or DER direction in the induction breaks it);
  * the EMF formula (A39) against the independently pinned divb=none scheme: with a
    uniform velocity and a field varying along one axis, every quadrant velocity is the
    same constant and the UCT-HLL EMF reduces to the 1-D HLL flux of the transverse
    field, so L(b) must equal divb=none's L(B) to roundoff, along each of the 3 axes
    (every component in both the p and q roles);
  * the whole UCT scheme (A38 quadrant velocities included): 5th-order convergence on
    the exact CP Alfven wave travelling obliquely across a 2-D grid, where field-CD is
    2nd order;
  * invariants: a uniform state stays exactly uniform; conservation of the hydro
    variables and of the mean field; with outflow sides (A42) div_H is still preserved
    in every cell, and the config-2 blast runs without floor events;
  * Kerr-Schild (A43): div_H preserved on the torus; with b = 0 the UCT step equals
    the field-CD step bit for bit.
"""
import math

import numpy as np
import pytest

import echo_inputs as I


def _cfg(orc, n, **kw):
    d = dict(n=tuple(n), divb=2)
    d.update(kw)
    return orc.Cfg(**d)


# ------------------------------------------------------------ A37 centring
def test_centre_interpolation_constant_and_order(orc):
    c = _cfg(orc, (8, 4, 4))
    b = np.full(c.shape(3), 0.7)
    assert np.array_equal(orc.uct_centre(c, b), b)  # weights sum to exactly 256/256
    errs = []
    for N in (16, 32):
        c = _cfg(orc, (N, 2, 2))
        xf = (np.arange(N) + 1.0) / N    # faces i + 1/2
        xc = (np.arange(N) + 0.5) / N
        b = np.zeros(c.shape(3))
        b[0] = np.sin(2 * np.pi * xf)[None, None, :]
        Bc = orc.uct_centre(c, b)
        errs.append(np.max(np.abs(Bc[0] - np.sin(2 * np.pi * xc)[None, None, :])))
        assert np.all(Bc[1:] == 0.0)
    assert math.log2(errs[0] / errs[1]) > 5.8, errs


# ------------------------------------------------------ A41 invariant
def _random_uct_state(orc, n, seed=3, amp=0.05):
    p = I.problem(0, n=n, seed=seed)
    p.params.update(modes=4, kmax=2, amp=amp)
    c = _cfg(orc, n)
    U, P, b = orc.set_prims_uct(c, I.initial_prims(p), I.face_field(p))
    return p, c, U, P, b


def test_divh_of_analytic_field_is_small_and_converges(orc):
    d = []
    for N in (16, 32):
        p, c, U, P, b = _random_uct_state(orc, (N, N, N))
        d.append(np.max(np.abs(orc.uct_divh(c, b))))
    assert d[1] < 1e-4 and math.log2(d[0] / d[1]) > 5.0, d


def test_divh_preserved_to_roundoff(orc):
    p, c, U, P, b = _random_uct_state(orc, (12, 10, 8))
    d0 = orc.uct_divh(c, b)
    scale = np.max(np.abs(b)) / min(c.dx(a) for a in range(3))
    for _ in range(3):
        dt = orc.max_dt(c, U, P, 0.4)
        U, P, b, cnt = orc.step_uct(c, dt, U, P, b)
        assert cnt == (0, 0)
        assert np.max(np.abs(orc.uct_divh(c, b) - d0)) < 200 * np.finfo(float).eps * scale
    # and it is a real constraint: the stage update of a single face breaks it
    L = orc.rhs_uct(c, U, P, b)
    assert np.max(np.abs(L[5:])) > 1e-3


def test_divh_preserved_with_outflow_boundaries(orc):
    # A42: b, the face data and the EMFs take the ghost rule of A13 (nearest owned face /
    # edge) on an outflow side; the ghost map along one axis commutes with the difference
    # operators along the others, so div_H is preserved in EVERY cell, boundary ones included
    n = (16, 14, 12)
    p = I.problem(0, n=n, seed=5)
    p.params.update(modes=4, kmax=2, amp=0.05)
    p.bc = ((1, 1), (1, 1), (1, 1))
    p.divb = 2
    c = orc.Cfg(**p.grid_kwargs())
    U, P, b = orc.set_prims_uct(c, I.initial_prims(p), I.face_field(p))
    d0 = orc.uct_divh(c, b)
    scale = np.max(np.abs(b)) / min(c.dx(a) for a in range(3))
    for _ in range(3):
        U, P, b, cnt = orc.step_uct(c, orc.max_dt(c, U, P, 0.4), U, P, b)
        assert cnt == (0, 0)
    assert np.max(np.abs(orc.uct_divh(c, b) - d0)) < 200 * np.finfo(float).eps * scale


def test_blast_runs_with_uct(orc):
    # config 2 (outflow blast, p jump 1000x) with UCT: 10 steps without floor events or
    # Newton failures, field divergence preserved
    n = (24, 24, 24)
    p = I.problem(2, n=n)
    p.divb = 2
    c = orc.Cfg(**p.grid_kwargs())
    U, P, b = orc.set_prims_uct(c, I.initial_prims(p), I.face_field(p))
    d0 = orc.uct_divh(c, b)
    for _ in range(10):
        U, P, b, cnt = orc.step_uct(c, orc.max_dt(c, U, P, p.cfl), U, P, b)
        assert cnt == (0, 0)
    assert np.max(np.abs(orc.uct_divh(c, b) - d0)) < 1e-12
    assert np.max(np.abs(b[1])) > 1e-3  # the explosion bent the field


def test_kerr_schild_uct(orc):
    # A43 (config 4, the torus in Kerr-Schild): div_H is preserved; and with b = 0 the
    # UCT step equals the field-CD step bit for bit (normal-field override, face metric,
    # sources and con2prim take identical paths; E = 0 keeps b exactly 0)
    p = I.problem(4, n=(48, 24, 16))
    p.divb = 2
    c = orc.Cfg(**p.grid_kwargs())
    U, P, b = orc.set_prims_uct(c, I.initial_prims(p), I.face_field(p))
    d0 = orc.uct_divh(c, b)
    scale = np.max(np.abs(b)) / min(c.dx(a) for a in range(3))
    for _ in range(3):
        U, P, b, _ = orc.step_uct(c, orc.max_dt(c, U, P, p.cfl), U, P, b)
    assert np.max(np.abs(orc.uct_divh(c, b) - d0)) < 200 * np.finfo(float).eps * scale
    P8 = I.initial_prims(p)
    P8[5:] = 0.0
    Uu, Pu, bu = orc.set_prims_uct(c, P8, np.zeros(c.shape(3)))
    c0 = orc.Cfg(**{**p.grid_kwargs(), "divb": 0})
    U0, P0 = orc.set_prims(c0, P8)
    dt = orc.max_dt(c0, U0, P0, p.cfl)
    Uu, Pu, bu, cu = orc.step_uct(c, dt, Uu, Pu, bu)
    U0, P0, c0n = orc.step(c0, dt, U0, P0)
    assert np.array_equal(Uu, U0) and np.array_equal(Pu, P0) and not np.any(bu) and cu == c0n


def test_uniform_state_exact(orc):
    c = _cfg(orc, (6, 5, 4))
    P8 = I.uniform_prims(c.n, 1.0, (0.1, -0.2, 0.05), 0.5, (0.3, 0.2, -0.4))
    b = np.ascontiguousarray(P8[5:8].copy())
    U, P, b = orc.set_prims_uct(c, P8, b)
    L = orc.rhs_uct(c, U, P, b)
    assert np.all(L == 0.0)
    U1, P1, b1, _ = orc.step_uct(c, 0.01, U, P, b)
    for a in (U1, P1, b1):
        for q in range(a.shape[0]):
            assert np.all(a[q] == a[q].flat[0])


def test_conservation(orc):
    p, c, U, P, b = _random_uct_state(orc, (10, 8, 12))
    s0 = [math.fsum(U[q].ravel()) for q in range(5)] + [math.fsum(b[a].ravel()) for a in range(3)]
    for _ in range(2):
        U, P, b, _ = orc.step_uct(c, orc.max_dt(c, U, P, 0.4), U, P, b)
    s1 = [math.fsum(U[q].ravel()) for q in range(5)] + [math.fsum(b[a].ravel()) for a in range(3)]
    for x0, x1, arr in zip(s0, s1, [U[q] for q in range(5)] + [b[a] for a in range(3)]):
        assert abs(x1 - x0) <= 1e-13 * np.sum(np.abs(arr)) + 1e-15


# ------------------------------------- A39 against the pinned divb=none scheme
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_emf_reduces_to_1d_hll(orc, axis):
    """uniform rho, p, v; B^t (t != axis) varying along `axis`, B^axis constant: the UCT
    rhs equals divb=none's (hydro and transverse field) to roundoff"""
    n = [4, 4, 4]
    n[axis] = 16
    shape = (n[2], n[1], n[0])
    x = (np.arange(n[axis]) + 0.5) / n[axis]
    prof = [np.sin(2 * np.pi * x) * 0.2, np.cos(4 * np.pi * x) * 0.15]
    P8 = I.uniform_prims(n, 1.0, (0.1, -0.15, 0.2), 0.8, (0.0, 0.0, 0.0))
    t1, t2 = (axis + 1) % 3, (axis + 2) % 3
    bshape = [1, 1, 1]
    bshape[2 - axis] = n[axis]
    P8[5 + axis] = 0.6
    P8[5 + t1] = np.broadcast_to(prof[0].reshape(bshape), shape)
    P8[5 + t2] = np.broadcast_to(prof[1].reshape(bshape), shape)
    c1 = orc.Cfg(n=tuple(n), divb=1)
    U1, Pp1 = orc.set_prims(c1, P8)
    L1 = orc.rhs(c1, U1, Pp1)
    c2 = _cfg(orc, n)
    b = np.ascontiguousarray(P8[5:8].copy())  # constant along the transverse axes: faces = centres
    U2, Pp2, b = orc.set_prims_uct(c2, P8, b)
    L2 = orc.rhs_uct(c2, U2, Pp2, b)
    for q in list(range(5)) + [5 + t1, 5 + t2]:
        scale = max(np.max(np.abs(L1[q])), 1e-3)
        assert np.max(np.abs(L2[q] - L1[q])) < 1e-12 * scale, (q, np.max(np.abs(L2[q] - L1[q])), scale)
    assert np.max(np.abs(L2[5 + axis])) < 1e-13  # the normal face field does not move
    assert np.max(np.abs(L1[5 + t1])) > 1e-2      # (the test has teeth)


# ------------------------------------------------ whole scheme convergence
def _alfven_oblique(orc, N, divb, tend=0.2):
    p = I.problem(1, n=(N, N, 1))
    p.hi = (1.0, 1.0, 1.0 / N)
    kdir = (1, 1, 0)
    X, Y, Z = I._coords(p, None, None)
    v, B = I.cp_alfven_fields(p, X, Y, Z, 0.0, kdir)
    shape = (1, N, N)
    P8 = np.ascontiguousarray(np.stack([np.ones(shape), *[np.broadcast_to(f, shape) for f in v], np.ones(shape),
                                        *[np.broadcast_to(f, shape) for f in B]]))
    c = orc.Cfg(n=(N, N, 1), hi=p.hi, divb=divb)
    if divb == 2:
        b = np.ascontiguousarray(I.face_field(p, direction=kdir))
        U, P, b = orc.set_prims_uct(c, P8, b)
    else:
        U, P = orc.set_prims(c, P8)
    nsteps = int(math.ceil(tend / (0.3 * (1.0 / N) ** (5.0 / 3.0))))
    dt = tend / nsteps
    for _ in range(nsteps):
        if divb == 2:
            U, P, b, _ = orc.step_uct(c, dt, U, P, b)
        else:
            U, P, _ = orc.step(c, dt, U, P)
    ve, Be = I.cp_alfven_fields(p, X, Y, Z, tend, kdir)
    P8e = orc.get_prims(c, U, P)
    return float(np.mean(np.abs(P8e[5] - Be[0])) + np.mean(np.abs(P8e[7] - Be[2])) + np.mean(np.abs(P8e[1] - ve[0])))


def test_alfven_oblique_convergence(orc):
    # P4 for f2: UCT moves B at the reconstruction order (nominal 5) on a wave crossing
    # both transverse directions of every edge; field-CD stays at 2
    e = [_alfven_oblique(orc, N, 2) for N in (16, 32)]
    assert math.log2(e[0] / e[1]) > 4.3, e
    ecd = [_alfven_oblique(orc, N, 0) for N in (16, 32)]
    assert math.log2(ecd[0] / ecd[1]) < 2.6 and e[1] < ecd[1] / 20, (e, ecd)


def test_uct_entry_points_refuse_other_setups(orc):
    p, c, U, P, b = _random_uct_state(orc, (6, 6, 6))
    with pytest.raises(orc.OracleError):
        orc.rhs_uct(orc.Cfg(n=(6, 6, 6), divb=0), U, P, b)
    with pytest.raises(orc.OracleError):
        orc.rhs(c, U, P)  # UCT needs the staggered field
