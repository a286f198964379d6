"""Pins of reading A44 (rec = 6): characteristic-wise WENO5 of the hydro primitives
(SURVEY.md §8(f) f3 "characteristic-wise reconstruction"; "high-order
reconstruction algorithms").  CPU only.

The oracle builds R (right eigenvectors of the flat relativistic-Euler Jacobian) from closed
forms and L = R^-1 by Gauss-Jordan.  The pins below check it against what the mathematics
fixes, with nothing retyped from the oracle:
* exactness: constant, linear and quadratic stencils give the exact interface values
  (point-form WENO5 candidates are exact on quadratics, and R L = I);
* the characteristic property: a stencil varying only along one eigenvector r of the
  Jacobian A = (dU/dq)^-1 dF/dq -- A built by finite differences of the oracle's pinned
  prim2cons / flux point functions, r from numpy's eigensolver -- yields face states that
  differ from the face state only along r (acoustic waves), or stay inside the
  lambda = v^n eigenspace (contact + shear);
* mirror symmetry, order 5 on smooth data, and the whole scheme's order on a sound wave.
"""
import math

import numpy as np
import pytest

import echo_inputs as I

G = 4.0 / 3.0


def cfg(orc, **kw):
    return orc.Cfg(rec=6, **kw)


def stencil(rows):
    st = np.zeros((6, 8))
    for m, r in enumerate(rows):
        st[m, :5] = r
        st[m, 5:] = (0.3, -0.1, 0.2)  # B (reconstructed component-wise, unused by char_rec)
    return st


def jacobian_q(orc, c, q, a):
    """A = (dU/dq)^-1 dF^a/dq in the sweep frame q = (rho, u~^n, u~^t1, u~^t2, p), by central
    differences of the oracle's prim2cons / flux point functions (B = 0, flat)."""
    comp = [a, (a + 1) % 3, (a + 2) % 3]
    perm = [0, 1 + comp[0], 1 + comp[1], 1 + comp[2], 4]   # frame -> state slots

    def to_state(qf):
        pr = np.zeros(8)
        pr[perm] = qf
        return pr

    def UF(qf):
        pr = to_state(qf)
        u = orc.prim2cons_pt(c, [0.5, 0.5, 0.5], pr)
        f = orc.flux_pt(c, [0.5, 0.5, 0.5], pr, a)
        return u[perm], f[perm]

    JU, JF = np.zeros((5, 5)), np.zeros((5, 5))
    for j in range(5):
        d = np.zeros(5)
        d[j] = 1e-6 * max(1.0, abs(q[j]))
        up, fp = UF(q + d)
        um, fm = UF(q - d)
        JU[:, j] = (up - um) / (2 * d[j])
        JF[:, j] = (fp - fm) / (2 * d[j])
    return np.linalg.solve(JU, JF)


def frame(q, a):
    """state slots (rho, u~^1..3, p) -> sweep frame (rho, u~^n, u~^t1, u~^t2, p) and back"""
    comp = [a, (a + 1) % 3, (a + 2) % 3]
    return np.array([q[0], q[1 + comp[0]], q[1 + comp[1]], q[1 + comp[2]], q[4]])


def random_q(rng):
    u = rng.uniform(-0.6, 0.6, 3)
    return np.array([10 ** rng.uniform(-1, 0.5), *u, 10 ** rng.uniform(-1.5, 0.5)])


def test_exact_on_constant_linear_quadratic(orc):
    rng = np.random.default_rng(1)
    c = cfg(orc)
    for _ in range(200):
        q0 = random_q(rng)
        sc = np.array([q0[0], 0.1, 0.1, 0.1, q0[4]])  # increments small against rho and p (stays physical)
        q1, q2 = 0.02 * sc * rng.normal(size=5), 0.002 * sc * rng.normal(size=5)
        for a in range(3):
            for rows in (lambda m: q0, lambda m: q0 + m * q1, lambda m: q0 + m * q1 + m * m * q2):
                st = stencil([rows(m) for m in range(6)])
                qL, qR = orc.charrec_face(c, st, a)
                exact = rows(2.5)  # the interface value of the polynomial at m = 2.5 (face i+1/2)
                assert np.allclose(qL, exact, rtol=1e-12, atol=1e-13), (a, qL, exact)
                assert np.allclose(qR, exact, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("a", [0, 1, 2])
def test_characteristic_property(orc, a):
    rng = np.random.default_rng(10 + a)
    c = cfg(orc)
    for _ in range(40):
        qs = random_q(rng)            # state slots
        qf = frame(qs, a)
        A = jacobian_q(orc, c, qf, a)
        lam, V = np.linalg.eig(A)
        lam, V = lam.real, V.real
        vn = qf[1] / math.sqrt(1 + qf[1:4] @ qf[1:4])
        # the two acoustic eigenvectors (simple eigenvalues) and the lambda = v^n eigenspace
        order = np.argsort(lam)
        ac = [order[0], order[4]]
        assert np.allclose(lam[order[1:4]], vn, atol=1e-6)
        # the lambda = v^n eigenspace as the null space of A - v^n I (SVD: a stable basis)
        E0 = np.linalg.svd(A - vn * np.eye(5))[2][2:].T
        # data varying along one direction r with f(2) = -f(3): the face mean is exactly qs
        f = np.array([0.3, -0.8, 1.0, -1.0, 0.7, -0.2])
        for k in ac:
            r = V[:, k] / np.max(np.abs(V[:, k])) * 0.05 * min(qs[0], qs[4])
            rows = [qf + f[m] * r for m in range(6)]
            st = stencil([back(x, a) for x in rows])
            qL, qR = orc.charrec_face(c, st, a)
            for out in (qL, qR):
                d = frame(out, a) - qf
                # parallel to r: the component orthogonal to r vanishes to rounding
                perp = d - (d @ r) / (r @ r) * r
                assert np.linalg.norm(perp) <= 1e-8 * np.linalg.norm(r), (k, perp)  # FD Jacobian: ~1e-10
            # and by the exact amount on a quadratic amplitude (f2(2) = -f2(3): same face mean)
            f2 = np.array([(m - 2.5) + 0.3 * ((m - 2.5) ** 2 - 0.25) for m in range(6)])
            st2 = stencil([back(qf + f2[m] * r, a) for m in range(6)])
            for out in orc.charrec_face(c, st2, a):
                assert np.allclose(frame(out, a), qf - 0.075 * r, rtol=1e-12, atol=1e-14)
        # a variation inside the lambda = v^n eigenspace stays inside it
        r = E0 @ rng.normal(size=3)
        r *= 0.05 * min(qs[0], qs[4]) / np.max(np.abs(r))
        rows = [qf + f[m] * r for m in range(6)]
        qL, qR = orc.charrec_face(c, stencil([back(x, a) for x in rows]), a)
        for out in (qL, qR):
            d = frame(out, a) - qf
            res = d - E0 @ np.linalg.lstsq(E0, d, rcond=None)[0]
            assert np.linalg.norm(res) <= 1e-8 * np.linalg.norm(r)


def back(qf, a):
    comp = [a, (a + 1) % 3, (a + 2) % 3]
    q = np.zeros(5)
    q[0], q[4] = qf[0], qf[4]
    for d in range(3):
        q[1 + comp[d]] = qf[1 + d]
    return q


def test_mirror_symmetry(orc):
    """Reflecting the stencil about the face and reversing the normal velocity swaps the
    left and right states (with the normal velocity reversed)."""
    rng = np.random.default_rng(3)
    c = cfg(orc)
    for _ in range(100):
        rows = [random_q(rng) for _ in range(6)]
        a = int(rng.integers(3))
        mir = []
        for m in range(6):
            q = rows[5 - m].copy()
            q[1 + a] = -q[1 + a]
            mir.append(q)
        qL, qR = orc.charrec_face(c, stencil(rows), a)
        mL, mR = orc.charrec_face(c, stencil(mir), a)
        for x, y in ((qL, mR), (qR, mL)):
            y = y.copy()
            y[1 + a] = -y[1 + a]
            assert np.allclose(x, y, rtol=1e-12, atol=1e-14)


def test_order_on_smooth_data(orc):
    c = cfg(orc)
    errs = []
    for N in (32, 64, 128):
        h = 1.0 / N
        x = (np.arange(-2, 4) + 0.5) * h  # cells i-2..i+3: cell i at h/2, the face i+1/2 at h
        errs_N = 0.0
        for x0 in np.linspace(0, 1, 7, endpoint=False):
            xs = x0 + x
            def q_at(z):
                return np.array([1 + 0.2 * np.sin(2 * np.pi * z), 0.3 * np.cos(2 * np.pi * z), 0.1 * np.sin(4 * np.pi * z),
                                 -0.2, 0.8 + 0.1 * np.cos(2 * np.pi * z)])
            st = stencil([q_at(z) for z in xs])
            qL, qR = orc.charrec_face(c, st, 0)
            exact = q_at(x0 + h)
            errs_N = max(errs_N, np.max(np.abs(qL - exact)), np.max(np.abs(qR - exact)))
        errs.append(errs_N)
    for e1, e2 in zip(errs, errs[1:]):
        assert math.log2(e1 / e2) > 4.5, errs


def test_sound_wave_self_convergence_characteristic(orc):
    """The whole scheme with rec = 6 on P5's smooth sound wave (B = 0): order > 4.5."""
    from tests.test_oracle_scheme import _sound, state

    c1 = []
    tend = 0.2
    for N in (24, 48, 96):
        c = orc.Cfg(n=(N, 1, 1), hi=(1.0, 1.0 / N, 1.0 / N), rec=6)
        U, P = state(orc, c, _sound(N))
        nsteps = int(math.ceil(tend / (0.5 * (1.0 / N) ** (5.0 / 3.0))))
        for _ in range(nsteps):
            U, P, _ = orc.step(c, tend / nsteps, U, P)
        rho = orc.get_prims(c, U, P)[0, 0, 0]
        x = (np.arange(N) + 0.5) / N
        c1.append(np.mean(rho * np.exp(-2j * np.pi * x)))
    e1, e2 = abs(c1[0] - c1[1]), abs(c1[1] - c1[2])
    assert math.log2(e1 / e2) > 4.5, (e1, e2)


def test_blast_runs_floor_free(orc):
    """Config 2's blast (p jump 1000x) at 40^3 for 10 steps with rec = 6: no floor fires."""
    p = I.problem(2, n=(40, 40, 40))
    p.rec = 6
    c = orc.Cfg(**p.grid_kwargs())
    U, P = orc.set_prims(c, I.initial_prims(p))
    cnt = [0, 0]
    for _ in range(10):
        U, P, k = orc.step(c, orc.max_dt(c, U, P, p.cfl), U, P)
        cnt[0] += k[0]
        cnt[1] += k[1]
    assert cnt == [0, 0] and float(P[4].max()) < 1.01  # (0.4 % overshoot at 40^3)


def test_refused_outside_its_scope(orc):
    """Reading A44 is flat-metric and not combined with UCT: the oracle refuses both."""
    p = I.problem(4, n=(16, 8, 8))
    p.rec = 6
    c = orc.Cfg(**p.grid_kwargs())
    U, P = orc.set_prims(c, I.initial_prims(p))
    with pytest.raises(orc.OracleError):
        orc.rhs(c, U, P)
