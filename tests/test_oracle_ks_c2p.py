"""Pins of the oracle's curved-metric prim<->cons pair (SURVEY.md §8(c) P9 applied to
the Kerr-Schild metric config 4 uses; BASELINE.json configs[4]; "the
equations of magneto-hydrodynamic in General Relativity").

The flat-metric pins (test_oracle_pointwise) cannot see a wrong index placement in
the metric contractions of con2prim (S^2 = gamma^{ij} S_i S_j, B_i = gamma_ij B^j,
v^i = gamma^{ij} v_j), since there gamma_ij = delta_ij.  Here:

1. the oracle's prim->cons at random Kerr-Schild points (a = 0.9, gamma_13 != 0) is
   checked against the conserved variables built from the 4-D stress-energy tensor
   T^{mu nu} = (rho h + b^2) u^mu u^nu + (p + b^2/2) g^{mu nu} - b^mu b^nu of the
   Eulerian observer n_mu = (-alpha, 0, 0, 0): D = rho W, S_i = alpha T^0_i,
   U = alpha^2 T^00 (a different route: no 3+1 identity of A1 is used);
2. prim -> cons -> con2prim round trips 10^4 random states at random Kerr-Schild
   points from a 1 % guess (the Newton solve of A8 in the curved metric).
CPU only; the metric itself is pinned by closed forms in test_oracle_pointwise.
"""
import math

import numpy as np
import pytest

GAMMA = 4.0 / 3.0
EPS = 2.0 ** -52


def kappa(met, pr, gamma=GAMMA):
    """(Z + B^2) / p of a state (rho, u~, p, B): the conditioning of p in con2prim."""
    ut, B = pr[1:4], pr[5:8]
    Z = (pr[0] + gamma / (gamma - 1) * pr[4]) * (1.0 + ut @ met["g"] @ ut)
    return (Z + B @ met["g"] @ B) / pr[4]


def ks(orc, a=0.9):
    # BASELINE.json configs[4]: Kerr-Schild, spin a = 0.9, x1 = ln r, x2 = theta, x3 = phi (A14)
    return orc.Cfg(metric=1, M=1.0, a=a, w_max=1e3)


def random_point(rng):
    r = math.exp(rng.uniform(math.log(1.2), math.log(60.0)))  # config 4's radial range (A14)
    th = rng.uniform(0.05 * math.pi, 0.95 * math.pi)
    ph = rng.uniform(0.0, 2.0 * math.pi)
    return np.array([math.log(r), th, ph])


def random_state(rng, met, wmax=10.0):
    """(rho, u~^i, p, B^i) with W in [1, wmax], p/rho in [1e-3, 1e2], B^2/(2p) in [1e-2, 1e2],
    directions random in the metric's own norm."""
    g = met["g"]
    W = rng.uniform(1.0, wmax)
    d = rng.normal(size=3)
    v = d / math.sqrt(d @ g @ d) * math.sqrt(1.0 - 1.0 / W ** 2)
    rho = 10 ** rng.uniform(-2, 1)
    p = rho * 10 ** rng.uniform(-3, 2)
    beta = 10 ** rng.uniform(-2, 2)
    e = rng.normal(size=3)
    B = e / math.sqrt(e @ g @ e) * math.sqrt(2 * p / beta)
    return np.array([rho, *(W * v), p, *B])


def covariant_cons(met, pr, gamma=GAMMA):
    """Non-densitised (D, S_i, tau, B^i) from T^{mu nu} (see the module docstring)."""
    al, be, g = met["alpha"], met["beta"], met["g"]
    rho, ut, p, B = pr[0], pr[1:4], pr[4], pr[5:8]
    W = math.sqrt(1.0 + ut @ g @ ut)
    v = ut / W
    u4 = np.concatenate([[W / al], ut - W * be / al])          # u^mu
    Bv = B @ g @ v
    b0 = W * Bv / al
    b4 = np.concatenate([[b0], B / W + W * Bv * (v - be / al)])  # b^mu
    g4 = np.zeros((4, 4))                                        # g_{mu nu}
    bl = g @ be
    g4[0, 0] = -al * al + be @ bl
    g4[0, 1:] = g4[1:, 0] = bl
    g4[1:, 1:] = g
    gi4 = np.zeros((4, 4))                                       # g^{mu nu}
    gi4[0, 0] = -1.0 / al ** 2
    gi4[0, 1:] = gi4[1:, 0] = be / al ** 2
    gi4[1:, 1:] = met["gi"] - np.outer(be, be) / al ** 2
    b2 = b4 @ g4 @ b4
    h = 1.0 + gamma / (gamma - 1.0) * p / rho
    T = (rho * h + b2) * np.outer(u4, u4) + (p + 0.5 * b2) * gi4 - np.outer(b4, b4)
    T0_low = T[0] @ g4                                           # T^0_nu
    D = rho * W
    S = al * T0_low[1:]
    U = al * al * T[0, 0]
    return np.array([D, *S, U - D, *B]), b2, W


def test_ks_points_have_offdiagonal_metric(orc):
    # the test points exercise the r-phi coupling of Kerr-Schild (gamma_13 != 0, A14)
    rng = np.random.default_rng(1)
    c = ks(orc)
    off = [abs(orc.metric(c, random_point(rng))["g"][0, 2]) for _ in range(200)]
    assert min(off) > 1e-3


def test_ks_prim2cons_matches_stress_energy_tensor(orc):
    rng = np.random.default_rng(11)
    c = ks(orc)
    worst = 0.0
    for _ in range(2000):
        x = random_point(rng)
        met = orc.metric(c, x)
        pr = random_state(rng, met)
        got = orc.prim2cons_pt(c, x, pr)
        ref, b2, W = covariant_cons(met, pr)
        # group scales (A16): D, S (lowered: compare against the S^i S_i norm), tau, B
        sS = math.sqrt(abs(ref[1:4] @ met["gi"] @ ref[1:4])) + 1e-300
        errs = (abs(got[0] / ref[0] - 1), np.max(np.abs(got[1:4] - ref[1:4])) / max(sS, np.max(np.abs(ref[1:4]))),
                abs(got[4] - ref[4]) / (ref[4] + ref[0]), np.max(np.abs(got[5:8] - ref[5:8])))
        worst = max(worst, *errs)
    # measured 6e-13: the rounding of the T^{mu nu} route itself (W <= 10)
    assert worst < 5e-12, worst


def test_ks_con2prim_roundtrip(orc):
    """P9 in Kerr-Schild: 10^4 random states at random points, prim -> cons -> prim from a
    1 % guess.  Error relative on rho and p, and on u~ scaled by max(1, |u~|) in the metric
    norm.  Bound per state: max(1e-13, 8 eps kappa) with kappa = (Z + B^2)/p, the condition
    number of recovering p from the total energy (p enters U only as Z - p + ...): measured
    e <= 2.8 eps kappa here and in the flat metric alike, so an index slip (an O(1) error,
    test_wrong_contraction_would_fail) cannot hide under it."""
    rng = np.random.default_rng(7)
    c = ks(orc)
    worst = 0.0
    iters = []
    for _ in range(10000):
        x = random_point(rng)
        met = orc.metric(c, x)
        pr = random_state(rng, met)
        u = orc.prim2cons_pt(c, x, pr)
        guess = pr.copy()
        guess[0] *= 1.01
        guess[4] *= 0.99
        st, out, it = orc.c2p_pt(c, x, u, guess)
        assert st == 0, (x, pr)
        iters.append(it)
        ut = pr[1:4]
        scale_u = max(1.0, math.sqrt(ut @ met["g"] @ ut))
        err = max(abs(out[0] / pr[0] - 1), abs(out[4] / pr[4] - 1), np.max(np.abs(out[1:4] - ut)) / scale_u)
        worst = max(worst, err / max(1e-13, 8 * EPS * kappa(met, pr)))
    assert worst <= 1.0, worst
    assert np.median(iters) <= 5 and max(iters) <= 30


def test_ks_con2prim_roundtrip_torus_states(orc):
    """The same at config 4's own states (torus and atmosphere: W <= 1.5, p/rho ~ 1e-4..1e-2,
    beta ~ 100), same per-state bound."""
    rng = np.random.default_rng(9)
    c = ks(orc)
    worst = 0.0
    for _ in range(5000):
        x = random_point(rng)
        met = orc.metric(c, x)
        g = met["g"]
        W = rng.uniform(1.0, 1.5)
        d = rng.normal(size=3)
        v = d / math.sqrt(d @ g @ d) * math.sqrt(1.0 - 1.0 / W ** 2)
        rho = 10 ** rng.uniform(-6, 0)
        p = rho * 10 ** rng.uniform(-4, -2)
        e = rng.normal(size=3)
        B = e / math.sqrt(e @ g @ e) * math.sqrt(2 * p / 100.0)
        pr = np.array([rho, *(W * v), p, *B])
        u = orc.prim2cons_pt(c, x, pr)
        guess = pr.copy()
        guess[0] *= 1.01
        guess[4] *= 0.99
        st, out, it = orc.c2p_pt(c, x, u, guess)
        assert st == 0
        ut = pr[1:4]
        scale_u = max(1.0, math.sqrt(ut @ g @ ut))
        err = max(abs(out[0] / pr[0] - 1), abs(out[4] / pr[4] - 1), np.max(np.abs(out[1:4] - ut)) / scale_u)
        worst = max(worst, err / max(1e-13, 8 * EPS * kappa(met, pr)))
    assert worst <= 1.0, worst


@pytest.mark.parametrize("which", ["S2_lowered", "B_not_lowered", "v_not_raised"])
def test_wrong_contraction_would_fail(orc, which):
    """The round trip detects each plausible index slip (a numpy Newton solve written from
    A8 with one contraction deliberately wrong does NOT reproduce the state, while the
    correct one does), so the pins above can fail."""
    rng = np.random.default_rng(5)
    c = ks(orc)
    bad = 0
    for _ in range(50):
        x = random_point(rng)
        met = orc.metric(c, x)
        pr = random_state(rng, met, wmax=3.0)
        u = orc.prim2cons_pt(c, x, pr)
        ok_r = _np_c2p(met, u, pr, None)
        assert np.max(np.abs(ok_r - pr[:5]) / np.maximum(1.0, np.abs(pr[:5]))) < 1e-9
        wrong = _np_c2p(met, u, pr, which)
        if np.max(np.abs(wrong - pr[:5]) / np.maximum(1.0, np.abs(pr[:5]))) > 1e-6:
            bad += 1
    assert bad >= 45


def _np_c2p(met, u, pr, slip, gamma=GAMMA):
    """Plain Newton in Z (A8) in numpy, optionally with one index slip."""
    g, gi = met["g"], met["gi"]
    D, S, tau, B = u[0], u[1:4], u[4], u[5:8]
    S2 = S @ (g if slip == "S2_lowered" else gi) @ S
    Bl = B if slip == "B_not_lowered" else g @ B
    B2 = B @ Bl
    SB = S @ B
    Ut = tau + D
    gm = (gamma - 1) / gamma
    W0 = math.sqrt(1 + pr[1:4] @ g @ pr[1:4])
    Z = (pr[0] + pr[4] / gm) * W0 ** 2 * 1.01
    for _ in range(60):
        def f(Z):
            v2 = (Z * Z * S2 + SB * SB * (2 * Z + B2)) / (Z * Z * (Z + B2) ** 2)
            v2 = min(v2, 1 - 1e-12)
            p = gm * (Z * (1 - v2) - D * math.sqrt(1 - v2))
            return Z - p + 0.5 * B2 * (1 + v2) - 0.5 * SB * SB / (Z * Z) - Ut
        h = 1e-7 * Z
        Zn = Z - f(Z) / ((f(Z + h) - f(Z - h)) / (2 * h))
        Z = Zn if Zn > 0 else 0.5 * Z
    v2 = min((Z * Z * S2 + SB * SB * (2 * Z + B2)) / (Z * Z * (Z + B2) ** 2), 1 - 1e-12)
    W = 1 / math.sqrt(1 - v2)
    vl = (S + SB * Bl / Z) / (Z + B2)
    vu = vl if slip == "v_not_raised" else gi @ vl
    return np.array([D / W, *(W * vu), gm * (Z * (1 - v2) - D / W)])
