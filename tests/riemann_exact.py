"""Exact solution of the 1-D Riemann problem of special-relativistic hydrodynamics (ideal gas,
no transverse velocity, B = 0): test infrastructure for pinning the oracle's shock-capturing
dynamics (the blast of config 2 has no exact solution; a shock tube does).

Written from the physics, not from the oracle (which it shares nothing with):
* rarefactions are isentropic simple waves: p / rho^Gamma constant and the Riemann invariant
  J = atanh(v) + s g(c) constant across the fan (s = +1 for the left-facing wave, -1 for the
  right-facing one), with g(c) = int c drho / rho = (2 / sqrt(Gamma - 1)) atanh(c / sqrt(Gamma - 1))
  for the ideal gas (d g / d rho = c / rho along the isentrope), and inside the fan the head-to-tail
  characteristic xi = (v - s c) / (1 - s v c);
* shocks satisfy the Rankine-Hugoniot conditions: the post-shock state on the Taub adiabat
  [h^2] = (h_b / rho_b + h_a / rho_a) [p], mass flux j^2 = -[p] / [h / rho], shock speed and
  post-shock velocity from the jump conditions of D and S (Marti & Mueller's closed forms);
* the star pressure joins the two waves' velocities (contact: p and v continuous).
Both branches are verified in tests/test_oracle_riemann.py against conservation itself: the shock
against F(U_b) - F(U_a) = V_s (U_b - U_a), the fan against dF/dxi = xi dU/dxi.
"""
import math

import numpy as np
from scipy.optimize import brentq


class Gas:
    def __init__(self, gamma):
        self.G = gamma
        self.k = gamma / (gamma - 1.0)

    def h(self, rho, p):
        return 1.0 + self.k * p / rho

    def cs(self, rho, p):
        return math.sqrt(self.G * p / (rho * self.h(rho, p)))

    def g(self, c):
        s = math.sqrt(self.G - 1.0)
        return 2.0 / s * math.atanh(c / s)

    def cons(self, rho, p, v):
        """(D, S, tau) and the x fluxes"""
        W = 1.0 / math.sqrt(1.0 - v * v)
        hh = self.h(rho, p)
        D, S, tau = rho * W, rho * hh * W * W * v, rho * hh * W * W - p - rho * W
        return np.array([D, S, tau]), np.array([D * v, S * v + p, S - D * v])


def rarefaction(gas, rho_a, p_a, v_a, p, s):
    """state (rho, v) reached from state a at pressure p through a simple wave (s = +1 left wave)"""
    rho = rho_a * (p / p_a) ** (1.0 / gas.G)
    J = math.atanh(v_a) + s * gas.g(gas.cs(rho_a, p_a))
    v = math.tanh(J - s * gas.g(gas.cs(rho, p)))
    return rho, v


def shock(gas, rho_a, p_a, v_a, p, s):
    """post-shock (rho, v, V_s) for pressure p > p_a, a the unshocked state; s = +1 the left wave
    (a left-facing shock, mass flux j < 0), s = -1 the right wave (j > 0)"""
    k, ha = gas.k, gas.h(rho_a, p_a)
    dp = p - p_a
    # Taub adiabat in x = 1 / rho_b with h_b = 1 + k p x: A x^2 + B x + C = 0
    A = k * k * p * p - k * p * dp
    B = 2.0 * k * p - dp
    C = 1.0 - ha * ha - ha * dp / rho_a
    disc = B * B - 4.0 * A * C
    x = max((-B + sg * math.sqrt(disc)) / (2.0 * A) for sg in (1.0, -1.0))
    rho_b = 1.0 / x
    hb = 1.0 + k * p * x
    j2 = -dp / (hb * x - ha / rho_a)
    j = -s * math.sqrt(j2)
    Wa = 1.0 / math.sqrt(1.0 - v_a * v_a)
    r2 = rho_a * rho_a * Wa * Wa
    Vs = (r2 * v_a + j * math.sqrt(j2 + rho_a * rho_a)) / (r2 + j2)
    Ws = 1.0 / math.sqrt(1.0 - Vs * Vs)
    v_b = (ha * Wa * v_a + Ws * dp / j) / (ha * Wa + dp * (Ws * v_a / j + 1.0 / (rho_a * Wa)))
    return rho_b, v_b, Vs


def wave(gas, rho_a, p_a, v_a, p, s):
    if p > p_a:
        rho, v, _ = shock(gas, rho_a, p_a, v_a, p, s)
    else:
        rho, v = rarefaction(gas, rho_a, p_a, v_a, p, s)
    return rho, v


class Riemann:
    """the exact solution for left / right states (rho, p, v), interface at xi = 0"""

    def __init__(self, gamma, L, R):
        self.gas = gas = Gas(gamma)
        self.L, self.R = L, R
        f = lambda p: wave(gas, *L, p, +1)[1] - wave(gas, *R, p, -1)[1]
        lo, hi = 1e-12 * min(L[1], R[1]), 1e3 * max(L[1], R[1])
        self.ps = brentq(f, lo, hi, xtol=1e-15, rtol=1e-15, maxiter=500)
        self.rhoL, self.vs = wave(gas, *L, self.ps, +1)
        self.rhoR, _ = wave(gas, *R, self.ps, -1)

    def _fan(self, side, xi):
        gas = self.gas
        rho_a, p_a, v_a = side
        s = +1 if side is self.L else -1
        def speed(p):
            rho, v = rarefaction(gas, rho_a, p_a, v_a, p, s)
            c = gas.cs(rho, p)
            return (v - s * c) / (1.0 - s * v * c) - xi
        lo, hi = sorted((self.ps, p_a))
        p = brentq(speed, lo, hi, xtol=1e-15, rtol=1e-15, maxiter=500)
        rho, v = rarefaction(gas, rho_a, p_a, v_a, p, s)
        return rho, p, v

    def sample(self, xi):
        """(rho, p, v) at xi = x / t"""
        gas = self.gas
        if xi < self.vs:  # left of the contact
            rho_a, p_a, v_a = self.L
            if self.ps > p_a:
                _, _, Vs = shock(gas, rho_a, p_a, v_a, self.ps, +1)
                return self.L if xi < Vs else (self.rhoL, self.ps, self.vs)
            ca, cs_ = gas.cs(rho_a, p_a), gas.cs(self.rhoL, self.ps)
            head = (v_a - ca) / (1.0 - v_a * ca)
            tail = (self.vs - cs_) / (1.0 - self.vs * cs_)
            if xi < head:
                return self.L
            if xi > tail:
                return (self.rhoL, self.ps, self.vs)
            return self._fan(self.L, xi)
        rho_a, p_a, v_a = self.R
        if self.ps > p_a:
            _, _, Vs = shock(gas, rho_a, p_a, v_a, self.ps, -1)
            return self.R if xi > Vs else (self.rhoR, self.ps, self.vs)
        ca, cs_ = gas.cs(rho_a, p_a), gas.cs(self.rhoR, self.ps)
        head = (v_a + ca) / (1.0 + v_a * ca)
        tail = (self.vs + cs_) / (1.0 + self.vs * cs_)
        if xi > head:
            return self.R
        if xi < tail:
            return (self.rhoR, self.ps, self.vs)
        return self._fan(self.R, xi)
