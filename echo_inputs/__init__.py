"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is shared by the oracle side (tests) and the product side
(bench.py, GPU tests).  It holds NONE of the method's arithmetic: it only
builds initial primitive states (rho, v^i, p, B^i) and the problem
description (grid, metric, EOS, floors).  The recipes are DESIGN.md §5
(SURVEY.md §8(d)); the paper's own workloads (512^3 / 1024^3
GRMHD runs; Fig. 1 torus) are unspecified, so these synthetic
states stand in for them.

Random numbers: splitmix64 (sequential, for Fourier-mode draws) and a
counter-based hash of (seed, global linear cell index) for per-cell white
noise, so inputs are independent of any thread/rank layout.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

MASK = (1 << 64) - 1
GAMMA = 4.0 / 3.0
PERIODIC, OUTFLOW = 0, 1
MINKOWSKI, KERR_SCHILD = 0, 1


# ----------------------------------------------------------------- RNG
class SplitMix64:
    def __init__(self, seed: int):
        self.s = seed & MASK

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform(self) -> float:  # [0, 1)
        return (self.next() >> 11) * (1.0 / (1 << 53))


def white_noise(seed: int, n_total: int, stream: int = 0) -> np.ndarray:
    """xi in [-1, 1) = hash(seed, stream, global linear index), numpy uint64 wrap-around."""
    with np.errstate(over="ignore"):
        idx = np.arange(n_total, dtype=np.uint64)
        z = idx * np.uint64(0x9E3779B97F4A7C15) + np.uint64(((seed * 0xD1B54A32D192ED03) ^ (stream * 0x8CB92BA72F3D8DD7)) & MASK)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))
    return 2.0 * u - 1.0


# ------------------------------------------------------------ problem
@dataclass
class Problem:
    """Grid + metric + EOS + floors + run length of one config."""

    name: str
    n: tuple
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)
    bc: tuple = ((PERIODIC, PERIODIC),) * 3
    metric: int = MINKOWSKI
    M: float = 1.0
    a: float = 0.0
    gamma: float = GAMMA
    rho_floor: float = 1e-8
    p_floor: float = 1e-10
    w_max: float = 50.0
    c2p_max_iter: int = 30
    c2p_tol: float = 1e-13
    rec: int = 0
    der: int = 6
    divb: int = 0
    der_jump: float = 0.5
    steps: int = 10
    cfl: float = 0.4
    dz: float = 0.0  # > 0: the z cell size itself (a z slab of a larger grid, echo.h echo_grid.dz)
    seed: int = 0
    params: dict = field(default_factory=dict)

    @property
    def ncells(self) -> int:
        return int(self.n[0]) * int(self.n[1]) * int(self.n[2])

    def grid_kwargs(self) -> dict:
        return dict(n=tuple(self.n), lo=tuple(self.lo), hi=tuple(self.hi), bc=tuple(tuple(b) for b in self.bc),
                    metric=self.metric, M=self.M, a=self.a, gamma=self.gamma, rho_floor=self.rho_floor,
                    p_floor=self.p_floor, w_max=self.w_max, c2p_max_iter=self.c2p_max_iter,
                    c2p_tol=self.c2p_tol, rec=self.rec, der=self.der, divb=self.divb, der_jump=self.der_jump,
                    **({"dz": self.dz} if self.dz > 0 else {}))

    def centres(self, a: int) -> np.ndarray:
        d = (self.hi[a] - self.lo[a]) / self.n[a]
        return self.lo[a] + (np.arange(self.n[a]) + 0.5) * d


def problem(cfg: int, n=None, seed=None) -> Problem:
    """BASELINE.json configs[cfg]; `n` overrides the grid (same physics, smaller grid)."""
    if cfg == 0:
        p = Problem("cfg0_turbulence32", (32, 32, 32), steps=10,
                    params=dict(modes=8, kmax=4, amp=0.05, vmax=0.1, B0=0.5))
    elif cfg == 1:
        p = Problem("cfg1_cp_alfven128", (128, 128, 128), steps=50, params=dict(eta=0.1, B0=1.0, noise=1e-6))
    elif cfg == 2:
        p = Problem("cfg2_blast256", (256, 256, 256), bc=((OUTFLOW, OUTFLOW),) * 3, steps=20,
                    params=dict(rho=1e-2, p_in=1.0, p_out=1e-3, radius=0.1, Bx=0.1, jitter=0.01))
    elif cfg == 3:
        p = Problem("cfg3_turbulence512", (512, 512, 512), steps=5,
                    params=dict(modes=32, kmax=8, amp=0.1, vmax=0.1, B0=0.5))
    elif cfg == 4:
        p = Problem("cfg4_ks_torus", (256, 128, 256), lo=(math.log(1.2), 0.05 * math.pi, 0.0),
                    hi=(math.log(60.0), 0.95 * math.pi, 2.0 * math.pi),
                    bc=((OUTFLOW, OUTFLOW), (OUTFLOW, OUTFLOW), (PERIODIC, PERIODIC)),
                    metric=KERR_SCHILD, M=1.0, a=0.9, rho_floor=1e-6, p_floor=1e-10, steps=10,
                    params=dict(r_in=7.0, r_max=12.0, K=0.01, beta=100.0, rho_atm=1e-6, p_atm=1e-10, pert=0.02))
    else:
        raise ValueError(f"unknown config {cfg}")
    p.seed = cfg if seed is None else seed
    p.params["cfg"] = cfg
    if n is not None:
        p.n = tuple(int(v) for v in n)
    return p


# -------------------------------------------------------- array helpers
def _backend(device):
    if device is None or device == "numpy":
        return None
    import torch  # plumbing only: IC evaluation on a device for the 512^3 bench state
    return torch


def _coords(p: Problem, torch, device):
    xs = [p.centres(a) for a in range(3)]
    if torch is None:
        return (xs[0][None, None, :], xs[1][None, :, None], xs[2][:, None, None])
    t = [torch.tensor(x, dtype=torch.float64, device=device) for x in xs]
    return (t[0].view(1, 1, -1), t[1].view(1, -1, 1), t[2].view(-1, 1, 1))


def draw_modes(rng: SplitMix64, nmodes: int, kmax: int):
    modes = []
    for _ in range(nmodes):
        while True:
            k = [int(rng.next() % (2 * kmax + 1)) - kmax for _ in range(3)]
            if any(k):
                break
        phi = 2.0 * math.pi * rng.uniform()
        w = 1.0 - rng.uniform()  # (0, 1]
        modes.append((k, phi, w))
    s = sum(abs(m[2]) for m in modes)
    return [(k, phi, w / s) for (k, phi, w) in modes]


def mode_sum(modes, X, Y, Z, torch=None, knorm=False):
    """M(x) = sum_m w_m sin(2 pi k_m . x + phi_m)  [optionally / (2 pi |k_m|)]."""
    sin = np.sin if torch is None else torch.sin
    out = 0.0
    for (k, phi, w) in modes:
        amp = w / (2.0 * math.pi * math.sqrt(k[0] ** 2 + k[1] ** 2 + k[2] ** 2)) if knorm else w
        out = out + amp * sin(2.0 * math.pi * (k[0] * X + k[1] * Y + k[2] * Z) + phi)
    return out


def _roll(a, s, axis, torch):
    return np.roll(a, s, axis=axis) if torch is None else torch.roll(a, s, dims=axis)


def curl_d2_periodic(A, dx, torch=None):
    """B = curl_D2 A on a periodic grid, arrays [n3][n2][n1]; axis 2 of the array is x."""
    def D(f, a):  # central difference along coordinate axis a
        ax = 2 - a
        return (_roll(f, -1, ax, torch) - _roll(f, 1, ax, torch)) / (2.0 * dx[a])
    Ax, Ay, Az = A
    return (D(Az, 1) - D(Ay, 2), D(Ax, 2) - D(Az, 0), D(Ay, 0) - D(Ax, 1))


def _stack(fields, torch):
    if torch is None:
        return np.ascontiguousarray(np.stack([np.broadcast_to(f, fields[0].shape) for f in fields]).astype(np.float64))
    return torch.stack([f.expand_as(fields[0]) for f in fields]).contiguous()


# --------------------------------------------------------------- ICs
def ic_turbulence(p: Problem, device=None):
    """configs 0 and 3: seeded multi-mode turbulence (SURVEY §8(d) cfg 0/3)."""
    torch = _backend(device)
    X, Y, Z = _coords(p, torch, device)
    prm = p.params
    rng = SplitMix64(p.seed)
    modes = [draw_modes(rng, prm["modes"], prm["kmax"]) for _ in range(8)]  # rho, p, v1..3, A1..3
    amp = prm["amp"]
    rho = 1.0 + amp * mode_sum(modes[0], X, Y, Z, torch)
    prs = 1.0 + amp * mode_sum(modes[1], X, Y, Z, torch)
    vs = [(prm["vmax"] / math.sqrt(3.0)) * mode_sum(modes[2 + c], X, Y, Z, torch) for c in range(3)]
    A = [amp * mode_sum(modes[5 + c], X, Y, Z, torch, knorm=True) for c in range(3)]
    dx = [(p.hi[a] - p.lo[a]) / p.n[a] for a in range(3)]
    B = curl_d2_periodic(A, dx, torch)
    Bx = B[0] + prm["B0"]
    return _stack([rho, vs[0], vs[1], vs[2], prs, Bx, B[1], B[2]], torch)


def cp_alfven_speed(eta: float, B0: float = 1.0, rho: float = 1.0, prs: float = 1.0, gamma: float = GAMMA) -> float:
    """v_A of the exact circularly-polarised Alfven wave: v_A^2 (rho h W^2 + B0^2) = B0^2,
    W^2 = 1/(1 - v_A^2 eta^2); solved by bisection."""
    rh = rho + gamma / (gamma - 1.0) * prs
    lo, hi = 0.0, 1.0
    for _ in range(200):
        va = 0.5 * (lo + hi)
        W2 = 1.0 / (1.0 - va * va * eta * eta)
        if va * va * (rh * W2 + B0 * B0) - B0 * B0 > 0:
            hi = va
        else:
            lo = va
    return 0.5 * (lo + hi)


def ic_cp_alfven(p: Problem, device=None, noise=True):
    """config 1: circularly polarised Alfven wave along (1,1,1)."""
    X, Y, Z = _coords(p, None, None)
    prm = p.params
    eta, B0 = prm["eta"], prm["B0"]
    va = cp_alfven_speed(eta, B0)
    phi = 2.0 * math.pi * (X + Y + Z)
    k = np.array([1.0, 1.0, 1.0]) / math.sqrt(3.0)
    e1 = np.array([1.0, -1.0, 0.0]) / math.sqrt(2.0)
    e2 = np.array([1.0, 1.0, -2.0]) / math.sqrt(6.0)
    c, s = np.cos(phi), np.sin(phi)
    B = [B0 * k[i] + eta * B0 * (c * e1[i] + s * e2[i]) for i in range(3)]
    v = [-va * eta * (c * e1[i] + s * e2[i]) for i in range(3)]
    shape = (p.n[2], p.n[1], p.n[0])
    rho = np.ones(shape)
    prs = np.ones(shape)
    if noise:
        prs = prs + prm["noise"] * white_noise(p.seed, p.ncells).reshape(shape)
    return _stack([rho, v[0], v[1], v[2], prs, B[0], B[1], B[2]], None)


def ic_blast(p: Problem, device=None):
    """config 2: relativistic MHD blast wave in an outflow box."""
    X, Y, Z = _coords(p, None, None)
    prm = p.params
    shape = (p.n[2], p.n[1], p.n[0])
    rho = prm["rho"] * (1.0 + prm["jitter"] * white_noise(p.seed, p.ncells).reshape(shape))
    r = np.sqrt((X - 0.5) ** 2 + (Y - 0.5) ** 2 + (Z - 0.5) ** 2)
    prs = np.where(r < prm["radius"], prm["p_in"], prm["p_out"]) * np.ones(shape)
    zero = np.zeros(shape)
    return _stack([rho, zero, zero, zero, prs, prm["Bx"] + zero, zero, zero], None)


# ------------------------------------------------ Kerr torus (IC only)
def _ks_metric_ic(M, a, r, th):
    """Kerr-Schild quantities in (ln r, theta, phi) needed to BUILD the torus IC
    (lapse, shift, 3-metric components, sqrt(gamma)).  IC arithmetic only."""
    s, c = np.sin(th), np.cos(th)
    rho2 = r * r + a * a * c * c
    z = 2.0 * M * r / rho2
    alpha = 1.0 / np.sqrt(1.0 + z)
    beta_r = z / (1.0 + z)
    g11 = r * r * (1.0 + z)
    g13 = r * (-a * (1.0 + z) * s * s)
    g22 = rho2
    g33 = s * s * (rho2 + a * a * (1.0 + z) * s * s)
    sqrtg = r * rho2 * s * np.sqrt(1.0 + z)
    return alpha, beta_r, (g11, g13, g22, g33), sqrtg


def torus_l_kepler(M, a, r):
    return math.sqrt(M) * (r * r - 2.0 * a * math.sqrt(M * r) + a * a) / (r ** 1.5 - 2.0 * M * math.sqrt(r) + a * math.sqrt(M))


def _bl_potential(M, a, ell, r, th):
    """W = ln(-u_t) of the constant-ell torus in Boyer-Lindquist; also u^t, u^phi."""
    s2 = np.sin(th) ** 2
    Sig = r * r + a * a * np.cos(th) ** 2
    Del = r * r - 2.0 * M * r + a * a
    Aa = (r * r + a * a) ** 2 - a * a * Del * s2
    gtt = -Aa / (Sig * Del)
    gtp = -2.0 * M * a * r / (Sig * Del)
    gpp = (Del - a * a * s2) / (Sig * Del * s2)
    q = gtt - 2.0 * ell * gtp + ell * ell * gpp
    with np.errstate(invalid="ignore", divide="ignore"):
        ut_low = -1.0 / np.sqrt(-q)
        Wp = np.log(-ut_low)
    u_phi_low = -ell * ut_low
    ut_up = gtt * ut_low + gtp * u_phi_low
    uphi_up = gtp * ut_low + gpp * u_phi_low
    return Wp, (q < 0) & (Del > 0), ut_up, uphi_up


def torus_hydro(p: Problem, r, th):
    """rho, p, v^1 (log-r), v^3 and the torus mask at (r, theta) arrays."""
    prm = p.params
    M, a, g = p.M, p.a, p.gamma
    ell = torus_l_kepler(M, a, prm["r_max"])
    W_in, _, _, _ = _bl_potential(M, a, ell, np.array(prm["r_in"]), np.array(math.pi / 2))
    Wp, ok, ut, uphi = _bl_potential(M, a, ell, r, th)
    with np.errstate(invalid="ignore", over="ignore"):
        h = np.exp(W_in - Wp)
    inside = ok & (r >= prm["r_in"]) & (h > 1.0)
    hh = np.where(inside, h, 1.0)
    rho = np.where(inside, ((hh - 1.0) * (g - 1.0) / (prm["K"] * g)) ** (1.0 / (g - 1.0)), 0.0)
    prs = prm["K"] * rho ** g
    alpha, beta_r, _, _ = _ks_metric_ic(M, a, r, th)
    with np.errstate(invalid="ignore", divide="ignore"):
        v_r = np.where(inside, beta_r / alpha, 0.0)  # u^r = 0
        v_phi = np.where(inside, uphi / (alpha * ut), 0.0)
    return rho, prs, v_r / r, v_phi, inside


def ic_torus(p: Problem, device=None):
    """config 4: constant-ell thick torus on Kerr-Schild (SURVEY §8(d) cfg 4, reading A15)."""
    return _torus(p)[0]


def _torus(p: Problem):
    """(prims8, rho_max, field scale) of config 4"""
    prm = p.params
    n1, n2, n3 = p.n
    d1 = (p.hi[0] - p.lo[0]) / n1
    d2 = (p.hi[1] - p.lo[1]) / n2
    # centres with one extra layer in x1, x2 (for the D2 curl of A_phi)
    x1 = p.lo[0] + (np.arange(-1, n1 + 1) + 0.5) * d1
    x2 = p.lo[1] + (np.arange(-1, n2 + 1) + 0.5) * d2
    R = np.exp(x1)[None, :]
    TH = x2[:, None]
    rho_e, prs_e, v1_e, v3_e, in_e = torus_hydro(p, R, TH)  # shape (n2+2, n1+2)
    rho_max = float(rho_e.max())
    Aphi = np.maximum(rho_e - 0.2 * rho_max, 0.0)
    sgB1 = (Aphi[2:, 1:-1] - Aphi[:-2, 1:-1]) / (2.0 * d2)   # sqrt(g) B^1 = d_theta A_phi
    sgB2 = -(Aphi[1:-1, 2:] - Aphi[1:-1, :-2]) / (2.0 * d1)  # sqrt(g) B^2 = -d_x1 A_phi
    rho = rho_e[1:-1, 1:-1]
    prs = prs_e[1:-1, 1:-1]
    v1 = v1_e[1:-1, 1:-1]
    v3 = v3_e[1:-1, 1:-1]
    inside = in_e[1:-1, 1:-1]
    r = np.exp(x1[1:-1])[None, :]
    th = x2[1:-1][:, None]
    alpha, beta_r, (g11, g13, g22, g33), sqrtg = _ks_metric_ic(p.M, p.a, r, th)
    B1 = sgB1 / sqrtg
    B2 = sgB2 / sqrtg
    # normalise to plasma beta: max p / max(b^2/2) over the torus
    v2 = g11 * v1 * v1 + 2.0 * g13 * v1 * v3 + g33 * v3 * v3
    W2 = 1.0 / (1.0 - v2)
    Bsq = g11 * B1 * B1 + g22 * B2 * B2
    vB = g11 * v1 * B1 + g13 * v3 * B1
    b2 = Bsq / W2 + vB * vB
    bmax = float(np.max(np.where(inside, b2, 0.0)))
    scale = 1.0
    if bmax > 0:
        pmax = float(np.max(np.where(inside, prs, 0.0)))
        scale = math.sqrt(pmax / (prm["beta"] * 0.5 * bmax))
        B1 = B1 * scale
        B2 = B2 * scale
    # atmosphere
    rho = np.where(inside, rho, prm["rho_atm"])
    prs = np.where(inside, prs, prm["p_atm"])
    v1 = np.where(inside, v1, 0.0)
    v3 = np.where(inside, v3, 0.0)
    shape = (n3, n2, n1)
    xi = white_noise(p.seed, p.ncells).reshape(shape)
    prs3 = np.broadcast_to(prs, shape) * np.where(np.broadcast_to(inside, shape), 1.0 + prm["pert"] * xi, 1.0)
    zero = np.zeros(shape)
    out = [np.broadcast_to(rho, shape), np.broadcast_to(v1, shape), zero, np.broadcast_to(v3, shape), prs3,
           np.broadcast_to(B1, shape), np.broadcast_to(B2, shape), zero]
    return np.ascontiguousarray(np.stack(out).astype(np.float64)), rho_max, scale


def _torus_face_field(p: Problem):
    """config 4 staggered field: A_phi = max(rho - 0.2 rho_max, 0) at the cell corners
    (x1 face, x2 face), its staggered curl sqrt(g) B^1 = d_theta A_phi at the x1 faces and
    sqrt(g) B^2 = -d_x1 A_phi at the x2 faces, with the cell-centred IC's beta scale"""
    _, rho_max, scale = _torus(p)
    n1, n2, n3 = p.n
    d1 = (p.hi[0] - p.lo[0]) / n1
    d2 = (p.hi[1] - p.lo[1]) / n2
    x1c = p.lo[0] + np.arange(n1 + 1) * d1   # faces -1/2 .. n1 - 1/2
    x2c = p.lo[1] + np.arange(n2 + 1) * d2
    rho_c = torus_hydro(p, np.exp(x1c)[None, :], x2c[:, None])[0]
    A = np.maximum(rho_c - 0.2 * rho_max, 0.0) * scale      # [n2 + 1][n1 + 1]
    b1 = (A[1:, 1:] - A[:-1, 1:]) / d2                      # face i + 1/2 = corner column i + 1
    b2 = -(A[1:, 1:] - A[1:, :-1]) / d1                     # face j + 1/2 = corner row j + 1
    shape = (n3, n2, n1)
    return [np.broadcast_to(b1, shape), np.broadcast_to(b2, shape), np.zeros(shape)]


def initial_prims(p: Problem, device=None, **kw):
    """prims8 [8][n3][n2][n1] (rho, v^1..3, p, B^1..3) for problem p (numpy, or torch on `device`)."""
    cfg = p.params["cfg"]
    if cfg in (0, 3):
        return ic_turbulence(p, device)
    if cfg == 1:
        return ic_cp_alfven(p, device, **kw)
    if cfg == 2:
        return ic_blast(p, device)
    if cfg == 4:
        return ic_torus(p, device)
    raise ValueError(cfg)


# ----------------------------------------------- staggered field (UCT, divb = 2)
def _coords_face(p: Problem, a: int, torch, device):
    """centre coordinates, except the face coordinates x_{i+1/2} along axis a"""
    xs = []
    for b in range(3):
        d = (p.hi[b] - p.lo[b]) / p.n[b]
        xs.append(p.lo[b] + (np.arange(p.n[b]) + (1.0 if b == a else 0.5)) * d)
    if torch is None:
        return (xs[0][None, None, :], xs[1][None, :, None], xs[2][:, None, None])
    t = [torch.tensor(x, dtype=torch.float64, device=device) for x in xs]
    return (t[0].view(1, 1, -1), t[1].view(1, -1, 1), t[2].view(-1, 1, 1))


def _curl_modes(modes_by_comp, a, X, Y, Z, amp, torch):
    """component a of the analytic curl of A^c = amp sum_m w_m sin(2 pi k_m.x + phi_m) / (2 pi |k_m|):
    d_j A^c = amp sum_m w_m (k_j / |k_m|) cos(...)"""
    cos = np.cos if torch is None else torch.cos
    def d(c, j):
        out = 0.0
        for (k, phi, w) in modes_by_comp[c]:
            kn = math.sqrt(k[0] ** 2 + k[1] ** 2 + k[2] ** 2)
            out = out + amp * w * (k[j] / kn) * cos(2.0 * math.pi * (k[0] * X + k[1] * Y + k[2] * Z) + phi)
        return out
    b1, b2 = (a + 1) % 3, (a + 2) % 3
    return d(b2, b1) - d(b1, b2)   # (curl A)^a = d_{a+1} A^{a+2} - d_{a+2} A^{a+1}


def face_field(p: Problem, device=None, direction=None):
    """UCT runs (divb = 2): sqrt(gamma) B^a at the centres of the faces i_a + 1/2,
    [3][n3][n2][n1], the ANALYTIC field of the config's initial condition sampled at the
    faces (turbulence: B0 x-hat + the exact curl of the same seeded vector potential,
    whose cell-centred counterpart ic_turbulence takes as a D2 curl; CP Alfven: the
    exact wave, along `direction` = integer (k1, k2, k3) if given, else (1, 1, 1); blast: the
    uniform B = Bx x-hat; torus: the staggered curl of A_phi at the cell corners)."""
    torch = _backend(device)
    cfg = p.params["cfg"]
    out = []
    if cfg in (0, 3):
        prm = p.params
        rng = SplitMix64(p.seed)
        modes = [draw_modes(rng, prm["modes"], prm["kmax"]) for _ in range(8)]
        for a in range(3):
            X, Y, Z = _coords_face(p, a, torch, device)
            b = _curl_modes(modes[5:8], a, X, Y, Z, prm["amp"], torch)
            out.append(b + (prm["B0"] if a == 0 else 0.0))
    elif cfg == 1:
        for a in range(3):
            X, Y, Z = _coords_face(p, a, None, None)
            out.append(cp_alfven_fields(p, X, Y, Z, 0.0, direction)[1][a])
    elif cfg == 2:
        for a in range(3):
            out.append(np.full((1, 1, 1), p.params["Bx"] if a == 0 else 0.0))
    elif cfg == 4:
        out = _torus_face_field(p)
    else:
        raise ValueError(f"face_field: no staggered-field recipe for config {cfg}")
    shape = (p.n[2], p.n[1], p.n[0])
    if torch is None:
        return np.ascontiguousarray(np.stack([np.broadcast_to(f, shape) for f in out]).astype(np.float64))
    return torch.stack([torch.as_tensor(np.ascontiguousarray(f) if isinstance(f, np.ndarray) else f,
                                        dtype=torch.float64, device=device).expand(shape) for f in out]).contiguous()


def cp_alfven_fields(p: Problem, X, Y, Z, t, direction=None):
    """(v, B) of the exact CP Alfven wave of config 1 along the integer wave vector
    `direction` (default (1,1,1)) at time t: phase 2 pi (k.x) - 2 pi |k| v_A t."""
    prm = p.params
    eta, B0 = prm["eta"], prm["B0"]
    va = cp_alfven_speed(eta, B0)
    kv = np.array(direction if direction is not None else (1, 1, 1), dtype=np.float64)
    kn = float(np.linalg.norm(kv))
    k = kv / kn
    # an orthonormal pair perpendicular to k
    t0 = np.array([0.0, 0.0, 1.0]) if abs(k[2]) < 0.9 else np.array([1.0, 0.0, 0.0])
    e1 = np.cross(k, t0)
    e1 /= np.linalg.norm(e1)
    e2 = np.cross(k, e1)
    phi = 2.0 * math.pi * (kv[0] * X + kv[1] * Y + kv[2] * Z) - 2.0 * math.pi * kn * va * t
    c, s = np.cos(phi), np.sin(phi)
    B = [B0 * k[i] + eta * B0 * (c * e1[i] + s * e2[i]) for i in range(3)]
    v = [-va * eta * (c * e1[i] + s * e2[i]) for i in range(3)]
    return v, B


def uniform_prims(n, rho=1.0, v=(0.0, 0.0, 0.0), prs=1.0, B=(0.0, 0.0, 0.0)) -> np.ndarray:
    shape = (n[2], n[1], n[0])
    vals = [rho, v[0], v[1], v[2], prs, B[0], B[1], B[2]]
    return np.ascontiguousarray(np.stack([np.full(shape, float(x)) for x in vals]))


def sample_cells(n, count: int, seed: int = 12345, include_corners: bool = True) -> np.ndarray:
    """seeded sample of cell indices (i,j,k), with the 8 domain corners and edge cells first."""
    rng = SplitMix64(seed)
    cells = []
    if include_corners:
        for k in (0, n[2] - 1):
            for j in (0, n[1] - 1):
                for i in (0, n[0] - 1):
                    cells.append((i, j, k))
    while len(cells) < count:
        cells.append(tuple(int(rng.next() % n[a]) for a in range(3)))
    return np.array(cells[:count], dtype=np.int64)
