"""Brute-force per-cell L(U) in mpmath (50 digits) — pin P6 for the oracle.

An independent transcription of DESIGN.md §3 (readings A1-A6, A12, A13, A25)
for tiny grids (4^3), written without looking at oracle/*.c structure:
every face flux is evaluated from the definition at 50 digits, metric
derivatives come from mpmath numerical differentiation (not from the oracle's
hand-derived formulas), and the 3x3 inverse / determinant from mpmath
matrices.  Used only by tests/test_oracle_bruteforce.py.
"""
from __future__ import annotations

import mpmath as mp

mp.mp.dps = 50


class Grid:
    def __init__(self, n, lo, hi, bc, metric=0, M=1, a=0, gamma=mp.mpf(4) / 3, rec=0, der=6, divb=0, der_jump=0.5):
        self.der_jump = der_jump
        self.n = list(n)
        self.lo = [mp.mpf(v) for v in lo]
        self.hi = [mp.mpf(v) for v in hi]
        self.bc = bc
        self.metric = metric
        self.M = mp.mpf(M)
        self.a = mp.mpf(a)
        self.gamma = mp.mpf(gamma)
        self.rec = rec
        self.der = der
        self.divb = divb

    def d(self, a):
        return (self.hi[a] - self.lo[a]) / self.n[a]

    def centre(self, a, i):
        return self.lo[a] + (i + mp.mpf(1) / 2) * self.d(a)

    def face(self, a, i):  # face i+1/2
        return self.lo[a] + (i + 1) * self.d(a)

    def wrap(self, a, i):
        n = self.n[a]
        if i < 0:
            return i % n if self.bc[a][0] == 0 else 0
        if i >= n:
            return i % n if self.bc[a][1] == 0 else n - 1
        return i


# ------------------------------------------------------------- metric
def _gamma_ij(G: Grid, x):
    if G.metric == 0:
        return mp.eye(3)
    r = mp.e ** x[0]
    th = x[1]
    s, c = mp.sin(th), mp.cos(th)
    rho2 = r ** 2 + G.a ** 2 * c ** 2
    z = 2 * G.M * r / rho2
    g = mp.matrix(3, 3)
    g[0, 0] = r ** 2 * (1 + z)
    g[0, 2] = g[2, 0] = r * (-G.a * (1 + z) * s ** 2)
    g[1, 1] = rho2
    g[2, 2] = s ** 2 * (rho2 + G.a ** 2 * (1 + z) * s ** 2)
    return g


def _alpha(G: Grid, x):
    if G.metric == 0:
        return mp.mpf(1)
    r = mp.e ** x[0]
    z = 2 * G.M * r / (r ** 2 + G.a ** 2 * mp.cos(x[1]) ** 2)
    return 1 / mp.sqrt(1 + z)


def _beta(G: Grid, x):
    if G.metric == 0:
        return [mp.mpf(0)] * 3
    r = mp.e ** x[0]
    z = 2 * G.M * r / (r ** 2 + G.a ** 2 * mp.cos(x[1]) ** 2)
    return [z / (1 + z) / r, mp.mpf(0), mp.mpf(0)]


class Met:
    def __init__(self, G: Grid, x, derivs=False):
        self.alpha = _alpha(G, x)
        self.beta = _beta(G, x)
        self.g = _gamma_ij(G, x)
        self.gi = self.g ** -1
        self.sqrtg = mp.sqrt(mp.det(self.g))
        if derivs:
            self.dalpha, self.dbeta, self.dg = [], [], []
            for k in range(3):
                def along(f, k=k):
                    return mp.diff(lambda t: f([x[m] if m != k else t for m in range(3)]), x[k])
                if G.metric == 0 or k == 2:
                    self.dalpha.append(mp.mpf(0))
                    self.dbeta.append([mp.mpf(0)] * 3)
                    self.dg.append(mp.zeros(3, 3))
                    continue
                self.dalpha.append(along(lambda y: _alpha(G, y)))
                self.dbeta.append([along(lambda y, i=i: _beta(G, y)[i]) for i in range(3)])
                dg = mp.zeros(3, 3)
                for i in range(3):
                    for j in range(3):
                        dg[i, j] = along(lambda y, i=i, j=j: _gamma_ij(G, y)[i, j])
                self.dg.append(dg)


# ------------------------------------------------------------- physics
def aux(m: Met, gam, pr):
    rho, ut, p, B = pr[0], pr[1:4], pr[4], pr[5:8]
    W = mp.sqrt(1 + sum(m.g[i, j] * ut[i] * ut[j] for i in range(3) for j in range(3)))
    v = [ut[i] / W for i in range(3)]
    vl = [sum(m.g[i, j] * v[j] for j in range(3)) for i in range(3)]
    Bl = [sum(m.g[i, j] * B[j] for j in range(3)) for i in range(3)]
    v2 = sum(vl[i] * v[i] for i in range(3))
    B2 = sum(Bl[i] * B[i] for i in range(3))
    vB = sum(vl[i] * B[i] for i in range(3))
    h = 1 + gam / (gam - 1) * p / rho
    Z = rho * h * W ** 2
    D = rho * W
    S = [(Z + B2) * vl[i] - vB * Bl[i] for i in range(3)]
    Su = [sum(m.gi[i, j] * S[j] for j in range(3)) for i in range(3)]
    E2 = B2 * v2 - vB ** 2
    U = Z - p + (E2 + B2) / 2
    # E^i = -eps^{ijk} v_j B_k with eps^{ijk} = [ijk]/sqrt(gamma)
    E = [-(vl[(i + 1) % 3] * Bl[(i + 2) % 3] - vl[(i + 2) % 3] * Bl[(i + 1) % 3]) / m.sqrtg for i in range(3)]
    Wst = [[Z * v[i] * v[j] - E[i] * E[j] - B[i] * B[j] + (p + (E2 + B2) / 2) * m.gi[i, j] for j in range(3)]
           for i in range(3)]
    return dict(W=W, v=v, vl=vl, v2=v2, B2=B2, vB=vB, h=h, Z=Z, D=D, S=S, Su=Su, U=U, tau=U - D, Wst=Wst)


def cons(m, gam, pr):
    q = aux(m, gam, pr)
    return [q["D"], *q["S"], q["tau"], *pr[5:8]]


def flux(m, gam, pr, j):
    q = aux(m, gam, pr)
    B = pr[5:8]
    a = m.alpha
    f = [(a * q["v"][j] - m.beta[j]) * q["D"]]
    for i in range(3):
        f.append(a * sum(q["Wst"][j][k] * m.g[k, i] for k in range(3)) - m.beta[j] * q["S"][i])
    f.append(a * (q["Su"][j] - q["D"] * q["v"][j]) - m.beta[j] * q["tau"])
    for i in range(3):
        f.append((a * q["v"][j] - m.beta[j]) * B[i] - (a * q["v"][i] - m.beta[i]) * B[j])
    return f


def speeds(m, gam, pr, j):
    q = aux(m, gam, pr)
    rho, p = pr[0], pr[4]
    cs2 = gam * p / (rho * q["h"])
    b2 = q["B2"] / q["W"] ** 2 + q["vB"] ** 2
    ca2 = b2 / (rho * q["h"] + b2)
    a2 = cs2 + ca2 - cs2 * ca2
    disc = a2 * (1 - q["v2"]) * (m.gi[j, j] * (1 - q["v2"] * a2) - q["v"][j] ** 2 * (1 - a2))
    sq = mp.sqrt(max(disc, 0))
    den = 1 - q["v2"] * a2
    return (m.alpha * (q["v"][j] * (1 - a2) - sq) / den - m.beta[j],
            m.alpha * (q["v"][j] * (1 - a2) + sq) / den - m.beta[j])


def hll(m, gam, pl, pr, j):
    uL, uR = cons(m, gam, pl), cons(m, gam, pr)
    fL, fR = flux(m, gam, pl, j), flux(m, gam, pr, j)
    lmL, lpL = speeds(m, gam, pl, j)
    lmR, lpR = speeds(m, gam, pr, j)
    sl = min(0, lmL, lmR)
    sr = max(0, lpL, lpR)
    if sr - sl > 0:
        F = [(sr * fL[q] - sl * fR[q] + sl * sr * (uR[q] - uL[q])) / (sr - sl) for q in range(8)]
    else:
        F = [(fL[q] + fR[q]) / 2 for q in range(8)]
    return [m.sqrtg * v for v in F]


def sources(m: Met, gam, pr):
    q = aux(m, gam, pr)
    s = [mp.mpf(0)] * 8
    for i in range(3):
        t1 = sum(q["Wst"][j][k] * m.dg[i][j, k] for j in range(3) for k in range(3))
        t2 = sum(q["S"][j] * m.dbeta[i][j] for j in range(3))
        s[1 + i] = m.alpha * t1 / 2 + t2 - q["U"] * m.dalpha[i]
    e1 = sum(q["Wst"][i][k] * sum(m.beta[j] * m.dg[j][i, k] for j in range(3)) / 2
             for i in range(3) for k in range(3))
    e2 = sum(sum(m.g[i, k] * q["Wst"][k][j] for k in range(3)) * m.dbeta[j][i] for i in range(3) for j in range(3))
    e3 = sum(q["Su"][j] * m.dalpha[j] for j in range(3))
    s[4] = e1 + e2 - e3
    return s


def weno(u, rec):
    eps = mp.mpf("1e-6")
    b0 = mp.mpf(13) / 12 * (u[0] - 2 * u[1] + u[2]) ** 2 + (u[0] - 4 * u[1] + 3 * u[2]) ** 2 / 4
    b1 = mp.mpf(13) / 12 * (u[1] - 2 * u[2] + u[3]) ** 2 + (u[1] - u[3]) ** 2 / 4
    b2 = mp.mpf(13) / 12 * (u[2] - 2 * u[3] + u[4]) ** 2 + (3 * u[2] - 4 * u[3] + u[4]) ** 2 / 4
    if rec == 0:
        q = [(3 * u[0] - 10 * u[1] + 15 * u[2]) / 8, (-u[1] + 6 * u[2] + 3 * u[3]) / 8, (3 * u[2] + 6 * u[3] - u[4]) / 8]
        d = [mp.mpf(1) / 16, mp.mpf(10) / 16, mp.mpf(5) / 16]
    else:
        q = [(2 * u[0] - 7 * u[1] + 11 * u[2]) / 6, (-u[1] + 5 * u[2] + 2 * u[3]) / 6, (2 * u[2] + 5 * u[3] - u[4]) / 6]
        d = [mp.mpf(1) / 10, mp.mpf(6) / 10, mp.mpf(3) / 10]
    al = [d[k] / (eps + b) ** 2 for k, b in enumerate((b0, b1, b2))]
    return sum(al[k] * q[k] for k in range(3)) / sum(al)


def mp5(u):
    """MP5 (Suresh & Huynh 1997) on point values, A33: always the median of the unlimited
    5-point interpolant and the MP interval (equivalent to the paper's early exit, which the
    oracle takes, because u_i and u_MP both lie in that interval)."""
    def minmod(*a):
        if all(x > 0 for x in a):
            return min(a)
        if all(x < 0 for x in a):
            return max(a)
        return mp.mpf(0)

    u_or = (3 * u[0] - 20 * u[1] + 90 * u[2] + 60 * u[3] - 5 * u[4]) / 128
    dm, d0, dp = u[0] - 2 * u[1] + u[2], u[1] - 2 * u[2] + u[3], u[2] - 2 * u[3] + u[4]
    m4p = minmod(4 * d0 - dp, 4 * dp - d0, d0, dp)
    m4m = minmod(4 * d0 - dm, 4 * dm - d0, d0, dm)
    ul = u[2] + 4 * (u[2] - u[1])
    md = (u[2] + u[3]) / 2 - m4p / 2
    lc = u[2] + (u[2] - u[1]) / 2 + mp.mpf(4) / 3 * m4m
    lo = max(min(u[2], u[3], md), min(u[2], ul, lc))
    hi = min(max(u[2], u[3], md), max(u[2], ul, lc))
    return sorted([u_or, lo, hi])[1] if lo <= hi else u_or + minmod(lo - u_or, hi - u_or)


def wenoz(u):
    """WENO-Z (Borges et al. 2008) on the point form, eps = 1e-40 (A34)."""
    eps = mp.mpf("1e-40")
    b = [mp.mpf(13) / 12 * (u[0] - 2 * u[1] + u[2]) ** 2 + (u[0] - 4 * u[1] + 3 * u[2]) ** 2 / 4,
         mp.mpf(13) / 12 * (u[1] - 2 * u[2] + u[3]) ** 2 + (u[1] - u[3]) ** 2 / 4,
         mp.mpf(13) / 12 * (u[2] - 2 * u[3] + u[4]) ** 2 + (3 * u[2] - 4 * u[3] + u[4]) ** 2 / 4]
    q = [(3 * u[0] - 10 * u[1] + 15 * u[2]) / 8, (-u[1] + 6 * u[2] + 3 * u[3]) / 8, (3 * u[2] + 6 * u[3] - u[4]) / 8]
    d = [mp.mpf(1) / 16, mp.mpf(10) / 16, mp.mpf(5) / 16]
    tau = abs(b[0] - b[2])
    al = [d[k] * (1 + tau / (b[k] + eps)) for k in range(3)]
    return sum(al[k] * q[k] for k in range(3)) / sum(al)


def mc2(u):
    """MC2 limited linear reconstruction (A35)."""
    dl, dr, dc = u[2] - u[1], u[3] - u[2], (u[3] - u[1]) / 2
    if dl > 0 and dr > 0:
        return u[2] + min(2 * dl, dc, 2 * dr) / 2
    if dl < 0 and dr < 0:
        return u[2] + max(2 * dl, dc, 2 * dr) / 2
    return u[2]


def ppm(u):
    """PPM on point values (A36): 4th-order interface interpolants kept between the
    neighbours, then the Colella-Woodward monotonicity constraints; u_R of cell i."""
    def face(a, b, c, d):
        v = (-a + 9 * b + 9 * c - d) / 16
        return min(max(v, min(b, c)), max(b, c))
    uR, uL, ui = face(u[1], u[2], u[3], u[4]), face(u[0], u[1], u[2], u[3]), u[2]
    if (uR - ui) * (ui - uL) <= 0:
        return ui
    du, m6 = uR - uL, 6 * (ui - (uL + uR) / 2)
    if -du * du > du * m6:
        uR = 3 * ui - 2 * uL
    return uR


def rec_left(u, rec):
    if rec == 5:
        return ppm(u)
    if rec == 4:
        return mc2(u)
    if rec == 3:
        return wenoz(u)
    return mp5(u) if rec == 2 else weno(u, rec)


def derf(F, order):
    if order == 6:
        return F[2] - (F[1] - 2 * F[2] + F[3]) / 24 + 3 * (F[0] - 4 * F[1] + 6 * F[2] - 4 * F[3] + F[4]) / 640
    if order == 4:
        return F[2] - (F[1] - 2 * F[2] + F[3]) / 24
    return F[2]


# --------------------------------------------- characteristic-wise WENO5 (A44)
def char_rec(G: Grid, st, ax):
    """Hydro face states (rho, u~^1..3, p) at face i+1/2 from prims st[0..5] of cells i-2..i+3:
    the right eigenvectors of the flat relativistic-Euler Jacobian at the mean of cells i, i+1,
    written in w = (rho, v^n, v^t1, v^t2, p) and pushed to q = (rho, u~^n, u~^t1, u~^t2, p) by
    du~ = W (I + W^2 v v^T) dv; L from mpmath's matrix inverse; WENO5 point form per field."""
    n, t1, t2 = ax, (ax + 1) % 3, (ax + 2) % 3
    order = [0, 1 + n, 1 + t1, 1 + t2, 4]            # frame slot -> state slot
    qs = [[cell[k] for k in order] for cell in st]
    qb = [(qs[2][k] + qs[3][k]) / 2 for k in range(5)]
    ut = qb[1:4]
    W = mp.sqrt(1 + sum(x * x for x in ut))
    v = [x / W for x in ut]
    vv = sum(x * x for x in v)
    rho, p, gam = qb[0], qb[4], G.gamma
    h = 1 + gam * p / ((gam - 1) * rho)
    c2 = gam * p / (rho * h)
    root = mp.sqrt(c2 * (1 - vv) * (1 - vv * c2 - v[0] ** 2 * (1 - c2)))
    Rw = mp.matrix(5, 5)
    for col, sgn in ((0, -1), (4, 1)):
        lam = (v[0] * (1 - c2) + sgn * root) / (1 - vv * c2)
        kap = (gam * p / rho) / (rho * h * W ** 2 * (lam - v[0]))
        Rw[0, col], Rw[1, col] = 1, kap * (1 - v[0] * lam)
        Rw[2, col], Rw[3, col], Rw[4, col] = -kap * lam * v[1], -kap * lam * v[2], gam * p / rho
    Rw[0, 1] = Rw[2, 2] = Rw[3, 3] = 1
    T = mp.eye(5)
    for i in range(3):
        for j in range(3):
            T[1 + i, 1 + j] = W * ((1 if i == j else 0) + W ** 2 * v[i] * v[j])
    R = T * Rw
    L = mp.inverse(R)
    cL, cR = [], []
    for k in range(5):
        ch = [sum(L[k, j] * qs[m][j] for j in range(5)) for m in range(6)]
        cL.append(weno(ch[0:5], 0))
        cR.append(weno(ch[5:0:-1], 0))
    fl = [sum(R[j, k] * cL[k] for k in range(5)) for j in range(5)]
    fr = [sum(R[j, k] * cR[k] for k in range(5)) for j in range(5)]
    outL, outR = [mp.mpf(0)] * 5, [mp.mpf(0)] * 5
    for f, slot in enumerate(order):
        outL[slot], outR[slot] = fl[f], fr[f]
    return outL, outR


# ------------------------------------------------------------- scheme
class Scheme:
    """L(U) on every owned cell of a tiny grid, from fp64 state arrays (converted exactly to mp)."""

    def __init__(self, G: Grid, U8, P5):
        self.G = G
        self.U8 = U8
        self.P5 = P5
        self._prim = {}
        self._face = {}
        self._H = {}

    def prim(self, i, j, k):
        G = self.G
        key = (G.wrap(0, i), G.wrap(1, j), G.wrap(2, k))
        if key not in self._prim:
            a, b, c = key
            m = Met(G, [G.centre(0, a), G.centre(1, b), G.centre(2, c)])
            pr = [mp.mpf(float(self.P5[q, c, b, a])) for q in range(5)]
            pr += [mp.mpf(float(self.U8[5 + q, c, b, a])) / m.sqrtg for q in range(3)]
            self._prim[key] = pr
        return self._prim[key]

    def face_flux(self, ax, cell):  # face cell[ax]+1/2, cell transverse owned
        key = (ax, tuple(cell))
        if key in self._face:
            return self._face[key]
        G = self.G
        st = []
        for mm in range(6):
            cc = list(cell)
            cc[ax] = cell[ax] - 2 + mm
            st.append(self.prim(*cc))
        rec = 0 if G.rec == 6 else G.rec
        qL = [rec_left([st[mm][v] for mm in range(5)], rec) for v in range(8)]
        qR = [rec_left([st[5 - mm][v] for mm in range(5)], rec) for v in range(8)]
        if G.rec == 6:  # A44: the hydro states from the characteristic fields
            hL, hR = char_rec(G, st, ax)
            qL[:5], qR[:5] = hL, hR
        if not qL[0] > 0:
            qL[0] = st[2][0]
        if not qL[4] > 0:
            qL[4] = st[2][4]
        if not qR[0] > 0:
            qR[0] = st[3][0]
        if not qR[4] > 0:
            qR[4] = st[3][4]
        x = [G.centre(b, cell[b]) for b in range(3)]
        x[ax] = G.face(ax, cell[ax])
        F = hll(Met(G, x), G.gamma, qL, qR, ax)
        # A31 jump flag of this face from the two cell-centre states it joins (fp64 inputs)
        a, b = st[2], st[3]
        dj = G.der_jump
        rough = dj > 0 and (abs(b[0] - a[0]) > dj * min(a[0], b[0]) or abs(b[4] - a[4]) > dj * min(a[4], b[4]))
        self._face[key] = (F, rough)
        return self._face[key]

    def H(self, ax, cell):
        key = (ax, tuple(cell))
        if key not in self._H:
            Fs = []
            for mm in range(5):
                cc = list(cell)
                cc[ax] = cell[ax] - 2 + mm
                Fs.append(self.face_flux(ax, cc))
            if any(r for _, r in Fs):
                self._H[key] = list(Fs[2][0])
            else:
                self._H[key] = [derf([Fs[mm][0][q] for mm in range(5)], self.G.der) for q in range(8)]
        return self._H[key]

    def axes(self, cell):
        G = self.G
        L = [mp.mpf(0)] * 8
        Om = [mp.mpf(0)] * 3
        for ax in range(3):
            cm = list(cell)
            cm[ax] -= 1
            Hp, Hm = self.H(ax, cell), self.H(ax, cm)
            d = G.d(ax)
            for q in range(5):
                L[q] -= (Hp[q] - Hm[q]) / d
            b1, b2 = (ax + 1) % 3, (ax + 2) % 3
            if G.divb == 1:
                L[5 + b1] -= (Hp[5 + b1] - Hm[5 + b1]) / d
                L[5 + b2] -= (Hp[5 + b2] - Hm[5 + b2]) / d
            else:
                Om[b2] -= (Hp[5 + b1] + Hm[5 + b1]) / 4
                Om[b1] += (Hp[5 + b2] + Hm[5 + b2]) / 4
        return L, Om

    def rhs_cell(self, cell):
        G = self.G
        L, _ = self.axes(cell)
        x = [G.centre(b, cell[b]) for b in range(3)]
        if G.metric != 0:
            m = Met(G, x, derivs=True)
            s = sources(m, G.gamma, self.prim(*cell))
            for q in range(1, 5):
                L[q] += m.sqrtg * s[q]
        if G.divb == 0:
            def om(ax, sgn, v):
                nb = list(cell)
                nb[ax] += sgn
                nb = [G.wrap(b, nb[b]) for b in range(3)]
                return self.axes(nb)[1][v]
            for i in range(3):
                j, k = (i + 1) % 3, (i + 2) % 3
                L[5 + i] = -(om(j, 1, k) - om(j, -1, k)) / (2 * G.d(j)) + (om(k, 1, j) - om(k, -1, j)) / (2 * G.d(k))
        return L


# ------------------------------------------------------------- UCT (divb = 2)
class SchemeUCT(Scheme):
    """UCT (readings A37-A43) written out from the readings: the staggered field
    b^a = sqrt(gamma) B^a at the face cell[a]+1/2, face data (V = alpha v - beta of both HLL
    states, a+ = max(0, lam+_L, lam+_R), a- = max(0, -lam-_L, -lam-_R)), the four-state
    UCT-HLL edge EMF with quadrant velocities averaged over the two double reconstructions,
    and L(b^p) = -d_q Dh E^c + d_c Dh E^q with (c, p, q) cyclic.  The hydro rhs is the
    base scheme's with the normal field of every face taken from b."""

    def __init__(self, G: Grid, U8, P5, b3):
        super().__init__(G, U8, P5)
        self.b3 = b3
        self._fd = {}
        self._E = {}

    def wrapc(self, cell):
        return [self.G.wrap(a, cell[a]) for a in range(3)]

    def b(self, a, cell):  # b^a at the face cell[a]+1/2
        i, j, k = self.wrapc(cell)
        return mp.mpf(float(self.b3[a, k, j, i]))

    def face_flux(self, ax, cell):
        key = (ax, tuple(cell))
        if key in self._face:
            return self._face[key]
        G = self.G
        st = []
        for mm in range(6):
            cc = list(cell)
            cc[ax] = cell[ax] - 2 + mm
            st.append(self.prim(*cc))
        qL = [rec_left([st[mm][v] for mm in range(5)], G.rec) for v in range(8)]
        qR = [rec_left([st[5 - mm][v] for mm in range(5)], G.rec) for v in range(8)]
        if not qL[0] > 0:
            qL[0] = st[2][0]
        if not qL[4] > 0:
            qL[4] = st[2][4]
        if not qR[0] > 0:
            qR[0] = st[3][0]
        if not qR[4] > 0:
            qR[4] = st[3][4]
        x = [G.centre(b, cell[b]) for b in range(3)]
        x[ax] = G.face(ax, cell[ax])
        m = Met(G, x)
        qL[5 + ax] = qR[5 + ax] = self.b(ax, cell) / m.sqrtg
        F = hll(m, G.gamma, qL, qR, ax)
        aL, aR = aux(m, G.gamma, qL), aux(m, G.gamma, qR)
        lmL, lpL = speeds(m, G.gamma, qL, ax)
        lmR, lpR = speeds(m, G.gamma, qR, ax)
        VL = [m.alpha * aL["v"][i] - m.beta[i] for i in range(3)]
        VR = [m.alpha * aR["v"][i] - m.beta[i] for i in range(3)]
        if list(cell) == self.wrapc(cell):  # face data of owned faces only (A42: ghosts = nearest owned)
            self._fd[(ax, tuple(cell))] = (VL, VR, max(0, lpL, lpR), max(0, -lmL, -lmR))
        a, bb = st[2], st[3]
        dj = G.der_jump
        rough = dj > 0 and (abs(bb[0] - a[0]) > dj * min(a[0], bb[0]) or abs(bb[4] - a[4]) > dj * min(a[4], bb[4]))
        self._face[key] = (F, rough)
        return self._face[key]

    def fd(self, ax, cell):
        key = (ax, tuple(self.wrapc(cell)))
        if key not in self._fd:
            w = self.wrapc(cell)
            self._face.pop((ax, tuple(w)), None)
            self.face_flux(ax, w)
        return self._fd[key]

    def emf(self, c, cell):
        """E^c at the edge (cell[p]+1/2, cell[q]+1/2, cell[c]), p = c+1, q = c+2; a ghost edge
        is the nearest owned one (A42: the cell ghost rule applied to the edge's cell)"""
        cell = self.wrapc(cell)
        key = (c, tuple(cell))
        if key in self._E:
            return self._E[key]
        G = self.G
        p, q = (c + 1) % 3, (c + 2) % 3

        def at(ax, d):
            cc = list(cell)
            cc[ax] += d
            return cc

        def pair(samples):  # one-sided values at +1/2 from samples at -2..3
            return rec_left(samples[0:5], G.rec), rec_left(samples[5:0:-1], G.rec)

        # p-faces: W = left state, E = right state, reconstructed along q -> (S, N)
        Wst = {}
        for side in (0, 1):
            for comp in (p, q):
                s = [self.fd(p, at(q, mm - 2))[side][comp] for mm in range(6)]
                Wst[(side, comp)] = pair(s)
        # q-faces: S = left state, N = right state, reconstructed along p -> (W, E)
        Sst = {}
        for side in (0, 1):
            for comp in (p, q):
                s = [self.fd(q, at(p, mm - 2))[side][comp] for mm in range(6)]
                Sst[(side, comp)] = pair(s)
        bpS, bpN = pair([self.b(p, at(q, mm - 2)) for mm in range(6)])
        bqW, bqE = pair([self.b(q, at(p, mm - 2)) for mm in range(6)])
        app = max(self.fd(p, cell)[2], self.fd(p, at(q, 1))[2])
        apm = max(self.fd(p, cell)[3], self.fd(p, at(q, 1))[3])
        aqp = max(self.fd(q, cell)[2], self.fd(q, at(p, 1))[2])
        aqm = max(self.fd(q, cell)[3], self.fd(q, at(p, 1))[3])

        def vel(we, sn, comp):  # quadrant (we: 0 W / 1 E, sn: 0 S / 1 N)
            return (Wst[(we, comp)][sn] + Sst[(sn, comp)][we]) / 2

        def equad(we, sn):
            bp = bpN if sn else bpS
            bq = bqE if we else bqW
            return vel(we, sn, q) * bp - vel(we, sn, p) * bq

        sp, sq = app + apm, aqp + aqm
        if sp > 0 and sq > 0:
            E = ((app * aqp * equad(0, 0) + app * aqm * equad(0, 1) + apm * aqp * equad(1, 0) + apm * aqm * equad(1, 1))
                 / (sp * sq) + app * apm * (bqE - bqW) / sp - aqp * aqm * (bpN - bpS) / sq)
        else:
            E = (equad(0, 0) + equad(0, 1) + equad(1, 0) + equad(1, 1)) / 4
        self._E[key] = E
        return E

    def rhs_cell(self, cell):
        G = self.G
        L, _ = self.axes(cell)
        x = [G.centre(b, cell[b]) for b in range(3)]
        if G.metric != 0:
            m = Met(G, x, derivs=True)
            s = sources(m, G.gamma, self.prim(*cell))
            for q in range(1, 5):
                L[q] += m.sqrtg * s[q]

        def Dh(c, ax, base, shift):
            vals = []
            for mm in range(5):
                cc = list(base)
                cc[ax] += mm - 2 + shift
                vals.append(self.emf(c, cc))
            return derf(vals, G.der)

        for p in range(3):
            c, q = (p + 2) % 3, (p + 1) % 3
            L[5 + p] = (-(Dh(c, q, cell, 0) - Dh(c, q, cell, -1)) / G.d(q)
                        + (Dh(q, c, cell, 0) - Dh(q, c, cell, -1)) / G.d(c))
        return L
