// cell_physics.cuh — per-cell device physics shared by the K3 kernels:
// con2prim Newton (A8, A27, A28), floors (A9) and the metric sources (a6).
#pragma once
#include "echo_dev.cuh"
#include "echo_kernels.h"

namespace echo {
constexpr int kCellThreads = 256;

ECHO_D void cell_ijk(const GridP& g, long long id, int& i, int& j, int& k) {
  long long r = id / g.n[0];
  i = (int)(id - r * g.n[0]);
  k = (int)(r / g.n[1]);
  j = (int)(r - (long long)k * g.n[1]);
}

template <bool KS>
struct MetAt;
template <>
struct MetAt<false> {
  using T = FlatMet;
  static ECHO_D T get(const MetTables&, int, int) { return FlatMet(); }
};
template <>
struct MetAt<true> {
  using T = GenMet;
  static ECHO_D T get(const MetTables& mt, int i, int j) { return load_met(cen_rec(mt, i, j)); }
};

// ----------------------------------------------------------- con2prim (A8)
// The Newton guess of A8: Z0 = rho h W^2 = (rho + Gamma/(Gamma-1) p)(1 + u~.u~) of the previous
// stage's primitives pr = (rho, u~^i, p).  In Minkowski K3 stores it in the otherwise unused P
// slot 5 when it writes the new primitives, so the next stage reads 8 bytes instead of 40.
template <class M>
ECHO_D double guess_Z(const M& m, const EosP& e, const double* pr) {
  double gu[3] = {pr[1], pr[2], pr[3]}, gl[3];
  m.lower(gu, gl);
  return (pr[0] + e.gfac * pr[4]) * (1.0 + gu[0] * gl[0] + gu[1] * gl[1] + gu[2] * gl[2]);
}
constexpr int kSlotZ = 5;  // P slot of the stored guess (Minkowski only: KS keeps B^i in slots 5..7)

// 1-D Newton in Z = rho h W^2 with the oracle's iteration rules (A8, A27, A28).
// u: non-densitised (D, S_i, tau, B^i); Z0: guess_Z of the previous primitives; out: (rho, u~^i, p).
template <class M>
ECHO_D int c2p_newton(const M& m, const EosP& e, const double* u, double Z0, double* out) {
  const double D = u[0], tau = u[4];
  const double S[3] = {u[1], u[2], u[3]};
  const double B[3] = {u[5], u[6], u[7]};
  const double Ut = tau + D;
  double Su[3], Bl[3];
  m.raise(S, Su);
  m.lower(B, Bl);
  const double S2 = S[0] * Su[0] + S[1] * Su[1] + S[2] * Su[2];
  const double B2 = B[0] * Bl[0] + B[1] * Bl[1] + B[2] * Bl[2];
  const double SB = S[0] * B[0] + S[1] * B[1] + S[2] * B[2];
  const double SB2 = SB * SB;
  double Z = Z0;
  bool polish = false, ok = false;
  for (int it = 1; it <= e.maxit; it++) {
    // 1/Z and 1/(Z + B^2) through one reciprocal; 1/sqrt(1 - v^2) from the rsqrt that gives sqrt(1 - v^2)
    const double ZB = Z + B2;
    const double r = frcp(Z * ZB);
    const double iZ = ZB * r, iZB = Z * r;
    const double iZ2 = iZ * iZ, iZB2 = iZB * iZB;
    double v2 = (Z * Z * S2 + SB2 * (2.0 * Z + B2)) * iZ2 * iZB2;
    bool clamped = false;
    if (v2 > e.v2max) { v2 = e.v2max; clamped = true; }
    const double omv2 = 1.0 - v2;
    const double rs = frsqrt(omv2);  // 1 - v^2 >= 1/W_max^2 > 0
    const double sq = omv2 * rs;
    const double p = e.gm * (Z * omv2 - D * sq);
    const double f = Z - p + 0.5 * B2 * (1.0 + v2) - 0.5 * SB2 * iZ2 - Ut;
    const double dv2 = clamped ? 0.0 : -2.0 * iZB2 * iZB * (S2 + SB2 * (3.0 * Z * Z + 3.0 * Z * B2 + B2 * B2) * iZ2 * iZ);
    const double dp = e.gm * (omv2 - Z * dv2 + D * dv2 * (0.5 * rs));
    const double df = 1.0 - dp + 0.5 * B2 * dv2 + SB2 * iZ2 * iZ;
    double Zn = Z - f * frcp(df);
    if (!(Zn > 0.0)) Zn = 0.5 * Z;
    const double dZ = fabs(Zn - Z);
    Z = Zn;
    if (!isfinite(Z)) return 1;
    if (polish) { ok = true; break; }
    if (dZ <= e.tol * Z) {
      polish = true;
      if (it == e.maxit) ok = true;
    }
  }
  if (!ok) return 1;
  const double ZB = Z + B2;
  const double r = frcp(Z * ZB);
  const double iZ = ZB * r, iZB = Z * r;
  double v2 = (Z * Z * S2 + SB2 * (2.0 * Z + B2)) * (iZ * iZ) * (iZB * iZB);
  if (v2 > e.v2max) v2 = e.v2max;
  const double omv2 = 1.0 - v2;
  const double W = frsqrt(omv2);
  const double sq = omv2 * W;
  out[0] = D * sq;
  out[4] = e.gm * (Z * omv2 - D * sq);
  double vl[3], vu[3];
#pragma unroll
  for (int i = 0; i < 3; i++) vl[i] = (S[i] + SB * Bl[i] * iZ) * iZB;
  m.raise(vl, vu);
#pragma unroll
  for (int i = 0; i < 3; i++) out[1 + i] = W * vu[i];
  if (!isfinite(out[0]) || !isfinite(out[4])) return 1;
  return 0;
}

// A9 floors on the densitised cons Uc (8); Z0 = guess_Z of the previous primitives; prev(P5)
// fills the previous primitives (called only when the Newton fails); Pout (5) out.
// Returns 0 (nothing), 1 (floor event), 2 (failure).
template <class M, class Prev>
ECHO_D int c2p_floors(const M& m, const EosP& e, double* Uc, double Z0, const Prev& prev, double* Pout) {
  const double isg = 1.0 / m.sqrtg();
  double u[8];
#pragma unroll
  for (int q = 0; q < 8; q++) u[q] = M::kFlat ? Uc[q] : Uc[q] * isg;
  double pr[5];
  int status = c2p_newton(m, e, u, Z0, pr);
  int ev = 0;
  if (status != 0) {
    double Pprev[5];
    prev(Pprev);
    double up[3] = {Pprev[1], Pprev[2], Pprev[3]}, ul[3];
    m.lower(up, ul);
    double Wp = sqrt(1.0 + up[0] * ul[0] + up[1] * ul[1] + up[2] * ul[2]);
    pr[1] = up[0]; pr[2] = up[1]; pr[3] = up[2];
    pr[0] = fmax(u[0] / Wp, e.rho_floor);
    pr[4] = fmax(Pprev[4], e.p_floor);
    ev = 2;
  } else {
    bool ch = false;
    if (pr[0] < e.rho_floor) { pr[0] = e.rho_floor; ch = true; }
    if (pr[4] < e.p_floor) { pr[4] = e.p_floor; ch = true; }
    double uu[3] = {pr[1], pr[2], pr[3]}, ul[3];
    m.lower(uu, ul);
    double Wu2 = 1.0 + uu[0] * ul[0] + uu[1] * ul[1] + uu[2] * ul[2];
    double Wu = sqrt(Wu2);
    if (Wu > e.w_max) {
      double sc = sqrt((e.w_max * e.w_max - 1.0) / (Wu * Wu - 1.0));
      pr[1] *= sc; pr[2] *= sc; pr[3] *= sc;
      ch = true;
    }
    ev = ch ? 1 : 0;
  }
  if (ev) {
    double p8[8] = {pr[0], pr[1], pr[2], pr[3], pr[4], u[5], u[6], u[7]};
    State s;
    make_state(m, e, p8, s);
    const double sg = m.sqrtg();
    Uc[0] = sg * s.D;
    Uc[1] = sg * s.S[0];
    Uc[2] = sg * s.S[1];
    Uc[3] = sg * s.S[2];
    Uc[4] = sg * s.tau;
  }
#pragma unroll
  for (int q = 0; q < 5; q++) Pout[q] = pr[q];
  return ev;
}

// ----------------------------------------------------- metric sources (a6)
// s(S_i) = 1/2 alpha W^{jk} d_i gamma_jk + S_j d_i beta^j - U d_i alpha
// s(tau) = 1/2 W^{ik} beta^j d_j gamma_ik + W_i^j d_j beta^i - S^j d_j alpha
// with W^{jk} = (Z+B^2) v^j v^k - (v.B)(B^j v^k + v^j B^k) - B^j B^k / W^2 + p_tot gamma^{jk};
// only d/dx1, d/dx2 are non-zero (stationary, axisymmetric metric).
ECHO_D void add_sources(const GenMet& m, const double* __restrict__ dr, const EosP& e, const double* pr, double* L) {
  State s;
  make_state(m, e, pr, s);
  const double ZB = s.tau + s.D + s.ptot;  // Z + B^2
  const double Ut = s.tau + s.D;
  double Wt[6];
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = a; b < 3; b++)
      Wt[sidx(a, b)] = ZB * s.v[a] * s.v[b] - s.vB * (s.B[a] * s.v[b] + s.v[a] * s.B[b]) - s.B[a] * s.B[b] * s.W2i +
                       s.ptot * m.gi[sidx(a, b)];
  double Su[3];
  m.raise(s.S, Su);
  // derivative records: dalpha[2], dbeta[2][3], dg[2][6]
  double dA[2], dB[2][3], dG[2][6];
#pragma unroll
  for (int k = 0; k < 2; k++) {
    dA[k] = __ldg(dr + k);
#pragma unroll
    for (int i = 0; i < 3; i++) dB[k][i] = __ldg(dr + 2 + 3 * k + i);
#pragma unroll
    for (int i = 0; i < 6; i++) dG[k][i] = __ldg(dr + 8 + 6 * k + i);
  }
  auto contract = [&](const double* dg) {  // W^{jk} dg_jk over the symmetric storage
    return Wt[0] * dg[0] + Wt[3] * dg[3] + Wt[5] * dg[5] + 2.0 * (Wt[1] * dg[1] + Wt[2] * dg[2] + Wt[4] * dg[4]);
  };
  const double sg = m.sqrtg();
  double e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll
  for (int k = 0; k < 2; k++) {
    double wdg = contract(dG[k]);
    double sdb = s.S[0] * dB[k][0] + s.S[1] * dB[k][1] + s.S[2] * dB[k][2];
    L[1 + k] += sg * (0.5 * m.a * wdg + sdb - Ut * dA[k]);
    e1 += 0.5 * m.b[k] * wdg;
    e3 += Su[k] * dA[k];
    // W_i^k d_k beta^i = sum_i gamma_il W^{lk} d_k beta^i
#pragma unroll
    for (int i = 0; i < 3; i++) {
      double Wik = m.g[sidx(i, 0)] * Wt[sidx(0, k)] + m.g[sidx(i, 1)] * Wt[sidx(1, k)] + m.g[sidx(i, 2)] * Wt[sidx(2, k)];
      e2 += Wik * dB[k][i];
    }
  }
  L[4] += sg * (e1 + e2 - e3);
}

// ------------------------------------------------- K3 per-cell pieces
// the 8 variables of one cell record (row-interleaved layout, echo_dev.cuh): stride n1
ECHO_D void ld8(const double* p, long long vs, double* o) {
#pragma unroll
  for (int v = 0; v < 8; v++) o[v] = p[v * vs];
}
ECHO_D void st8(double* p, long long vs, const double* o) {
#pragma unroll
  for (int v = 0; v < 8; v++) p[v * vs] = o[v];
}
// primitives of a cell into P: the 5 hydro ones, plus B^i (= U_B / sqrt(g)) only in a curved
// metric — in Minkowski B^i = U_B and every reader takes it from U
template <bool KS>
ECHO_D void st_prims(double* p, long long vs, const double* o) {
#pragma unroll
  for (int v = 0; v < (KS ? 8 : 5); v++) p[v * vs] = o[v];
}

// L(U) of cell (i, j, k) from the sweep accumulator R (rows a5, a6): hydro rhs
// from R plus the metric sources (KS), and L(sqrt(g) B^c) = -D_{c+1} Omega_{c+2}
// + D_{c+2} Omega_{c+1} (field-CD, A6, A26) or the B rhs from R (divb none).
// Pp: stage-input primitives of the cell (all 8 for KS, 5 otherwise).
template <bool KS, bool DIVB_NONE, class M>
ECHO_D void cell_L(const GridP& g, const EosP& e, const MetTables& mt, const M& m, const double* __restrict__ R,
                   long long rb, int i, int j, int k, const double* Pp, double* L) {
  const long long vs = g.vs;
  double Rv[8];
  ld8(R + rb, vs, Rv);
#pragma unroll
  for (int q = 0; q < 5; q++) L[q] = Rv[q];
  if constexpr (KS) add_sources(m, der_rec(mt, i, j), e, Pp, L);
  if (DIVB_NONE) {
#pragma unroll
    for (int c = 0; c < 3; c++) L[5 + c] = Rv[5 + c];
  } else {
    // Neighbour offsets in the record layout with the ghost rule for a +-1
    // step (periodic: wrap to the other end; outflow: the cell itself), branch free.
    const int ci[3] = {i, j, k};
    const long long stride[3] = {1, g.pitch, (long long)g.n[1] * g.pitch};
    long long om_off[3][2];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const long long wrap = (long long)(g.n[a] - 1) * stride[a];
      // (slab mode, z: an inter-slab side reads the stored ghost plane, whose EMF the sweeps computed)
      om_off[a][0] = (ci[a] > 0) ? -stride[a] : (g.bc[a][0] == 0 ? wrap : (g.bc[a][0] == 2 ? -stride[a] : 0));
      om_off[a][1] = (ci[a] < g.n[a] - 1) ? stride[a] : (g.bc[a][1] == 0 ? -wrap : (g.bc[a][1] == 2 ? stride[a] : 0));
    }
    double onb[3][2][2];  // [axis][-/+][which of the two Omega components used along it]
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int sgn = 0; sgn < 2; sgn++) {
        const double* base = R + rb + om_off[a][sgn];
        onb[a][sgn][0] = base[(5 + (a + 1) % 3) * vs];  // Omega_{a+1}
        onb[a][sgn][1] = base[(5 + (a + 2) % 3) * vs];  // Omega_{a+2}
      }
#pragma unroll
    for (int c = 0; c < 3; c++) {
      const int a1 = (c + 1) % 3, a2 = (c + 2) % 3;
      // Omega_{c+2} along a1 = c+1 is component (a1 + 1) % 3 -> index 0 of onb[a1];
      // Omega_{c+1} along a2 = c+2 is component (a2 + 2) % 3 -> index 1 of onb[a2]
      L[5 + c] = -(onb[a1][1][0] - onb[a1][0][0]) * (0.5 * g.idx[a1]) +
                 (onb[a2][1][1] - onb[a2][0][1]) * (0.5 * g.idx[a2]);
    }
  }
}

// per-cell CFL rate sum_a max(|lambda+_a|, |lambda-_a|)/Delta_a (a9, A11) of prims pr (with B)
template <class M>
ECHO_D double cfl_rate(const M& m, const GridP& g, const EosP& e, const double* pr) {
  State s;
  make_state(m, e, pr, s);
  double val = 0.0;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    double lm, lp;
    speeds(m, e, pr, s, a, lm, lp);
    val += fmax(fabs(lp), fabs(lm)) * g.idx[a];
  }
  if (!(val == val)) val = __longlong_as_double(0x7ff0000000000000LL);  // NaN -> +inf (flagged on host)
  return val;
}

// One RK stage of cell (i, j, k) (rows a5-a8, and a9 when want_rate):
// U^{s+1} = RK_s(U^n, U^s, L) into Uout, then con2prim + floors -> P (st_prims; in place:
// the stage-input P of the cell is the Newton guess).  Returns the A9 event
// code (0 none, 1 floor, 2 failure); rate = CFL rate of the new state.
template <bool KS, bool DIVB_NONE>
ECHO_D int stage_cell(const GridP& g, const EosP& e, const MetTables& mt, int s, double dt, const double* __restrict__ R,
                      const double* Un, const double* Us, double* Uout, double* P, int i, int j, int k,
                      bool want_rate, double& rate, const GhostLinks* gl = nullptr) {
  const auto m = MetAt<KS>::get(mt, i, j);
  const long long rb = rec_base(g, i, j, k), vs = g.vs;
  double Pp[8];
  double Z0;
  if (KS) {
    ld8(P + rb, vs, Pp);  // rho, u~, p, B of the stage input (B for the sources)
    Z0 = guess_Z(m, e, Pp);
  } else {
    Z0 = P[rb + kSlotZ * vs];  // the stored Newton guess (the primitives only on a failure)
  }
  double L[8];
  cell_L<KS, DIVB_NONE>(g, e, mt, m, R, rb, i, j, k, Pp, L);
  double Uo[8];
  ld8(Un + rb, vs, Uo);
  if (s == 1) {
#pragma unroll
    for (int q = 0; q < 8; q++) Uo[q] = Uo[q] + dt * L[q];
  } else {
    double us[8];
    ld8(Us + rb, vs, us);
    if (s == 2) {
#pragma unroll
      for (int q = 0; q < 8; q++) Uo[q] = 0.75 * Uo[q] + 0.25 * (us[q] + dt * L[q]);
    } else {
#pragma unroll
      for (int q = 0; q < 8; q++) Uo[q] = (1.0 / 3.0) * Uo[q] + (2.0 / 3.0) * (us[q] + dt * L[q]);
    }
  }
  double Po[8];
  const int ev = c2p_floors(m, e, Uo, Z0, [&](double* pv) {
#pragma unroll
    for (int v = 0; v < 5; v++) pv[v] = KS ? Pp[v] : P[rb + v * vs];
  }, Po);
  const double isg = !KS ? 1.0 : frcp(m.sqrtg());
#pragma unroll
  for (int c = 0; c < 3; c++) Po[5 + c] = !KS ? Uo[5 + c] : Uo[5 + c] * isg;
  st8(Uout + rb, vs, Uo);
  st_prims<KS>(P + rb, vs, Po);
  if (!KS) P[rb + kSlotZ * vs] = guess_Z(m, e, Po);  // the next stage's Newton guess
  if (want_rate) rate = fmax(rate, cfl_rate(m, g, e, Po));  // a9 fused: CFL rate of the new state
  if (gl && gl->on) {  // slab mode: the fused ghost exchange (echo_halo_link) and outflow replication
    const long long plane = (long long)g.n[1] * g.pitch;
    if (k < kZH && gl->dstP[0]) {
      st_prims<KS>(gl->dstP[0] + rb, vs, Po);
      st8(gl->dstU[0] + rb, vs, Uo);
    }
    if (k >= g.n[2] - kZH && gl->dstP[1]) {
      st_prims<KS>(gl->dstP[1] + rb, vs, Po);
      st8(gl->dstU[1] + rb, vs, Uo);
    }
    if (k == 0 && gl->replicate[0])
      for (int h = 1; h <= kZH; h++) {
        st_prims<KS>(P + rb - h * plane, vs, Po);
        st8(Uout + rb - h * plane, vs, Uo);
      }
    if (k == g.n[2] - 1 && gl->replicate[1])
      for (int h = 1; h <= kZH; h++) {
        st_prims<KS>(P + rb + h * plane, vs, Po);
        st8(Uout + rb + h * plane, vs, Uo);
      }
  }
  return ev;
}

}  // namespace echo
