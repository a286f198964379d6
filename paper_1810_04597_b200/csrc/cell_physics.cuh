// cell_physics.cuh — per-cell device physics shared by the K3 kernels:
// con2prim Newton (A8, A27, A28), floors (A9) and the metric sources (a6).
#pragma once
#include "echo_dev.cuh"

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
// 1-D Newton in Z = rho h W^2 with the oracle's iteration rules (A8, A27, A28).
// u: non-densitised (D, S_i, tau, B^i); guess: (rho, u~^i, p); out: (rho, u~^i, p).
template <class M>
ECHO_D int c2p_newton(const M& m, const EosP& e, const double* u, const double* guess, double* out) {
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
  double gu[3] = {guess[1], guess[2], guess[3]}, gl[3];
  m.lower(gu, gl);
  double Z = (guess[0] + e.gfac * guess[4]) * (1.0 + gu[0] * gl[0] + gu[1] * gl[1] + gu[2] * gl[2]);
  bool polish = false, ok = false;
  for (int it = 1; it <= e.maxit; it++) {
    const double iZ = frcp(Z);
    const double ZB = Z + B2;
    const double iZB = frcp(ZB);
    const double iZ2 = iZ * iZ, iZB2 = iZB * iZB;
    double v2 = (Z * Z * S2 + SB2 * (2.0 * Z + B2)) * iZ2 * iZB2;
    bool clamped = false;
    if (v2 > e.v2max) { v2 = e.v2max; clamped = true; }
    const double sq = fsqrt(1.0 - v2);
    const double p = e.gm * (Z * (1.0 - v2) - D * sq);
    const double f = Z - p + 0.5 * B2 * (1.0 + v2) - 0.5 * SB2 * iZ2 - Ut;
    const double dv2 = clamped ? 0.0 : -2.0 * iZB2 * iZB * (S2 + SB2 * (3.0 * Z * Z + 3.0 * Z * B2 + B2 * B2) * iZ2 * iZ);
    const double dp = e.gm * ((1.0 - v2) - Z * dv2 + D * dv2 * (0.5 * frcp(sq)));
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
  const double iZ = frcp(Z);
  const double ZB = Z + B2;
  const double iZB = frcp(ZB);
  double v2 = (Z * Z * S2 + SB2 * (2.0 * Z + B2)) * (iZ * iZ) * (iZB * iZB);
  if (v2 > e.v2max) v2 = e.v2max;
  const double sq = fsqrt(1.0 - v2);
  const double W = frcp(sq);
  out[0] = D * sq;
  out[4] = e.gm * (Z * (1.0 - v2) - D * sq);
  double vl[3], vu[3];
#pragma unroll
  for (int i = 0; i < 3; i++) vl[i] = (S[i] + SB * Bl[i] * iZ) * iZB;
  m.raise(vl, vu);
#pragma unroll
  for (int i = 0; i < 3; i++) out[1 + i] = W * vu[i];
  if (!isfinite(out[0]) || !isfinite(out[4])) return 1;
  return 0;
}

// A9 floors on the densitised cons Uc (8); Pprev (5) in, Pout (5) out.
// Returns 0 (nothing), 1 (floor event), 2 (failure).
template <class M>
ECHO_D int c2p_floors(const M& m, const EosP& e, double* Uc, const double* Pprev, double* Pout) {
  const double isg = 1.0 / m.sqrtg();
  double u[8];
#pragma unroll
  for (int q = 0; q < 8; q++) u[q] = M::kFlat ? Uc[q] : Uc[q] * isg;
  double pr[5];
  int status = c2p_newton(m, e, u, Pprev, pr);
  int ev = 0;
  if (status != 0) {
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

}  // namespace echo
