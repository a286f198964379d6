// echo_dev.cuh — device-side parameters and point-wise GRMHD physics for the
// sm_100a kernels.  Formulas: DESIGN.md §2 and readings A1-A30 (the paper,
// PAPER.md:19, names the equations but prints none).  Written for the FP64
// pipe: reciprocals computed once, products of the WENO smoothness factors
// instead of three divisions, the stress written through b^2 (no E field).
#pragma once
#include <cstdint>

#define ECHO_HD __host__ __device__ __forceinline__
#define ECHO_D __device__ __forceinline__

namespace echo {

constexpr int kG = 5;  // halo: WENO5 (3) + DER6 (2), A12
constexpr int kZH = 6; // stored z ghost planes per side in slab mode (kG + 1: the sweeps also
                       // produce the EMF on the first ghost plane, which the field-CD curl reads)
constexpr int kZHU = 8;  // UCT slabs: the induction's DER needs the edge EMFs 3 planes into the
                         // halo, their z reconstructions face data 5 planes in, whose HLL states
                         // the primitives 7 planes in (+1: the staggered b^z of the last face)

// FP64 constants that are not exact in a 32-bit-high-word immediate live in the
// constant bank, so every DFMA takes them as a c[][] operand (otherwise the
// compiler rebuilds each one with a pair of UMOVs at every use).
//   [0..2] DER6 symmetric-sum weights 1067/960, -29/480, 3/640; [3..4] DER4 13/12, -1/24
//   [5] WENO5 eps scaled by 3 (weno5_both), [6] 1/6 (FV candidates), [7] 4/3 (MP5 u_lc),
//   [8] WENO-Z eps scaled by 3, [9] [10] point-form WENO5 eps scaled by 3/4 and -1.5 x that
static __constant__ double kCst[11] = {1067.0 / 960.0, -29.0 / 480.0, 3.0 / 640.0, 13.0 / 12.0, -1.0 / 24.0,
                                       3.0e-6, 1.0 / 6.0, 4.0 / 3.0, 3.0e-40, 0.75e-6, -1.125e-6};

struct GridP {
  int n[3];
  long long N;      // cells per field
  double lo[3];
  double dx[3];     // (hi - lo) / n
  double idx[3];    // 1 / dx
  int bc[3][2];     // 0 periodic, 1 outflow, 2 halo (z only: planes filled by the caller, echo_halo_*)
  int zhalo;        // stored z ghost planes per side (0: none; kZH, or kZHU with UCT), filled by the caller
                    // before each stage
  int rec, der, divb;
  double der_jump;  // A31 DER shock switch (+inf: off; the host maps <= 0 to +inf)
  long long vs;     // variable stride inside a row: n1 rounded up to even (16-byte aligned variables, TMA)
  long long pitch;  // doubles per (j, k) row of a record array: 8 vs + padding
};

struct EosP {
  double gamma;
  double gfac;      // Gamma / (Gamma - 1)
  double gm;        // (Gamma - 1) / Gamma
  double rho_floor, p_floor, w_max, v2max;
  int maxit;
  double tol;
};

// ----------------------------------------------------------- metric types
// Symmetric 3x3 stored as (00, 01, 02, 11, 12, 22).
ECHO_HD int sidx(int i, int j) {
  return (i <= j) ? (i == 0 ? j : (i == 1 ? 2 + j : 5)) : (j == 0 ? i : (j == 1 ? 2 + i : 5));
}

// Flat (Minkowski, Cartesian): every metric operation compiles away.
struct FlatMet {
  ECHO_D double alpha() const { return 1.0; }
  ECHO_D double beta(int) const { return 0.0; }
  ECHO_D double sqrtg() const { return 1.0; }
  ECHO_D double gi_diag(int) const { return 1.0; }
  ECHO_D void lower(const double* v, double* vl) const { vl[0] = v[0]; vl[1] = v[1]; vl[2] = v[2]; }
  ECHO_D void raise(const double* v, double* vu) const { vu[0] = v[0]; vu[1] = v[1]; vu[2] = v[2]; }
  static constexpr bool kFlat = true;
};

// General stationary 3+1 metric at one point (Kerr-Schild tables).
struct GenMet {
  double a, b[3], g[6], gi[6], sg;
  ECHO_D double alpha() const { return a; }
  ECHO_D double beta(int i) const { return b[i]; }
  ECHO_D double sqrtg() const { return sg; }
  ECHO_D double gi_diag(int j) const { return gi[sidx(j, j)]; }
  ECHO_D void lower(const double* v, double* vl) const {
    vl[0] = g[0] * v[0] + g[1] * v[1] + g[2] * v[2];
    vl[1] = g[1] * v[0] + g[3] * v[1] + g[4] * v[2];
    vl[2] = g[2] * v[0] + g[4] * v[1] + g[5] * v[2];
  }
  ECHO_D void raise(const double* v, double* vu) const {
    vu[0] = gi[0] * v[0] + gi[1] * v[1] + gi[2] * v[2];
    vu[1] = gi[1] * v[0] + gi[3] * v[1] + gi[4] * v[2];
    vu[2] = gi[2] * v[0] + gi[4] * v[1] + gi[5] * v[2];
  }
  static constexpr bool kFlat = false;
};

// Table record sizes (doubles).  Face/centre value record: alpha, beta[3], g[6], gi[6], sqrtg.
constexpr int kMetRec = 17;
// Centre derivative record: dalpha[2], dbeta[2][3], dg[2][6]  (d/dx1, d/dx2; d/dx3 = 0).
constexpr int kDerRec = 20;

ECHO_D GenMet load_met(const double* __restrict__ rec) {
  GenMet m;
  m.a = __ldg(rec + 0);
#pragma unroll
  for (int i = 0; i < 3; i++) m.b[i] = __ldg(rec + 1 + i);
#pragma unroll
  for (int i = 0; i < 6; i++) m.g[i] = __ldg(rec + 4 + i);
#pragma unroll
  for (int i = 0; i < 6; i++) m.gi[i] = __ldg(rec + 10 + i);
  m.sg = __ldg(rec + 16);
  return m;
}

// Kerr-Schild tables (device pointers), all phi-independent (2-D in x1, x2),
// extended by kG ghost layers so that ghost positions are covered.
struct MetTables {
  const double* cen;   // [(j+G)*(n1+2G) + (i+G)][kMetRec]       cell centres
  const double* der;   // [(j+G)*(n1+2G) + (i+G)][kDerRec]       centre derivatives
  const double* f0;    // [(j+G)*(n1+2G+1) + (i+G)][kMetRec]     x1-face i-1/2, i in [-G, n1+G]
  const double* f1;    // [(j+G)*(n1+2G) + (i+G)][kMetRec]       x2-face j-1/2, j in [-G, n2+G]
  int w0;              // n1 + 2G
};

ECHO_D const double* cen_rec(const MetTables& t, int i, int j) {
  return t.cen + ((long long)(j + kG) * t.w0 + (i + kG)) * kMetRec;
}
ECHO_D const double* der_rec(const MetTables& t, int i, int j) {
  return t.der + ((long long)(j + kG) * t.w0 + (i + kG)) * kDerRec;
}
// face i-1/2 along x1 at row j
ECHO_D const double* f0_rec(const MetTables& t, int i, int j) {
  return t.f0 + ((long long)(j + kG) * (t.w0 + 1) + (i + kG)) * kMetRec;
}
// face j-1/2 along x2 at column i
ECHO_D const double* f1_rec(const MetTables& t, int i, int j) {
  return t.f1 + ((long long)(j + kG) * t.w0 + (i + kG)) * kMetRec;
}

// ------------------------------------------------ FP64 reciprocal / rsqrt
// MUFU seed (rcp/rsqrt.approx.ftz.f64: relative error <= 1e-6, measured in
// tools/rcp_accuracy.cu) + one higher-order correction: with e = 1 - x y0,
// 1/x = y0 (1 + e + e^2 + ...) -> y0 + y0 (e + e^2), truncation |e|^3 <= 1e-18;
// with r = 1 - x y0^2, 1/sqrt(x) = y0 (1 + r/2 + 3 r^2/8 + ...), truncation ~|r|^3.
// Both are within 1-1.3 ulp of the correctly rounded results over 1.2e9 samples
// (profiles/rcp_accuracy.json).  Arguments here are always positive, normal and
// finite (sums of squares, 1 - v^2 a^2, ...).
ECHO_D double frcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}
ECHO_D double frsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double r = fma(-x * y, y, 1.0);
  return fma(y * r, fma(0.375, r, 0.5), y);
}
// min / max by compare-select (operands are finite: no NaN handling needed, unlike fmin)
ECHO_D double dmin(double a, double b) { return a < b ? a : b; }
ECHO_D double dmax(double a, double b) { return a > b ? a : b; }
ECHO_D double fsqrt(double x) { return x > 0.0 ? x * frsqrt(x) : 0.0; }

// ------------------------------------------------------- device layout
// Every per-cell record (P, U, R: 8 doubles) is stored row-interleaved,
// [k][j][var][i]: element (var, i, j, k) at (k n2 + j) pitch + var vs + i.  x stays
// unit-stride (coalesced, 16-B pairs), and one (j, k) row holds all 8 variables
// (8 n1 doubles), so a z-pencil touches one 2 MB page per plane instead of 8.
// vs = n1 rounded up to even; rows are padded to `pitch` = 8 vs + 8 doubles so plane
// strides are not powers of two.
ECHO_HD long long rec_base(const GridP& g, int i, int j, int k) {
  return ((long long)k * g.n[1] + j) * g.pitch + i;
}
ECHO_HD long long rec_base_id(const GridP& g, long long id) {  // id = linear cell index (x fastest)
  const long long r = id / g.n[0];
  return r * g.pitch + (id - r * g.n[0]);
}

// --------------------------------------------------------------- indices
ECHO_D int map_index(int i, int n, int bclo, int bchi) {  // ghost rule A12/A13
  // (bc 2: a slab side whose ghost planes are stored: the index itself)
  if (i < 0) return bclo == 0 ? ((i % n) + n) % n : (bclo == 2 ? i : 0);
  if (i >= n) return bchi == 0 ? (i % n) : (bchi == 2 ? i : n - 1);
  return i;
}

// ------------------------------------------------------- one state's physics
// Everything the flux, conserved vector and speeds of one primitive state need.
struct State {
  double W2i;        // 1/W^2
  double v[3];       // v^i
  double vl[3];      // v_i
  double v2;
  double B[3];       // B^i
  double Bl[3];      // B_i
  double B2, vB, b2;
  double rhoh, ptot;
  double ZB;         // Z + B^2 (= tau + D + p_tot)
  double D, S[3], tau;
};

template <class M>
ECHO_D void make_state(const M& m, const EosP& e, const double* pr, State& s) {
  // pr: rho, u~^1..3, p, B^1..3
  double ut[3] = {pr[1], pr[2], pr[3]};
  double ul[3];
  m.lower(ut, ul);
  double u2 = ut[0] * ul[0] + ut[1] * ul[1] + ut[2] * ul[2];
  double W2 = 1.0 + u2;
  double iW = frsqrt(W2);
  double W = W2 * iW;
  s.W2i = iW * iW;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    s.v[i] = ut[i] * iW;
    s.vl[i] = ul[i] * iW;
    s.B[i] = pr[5 + i];
  }
  s.v2 = u2 * s.W2i;
  m.lower(s.B, s.Bl);
  s.B2 = s.B[0] * s.Bl[0] + s.B[1] * s.Bl[1] + s.B[2] * s.Bl[2];
  s.vB = s.vl[0] * s.B[0] + s.vl[1] * s.B[1] + s.vl[2] * s.B[2];
  s.b2 = s.B2 * s.W2i + s.vB * s.vB;
  s.rhoh = pr[0] + e.gfac * pr[4];
  s.ptot = pr[4] + 0.5 * s.b2;
  s.ZB = fma(s.rhoh, W2, s.B2);  // Z + B^2, Z = rho h W^2
  s.D = pr[0] * W;
#pragma unroll
  for (int i = 0; i < 3; i++) s.S[i] = fma(s.ZB, s.vl[i], -s.vB * s.Bl[i]);
  // U = Z - p + (E^2 + B^2)/2 = Z + B^2 - p_tot  (E^2 = B^2 - b^2)
  s.tau = (s.ZB - s.ptot) - s.D;
}

// fast-speed bound along axis j (A4).  With N = Gamma p + b^2 and Dn = rho h + b^2,
// a^2 = cs^2 + cA^2 - cs^2 cA^2 = N / Dn, and the reading's
//   lambda = alpha [v^j (1 - a^2) +- sqrt(a^2 (1 - v^2) [g^jj (1 - v^2 a^2) - v^j v^j (1 - a^2)])] / (1 - v^2 a^2) - beta^j
// multiplied through by Dn (exact in real arithmetic):
//   lambda = alpha [v^j (Dn - N) +- sqrt(N (1 - v^2) [g^jj (Dn - v^2 N) - v^j v^j (Dn - N)])] / (Dn - v^2 N) - beta^j
// (one reciprocal and one square root per state).
template <class M>
ECHO_D void speeds(const M& m, const EosP& e, const double* pr, const State& s, int j, double& lm, double& lp) {
  const double N = fma(e.gamma, pr[4], s.b2);
  const double Dn = s.rhoh + s.b2;
  const double vj = s.v[j];
  const double DmN = Dn - N;
  const double den = fma(-s.v2, N, Dn);
  // 1 - v^2 = 1 / W^2 (exact in real arithmetic)
  // (flat: den - v_j^2 (Dn - N) as one FMA)
  const double Q = (N * s.W2i) * (M::kFlat ? fma(-vj * vj, DmN, den) : fma(m.gi_diag(j), den, -vj * vj * DmN));
  const double sq = fsqrt(Q);
  const double iden = M::kFlat ? frcp(den) : m.alpha() * frcp(den);
  const double c0 = M::kFlat ? vj * (DmN * iden) : fma(vj * DmN, iden, -m.beta(j));
  lp = fma(sq, iden, c0);
  lm = fma(-sq, iden, c0);
}

// densitised HLL flux (7 comps) between two reconstructed states at one face (A4), times
// `scale` (the sweeps pass 1/Delta_a, so the flux difference of the DER values needs no
// multiply: DER is linear)
// fs (UCT, A38, A43): if not NULL, V^1..3 = alpha v^i - beta^i of the left and of the right
// state, a+ = S_R, a- = -S_L
template <class M>
ECHO_D void hll_face(const M& m, const EosP& e, const double* pl, const double* pr, int AX, double* F,
                     double* fs = nullptr, double scale = 1.0) {
  State sl, sr;
  make_state(m, e, pl, sl);
  make_state(m, e, pr, sr);
  double uL[7], fL[7], uR[7], fR[7];
  cons_flux(m, sl, AX, uL, fL);
  cons_flux(m, sr, AX, uR, fR);
  double lmL, lpL, lmR, lpR;
  speeds(m, e, pl, sl, AX, lmL, lpL);
  speeds(m, e, pr, sr, AX, lmR, lpR);
  const double sL = dmin(0.0, dmin(lmL, lmR));
  const double sR = dmax(0.0, dmax(lpL, lpR));
  if (fs) {  // A43: the transport velocity V^i = alpha v^i - beta^i of each state
#pragma unroll
    for (int i = 0; i < 3; i++) {
      fs[i] = fma(m.alpha(), sl.v[i], -m.beta(i));
      fs[3 + i] = fma(m.alpha(), sr.v[i], -m.beta(i));
    }
    fs[6] = sR;
    fs[7] = -sL;
  }
  const double den = sR - sL;
  if (den > 0.0) {
    const double inv = (M::kFlat ? scale : m.sqrtg() * scale) * frcp(den);
    const double a = sR * inv, b = sL * inv, c = a * sL;
#pragma unroll
    for (int q = 0; q < 7; q++) F[q] = fma(c, uR[q] - uL[q], fma(a, fL[q], -b * fR[q]));
  } else {
#pragma unroll
    for (int q = 0; q < 7; q++) F[q] = (fL[q] + fR[q]) * (0.5 * m.sqrtg() * scale);
  }
}

// Non-densitised conserved vector (7 used comps along axis j: D, S_1..3, tau, B^{j+1}, B^{j+2})
// and flux along j.  Momentum flux through the b^2 identity (E^2 = B^2 - b^2)
//   W^j_i = v_i S^j + p_tot delta^j_i - B_i (B^j / W^2 + (v.B) v^j),
//   S^j = (Z + B^2) v^j - (v.B) B^j.
template <class M>
ECHO_D void cons_flux(const M& m, const State& s, int j, double* u, double* f) {
  const double a = m.alpha();
  const double bj = m.beta(j);
  const double Vj = a * s.v[j] - bj;
  const double bbar = s.B[j] * s.W2i + s.vB * s.v[j];
  // S^j = (Z + B^2) v^j - (v.B) B^j (flat: S^j = S_j)
  const double Sj = M::kFlat ? s.S[j] : fma(s.ZB, s.v[j], -s.vB * s.B[j]);
  u[0] = s.D;
  f[0] = Vj * s.D;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    u[1 + i] = s.S[i];
    f[1 + i] = a * (s.vl[i] * Sj - s.Bl[i] * bbar) - bj * s.S[i] + (i == j ? a * s.ptot : 0.0);
  }
  u[4] = s.tau;
  f[4] = a * (Sj - s.D * s.v[j]) - bj * s.tau;
  const int j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  u[5] = s.B[j1];
  u[6] = s.B[j2];
  f[5] = Vj * s.B[j1] - (a * s.v[j1] - m.beta(j1)) * s.B[j];
  f[6] = Vj * s.B[j2] - (a * s.v[j2] - m.beta(j2)) * s.B[j];
}

// --------------------------------------------------------------- WENO5 (A2)
// Left state at i+1/2 and right state at i-1/2 from u[-2..2] of one cell and one
// variable.  beta_k are shared by both faces; alpha_k = d_k/(eps+beta_k)^2 is
// evaluated through the products s_l s_m so one division per face remains.
// Arithmetic rearrangements (all exact in real arithmetic, rounding-level in fp64):
//  * beta_k scaled by 3 with eps -> 3 eps: the weights only depend on ratios of
//    (eps + beta_k)^2, so the common factor 9 cancels;
//  * the ideal weights d_k and the candidates' 1/8 are folded into the candidate
//    coefficients (all exact binary fractions for the point-value form).
//  * everything is written in the first differences dmm = u_{-1}-u_{-2},
//    dm = u_0-u_{-1}, dp = u_1-u_0, dpp = u_2-u_1: the second differences of the
//    smoothness indicators are d2m = dm-dmm, d2c = dp-dm, d2p = dpp-dp, and
//    (u_{-2} - 4u_{-1} + 3u_0) = d2m + 2dm, (u_{-1} - u_1) = -(dm + dp),
//    (3u_0 - 4u_1 + u_2) = d2p - 2dp; since sum(omega) = 1 each face value is
//    u_0 + sum_k omega_k (q_k - u_0) with the candidate increments q_k - u_0
//    linear in the differences (2 flops each instead of 5).
// REC 0: point form (A2), 1: finite-volume form, 3: WENO-Z weights on the point form (A34)
template <int REC>
ECHO_D void weno5_both(double um2, double um1, double u0, double up1, double up2, double& qL, double& qR) {
  const double eps3 = REC == 3 ? kCst[8] : kCst[5];
  const double dmm = um1 - um2, dm = u0 - um1, dp = up1 - u0, dpp = up2 - up1;
  // 3 beta_k as quadratic forms of the first differences (12 beta_k = 13 t^2 + 3 tb^2):
  //   3 beta_0 = 10 dm^2 - 11 dm dmm + 4 dmm^2
  //   3 beta_1 =  4 dm^2 -  5 dm dp  + 4 dp^2
  //   3 beta_2 = 10 dp^2 - 11 dp dpp + 4 dpp^2
  // (positive definite, so no cancellation beyond a few ulp); eps -> 3 eps.
  const double m2 = dm * dm, p2 = dp * dp;
  double s0, s1, s2;
  if constexpr (REC == 0) {
    // point form: the three scaled by 1/4 (the weights depend on ratios only), eps -> 3 eps / 4,
    // written so that every coefficient-1 term rides in an FMA (10 operations instead of 14):
    //   s0 = dmm (dmm - 2.75 dm) + 2.5 dm^2 + e,  s1 = dm (dm - 1.25 dp) + dp^2 + e,
    //   s2 = dpp (dpp - 2.75 dp) + 2.5 dp^2 + e = dpp (...) + 2.5 (dp^2 + e) - 1.5 e
    const double e4 = kCst[9];
    const double pe = fma(dp, dp, e4);
    s0 = fma(dmm, fma(-2.75, dm, dmm), fma(2.5, m2, e4));
    s1 = fma(dm, fma(-1.25, dp, dm), pe);
    s2 = fma(dpp, fma(-2.75, dp, dpp), fma(2.5, pe, kCst[10]));
  } else {
    s0 = fma(10.0, m2, fma(dmm, fma(4.0, dmm, -11.0 * dm), eps3));
    s1 = fma(4.0, m2, fma(4.0, p2, fma(-5.0 * dm, dp, eps3)));
    s2 = fma(10.0, p2, fma(dpp, fma(4.0, dpp, -11.0 * dp), eps3));
  }
  if constexpr (REC == 3) {
    // WENO-Z: alpha_k = d_k (1 + tau5 / s_k), tau5 = |s_0 - s_2| (the common factor 3 of s_k and
    // tau5 cancels); times s_0 s_1 s_2: A_k = (s_k + tau5) prod_{l != k} s_l.  The mirror face
    // swaps s_0 and s_2, i.e. A_0 <-> A_2, with the same candidate increments as the point form.
    const double tau = fabs(s0 - s2);
    const double A0 = (s0 + tau) * (s1 * s2), A1 = (s1 + tau) * (s0 * s2), A2 = (s2 + tau) * (s0 * s1);
    const double C0 = fma(0.875, dm, -0.375 * dmm), C1 = fma(1.25, dm, 3.75 * dp), C2 = fma(3.125, dp, -0.625 * dpp);
    const double E0 = fma(0.375, dpp, -0.875 * dp), E1 = fma(-1.25, dp, -3.75 * dm), E2 = fma(0.625, dmm, -3.125 * dm);
    const double SL = fma(10.0, A1, fma(5.0, A2, A0)), SR = fma(10.0, A1, fma(5.0, A0, A2));
    const double NL = fma(A2, C2, fma(A1, C1, A0 * C0));
    const double NR = fma(A0, E2, fma(A1, E1, A2 * E0));
    const double inv = frcp(SL * SR);
    qL = fma(NL, SR * inv, u0);
    qR = fma(NR, SL * inv, u0);
    return;
  }
  s0 *= s0;
  s1 *= s1;
  s2 *= s2;
  const double p01 = s0 * s1, p02 = s0 * s2, p12 = s1 * s2;
  double C0, C1, C2, E0, E1, E2, SL, SR;  // d_k (q_k - u0) for the left / right faces
  if (REC == 0) {
    // point form, d = (1, 10, 5)/16 (the 16 cancels):
    //   q0-u0 = (7dm - 3dmm)/8, q1-u0 = (dm + 3dp)/8, q2-u0 = (5dp - dpp)/8, right = mirror
    C0 = fma(0.875, dm, -0.375 * dmm);
    C1 = fma(1.25, dm, 3.75 * dp);
    C2 = fma(3.125, dp, -0.625 * dpp);
    E0 = fma(0.375, dpp, -0.875 * dp);
    E1 = fma(-1.25, dp, -3.75 * dm);
    E2 = fma(0.625, dmm, -3.125 * dm);
    SL = fma(5.0, p01, fma(10.0, p02, p12));
    SR = fma(5.0, p12, fma(10.0, p02, p01));
  } else {
    // finite-volume form, d = (1, 6, 3)/10 (the 10 cancels):
    //   q0-u0 = (5dm - 2dmm)/6, q1-u0 = (dm + 2dp)/6, q2-u0 = (4dp - dpp)/6, right = mirror
    const double k = kCst[6];
    C0 = k * fma(5.0, dm, -2.0 * dmm);
    C1 = fma(1.0, dm, 2.0 * dp);
    C2 = 0.5 * fma(4.0, dp, -dpp);
    E0 = k * fma(2.0, dpp, -5.0 * dp);
    E1 = fma(-1.0, dp, -2.0 * dm);
    E2 = 0.5 * fma(-4.0, dm, dmm);
    SL = fma(3.0, p01, fma(6.0, p02, p12));
    SR = fma(3.0, p12, fma(6.0, p02, p01));
  }
  // left: alpha_k ~ d_k / s_k ~ (p12, d1 p02, d2 p01); right (mirror): (p01, d1 p02, d2 p12)
  double NL, NR;
  if (REC == 0) {
    // C1 = 1.25 (dm + 3 dp), E1 = -1.25 (dp + 3 dm): the common 1.25 rides on p02 (one multiply
    // instead of two)
    const double q02 = 1.25 * p02;
    NL = fma(p01, C2, fma(q02, fma(3.0, dp, dm), p12 * C0));
    NR = fma(p12, E2, fma(-q02, fma(3.0, dm, dp), p01 * E0));
  } else {
    NL = fma(p01, C2, fma(p02, C1, p12 * C0));
    NR = fma(p12, E2, fma(p02, E1, p01 * E0));
  }
#ifdef ECHO_WENO_TWO_RCP
  // two independent reciprocals (same FP64 count, one more MUFU, a dependency chain 2 shorter)
  qL = fma(NL, frcp(SL), u0);
  qR = fma(NR, frcp(SR), u0);
#else
  // both normalisations through one reciprocal: 1/(SL SR)
  const double inv = frcp(SL * SR);
  qL = fma(NL, SR * inv, u0);
  qR = fma(NR, SL * inv, u0);
#endif
}

// --------------------------------------------------------------- MP5 (A33)
// Suresh & Huynh (1997) on point values: left state at i+1/2 = median(u_OR, u_min, u_max)
// with u_OR the 5-point interpolant (3, -20, 90, 60, -5)/128 (the paper's early exit for
// (u_OR - u_i)(u_OR - u_MP) <= 0 returns the same value, A33).  The right state at i-1/2
// is the mirror; the second differences and their M4 limits are shared by both faces
// (the mirror maps d_{i-1} <-> d_{i+1} and M4_{i+1/2} <-> M4_{i-1/2}).
// minmod through signs (copysign and fabs are sign-bit operations): the sign factor is
// exactly -1, 0 or 1, and an argument +-0 gives 0 through the magnitude minimum, so
// the values equal the oracle's branch form bit for bit
ECHO_D double mm2(double a, double b) {
  return (copysign(0.5, a) + copysign(0.5, b)) * dmin(fabs(a), fabs(b));
}
ECHO_D double mm4(double a, double b, double c, double d) {
  const double sa = copysign(1.0, a);
  const double s = (sa + copysign(1.0, b)) * fabs((sa + copysign(1.0, c)) * (sa + copysign(1.0, d)));  // -8, 0, 8
  return (0.125 * s) * dmin(dmin(fabs(a), fabs(b)), dmin(fabs(c), fabs(d)));
}
// one face from the stencil (um2, um1, u0, up1, up2), M4 at the face (m4f) and at the
// opposite face (m4b)
ECHO_D double mp5_face(double um2, double um1, double u0, double up1, double up2, double m4f, double m4b) {
  const double u_or = (3.0 * um2 - 20.0 * um1 + 90.0 * u0 + 60.0 * up1 - 5.0 * up2) * 0.0078125;  // /128
  const double dl = u0 - um1;
  const double u_ul = fma(4.0, dl, u0);
  const double u_md = fma(-0.5, m4f, 0.5 * (u0 + up1));
  const double u_lc = fma(kCst[7], m4b, fma(0.5, dl, u0));
  // max(min(u0, up1, u_md), min(u0, u_ul, u_lc)) = min(u0, max(min(up1, u_md), min(u_ul, u_lc))), exact
  const double u_min = dmin(u0, dmax(dmin(up1, u_md), dmin(u_ul, u_lc)));
  const double u_max = dmax(u0, dmin(dmax(up1, u_md), dmax(u_ul, u_lc)));
  return u_or + mm2(u_min - u_or, u_max - u_or);
}
ECHO_D void mp5_both(double um2, double um1, double u0, double up1, double up2, double& qL, double& qR) {
  const double dm = um2 - 2.0 * um1 + u0, d0 = um1 - 2.0 * u0 + up1, dp = u0 - 2.0 * up1 + up2;
  const double m4p = mm4(4.0 * d0 - dp, 4.0 * dp - d0, d0, dp);  // at i+1/2
  const double m4m = mm4(4.0 * d0 - dm, 4.0 * dm - d0, d0, dm);  // at i-1/2
  qL = mp5_face(um2, um1, u0, up1, up2, m4p, m4m);
  qR = mp5_face(up2, up1, u0, um1, um2, m4m, m4p);
}

// MC2 (A35): u_i +- slope/2 with the monotonized-central slope; the mirror face has the
// negated slope exactly (minmod is odd)
ECHO_D void mc2_both(double um1, double u0, double up1, double& qL, double& qR) {
  const double dl = u0 - um1, dr = up1 - u0, dc = 0.5 * (up1 - um1);
  double slope = 0.0;
  if (dl > 0.0 && dr > 0.0) slope = dmin(dmin(2.0 * dl, dc), 2.0 * dr);
  else if (dl < 0.0 && dr < 0.0) slope = dmax(dmax(2.0 * dl, dc), 2.0 * dr);
  qL = u0 + 0.5 * slope;
  qR = u0 + 0.5 * -slope;
}

// PPM (A36): the limiter's decisions are discontinuous, so every quantity that enters one is
// evaluated with explicitly rounded operations in the oracle's order (no FMA contraction):
// the decisions, and hence the states, match the oracle's bit for bit.
ECHO_D double ppm_face(double a, double b, double c, double d) {  // interface between b and c
  double v = __dmul_rn(__dsub_rn(__dadd_rn(__dadd_rn(-a, __dmul_rn(9.0, b)), __dmul_rn(9.0, c)), d), 0.0625);
  const double lo = dmin(b, c), hi = dmax(b, c);
  v = dmax(v, lo);
  return dmin(v, hi);
}
ECHO_D double ppm_right_of(double uL, double ui, double uR) {  // the constrained u_R of a cell
  if (!(__dmul_rn(__dsub_rn(uR, ui), __dsub_rn(ui, uL)) > 0.0)) return ui;
  const double du = __dsub_rn(uR, uL);
  const double m6 = __dmul_rn(6.0, __dsub_rn(ui, __dmul_rn(0.5, __dadd_rn(uL, uR))));
  if (-__dmul_rn(du, du) > __dmul_rn(du, m6)) return __dsub_rn(__dmul_rn(3.0, ui), __dmul_rn(2.0, uL));
  return uR;
}
ECHO_D void ppm_both(double um2, double um1, double u0, double up1, double up2, double& qL, double& qR) {
  // left state at i+1/2: u_R of cell i from the stencil (um2..up2); right state at i-1/2:
  // u_R of the mirrored stencil (up2..um2), i.e. its interfaces evaluated in the mirror order
  qL = ppm_right_of(ppm_face(um2, um1, u0, up1), u0, ppm_face(um1, u0, up1, up2));
  qR = ppm_right_of(ppm_face(up2, up1, u0, um1), u0, ppm_face(up1, u0, um1, um2));
}

// ----------------------------------------- characteristic-wise WENO5 (rec = 6, A44)
// One face of WENO5 point form (A2): the left-biased value at i+1/2 from u_{i-2..i+2} (the right
// state at i+1/2 is this of the mirrored stencil u_{i+3..i-1}).  The same normalisation as
// weno5_both (beta / 4, eps -> 3 eps / 4).
ECHO_D double weno5_one(double um2, double um1, double u0, double up1, double up2) {
  const double dmm = um1 - um2, dm = u0 - um1, dp = up1 - u0, dpp = up2 - up1;
  const double e4 = kCst[9];
  const double pe = fma(dp, dp, e4);
  double s0 = fma(dmm, fma(-2.75, dm, dmm), fma(2.5, dm * dm, e4));
  double s1 = fma(dm, fma(-1.25, dp, dm), pe);
  double s2 = fma(dpp, fma(-2.75, dp, dpp), fma(2.5, pe, kCst[10]));
  s0 *= s0;
  s1 *= s1;
  s2 *= s2;
  const double p01 = s0 * s1, p02 = s0 * s2, p12 = s1 * s2;
  const double C0 = fma(0.875, dm, -0.375 * dmm), C1 = fma(1.25, dm, 3.75 * dp), C2 = fma(3.125, dp, -0.625 * dpp);
  const double SL = fma(5.0, p01, fma(10.0, p02, p12));
  const double NL = fma(p01, C2, fma(p02, C1, p12 * C0));
  return fma(NL, frcp(SL), u0);
}

// Reading A44 at one face i+1/2 along the sweep axis: q[m] = (rho, u~^n, u~^t1, u~^t2, p) of cells
// i-2+m, m = 0..5, in the sweep's frame.  Projection with the closed-form LEFT eigenvectors of the
// flat relativistic-Euler Jacobian at the mean of cells i and i+1 (the oracle inverts the right
// ones numerically; exact in real arithmetic):
//   w = (rho, v^n, v^t1, v^t2, p):  l_- = (0, -1, 0, 0, a_+/g) / Da,  l_0 = (1, 0, 0, 0, -1/g),
//   l_t1 = (0, -v^t1 T, 1, 0, -v^t1 X),  l_t2 likewise,  l_+ = (0, 1, 0, 0, -a_-/g) / Da,
//   a_+- = k_+-(1 - v^n lambda_+-), t_+- = -k_+- lambda_+-, k_+- = g / (rho h W^2 (lambda_+- - v^n)),
//   g = Gamma p / rho, Da = a_+ - a_-, T = (t_+ - t_-) / Da, X = (t_- a_+ - t_+ a_-) / (g Da);
//   in q (du~ = W (I + W^2 v v^T) dv) a row (l_rho, l_v, l_p) becomes (l_rho, (l_v - (l_v.v) v)/W, l_p).
// WENO5 per characteristic field, then back with the right eigenvectors:
//   rho = c_- + c_0 + c_+,  p = g (c_- + c_+),  u~ = W (z + W^2 v (v.z)),
//   z = (c_- a_- + c_+ a_+, v^t1 (c_- t_- + c_+ t_+) + c_t1, v^t2 (c_- t_- + c_+ t_+) + c_t2).
// fL / fR: the left / right hydro states at the face, frame order.
ECHO_D void char_face(const EosP& e, const double (&q)[6][5], double* fL, double* fR) {
  double qb[5];
#pragma unroll
  for (int k = 0; k < 5; k++) qb[k] = 0.5 * (q[2][k] + q[3][k]);
  const double u2 = fma(qb[1], qb[1], fma(qb[2], qb[2], qb[3] * qb[3]));
  const double W2 = 1.0 + u2;
  const double iW = frsqrt(W2);
  const double W = W2 * iW;
  const double v[3] = {qb[1] * iW, qb[2] * iW, qb[3] * iW};
  const double v2 = u2 * (iW * iW);
  const double rho = qb[0], p = qb[4];
  const double rhoh = fma(e.gfac, p, rho);
  const double irho = frcp(rho * rhoh);                  // 1/rho and 1/(rho h) from one reciprocal
  const double g = e.gamma * p * (rhoh * irho);          // Gamma p / rho
  const double cs2 = e.gamma * p * (rho * irho);         // Gamma p / (rho h)
  const double den = fma(-v2, cs2, 1.0);
  const double disc = cs2 * (1.0 - v2) * fma(-v[0] * v[0], 1.0 - cs2, den);
  const double sq = fsqrt(disc);
  const double iden = frcp(den);
  const double b = v[0] * (1.0 - cs2) * iden;
  const double lp = fma(sq, iden, b), lm = fma(-sq, iden, b);
  // k_+- = g / (rho h W^2 (lambda_+- - v^n)) through one reciprocal of the product
  const double dp_ = lp - v[0], dm_ = lm - v[0];
  const double ir = frcp(rhoh * W2 * dp_ * dm_);
  const double kp = g * dm_ * ir, km = g * dp_ * ir;
  const double ap = kp * fma(-v[0], lp, 1.0), am = km * fma(-v[0], lm, 1.0);
  const double tp = -kp * lp, tm = -km * lm;
  const double iDa = frcp(ap - am);
  const double ig = frcp(g);
  const double T = (tp - tm) * iDa, X = (tm * ap - tp * am) * (ig * iDa);
  // left eigenvectors in q: e_ = (e_n - v^n v) / (W Da) for l_+ (l_- = -e_), l_t1, l_t2
  const double iWD = iW * iDa;
  const double en[3] = {(1.0 - v[0] * v[0]) * iWD, -v[0] * v[1] * iWD, -v[0] * v[2] * iWD};
  double lt[2][3];
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const double vt = v[1 + k];
    const double lv[3] = {-vt * T, k == 0 ? 1.0 : 0.0, k == 0 ? 0.0 : 1.0};
    const double dot = vt * fma(-T, v[0], 1.0);         // l_v . v
#pragma unroll
    for (int d = 0; d < 3; d++) lt[k][d] = fma(-dot, v[d], lv[d]) * iW;
  }
  const double pm = ap * ig * iDa, pp = -am * ig * iDa;  // p coefficients of l_- and l_+
  double cl[5], cr[5];  // characteristic face values: -, 0, t1, t2, +
#pragma unroll
  for (int k = 0; k < 5; k++) {
    double ch[6];
#pragma unroll
    for (int m = 0; m < 6; m++) {
      const double eu = fma(en[0], q[m][1], fma(en[1], q[m][2], en[2] * q[m][3]));
      if (k == 0) ch[m] = fma(pm, q[m][4], -eu);
      else if (k == 4) ch[m] = fma(pp, q[m][4], eu);
      else if (k == 1) ch[m] = fma(-ig, q[m][4], q[m][0]);
      else {
        const double* l = lt[k - 2];
        ch[m] = fma(-v[k - 1] * X, q[m][4], fma(l[0], q[m][1], fma(l[1], q[m][2], l[2] * q[m][3])));
      }
    }
    cl[k] = weno5_one(ch[0], ch[1], ch[2], ch[3], ch[4]);
    cr[k] = weno5_one(ch[5], ch[4], ch[3], ch[2], ch[1]);
  }
  auto back = [&](const double* c, double* f) {
    f[0] = c[0] + c[1] + c[4];
    f[4] = g * (c[0] + c[4]);
    const double tt = fma(c[0], tm, c[4] * tp);
    const double z[3] = {fma(c[0], am, c[4] * ap), fma(v[1], tt, c[2]), fma(v[2], tt, c[3])};
    const double vz = W2 * fma(v[0], z[0], fma(v[1], z[1], v[2] * z[2]));
#pragma unroll
    for (int d = 0; d < 3; d++) f[1 + d] = W * fma(vz, v[d], z[d]);
  };
  back(cl, fL);
  back(cr, fR);
}

// reconstruction switch: REC 0/1 WENO5 (point / finite-volume form), 2 MP5, 3 WENO-Z, 4 MC2, 5 PPM
template <int REC>
ECHO_D void rec_both(double um2, double um1, double u0, double up1, double up2, double& qL, double& qR) {
  if constexpr (REC == 5) ppm_both(um2, um1, u0, up1, up2, qL, qR);
  else if constexpr (REC == 4) mc2_both(um1, u0, up1, qL, qR);
  else if constexpr (REC == 2) mp5_both(um2, um1, u0, up1, up2, qL, qR);
  else weno5_both<REC>(um2, um1, u0, up1, up2, qL, qR);
}

// --------------------------------------------------------------- DER (A5)
// H = F0 - d2F/24 + 3 d4F/640 collected by symmetric sums:
//   H = (1067/960) F0 - (29/480)(F-1 + F+1) + (3/640)(F-2 + F+2)
template <int DER>
ECHO_D double der5(double Fm2, double Fm1, double F0, double Fp1, double Fp2) {
  if (DER == 6) return fma(kCst[2], Fm2 + Fp2, fma(kCst[1], Fm1 + Fp1, kCst[0] * F0));
  if (DER == 4) return fma(kCst[4], Fm1 + Fp1, kCst[3] * F0);
  return F0;
}

}  // namespace echo
