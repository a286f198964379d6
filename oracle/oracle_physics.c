/*
 * oracle_physics.c — ORACLE (test infrastructure only; see oracle.h).
 *
 * Point-wise ideal GRMHD in the 3+1 conservative form of the ECHO family
 * (ref. [1] of PAPER.md:104, not in the container; formulas restated from the
 * standard literature as DESIGN.md reading A1, SURVEY.md §8(c) "Equations"):
 *
 *   W = sqrt(1 + gamma_ij u~^i u~^j),  v^i = u~^i / W,  v^2 = v_i v^i
 *   h = 1 + Gamma p / ((Gamma-1) rho),  Z = rho h W^2
 *   E^i = -eps^{ijk} v_j B_k  (eps^{ijk} = [ijk]/sqrt(gamma)),
 *   E^2 = B^2 v^2 - (v.B)^2
 *   D = rho W,  S_i = (Z + B^2) v_i - (v.B) B_i,
 *   U = Z - p + (E^2 + B^2)/2,  tau = U - D                       [A10]
 *   W^{ij} = Z v^i v^j - E^i E^j - B^i B^j + (p + (E^2+B^2)/2) gamma^{ij}
 *   fluxes along j:  f(D) = (alpha v^j - beta^j) D
 *                    f(S_i) = alpha W^j_i - beta^j S_i
 *                    f(tau) = alpha (S^j - D v^j) - beta^j tau
 *                    f(B^i) = (alpha v^j - beta^j) B^i - (alpha v^i - beta^i) B^j
 *   sources (stationary metric):
 *     s(S_i) = 1/2 alpha W^{jk} d_i gamma_jk + S_j d_i beta^j - U d_i alpha
 *     s(tau) = 1/2 W^{ik} beta^j d_j gamma_ik + W_i^j d_j beta^i - S^j d_j alpha
 *   fast-speed bound (A4), HLL (A4), con2prim Newton in Z (A8).
 */
#include <math.h>
#include <string.h>
#include "oracle_internal.h"

void orc_aux_eval(const orc_met* m, double gam, const double pr[8], orc_aux* q) {
  const double rho = pr[0], p = pr[4];
  const double* ut = pr + 1;
  const double* B = pr + 5;
  double u2 = 0.0;
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) u2 += m->g[i][j] * ut[i] * ut[j];
  q->W = sqrt(1.0 + u2);
  for (int i = 0; i < 3; i++) q->v[i] = ut[i] / q->W;
  for (int i = 0; i < 3; i++) {
    q->vl[i] = 0.0;
    q->Bl[i] = 0.0;
    for (int j = 0; j < 3; j++) {
      q->vl[i] += m->g[i][j] * q->v[j];
      q->Bl[i] += m->g[i][j] * B[j];
    }
  }
  q->v2 = 0.0;
  q->B2 = 0.0;
  q->vB = 0.0;
  for (int i = 0; i < 3; i++) {
    q->v2 += q->vl[i] * q->v[i];
    q->B2 += q->Bl[i] * B[i];
    q->vB += q->vl[i] * B[i];
  }
  q->h = 1.0 + gam / (gam - 1.0) * p / rho;
  q->Z = rho * q->h * q->W * q->W;
  q->D = rho * q->W;
  for (int i = 0; i < 3; i++) q->S[i] = (q->Z + q->B2) * q->vl[i] - q->vB * q->Bl[i];
  for (int i = 0; i < 3; i++) {
    q->Su[i] = 0.0;
    for (int j = 0; j < 3; j++) q->Su[i] += m->gi[i][j] * q->S[j];
  }
  q->E2 = q->B2 * q->v2 - q->vB * q->vB;
  q->U = q->Z - p + 0.5 * (q->E2 + q->B2);
  q->tau = q->U - q->D;
  q->E[0] = -(q->vl[1] * q->Bl[2] - q->vl[2] * q->Bl[1]) / m->sqrtg;
  q->E[1] = -(q->vl[2] * q->Bl[0] - q->vl[0] * q->Bl[2]) / m->sqrtg;
  q->E[2] = -(q->vl[0] * q->Bl[1] - q->vl[1] * q->Bl[0]) / m->sqrtg;
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++)
      q->Wst[i][j] = q->Z * q->v[i] * q->v[j] - q->E[i] * q->E[j] - B[i] * B[j]
                   + (p + 0.5 * (q->E2 + q->B2)) * m->gi[i][j];
}

void orc_p2c(const orc_met* m, double gam, const double pr[8], double u[8]) {
  orc_aux q;
  orc_aux_eval(m, gam, pr, &q);
  u[0] = q.D;
  for (int i = 0; i < 3; i++) u[1 + i] = q.S[i];
  u[4] = q.tau;
  for (int i = 0; i < 3; i++) u[5 + i] = pr[5 + i];
}

void orc_flux(const orc_met* m, double gam, const double pr[8], int j, double f[8]) {
  orc_aux q;
  orc_aux_eval(m, gam, pr, &q);
  const double* B = pr + 5;
  const double a = m->alpha;
  f[0] = (a * q.v[j] - m->beta[j]) * q.D;
  for (int i = 0; i < 3; i++) {
    double Wmix = 0.0; /* W^j_i = W^{jk} gamma_ki */
    for (int k = 0; k < 3; k++) Wmix += q.Wst[j][k] * m->g[k][i];
    f[1 + i] = a * Wmix - m->beta[j] * q.S[i];
  }
  f[4] = a * (q.Su[j] - q.D * q.v[j]) - m->beta[j] * q.tau;
  for (int i = 0; i < 3; i++)
    f[5 + i] = (a * q.v[j] - m->beta[j]) * B[i] - (a * q.v[i] - m->beta[i]) * B[j];
}

/* A4: c_s^2 = Gamma p/(rho h), b^2 = B^2/W^2 + (v.B)^2, c_A^2 = b^2/(rho h + b^2),
 * a^2 = c_s^2 + c_A^2 - c_s^2 c_A^2,
 * lambda+- = alpha [v^j (1-a^2) +- sqrt(a^2 (1-v^2) [gamma^jj (1 - v^2 a^2) - v^j v^j (1-a^2)])]
 *            / (1 - v^2 a^2) - beta^j */
void orc_speeds(const orc_met* m, double gam, const double pr[8], int j, double* lm, double* lp) {
  orc_aux q;
  orc_aux_eval(m, gam, pr, &q);
  double rho = pr[0], p = pr[4];
  double cs2 = gam * p / (rho * q.h);
  double b2 = q.B2 / (q.W * q.W) + q.vB * q.vB;
  double ca2 = b2 / (rho * q.h + b2);
  double a2 = cs2 + ca2 - cs2 * ca2;
  double disc = a2 * (1.0 - q.v2) * (m->gi[j][j] * (1.0 - q.v2 * a2) - q.v[j] * q.v[j] * (1.0 - a2));
  if (disc < 0.0) disc = 0.0;
  double sq = sqrt(disc);
  double den = 1.0 - q.v2 * a2;
  *lp = m->alpha * (q.v[j] * (1.0 - a2) + sq) / den - m->beta[j];
  *lm = m->alpha * (q.v[j] * (1.0 - a2) - sq) / den - m->beta[j];
}

/* A4: two-wave HLL, S_L = min(0, lam-_L, lam-_R), S_R = max(0, lam+_L, lam+_R),
 * F = (S_R F_L - S_L F_R + S_L S_R (U_R - U_L)) / (S_R - S_L), then densitised. */
void orc_hll(const orc_met* m, double gam, const double pl[8], const double prr[8], int j, double F[8]) {
  double uL[8], uR[8], fL[8], fR[8], lmL, lpL, lmR, lpR;
  orc_p2c(m, gam, pl, uL);
  orc_p2c(m, gam, prr, uR);
  orc_flux(m, gam, pl, j, fL);
  orc_flux(m, gam, prr, j, fR);
  orc_speeds(m, gam, pl, j, &lmL, &lpL);
  orc_speeds(m, gam, prr, j, &lmR, &lpR);
  double sl = fmin(0.0, fmin(lmL, lmR));
  double sr = fmax(0.0, fmax(lpL, lpR));
  for (int q = 0; q < 8; q++) {
    double Fq;
    if (sr - sl > 0.0)
      Fq = (sr * fL[q] - sl * fR[q] + sl * sr * (uR[q] - uL[q])) / (sr - sl);
    else
      Fq = 0.5 * (fL[q] + fR[q]);
    F[q] = m->sqrtg * Fq;
  }
}

void orc_sources(const orc_met* m, const orc_metd* d, double gam, const double pr[8], double s[8]) {
  orc_aux q;
  orc_aux_eval(m, gam, pr, &q);
  for (int k = 0; k < 8; k++) s[k] = 0.0;
  for (int i = 0; i < 3; i++) {
    double t1 = 0.0, t2 = 0.0;
    for (int j = 0; j < 3; j++)
      for (int k = 0; k < 3; k++) t1 += q.Wst[j][k] * d->dg[i][j][k];
    for (int j = 0; j < 3; j++) t2 += q.S[j] * d->dbeta[i][j];
    s[1 + i] = 0.5 * m->alpha * t1 + t2 - q.U * d->dalpha[i];
  }
  double e1 = 0.0, e2 = 0.0, e3 = 0.0;
  for (int i = 0; i < 3; i++)
    for (int k = 0; k < 3; k++) {
      double bdg = 0.0; /* beta^j d_j gamma_ik */
      for (int j = 0; j < 3; j++) bdg += m->beta[j] * d->dg[j][i][k];
      e1 += 0.5 * q.Wst[i][k] * bdg;
    }
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      double Wmix = 0.0; /* W_i^j = gamma_ik W^{kj} */
      for (int k = 0; k < 3; k++) Wmix += m->g[i][k] * q.Wst[k][j];
      e2 += Wmix * d->dbeta[j][i];
    }
  for (int j = 0; j < 3; j++) e3 += q.Su[j] * d->dalpha[j];
  s[4] = e1 + e2 - e3;
}

/* A8: 1-D Newton in Z = rho h W^2 on the non-densitised cons u (D,S_i,tau,B^i).
 *   v^2(Z) = [Z^2 S^2 + (S.B)^2 (2Z + B^2)] / [Z^2 (Z + B^2)^2]  (clamped <= 1 - 1/Wmax^2)
 *   p(Z)   = (Gamma-1)/Gamma [Z (1-v^2) - D sqrt(1-v^2)]
 *   f(Z)   = Z - p + B^2 (1+v^2)/2 - (S.B)^2/(2 Z^2) - U,   U = tau + D
 *   f'(Z)  = 1 - p' + B^2 v2'/2 + (S.B)^2/Z^3
 *   p'     = (Gamma-1)/Gamma [(1-v^2) - Z v2' + D v2'/(2 sqrt(1-v^2))]
 *   v2'    = -2/(Z+B^2)^3 [S^2 + (S.B)^2 (3Z^2 + 3Z B^2 + B^4)/Z^3]   (0 when clamped)
 * Z <- Z - f/f'; a non-positive new Z is replaced by Z/2.  Converged when
 * |dZ| <= tol Z; then exactly one more (polish) iteration; cap c2p_max_iter. */
int orc_c2p(const orc_cfg* c, const orc_met* m, const double u[8], const double guess[8],
            double out[8], int* iters) {
  const double gam = c->gamma, gm = (gam - 1.0) / gam;
  const double D = u[0], tau = u[4];
  const double* S = u + 1;
  const double* B = u + 5;
  double U = tau + D;
  double S2 = 0.0, B2 = 0.0, SB = 0.0, Bl[3];
  for (int i = 0; i < 3; i++) {
    Bl[i] = 0.0;
    for (int j = 0; j < 3; j++) {
      S2 += m->gi[i][j] * S[i] * S[j];
      Bl[i] += m->g[i][j] * B[j];
    }
  }
  for (int i = 0; i < 3; i++) {
    B2 += Bl[i] * B[i];
    SB += S[i] * B[i];
  }
  double v2max = 1.0 - 1.0 / (c->w_max * c->w_max);
  /* initial guess from the previous primitive state */
  double ug2 = 0.0;
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) ug2 += m->g[i][j] * guess[1 + i] * guess[1 + j];
  double hg = 1.0 + gam / (gam - 1.0) * guess[4] / guess[0];
  double Z = guess[0] * hg * (1.0 + ug2);
  int polish = 0, ok = 0;
  *iters = 0;
  for (int it = 1; it <= c->c2p_max_iter; it++) {
    double Z2 = Z * Z, ZB = Z + B2;
    double v2 = (Z2 * S2 + SB * SB * (2.0 * Z + B2)) / (Z2 * ZB * ZB);
    int clamped = 0;
    if (v2 > v2max) {
      v2 = v2max;
      clamped = 1;
    }
    double sq = sqrt(1.0 - v2);
    double p = gm * (Z * (1.0 - v2) - D * sq);
    double f = Z - p + 0.5 * B2 * (1.0 + v2) - SB * SB / (2.0 * Z2) - U;
    double dv2 = clamped ? 0.0
                         : -2.0 / (ZB * ZB * ZB) * (S2 + SB * SB * (3.0 * Z2 + 3.0 * Z * B2 + B2 * B2) / (Z2 * Z));
    double dp = gm * ((1.0 - v2) - Z * dv2 + D * dv2 / (2.0 * sq));
    double df = 1.0 - dp + 0.5 * B2 * dv2 + SB * SB / (Z2 * Z);
    double Zn = Z - f / df;
    if (!(Zn > 0.0)) Zn = 0.5 * Z;
    double dZ = fabs(Zn - Z);
    Z = Zn;
    *iters = it;
    if (!isfinite(Z)) return 1;
    if (polish) {
      ok = 1;
      break;
    }
    if (dZ <= c->c2p_tol * Z) {
      polish = 1;
      if (it == c->c2p_max_iter) ok = 1;
    }
  }
  if (!ok) return 1;
  double Z2 = Z * Z, ZB = Z + B2;
  double v2 = (Z2 * S2 + SB * SB * (2.0 * Z + B2)) / (Z2 * ZB * ZB);
  if (v2 > v2max) v2 = v2max;
  double sq = sqrt(1.0 - v2);
  double W = 1.0 / sq;
  out[0] = D / W;
  out[4] = gm * (Z * (1.0 - v2) - D * sq);
  double vl[3];
  for (int i = 0; i < 3; i++) vl[i] = (S[i] + SB * Bl[i] / Z) / (Z + B2);
  for (int i = 0; i < 3; i++) {
    double vu = 0.0;
    for (int j = 0; j < 3; j++) vu += m->gi[i][j] * vl[j];
    out[1 + i] = W * vu;
  }
  for (int i = 0; i < 3; i++) out[5 + i] = B[i];
  if (!isfinite(out[0]) || !isfinite(out[4])) return 1;
  return 0;
}

/* A9 floors, applied in order; every change is counted, never silent. */
void orc_c2p_floors(const orc_cfg* c, const orc_met* m, double Uc[8], const double Pprev[5],
                    double Pout[5], long long* nfloor, long long* nfail) {
  double u[8], guess[8], pr[8];
  for (int q = 0; q < 8; q++) u[q] = Uc[q] / m->sqrtg;
  for (int q = 0; q < 5; q++) guess[q] = Pprev[q];
  for (int q = 5; q < 8; q++) guess[q] = u[q];
  int it;
  int status = orc_c2p(c, m, u, guess, pr, &it);
  int changed = 0;
  if (status != 0) {
    for (int i = 0; i < 3; i++) pr[1 + i] = Pprev[1 + i];
    double u2 = 0.0;
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++) u2 += m->g[i][j] * Pprev[1 + i] * Pprev[1 + j];
    double Wp = sqrt(1.0 + u2);
    pr[0] = fmax(u[0] / Wp, c->rho_floor);
    pr[4] = fmax(Pprev[4], c->p_floor);
    for (int i = 0; i < 3; i++) pr[5 + i] = u[5 + i];
    *nfail += 1;
    changed = 1;
  } else {
    if (pr[0] < c->rho_floor) {
      pr[0] = c->rho_floor;
      changed = 1;
    }
    if (pr[4] < c->p_floor) {
      pr[4] = c->p_floor;
      changed = 1;
    }
    double u2 = 0.0;
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++) u2 += m->g[i][j] * pr[1 + i] * pr[1 + j];
    double Wu = sqrt(1.0 + u2);
    if (Wu > c->w_max) {
      double sc = sqrt((c->w_max * c->w_max - 1.0) / (Wu * Wu - 1.0));
      for (int i = 0; i < 3; i++) pr[1 + i] *= sc;
      changed = 1;
    }
    if (changed) *nfloor += 1;
  }
  if (changed) {
    double cons[8];
    orc_p2c(m, c->gamma, pr, cons);
    for (int q = 0; q < 5; q++) Uc[q] = m->sqrtg * cons[q];
  }
  for (int q = 0; q < 5; q++) Pout[q] = pr[q];
}

/* ---- exported point-wise wrappers ---- */
int orc_prim2cons_pt(const orc_cfg* c, const double x[3], const double pr[8], double u[8]) {
  orc_met m;
  orc_met_eval(c, x, &m);
  orc_p2c(&m, c->gamma, pr, u);
  return 0;
}
int orc_flux_pt(const orc_cfg* c, const double x[3], const double pr[8], int dir, double f[8]) {
  orc_met m;
  orc_met_eval(c, x, &m);
  orc_flux(&m, c->gamma, pr, dir, f);
  return 0;
}
int orc_speeds_pt(const orc_cfg* c, const double x[3], const double pr[8], int dir, double lam[2]) {
  orc_met m;
  orc_met_eval(c, x, &m);
  orc_speeds(&m, c->gamma, pr, dir, &lam[0], &lam[1]);
  return 0;
}
int orc_hll_pt(const orc_cfg* c, const double x[3], const double pl[8], const double prr[8], int dir,
               double F[8]) {
  orc_met m;
  orc_met_eval(c, x, &m);
  orc_hll(&m, c->gamma, pl, prr, dir, F);
  return 0;
}
int orc_sources_pt(const orc_cfg* c, const double x[3], const double pr[8], double s[8]) {
  orc_met m;
  orc_metd d;
  orc_met_eval(c, x, &m);
  orc_met_deriv_eval(c, x, &d);
  orc_sources(&m, &d, c->gamma, pr, s);
  return 0;
}
int orc_c2p_pt(const orc_cfg* c, const double x[3], const double u[8], const double guess[8],
               double pr_out[8], int* iters) {
  orc_met m;
  orc_met_eval(c, x, &m);
  return orc_c2p(c, &m, u, guess, pr_out, iters);
}
