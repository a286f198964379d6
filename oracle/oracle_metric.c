/*
 * oracle_metric.c — ORACLE (test infrastructure only; see oracle.h header).
 *
 * The 3+1 split of the stationary background metric: lapse alpha, shift
 * beta^i, spatial metric gamma_ij, its inverse and sqrt(det gamma), plus the
 * coordinate derivatives the source terms need.
 *
 *  Minkowski (Cartesian x,y,z): alpha=1, beta=0, gamma=delta.   [DESIGN A1]
 *  Kerr-Schild (ingoing), spin a, mass M, in coordinates
 *  x1 = ln r, x2 = theta, x3 = phi                               [DESIGN A14]
 *    rho_K^2 = r^2 + a^2 cos^2(theta),  z = 2 M r / rho_K^2
 *    alpha = (1+z)^(-1/2),  beta^r = z/(1+z),  beta^theta = beta^phi = 0
 *    gamma_rr = 1+z, gamma_rphi = -a (1+z) sin^2,  gamma_thth = rho_K^2,
 *    gamma_phph = sin^2 (rho_K^2 + a^2 (1+z) sin^2)
 *  and with dr = r dx1:  gamma_11 = r^2 gamma_rr, gamma_13 = r gamma_rphi,
 *  beta^1 = beta^r / r.  The paper states only "General Relativity"
 *   and the torus run of Fig. 1; BASELINE.json
 *  config 4 names the Kerr-Schild (r,theta,phi) grid.
 *
 * gamma^ij and sqrt(gamma) are computed by their plain definitions (cofactor
 * inverse, sqrt of the determinant); the derivatives d/dx1 = r d/dr and
 * d/dx2 = d/dtheta are written out by hand below (pinned in tests against
 * finite differences and against d ln sqrt(gamma) = 1/2 gamma^ij d gamma_ij).
 */
#include <math.h>
#include <string.h>
#include "oracle_internal.h"

static void inverse3(const double g[3][3], double gi[3][3], double* det) {
  double c00 = g[1][1] * g[2][2] - g[1][2] * g[2][1];
  double c01 = g[1][2] * g[2][0] - g[1][0] * g[2][2];
  double c02 = g[1][0] * g[2][1] - g[1][1] * g[2][0];
  double d = g[0][0] * c00 + g[0][1] * c01 + g[0][2] * c02;
  gi[0][0] = c00 / d;
  gi[1][0] = c01 / d;
  gi[2][0] = c02 / d;
  gi[0][1] = (g[0][2] * g[2][1] - g[0][1] * g[2][2]) / d;
  gi[1][1] = (g[0][0] * g[2][2] - g[0][2] * g[2][0]) / d;
  gi[2][1] = (g[0][1] * g[2][0] - g[0][0] * g[2][1]) / d;
  gi[0][2] = (g[0][1] * g[1][2] - g[0][2] * g[1][1]) / d;
  gi[1][2] = (g[0][2] * g[1][0] - g[0][0] * g[1][2]) / d;
  gi[2][2] = (g[0][0] * g[1][1] - g[0][1] * g[1][0]) / d;
  *det = d;
}

void orc_met_eval(const orc_cfg* c, const double x[3], orc_met* m) {
  memset(m, 0, sizeof(*m));
  if (c->metric == ORC_MINKOWSKI) {
    m->alpha = 1.0;
    for (int i = 0; i < 3; i++) m->g[i][i] = 1.0;
  } else {
    double M = c->M, a = c->a;
    double r = exp(x[0]), th = x[1];
    double s = sin(th), co = cos(th);
    double rho2 = r * r + a * a * co * co;
    double z = 2.0 * M * r / rho2;
    double g_rr = 1.0 + z;
    double g_rph = -a * (1.0 + z) * s * s;
    double g_thth = rho2;
    double g_phph = s * s * (rho2 + a * a * (1.0 + z) * s * s);
    m->alpha = 1.0 / sqrt(1.0 + z);
    m->beta[0] = z / (1.0 + z) / r;
    m->g[0][0] = r * r * g_rr;
    m->g[0][2] = r * g_rph;
    m->g[2][0] = r * g_rph;
    m->g[1][1] = g_thth;
    m->g[2][2] = g_phph;
  }
  double det;
  inverse3(m->g, m->gi, &det);
  m->sqrtg = sqrt(det);
}

void orc_met_deriv_eval(const orc_cfg* c, const double x[3], orc_metd* d) {
  memset(d, 0, sizeof(*d));
  if (c->metric == ORC_MINKOWSKI) return;
  double M = c->M, a = c->a;
  double r = exp(x[0]), th = x[1];
  double s = sin(th), co = cos(th);
  double rho2 = r * r + a * a * co * co;
  double z = 2.0 * M * r / rho2;
  /* partial derivatives with respect to r and theta */
  double drho2_r = 2.0 * r;
  double drho2_t = -2.0 * a * a * co * s;
  double dz_r = 2.0 * M / rho2 - 2.0 * M * r * drho2_r / (rho2 * rho2);
  double dz_t = -2.0 * M * r * drho2_t / (rho2 * rho2);
  double dz[2] = {r * dz_r, dz_t}; /* d/dx1 = r d/dr, d/dx2 = d/dtheta */
  double drho2[2] = {r * drho2_r, drho2_t};
  for (int k = 0; k < 2; k++) {
    /* alpha = (1+z)^-1/2 */
    d->dalpha[k] = -0.5 * pow(1.0 + z, -1.5) * dz[k];
  }
  /* beta^1 = z / ((1+z) r) */
  double br = z / (1.0 + z);
  double dbr_r = dz_r / ((1.0 + z) * (1.0 + z));
  double dbr_t = dz_t / ((1.0 + z) * (1.0 + z));
  d->dbeta[0][0] = r * (dbr_r / r - br / (r * r)); /* r d/dr (beta^r / r) */
  d->dbeta[1][0] = dbr_t / r;
  /* gamma_11 = r^2 (1+z) */
  d->dg[0][0][0] = r * (2.0 * r * (1.0 + z) + r * r * dz_r);
  d->dg[1][0][0] = r * r * dz_t;
  /* gamma_13 = -a r (1+z) sin^2 */
  d->dg[0][0][2] = r * (-a * s * s * ((1.0 + z) + r * dz_r));
  d->dg[1][0][2] = -a * r * (dz_t * s * s + (1.0 + z) * 2.0 * s * co);
  d->dg[0][2][0] = d->dg[0][0][2];
  d->dg[1][2][0] = d->dg[1][0][2];
  /* gamma_22 = rho2 */
  d->dg[0][1][1] = drho2[0];
  d->dg[1][1][1] = drho2[1];
  /* gamma_33 = sin^2 (rho2 + a^2 (1+z) sin^2) */
  d->dg[0][2][2] = s * s * (drho2[0] + a * a * dz[0] * s * s);
  d->dg[1][2][2] = 2.0 * s * co * (rho2 + a * a * (1.0 + z) * s * s)
                 + s * s * (drho2[1] + a * a * dz[1] * s * s + a * a * (1.0 + z) * 2.0 * s * co);
}

int orc_metric(const orc_cfg* c, const double x[3], double out[23]) {
  orc_met m;
  orc_met_eval(c, x, &m);
  out[0] = m.alpha;
  for (int i = 0; i < 3; i++) out[1 + i] = m.beta[i];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      out[4 + 3 * i + j] = m.g[i][j];
      out[13 + 3 * i + j] = m.gi[i][j];
    }
  out[22] = m.sqrtg;
  return 0;
}

int orc_metric_deriv(const orc_cfg* c, const double x[3], double out[39]) {
  orc_metd d;
  orc_met_deriv_eval(c, x, &d);
  for (int k = 0; k < 3; k++) {
    out[k] = d.dalpha[k];
    for (int i = 0; i < 3; i++) out[3 + 3 * k + i] = d.dbeta[k][i];
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++) out[12 + 9 * k + 3 * i + j] = d.dg[k][i][j];
  }
  return 0;
}
