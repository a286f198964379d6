/*
 * oracle_scheme.c — ORACLE (test infrastructure only; see oracle.h).
 *
 * Grid-level algorithm of one SSP-RK3 stage, in the order of DESIGN.md §2
 * (SURVEY.md §8(c) "Stage algorithm"):
 *   1. ghost fill of the 8 primitives (rho, u~^i, p, B^i = U_B/sqrt(gamma)),
 *      g = 5 deep, axis-sequential, ghost(i) = owned(((i mod n)+n) mod n) for
 *      periodic, owned(clamp(i,0,n-1)) for outflow            [A12, A13]
 *   2. for axis a = 1,2,3: per line, every face i+1/2, i = -3..n+1:
 *      WENO5 (or MP5, rec=2, A33) of the 8 primitives (left state from cells
 *      i-2..i+2, right state the mirror from cells i+3..i-1) [A2, A3],
 *      positivity fallback [A25],
 *      HLL flux with the face metric [A4]; DER correction of the face fluxes
 *      [A5]; L_q -= (H_{i+1/2} - H_{i-1/2}) / Delta_a for the 5 hydro vars;
 *      field-CD EMF contributions Omega (or, divb=none, B flux differences) [A6]
 *   3. L += sqrt(gamma) s  (metric sources at cell centres)
 *   4. L(sqrt(gamma) B^i) = -D_j Omega_k + D_k Omega_j, (i,j,k) cyclic,
 *      Omega ghosts filled with the same boundary rule      [A6]
 *   5. RK combine in the literal SPEC.md:154 forms             [A7]
 *   6. con2prim + floors                                       [A8, A9]
 * Two evaluation paths share the face/cell functions bit for bit: the full
 * grid (padded arrays) and the per-cell path (index-mapped reads) used for
 * sampled parity at full size; a pin test checks they agree bitwise.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include "oracle_internal.h"

#define G ORC_G

static int nthreads_of(const orc_cfg* c) {
#ifdef _OPENMP
  return c->nthreads > 0 ? c->nthreads : omp_get_max_threads();
#else
  (void)c;
  return 1;
#endif
}

static double dx_of(const orc_cfg* c, int a) { return (c->hi[a] - c->lo[a]) / c->n[a]; }
static double centre_of(const orc_cfg* c, int a, long long i) { return c->lo[a] + (i + 0.5) * dx_of(c, a); }
static double face_of(const orc_cfg* c, int a, long long i) { return c->lo[a] + (i + 1) * dx_of(c, a); } /* face i+1/2 */

/* ghost index rule (A12/A13) */
static long long map_index(const orc_cfg* c, int a, long long i) {
  long long n = c->n[a];
  if (i < 0) {
    if (c->bc[a][0] == ORC_BC_PERIODIC) return ((i % n) + n) % n;
    return 0;
  }
  if (i >= n) {
    if (c->bc[a][1] == ORC_BC_PERIODIC) return ((i % n) + n) % n;
    return n - 1;
  }
  return i;
}

static long long ncells(const orc_cfg* c) { return (long long)c->n[0] * c->n[1] * c->n[2]; }
static long long lin(const orc_cfg* c, long long i, long long j, long long k) {
  return (k * c->n[1] + j) * c->n[0] + i;
}

/* ------------------------------------------------------------------ */
/* Reconstruction and DER (A2, A5)                                     */
/* ------------------------------------------------------------------ */
double orc_weno5_left(const double u[5], int rec) {
  const double eps = 1e-6;
  double b0 = 13.0 / 12.0 * (u[0] - 2.0 * u[1] + u[2]) * (u[0] - 2.0 * u[1] + u[2])
            + 0.25 * (u[0] - 4.0 * u[1] + 3.0 * u[2]) * (u[0] - 4.0 * u[1] + 3.0 * u[2]);
  double b1 = 13.0 / 12.0 * (u[1] - 2.0 * u[2] + u[3]) * (u[1] - 2.0 * u[2] + u[3])
            + 0.25 * (u[1] - u[3]) * (u[1] - u[3]);
  double b2 = 13.0 / 12.0 * (u[2] - 2.0 * u[3] + u[4]) * (u[2] - 2.0 * u[3] + u[4])
            + 0.25 * (3.0 * u[2] - 4.0 * u[3] + u[4]) * (3.0 * u[2] - 4.0 * u[3] + u[4]);
  double q0, q1, q2, d0, d1, d2;
  if (rec == 0) { /* point-value interpolation form (A2) */
    q0 = (3.0 * u[0] - 10.0 * u[1] + 15.0 * u[2]) / 8.0;
    q1 = (-u[1] + 6.0 * u[2] + 3.0 * u[3]) / 8.0;
    q2 = (3.0 * u[2] + 6.0 * u[3] - u[4]) / 8.0;
    d0 = 1.0 / 16.0;
    d1 = 10.0 / 16.0;
    d2 = 5.0 / 16.0;
  } else { /* finite-volume form */
    q0 = (2.0 * u[0] - 7.0 * u[1] + 11.0 * u[2]) / 6.0;
    q1 = (-u[1] + 5.0 * u[2] + 2.0 * u[3]) / 6.0;
    q2 = (2.0 * u[2] + 5.0 * u[3] - u[4]) / 6.0;
    d0 = 1.0 / 10.0;
    d1 = 6.0 / 10.0;
    d2 = 3.0 / 10.0;
  }
  double a0 = d0 / ((eps + b0) * (eps + b0));
  double a1 = d1 / ((eps + b1) * (eps + b1));
  double a2 = d2 / ((eps + b2) * (eps + b2));
  double w0 = a0 / (a0 + a1 + a2);
  double w1 = a1 / (a0 + a1 + a2);
  double w2 = a2 / (a0 + a1 + a2);
  return w0 * q0 + w1 * q1 + w2 * q2;
}

/* MP5 (Suresh & Huynh 1997, J. Comput. Phys. 136, 83: eqs. 2.12 and 2.19-2.21 in
 * their order), left-biased value at i+1/2 from u[0..4] = u_{i-2..i+2}; SURVEY §8(f)
 * f3 ("other high-order reconstruction algorithms").  Reading A33: point
 * values, so the unlimited value u_OR is the 5-point interpolant at i+1/2,
 * (3 u_{i-2} - 20 u_{i-1} + 90 u_i + 60 u_{i+1} - 5 u_{i+2}) / 128; alpha = 4;
 * the no-limiting test uses eps = 0. */
static double minmod2(double a, double b) {
  if (a > 0.0 && b > 0.0) return a < b ? a : b;
  if (a < 0.0 && b < 0.0) return a > b ? a : b;
  return 0.0;
}
static double minmod4(double a, double b, double c, double d) {
  if (a > 0.0 && b > 0.0 && c > 0.0 && d > 0.0) return fmin(fmin(a, b), fmin(c, d));
  if (a < 0.0 && b < 0.0 && c < 0.0 && d < 0.0) return fmax(fmax(a, b), fmax(c, d));
  return 0.0;
}
static double median3(double a, double b, double c) { return a + minmod2(b - a, c - a); }
static double min3(double a, double b, double c) { return fmin(a, fmin(b, c)); }
static double max3(double a, double b, double c) { return fmax(a, fmax(b, c)); }

double orc_mp5_left(const double u[5]) {
  const double alpha = 4.0;
  /* (2.12) the unlimited value and the monotonicity-preserving bound */
  const double u_or = (3.0 * u[0] - 20.0 * u[1] + 90.0 * u[2] + 60.0 * u[3] - 5.0 * u[4]) / 128.0;
  const double u_mp = u[2] + minmod2(u[3] - u[2], alpha * (u[2] - u[1]));
  if ((u_or - u[2]) * (u_or - u_mp) <= 0.0) return u_or;
  /* (2.19) second differences and their M4 limits at i+1/2 and i-1/2 */
  const double dm = u[0] - 2.0 * u[1] + u[2];
  const double d0 = u[1] - 2.0 * u[2] + u[3];
  const double dp = u[2] - 2.0 * u[3] + u[4];
  const double dm4_p = minmod4(4.0 * d0 - dp, 4.0 * dp - d0, d0, dp);
  const double dm4_m = minmod4(4.0 * d0 - dm, 4.0 * dm - d0, d0, dm);
  /* (2.20) upper limit, median, large curvature */
  const double u_ul = u[2] + alpha * (u[2] - u[1]);
  const double u_av = 0.5 * (u[2] + u[3]);
  const double u_md = u_av - 0.5 * dm4_p;
  const double u_lc = u[2] + 0.5 * (u[2] - u[1]) + 4.0 / 3.0 * dm4_m;
  /* (2.21) the limit interval and the limited value */
  const double u_min = fmax(min3(u[2], u[3], u_md), min3(u[2], u_ul, u_lc));
  const double u_max = fmin(max3(u[2], u[3], u_md), max3(u[2], u_ul, u_lc));
  return median3(u_or, u_min, u_max);
}

/* WENO-Z (Borges, Carmona, Costa & Don 2008, J. Comput. Phys. 227, 3191: eqs. 24-28),
 * point-value candidates and ideal weights as WENO5 (A2), the same Jiang-Shu beta_k;
 * alpha_k = d_k (1 + tau5 / (beta_k + eps)) with tau5 = |beta_0 - beta_2|, eps = 1e-40
 * (their value; reading A34).  Left-biased value at i+1/2 from u[0..4] = u_{i-2..i+2}. */
double orc_wenoz_left(const double u[5]) {
  const double eps = 1e-40;
  double b0 = 13.0 / 12.0 * (u[0] - 2.0 * u[1] + u[2]) * (u[0] - 2.0 * u[1] + u[2])
            + 0.25 * (u[0] - 4.0 * u[1] + 3.0 * u[2]) * (u[0] - 4.0 * u[1] + 3.0 * u[2]);
  double b1 = 13.0 / 12.0 * (u[1] - 2.0 * u[2] + u[3]) * (u[1] - 2.0 * u[2] + u[3])
            + 0.25 * (u[1] - u[3]) * (u[1] - u[3]);
  double b2 = 13.0 / 12.0 * (u[2] - 2.0 * u[3] + u[4]) * (u[2] - 2.0 * u[3] + u[4])
            + 0.25 * (3.0 * u[2] - 4.0 * u[3] + u[4]) * (3.0 * u[2] - 4.0 * u[3] + u[4]);
  double q0 = (3.0 * u[0] - 10.0 * u[1] + 15.0 * u[2]) / 8.0;
  double q1 = (-u[1] + 6.0 * u[2] + 3.0 * u[3]) / 8.0;
  double q2 = (3.0 * u[2] + 6.0 * u[3] - u[4]) / 8.0;
  double tau5 = fabs(b0 - b2);
  double a0 = 1.0 / 16.0 * (1.0 + tau5 / (b0 + eps));
  double a1 = 10.0 / 16.0 * (1.0 + tau5 / (b1 + eps));
  double a2 = 5.0 / 16.0 * (1.0 + tau5 / (b2 + eps));
  return (a0 * q0 + a1 * q1 + a2 * q2) / (a0 + a1 + a2);
}

/* MC2: the monotonized-central limited linear reconstruction (van Leer 1977), the
 * "limited" second-order entry of SURVEY f3 (reading A35): left value at i+1/2 =
 * u_i + slope/2 with slope = minmod(2 (u_i - u_{i-1}), (u_{i+1} - u_{i-1}) / 2,
 * 2 (u_{i+1} - u_i)); uses u[1..3] of the 5-point stencil. */
double orc_mc2_left(const double u[5]) {
  const double dl = u[2] - u[1], dr = u[3] - u[2], dc = 0.5 * (u[3] - u[1]);
  double slope;
  if (dl > 0.0 && dr > 0.0) slope = fmin(fmin(2.0 * dl, dc), 2.0 * dr);
  else if (dl < 0.0 && dr < 0.0) slope = fmax(fmax(2.0 * dl, dc), 2.0 * dr);
  else slope = 0.0;
  return u[2] + 0.5 * slope;
}

/* PPM (Colella & Woodward 1984, J. Comput. Phys. 54, 174: eqs. 1.6-1.10) on point values
 * (reading A36): the interface values of cell i are the 4th-order point interpolants
 * (-u_{i-1} + 9 u_i + 9 u_{i+1} - u_{i+2}) / 16 at i+1/2 (and the mirror at i-1/2),
 * kept between the neighbouring cells (eq. 1.8's role: min/max of u_i, u_{i+1}); then the
 * monotonicity constraints of eq. 1.10: a local extremum flattens both to u_i; an
 * interface value that would put an extremum of the parabola inside the cell is reset
 * (u_R = 3 u_i - 2 u_L, or u_L = 3 u_i - 2 u_R).  Contact steepening and flattening
 * (CW84 §1 eqs. 1.14-1.17) are not used.  Returns the left state at i+1/2 (u_R of cell i). */
static double ppm_face(double a, double b, double c, double d) {  /* interface between b and c */
  double v = (-a + 9.0 * b + 9.0 * c - d) / 16.0;
  const double lo = fmin(b, c), hi = fmax(b, c);
  if (v < lo) v = lo;
  if (v > hi) v = hi;
  return v;
}
double orc_ppm_left(const double u[5]) {
  double uR = ppm_face(u[1], u[2], u[3], u[4]); /* i+1/2 */
  double uL = ppm_face(u[0], u[1], u[2], u[3]); /* i-1/2 */
  const double ui = u[2];
  if ((uR - ui) * (ui - uL) <= 0.0) return ui;
  const double du = uR - uL, m6 = 6.0 * (ui - 0.5 * (uL + uR));
  if (du * m6 > du * du) uL = 3.0 * ui - 2.0 * uR;
  if (-du * du > du * m6) uR = 3.0 * ui - 2.0 * uL;
  return uR;
}

/* reconstruction switch: rec 0/1 WENO5 (point / finite-volume form), 2 MP5, 3 WENO-Z, 4 MC2, 5 PPM */
static double orc_rec_left(const double u[5], int rec) {
  if (rec == 5) return orc_ppm_left(u);
  if (rec == 4) return orc_mc2_left(u);
  if (rec == 3) return orc_wenoz_left(u);
  return rec == 2 ? orc_mp5_left(u) : orc_weno5_left(u, rec);
}

double orc_der(const double F[5], int der) {
  if (der == 6)
    return F[2] - (F[1] - 2.0 * F[2] + F[3]) / 24.0
         + 3.0 * (F[0] - 4.0 * F[1] + 6.0 * F[2] - 4.0 * F[3] + F[4]) / 640.0;
  if (der == 4) return F[2] - (F[1] - 2.0 * F[2] + F[3]) / 24.0;
  return F[2];
}

/* A31: does the face between cells with prims pa, pb join a jump in rho or p? */
static int rough_face(const orc_cfg* c, const double pa[8], const double pb[8]) {
  if (!(c->der_jump > 0.0)) return 0;
  return fabs(pb[0] - pa[0]) > c->der_jump * fmin(pa[0], pb[0]) ||
         fabs(pb[4] - pa[4]) > c->der_jump * fmin(pa[4], pb[4]);
}

/* DER flux at a face from the 5 face fluxes F5[m][q] (faces i-3/2..i+5/2) and
 * their roughness flags: the plain flux if any face of the stencil is rough (A31). */
static void der_face(const orc_cfg* c, const double F5[5][8], const int rough5[5], double H[8]) {
  int any = 0;
  for (int m = 0; m < 5; m++) any |= rough5[m];
  for (int q = 0; q < 8; q++) {
    double f5[5];
    for (int m = 0; m < 5; m++) f5[m] = F5[m][q];
    H[q] = any ? F5[2][q] : orc_der(f5, c->der);
  }
}

/* ------------------------------------------------------------------ */
/* rec = 6: characteristic-wise WENO5 of the hydro primitives (A44)     */
/* ------------------------------------------------------------------ */
/* Plain Gauss-Jordan inverse with partial pivoting of an n x n matrix (n <= 5). */
static void invert5(int n, const double A[5][5], double X[5][5]) {
  double M[5][10];
  for (int i = 0; i < n; i++)
    for (int j = 0; j < 2 * n; j++) M[i][j] = j < n ? A[i][j] : (j - n == i ? 1.0 : 0.0);
  for (int col = 0; col < n; col++) {
    int piv = col;
    for (int r = col + 1; r < n; r++)
      if (fabs(M[r][col]) > fabs(M[piv][col])) piv = r;
    if (piv != col)
      for (int j = 0; j < 2 * n; j++) {
        double t = M[col][j];
        M[col][j] = M[piv][j];
        M[piv][j] = t;
      }
    double d = M[col][col];
    for (int j = 0; j < 2 * n; j++) M[col][j] /= d;
    for (int r = 0; r < n; r++) {
      if (r == col) continue;
      double f = M[r][col];
      for (int j = 0; j < 2 * n; j++) M[r][j] -= f * M[col][j];
    }
  }
  for (int i = 0; i < n; i++)
    for (int j = 0; j < n; j++) X[i][j] = M[i][n + j];
}

/* Reading A44, step by step.  q = (rho, u~^n, u~^t1, u~^t2, p) with n = a, t1 = a+1, t2 = a+2
 * (cyclic), the hydro primitives of A3 in the sweep's own frame.  Flat metric only.
 *  1. face state qbar = (q_i + q_{i+1}) / 2 (cells st[2], st[3]);
 *  2. its right eigenvectors, the flat-space relativistic-Euler Jacobian A = (dU/dq)^-1 dF^n/dq
 *     with B = 0: in w = (rho, v^n, v^t1, v^t2, p) they are (SURVEY §8(c) A4 gives the speeds)
 *       r_-  = (1, k_-(1 - v^n l_-), -k_- l_- v^t1, -k_- l_- v^t2, G p / rho),  l_- = lambda_-
 *       r_0  = (1, 0, 0, 0, 0)       (contact: lambda = v^n)
 *       r_t1 = (0, 0, 1, 0, 0), r_t2 = (0, 0, 0, 1, 0)   (shear: lambda = v^n)
 *       r_+  as r_- with lambda_+,   k_+- = (G p / rho) / (rho h W^2 (lambda_+- - v^n));
 *     mapped to q by dq = blockdiag(1, W (I + W^2 v v^T), 1) dw;
 *  3. L = R^-1 (Gauss-Jordan);
 *  4. characteristic variables c_k(m) = L_k . q_m of cells m = i-2 .. i+3;
 *  5. WENO5 point form (A2) of each: c_k^L from m = 0..4, c_k^R the mirror from m = 5..1;
 *  6. q^L = R c^L, q^R = R c^R.
 * Writes the 5 hydro slots of qL, qR (the order rho, u~^1, u~^2, u~^3, p of the state). */
static void char_rec_face(const orc_cfg* c, const double st[6][8], int a, double qL[8], double qR[8]) {
  const double G_ = c->gamma;
  const int comp[3] = {a, (a + 1) % 3, (a + 2) % 3};
  double qs[6][5];
  for (int m = 0; m < 6; m++) {
    qs[m][0] = st[m][0];
    for (int d = 0; d < 3; d++) qs[m][1 + d] = st[m][1 + comp[d]];
    qs[m][4] = st[m][4];
  }
  /* 1. */
  double qb[5];
  for (int v = 0; v < 5; v++) qb[v] = 0.5 * (qs[2][v] + qs[3][v]);
  const double rho = qb[0], p = qb[4];
  const double uu = qb[1] * qb[1] + qb[2] * qb[2] + qb[3] * qb[3];
  const double W = sqrt(1.0 + uu);
  double v[3];
  for (int d = 0; d < 3; d++) v[d] = qb[1 + d] / W;
  const double v2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  const double h = 1.0 + G_ / (G_ - 1.0) * p / rho;
  const double cs2 = G_ * p / (rho * h);
  const double gp = G_ * p / rho;
  /* 2. */
  const double disc = cs2 * (1.0 - v2) * (1.0 - v2 * cs2 - v[0] * v[0] * (1.0 - cs2));
  const double lam[2] = {(v[0] * (1.0 - cs2) - sqrt(disc)) / (1.0 - v2 * cs2),
                         (v[0] * (1.0 - cs2) + sqrt(disc)) / (1.0 - v2 * cs2)};
  double Rw[5][5] = {{0}};
  for (int s = 0; s < 2; s++) {
    const int col = s == 0 ? 0 : 4;
    const double k = gp / (rho * h * W * W * (lam[s] - v[0]));
    Rw[0][col] = 1.0;
    Rw[1][col] = k * (1.0 - v[0] * lam[s]);
    Rw[2][col] = -k * lam[s] * v[1];
    Rw[3][col] = -k * lam[s] * v[2];
    Rw[4][col] = gp;
  }
  Rw[0][1] = 1.0;
  Rw[2][2] = 1.0;
  Rw[3][3] = 1.0;
  double Mv[3][3];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) Mv[i][j] = W * ((i == j ? 1.0 : 0.0) + W * W * v[i] * v[j]);
  double R[5][5];
  for (int col = 0; col < 5; col++) {
    R[0][col] = Rw[0][col];
    R[4][col] = Rw[4][col];
    for (int i = 0; i < 3; i++) {
      double sum = 0.0;
      for (int j = 0; j < 3; j++) sum += Mv[i][j] * Rw[1 + j][col];
      R[1 + i][col] = sum;
    }
  }
  /* 3. */
  double L[5][5];
  invert5(5, R, L);
  /* 4.-5. */
  double cL[5], cR[5];
  for (int k = 0; k < 5; k++) {
    double ch[6];
    for (int m = 0; m < 6; m++) {
      double sum = 0.0;
      for (int vv = 0; vv < 5; vv++) sum += L[k][vv] * qs[m][vv];
      ch[m] = sum;
    }
    double l[5], r[5];
    for (int m = 0; m < 5; m++) l[m] = ch[m];
    for (int m = 0; m < 5; m++) r[m] = ch[5 - m];
    cL[k] = orc_weno5_left(l, 0);
    cR[k] = orc_weno5_left(r, 0);
  }
  /* 6. */
  double fl[5], fr[5];
  for (int vv = 0; vv < 5; vv++) {
    double sl = 0.0, sr = 0.0;
    for (int k = 0; k < 5; k++) {
      sl += R[vv][k] * cL[k];
      sr += R[vv][k] * cR[k];
    }
    fl[vv] = sl;
    fr[vv] = sr;
  }
  qL[0] = fl[0];
  qR[0] = fr[0];
  qL[4] = fl[4];
  qR[4] = fr[4];
  for (int d = 0; d < 3; d++) {
    qL[1 + comp[d]] = fl[1 + d];
    qR[1 + comp[d]] = fr[1 + d];
  }
}

int orc_charrec_face_pt(const orc_cfg* c, const double st[48], int a, double qL[8], double qR[8]) {
  double s6[6][8];
  for (int m = 0; m < 6; m++)
    for (int v = 0; v < 8; v++) s6[m][v] = st[8 * m + v];
  for (int v = 0; v < 8; v++) qL[v] = qR[v] = 0.0;
  char_rec_face(c, s6, a, qL, qR);
  return 0;
}

/* Face flux at face i+1/2 from the stencil st[m][v] = prims of cells i-2+m,
 * m = 0..5, v = 0..7; xf = face coordinates; a = axis.  Shared by both paths.
 * UCT (divb = 2, A37): bnorm -> the staggered sqrt(gamma) B^a of this face, whose
 * B^a = bnorm / sqrt(gamma_face) replaces both reconstructed normal components, and
 * fs (if not NULL) receives the face data of the EMF step (A38, A43): V^1..3 =
 * alpha v^i - beta^i of the left state, V^1..3 of the right state, a+ = S_R,
 * a- = -S_L of the HLL flux (A4).
 * Returns the A31 roughness flag of the face. */
static int face_flux(const orc_cfg* c, const double st[6][8], const double xf[3], int a, double F[8],
                     const double* bnorm, double fs[8]) {
  double qL[8], qR[8];
  for (int v = (c->rec == 6 ? 5 : 0); v < 8; v++) {  /* rec 6: B^i component-wise WENO5 (A44) */
    double l[5], r[5];
    for (int m = 0; m < 5; m++) l[m] = st[m][v];     /* cells i-2 .. i+2 */
    for (int m = 0; m < 5; m++) r[m] = st[5 - m][v]; /* cells i+3 .. i-1 (mirror) */
    qL[v] = orc_rec_left(l, c->rec == 6 ? 0 : c->rec);
    qR[v] = orc_rec_left(r, c->rec == 6 ? 0 : c->rec);
  }
  if (c->rec == 6) char_rec_face(c, st, a, qL, qR); /* the hydro states (A44) */
  /* A25 positivity fallback: a non-positive reconstructed rho or p takes the
   * value of the cell the state was reconstructed in */
  if (!(qL[0] > 0.0)) qL[0] = st[2][0];
  if (!(qL[4] > 0.0)) qL[4] = st[2][4];
  if (!(qR[0] > 0.0)) qR[0] = st[3][0];
  if (!(qR[4] > 0.0)) qR[4] = st[3][4];
  orc_met m;
  orc_met_eval(c, xf, &m);
  if (bnorm) qL[5 + a] = qR[5 + a] = *bnorm / m.sqrtg; /* b = sqrt(gamma) B at the face (A37) */
  orc_hll(&m, c->gamma, qL, qR, a, F);
  if (fs) {
    orc_aux al, ar;
    orc_aux_eval(&m, c->gamma, qL, &al);
    orc_aux_eval(&m, c->gamma, qR, &ar);
    double lmL, lpL, lmR, lpR;
    orc_speeds(&m, c->gamma, qL, a, &lmL, &lpL);
    orc_speeds(&m, c->gamma, qR, a, &lmR, &lpR);
    for (int i = 0; i < 3; i++) { /* A43: the transport velocity V^i = alpha v^i - beta^i */
      fs[i] = m.alpha * al.v[i] - m.beta[i];
      fs[3 + i] = m.alpha * ar.v[i] - m.beta[i];
    }
    fs[6] = fmax(0.0, fmax(lpL, lpR));   /* a+ = S_R */
    fs[7] = -fmin(0.0, fmin(lmL, lmR));  /* a- = -S_L */
  }
  return rough_face(c, st[2], st[3]);
}

/* prims (8) of an owned cell from the state arrays */
static void owned_prim(const orc_cfg* c, const double* U8, const double* P5, long long i, long long j,
                       long long k, double out[8]) {
  long long N = ncells(c), id = lin(c, i, j, k);
  double x[3] = {centre_of(c, 0, i), centre_of(c, 1, j), centre_of(c, 2, k)};
  orc_met m;
  orc_met_eval(c, x, &m);
  for (int q = 0; q < 5; q++) out[q] = P5[q * N + id];
  for (int q = 0; q < 3; q++) out[5 + q] = U8[(5 + q) * N + id] / m.sqrtg;
}

/* ------------------------------------------------------------------ */
/* Full-grid right-hand side                                           */
/* ------------------------------------------------------------------ */
typedef struct {
  long long N[3];
  double* a; /* [8][N2][N1][N0] */
} padded;

static double* pget(padded* p, int v, long long i, long long j, long long k) {
  return &p->a[(((long long)v * p->N[2] + (k + G)) * p->N[1] + (j + G)) * p->N[0] + (i + G)];
}

static void ghost_fill(const orc_cfg* c, padded* P) {
  int nt = nthreads_of(c);
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2];
  /* axis 0 ghosts on owned (j,k) */
#pragma omp parallel for num_threads(nt) schedule(static)
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = -G; i < n0 + G; i++) {
        if (i >= 0 && i < n0) continue;
        long long s = map_index(c, 0, i);
        for (int v = 0; v < 8; v++) *pget(P, v, i, j, k) = *pget(P, v, s, j, k);
      }
  /* axis 1 ghosts on every i (including axis-0 ghosts), owned k */
#pragma omp parallel for num_threads(nt) schedule(static)
  for (long long k = 0; k < n2; k++)
    for (long long j = -G; j < n1 + G; j++) {
      if (j >= 0 && j < n1) continue;
      long long s = map_index(c, 1, j);
      for (long long i = -G; i < n0 + G; i++)
        for (int v = 0; v < 8; v++) *pget(P, v, i, j, k) = *pget(P, v, i, s, k);
    }
  /* axis 2 ghosts everywhere */
#pragma omp parallel for num_threads(nt) schedule(static)
  for (long long k = -G; k < n2 + G; k++) {
    if (k >= 0 && k < n2) continue;
    long long s = map_index(c, 2, k);
    for (long long j = -G; j < n1 + G; j++)
      for (long long i = -G; i < n0 + G; i++)
        for (int v = 0; v < 8; v++) *pget(P, v, i, j, k) = *pget(P, v, i, j, s);
  }
}

/* Omega arrays padded by one cell per side */
typedef struct {
  long long N[3];
  double* a; /* [3][n2+2][n1+2][n0+2] */
} omega_t;
static double* oget(omega_t* o, int v, long long i, long long j, long long k) {
  return &o->a[(((long long)v * o->N[2] + (k + 1)) * o->N[1] + (j + 1)) * o->N[0] + (i + 1)];
}

/* accumulate the contribution of axis a at one cell: hydro rhs and Omega / B rhs.
 * Hp, Hm = DER fluxes at faces i+1/2 and i-1/2 of the cell. */
static void accumulate_axis(const orc_cfg* c, int a, const double Hp[8], const double Hm[8], double L[8],
                            double Om[3]) {
  double d = dx_of(c, a);
  for (int q = 0; q < 5; q++) L[q] = L[q] - (Hp[q] - Hm[q]) / d;
  int b1 = (a + 1) % 3, b2 = (a + 2) % 3;
  if (c->divb == 2) return; /* UCT: the field is updated from edge EMFs (uct_induction) */
  if (c->divb == 1) {
    L[5 + b1] = L[5 + b1] - (Hp[5 + b1] - Hm[5 + b1]) / d;
    L[5 + b2] = L[5 + b2] - (Hp[5 + b2] - Hm[5 + b2]) / d;
  } else {
    /* field-CD (A6): axis-a flux of B^{a+1} -> -1/4 into Omega_{a+2};
     *                axis-a flux of B^{a+2} -> +1/4 into Omega_{a+1} */
    Om[b2] = Om[b2] - 0.25 * (Hp[5 + b1] + Hm[5 + b1]);
    Om[b1] = Om[b1] + 0.25 * (Hp[5 + b2] + Hm[5 + b2]);
  }
}

static void add_sources(const orc_cfg* c, const double pr[8], const double x[3], double L[8]) {
  orc_met m;
  orc_metd d;
  orc_met_eval(c, x, &m);
  orc_met_deriv_eval(c, x, &d);
  double s[8];
  orc_sources(&m, &d, c->gamma, pr, s);
  for (int q = 1; q < 5; q++) L[q] = L[q] + m.sqrtg * s[q];
}

/* L(sqrt(gamma) B^i) = -(Om_k(j+1) - Om_k(j-1))/(2 D_j) + (Om_j(k+1) - Om_j(k-1))/(2 D_k),
 * (i,j,k) cyclic.  om(v, axis, +-1) returns Omega_v at the neighbour. */
static void curl_from(const orc_cfg* c, const double onb[3][3][2], double L[8]) {
  /* onb[v][axis][0:-1, 1:+1] */
  for (int i = 0; i < 3; i++) {
    int j = (i + 1) % 3, k = (i + 2) % 3;
    L[5 + i] = -(onb[k][j][1] - onb[k][j][0]) / (2.0 * dx_of(c, j))
             + (onb[j][k][1] - onb[j][k][0]) / (2.0 * dx_of(c, k));
  }
}

static void uct_emf_induction(const orc_cfg* c, const double* FS, const double* b3, double* L8);

/* L(U) on every owned cell; UCT (b3 != NULL): slots 5..7 receive L(b^a) at the faces */
static int rhs_full(const orc_cfg* c, const double* U8, const double* P5, const double* b3, double* L8) {
  if (c->rec == 6 && (c->metric != ORC_MINKOWSKI || c->divb == 2)) return -1; /* A44: flat, no UCT */
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2], N = ncells(c);
  int nt = nthreads_of(c);
  double* FS = NULL; /* UCT face data [axis][8][N] of the faces i_a + 1/2 owned by the cells */
  if (b3) {
    FS = (double*)malloc(sizeof(double) * 24 * N);
    if (!FS) return -3;
  }
  padded P;
  P.N[0] = n0 + 2 * G;
  P.N[1] = n1 + 2 * G;
  P.N[2] = n2 + 2 * G;
  P.a = (double*)malloc(sizeof(double) * 8 * P.N[0] * P.N[1] * P.N[2]);
  omega_t O;
  O.N[0] = n0 + 2;
  O.N[1] = n1 + 2;
  O.N[2] = n2 + 2;
  O.a = (double*)calloc((size_t)3 * O.N[0] * O.N[1] * O.N[2], sizeof(double));
  if (!P.a || !O.a) {
    free(P.a);
    free(O.a);
    free(FS);
    return -3;
  }
  /* 1. owned primitives, then ghosts */
#pragma omp parallel for num_threads(nt) schedule(static)
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        double pr[8];
        owned_prim(c, U8, P5, i, j, k, pr);
        for (int v = 0; v < 8; v++) *pget(&P, v, i, j, k) = pr[v];
      }
  ghost_fill(c, &P);
  for (long long q = 0; q < 8 * N; q++) L8[q] = 0.0;

  /* 2. axis sweeps, a = 0,1,2 in this order */
  for (int a = 0; a < 3; a++) {
    int t1 = (a + 1) % 3, t2 = (a + 2) % 3;
    long long na = c->n[a], nl = (long long)c->n[t1] * c->n[t2];
#pragma omp parallel for num_threads(nt) schedule(static)
    for (long long line = 0; line < nl; line++) {
      long long cell[3];
      cell[t1] = line % c->n[t1];
      cell[t2] = line / c->n[t1];
      double* F = (double*)malloc(sizeof(double) * 8 * (na + 5));
      int* rf = (int*)malloc(sizeof(int) * (na + 5));
      double* H = (double*)malloc(sizeof(double) * 8 * (na + 1));
      for (long long fi = -3; fi < na + 2; fi++) { /* face fi+1/2 */
        double st[6][8];
        for (int m = 0; m < 6; m++) {
          long long cc[3] = {cell[0], cell[1], cell[2]};
          cc[a] = fi - 2 + m;
          for (int v = 0; v < 8; v++) st[m][v] = *pget(&P, v, cc[0], cc[1], cc[2]);
        }
        double xf[3];
        xf[a] = face_of(c, a, fi);
        xf[t1] = centre_of(c, t1, cell[t1]);
        xf[t2] = centre_of(c, t2, cell[t2]);
        const double* bnorm = NULL;
        double* fs = NULL;
        if (b3) { /* the face fi+1/2 is owned by cell fi (wrapped) */
          long long cf[3] = {cell[0], cell[1], cell[2]};
          cf[a] = map_index(c, a, fi);
          const long long idf = lin(c, cf[0], cf[1], cf[2]);
          bnorm = &b3[a * N + idf];
          if (fi >= 0 && fi < na) fs = &FS[(a * 8) * N + idf]; /* stride N between the 8 entries */
        }
        double fsv[8];
        rf[fi + 3] = face_flux(c, st, xf, a, &F[8 * (fi + 3)], bnorm, fs ? fsv : NULL);
        if (fs)
          for (int m = 0; m < 8; m++) fs[m * N] = fsv[m];
      }
      for (long long hi = -1; hi < na; hi++) { /* DER flux at face hi+1/2 */
        double F5[5][8];
        int r5[5];
        for (int m = 0; m < 5; m++) {
          for (int q = 0; q < 8; q++) F5[m][q] = F[8 * (hi - 2 + m + 3) + q];
          r5[m] = rf[hi - 2 + m + 3];
        }
        der_face(c, F5, r5, &H[8 * (hi + 1)]);
      }
      for (long long i = 0; i < na; i++) {
        long long cc[3] = {cell[0], cell[1], cell[2]};
        cc[a] = i;
        long long id = lin(c, cc[0], cc[1], cc[2]);
        double L[8], Om[3];
        for (int q = 0; q < 8; q++) L[q] = L8[q * N + id];
        for (int q = 0; q < 3; q++) Om[q] = *oget(&O, q, cc[0], cc[1], cc[2]);
        accumulate_axis(c, a, &H[8 * (i + 1)], &H[8 * i], L, Om);
        for (int q = 0; q < 8; q++) L8[q * N + id] = L[q];
        for (int q = 0; q < 3; q++) *oget(&O, q, cc[0], cc[1], cc[2]) = Om[q];
      }
      free(F);
      free(rf);
      free(H);
    }
  }

  /* 3. metric sources at cell centres */
#pragma omp parallel for num_threads(nt) schedule(static)
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        long long id = lin(c, i, j, k);
        double x[3] = {centre_of(c, 0, i), centre_of(c, 1, j), centre_of(c, 2, k)};
        double pr[8], L[8];
        for (int v = 0; v < 8; v++) pr[v] = *pget(&P, v, i, j, k);
        for (int q = 0; q < 8; q++) L[q] = L8[q * N + id];
        add_sources(c, pr, x, L);
        for (int q = 0; q < 8; q++) L8[q * N + id] = L[q];
      }

  /* 4. UCT: edge EMFs and the staggered-field rhs; field-CD: curl with Omega ghosts
   *    filled by the same rule */
  if (b3) uct_emf_induction(c, FS, b3, L8);
  if (c->divb == 0) {
    for (long long k = -1; k <= n2; k++)
      for (long long j = -1; j <= n1; j++)
        for (long long i = -1; i <= n0; i++) {
          if (i >= 0 && i < n0 && j >= 0 && j < n1 && k >= 0 && k < n2) continue;
          long long si = map_index(c, 0, i), sj = map_index(c, 1, j), sk = map_index(c, 2, k);
          for (int v = 0; v < 3; v++) *oget(&O, v, i, j, k) = *oget(&O, v, si, sj, sk);
        }
#pragma omp parallel for num_threads(nt) schedule(static)
    for (long long k = 0; k < n2; k++)
      for (long long j = 0; j < n1; j++)
        for (long long i = 0; i < n0; i++) {
          long long id = lin(c, i, j, k);
          double onb[3][3][2];
          for (int v = 0; v < 3; v++) {
            onb[v][0][0] = *oget(&O, v, i - 1, j, k);
            onb[v][0][1] = *oget(&O, v, i + 1, j, k);
            onb[v][1][0] = *oget(&O, v, i, j - 1, k);
            onb[v][1][1] = *oget(&O, v, i, j + 1, k);
            onb[v][2][0] = *oget(&O, v, i, j, k - 1);
            onb[v][2][1] = *oget(&O, v, i, j, k + 1);
          }
          double L[8];
          for (int q = 0; q < 8; q++) L[q] = L8[q * N + id];
          curl_from(c, onb, L);
          for (int q = 0; q < 8; q++) L8[q * N + id] = L[q];
        }
  }
  free(P.a);
  free(O.a);
  free(FS);
  return 0;
}

int orc_rhs(const orc_cfg* c, const double* U8, const double* P5, double* L8) {
  if (c->divb == 2) return -1; /* UCT needs the staggered field: orc_rhs_uct */
  return rhs_full(c, U8, P5, NULL, L8);
}

/* ------------------------------------------------------------------ */
/* Per-cell path (index-mapped reads), for sampled parity at full size */
/* ------------------------------------------------------------------ */
static void prim_at(const orc_cfg* c, const double* U8, const double* P5, long long i, long long j, long long k,
                    double out[8]) {
  owned_prim(c, U8, P5, map_index(c, 0, i), map_index(c, 1, j), map_index(c, 2, k), out);
}

/* DER flux at face (cell[a])+1/2 of the line through cell */
static void hhat_at(const orc_cfg* c, const double* U8, const double* P5, int a, const long long cell[3],
                    double H[8]) {
  int t1 = (a + 1) % 3, t2 = (a + 2) % 3;
  double F[5][8];
  int r5[5];
  for (int f = 0; f < 5; f++) {
    long long fi = cell[a] - 2 + f;
    double st[6][8];
    for (int m = 0; m < 6; m++) {
      long long cc[3] = {cell[0], cell[1], cell[2]};
      cc[a] = fi - 2 + m;
      prim_at(c, U8, P5, cc[0], cc[1], cc[2], st[m]);
    }
    double xf[3];
    xf[a] = face_of(c, a, fi);
    xf[t1] = centre_of(c, t1, cell[t1]);
    xf[t2] = centre_of(c, t2, cell[t2]);
    r5[f] = face_flux(c, st, xf, a, F[f], NULL, NULL);
  }
  der_face(c, F, r5, H);
}

/* hydro/divb-none rhs and Omega of an owned cell, sweeps in axis order */
static void axes_at(const orc_cfg* c, const double* U8, const double* P5, const long long cell[3], double L[8],
                    double Om[3]) {
  for (int q = 0; q < 8; q++) L[q] = 0.0;
  for (int q = 0; q < 3; q++) Om[q] = 0.0;
  for (int a = 0; a < 3; a++) {
    double Hp[8], Hm[8];
    long long cm[3] = {cell[0], cell[1], cell[2]};
    cm[a] -= 1;
    hhat_at(c, U8, P5, a, cell, Hp);
    hhat_at(c, U8, P5, a, cm, Hm);
    accumulate_axis(c, a, Hp, Hm, L, Om);
  }
}

static void rhs_cell(const orc_cfg* c, const double* U8, const double* P5, const long long cell[3], double L[8]) {
  double Om[3];
  axes_at(c, U8, P5, cell, L, Om);
  double pr[8];
  owned_prim(c, U8, P5, cell[0], cell[1], cell[2], pr);
  double x[3] = {centre_of(c, 0, cell[0]), centre_of(c, 1, cell[1]), centre_of(c, 2, cell[2])};
  add_sources(c, pr, x, L);
  if (c->divb == 0) {
    double onb[3][3][2];
    for (int ax = 0; ax < 3; ax++)
      for (int s = 0; s < 2; s++) {
        long long nb[3] = {cell[0], cell[1], cell[2]};
        nb[ax] += s ? 1 : -1;
        for (int b = 0; b < 3; b++) nb[b] = map_index(c, b, nb[b]);
        double Ld[8], Omn[3];
        axes_at(c, U8, P5, nb, Ld, Omn);
        for (int v = 0; v < 3; v++) onb[v][ax][s] = Omn[v];
      }
    curl_from(c, onb, L);
  }
}

int orc_rhs_cells(const orc_cfg* c, const double* U8, const double* P5, long long ncell, const long long* idx,
                  double* out) {
  if (c->divb == 2) return -1; /* UCT: full-grid path only */
  if (c->rec == 6 && c->metric != ORC_MINKOWSKI) return -1; /* A44: flat metric only */
  int nt = nthreads_of(c);
#pragma omp parallel for num_threads(nt) schedule(dynamic)
  for (long long m = 0; m < ncell; m++) rhs_cell(c, U8, P5, &idx[3 * m], &out[8 * m]);
  return 0;
}

/* ------------------------------------------------------------------ */
/* RK stage (A7) + con2prim/floors (A8, A9)                            */
/* ------------------------------------------------------------------ */
static void combine(int s, double dt, const double Un[8], const double Us[8], const double L[8], double Uo[8]) {
  for (int q = 0; q < 8; q++) {
    if (s == 1)
      Uo[q] = Un[q] + dt * L[q];
    else if (s == 2)
      Uo[q] = 0.75 * Un[q] + 0.25 * (Us[q] + dt * L[q]);
    else
      Uo[q] = (1.0 / 3.0) * Un[q] + (2.0 / 3.0) * (Us[q] + dt * L[q]);
  }
}

static void update_cell(const orc_cfg* c, int s, double dt, const double* Un, const double* Us, const double* Ps,
                        long long i, long long j, long long k, const double L[8], double Uo[8], double Po[5],
                        long long* nfl, long long* nfa) {
  long long N = ncells(c), id = lin(c, i, j, k);
  double un[8], us[8], pp[5];
  for (int q = 0; q < 8; q++) {
    un[q] = Un[q * N + id];
    us[q] = Us[q * N + id];
  }
  for (int q = 0; q < 5; q++) pp[q] = Ps[q * N + id];
  combine(s, dt, un, us, L, Uo);
  double x[3] = {centre_of(c, 0, i), centre_of(c, 1, j), centre_of(c, 2, k)};
  orc_met m;
  orc_met_eval(c, x, &m);
  orc_c2p_floors(c, &m, Uo, pp, Po, nfl, nfa);
}

int orc_stage(const orc_cfg* c, int s, double dt, const double* Un, const double* Us, const double* Ps,
              double* Uout, double* Pout, orc_counts* cnt) {
  long long N = ncells(c);
  double* L8 = (double*)malloc(sizeof(double) * 8 * N);
  if (!L8) return -3;
  int rc = orc_rhs(c, Us, Ps, L8);
  if (rc) {
    free(L8);
    return rc;
  }
  long long nfl = 0, nfa = 0;
  int nt = nthreads_of(c);
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2];
#pragma omp parallel for num_threads(nt) schedule(static) reduction(+ : nfl, nfa)
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        long long id = lin(c, i, j, k);
        double L[8], Uo[8], Po[5];
        for (int q = 0; q < 8; q++) L[q] = L8[q * N + id];
        update_cell(c, s, dt, Un, Us, Ps, i, j, k, L, Uo, Po, &nfl, &nfa);
        for (int q = 0; q < 8; q++) Uout[q * N + id] = Uo[q];
        for (int q = 0; q < 5; q++) Pout[q * N + id] = Po[q];
      }
  free(L8);
  if (cnt) {
    cnt->floor_events += nfl;
    cnt->c2p_failures += nfa;
  }
  return 0;
}

int orc_stage_cells(const orc_cfg* c, int s, double dt, const double* Un, const double* Us, const double* Ps,
                    long long ncell, const long long* idx, double* Uout, double* Pout, orc_counts* cnt) {
  if (c->divb == 2) return -1; /* UCT: full-grid path only */
  if (c->rec == 6 && c->metric != ORC_MINKOWSKI) return -1; /* A44: flat metric only */
  long long nfl = 0, nfa = 0;
  int nt = nthreads_of(c);
#pragma omp parallel for num_threads(nt) schedule(dynamic) reduction(+ : nfl, nfa)
  for (long long m = 0; m < ncell; m++) {
    double L[8];
    rhs_cell(c, Us, Ps, &idx[3 * m], L);
    update_cell(c, s, dt, Un, Us, Ps, idx[3 * m], idx[3 * m + 1], idx[3 * m + 2], L, &Uout[8 * m],
                &Pout[5 * m], &nfl, &nfa);
  }
  if (cnt) {
    cnt->floor_events += nfl;
    cnt->c2p_failures += nfa;
  }
  return 0;
}

int orc_step(const orc_cfg* c, double dt, double* U8, double* P5, orc_counts* cnt) {
  long long N = ncells(c);
  double* U1 = (double*)malloc(sizeof(double) * 8 * N);
  double* P1 = (double*)malloc(sizeof(double) * 5 * N);
  double* U2 = (double*)malloc(sizeof(double) * 8 * N);
  double* P2 = (double*)malloc(sizeof(double) * 5 * N);
  if (!U1 || !P1 || !U2 || !P2) {
    free(U1);
    free(P1);
    free(U2);
    free(P2);
    return -3;
  }
  int rc = orc_stage(c, 1, dt, U8, U8, P5, U1, P1, cnt);
  if (!rc) rc = orc_stage(c, 2, dt, U8, U1, P1, U2, P2, cnt);
  if (!rc) rc = orc_stage(c, 3, dt, U8, U2, P2, U8, P5, cnt);
  free(U1);
  free(P1);
  free(U2);
  free(P2);
  return rc;
}

/* ------------------------------------------------------------------ */
/* CFL (SPEC.md:163 form, A11), con2prim, div B, set/get               */
/* ------------------------------------------------------------------ */
int orc_max_dt(const orc_cfg* c, const double* U8, const double* P5, double cfl, double* dt) {
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2];
  int nt = nthreads_of(c);
  double mx = 0.0;
#pragma omp parallel for num_threads(nt) schedule(static) reduction(max : mx)
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        double pr[8];
        owned_prim(c, U8, P5, i, j, k, pr);
        double x[3] = {centre_of(c, 0, i), centre_of(c, 1, j), centre_of(c, 2, k)};
        orc_met m;
        orc_met_eval(c, x, &m);
        double sum = 0.0;
        for (int a = 0; a < 3; a++) {
          double lm, lp;
          orc_speeds(&m, c->gamma, pr, a, &lm, &lp);
          sum += fmax(fabs(lp), fabs(lm)) / dx_of(c, a);
        }
        if (sum > mx) mx = sum;
      }
  if (!(mx > 0.0)) return -1;
  *dt = cfl / mx;
  return 0;
}

int orc_con2prim(const orc_cfg* c, double* U8, double* P5, orc_counts* cnt) {
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2], N = ncells(c);
  int nt = nthreads_of(c);
  long long nfl = 0, nfa = 0;
#pragma omp parallel for num_threads(nt) schedule(static) reduction(+ : nfl, nfa)
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        long long id = lin(c, i, j, k);
        double x[3] = {centre_of(c, 0, i), centre_of(c, 1, j), centre_of(c, 2, k)};
        orc_met m;
        orc_met_eval(c, x, &m);
        double Uc[8], pp[5], po[5];
        for (int q = 0; q < 8; q++) Uc[q] = U8[q * N + id];
        for (int q = 0; q < 5; q++) pp[q] = P5[q * N + id];
        orc_c2p_floors(c, &m, Uc, pp, po, &nfl, &nfa);
        for (int q = 0; q < 8; q++) U8[q * N + id] = Uc[q];
        for (int q = 0; q < 5; q++) P5[q * N + id] = po[q];
      }
  if (cnt) {
    cnt->floor_events += nfl;
    cnt->c2p_failures += nfa;
  }
  return 0;
}

double orc_divb(const orc_cfg* c, const double* U8) {
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2], N = ncells(c);
  double mx = 0.0;
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        long long ci[3] = {i, j, k};
        double div = 0.0;
        for (int a = 0; a < 3; a++) {
          long long p[3] = {i, j, k}, m[3] = {i, j, k};
          p[a] = map_index(c, a, ci[a] + 1);
          m[a] = map_index(c, a, ci[a] - 1);
          div += (U8[(5 + a) * N + lin(c, p[0], p[1], p[2])] - U8[(5 + a) * N + lin(c, m[0], m[1], m[2])])
               / (2.0 * dx_of(c, a));
        }
        if (fabs(div) > mx) mx = fabs(div);
      }
  return mx;
}

int orc_set_prims(const orc_cfg* c, const double* P8, double* U8, double* P5, long long* bad) {
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2], N = ncells(c);
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        long long id = lin(c, i, j, k);
        double x[3] = {centre_of(c, 0, i), centre_of(c, 1, j), centre_of(c, 2, k)};
        orc_met m;
        orc_met_eval(c, x, &m);
        double v[3] = {P8[1 * N + id], P8[2 * N + id], P8[3 * N + id]};
        double v2 = 0.0;
        for (int a = 0; a < 3; a++)
          for (int b = 0; b < 3; b++) v2 += m.g[a][b] * v[a] * v[b];
        double rho = P8[0 * N + id], p = P8[4 * N + id];
        if (!(rho > 0.0) || !(p > 0.0) || !(v2 < 1.0)) {
          if (bad) *bad = id;
          return -5;
        }
        double W = 1.0 / sqrt(1.0 - v2);
        double pr[8] = {rho, W * v[0], W * v[1], W * v[2], p, P8[5 * N + id], P8[6 * N + id], P8[7 * N + id]};
        double u[8];
        orc_p2c(&m, c->gamma, pr, u);
        for (int q = 0; q < 8; q++) U8[q * N + id] = m.sqrtg * u[q];
        for (int q = 0; q < 5; q++) P5[q * N + id] = pr[q];
      }
  return 0;
}

int orc_get_prims(const orc_cfg* c, const double* U8, const double* P5, double* P8) {
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2], N = ncells(c);
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        long long id = lin(c, i, j, k);
        double pr[8];
        owned_prim(c, U8, P5, i, j, k, pr);
        double x[3] = {centre_of(c, 0, i), centre_of(c, 1, j), centre_of(c, 2, k)};
        orc_met m;
        orc_met_eval(c, x, &m);
        double u2 = 0.0;
        for (int a = 0; a < 3; a++)
          for (int b = 0; b < 3; b++) u2 += m.g[a][b] * pr[1 + a] * pr[1 + b];
        double W = sqrt(1.0 + u2);
        P8[0 * N + id] = pr[0];
        for (int a = 0; a < 3; a++) P8[(1 + a) * N + id] = pr[1 + a] / W;
        P8[4 * N + id] = pr[4];
        for (int a = 0; a < 3; a++) P8[(5 + a) * N + id] = pr[5 + a];
      }
  return 0;
}

/* ------------------------------------------------------------------ */
/* UCT: staggered field + upwind constrained transport (divb = 2;      */
/* SURVEY.md §8(f) f2; readings A37-A43).  Periodic or     */
/* outflow axes, any metric.  b3[a][N]: sqrt(gamma) B^a at the face i_a + 1/2     */
/* owned by cell i (x1 fastest); E3[c][N]: EMF E^c at the edge         */
/* (i_p + 1/2, i_q + 1/2, i_c) owned by cell i, (c, p, q) cyclic.      */
/* ------------------------------------------------------------------ */
/* linear index of cell x + d e_a with every index wrapped (A13) */
static long long lin_shift(const orc_cfg* c, const long long x[3], int a, long long d) {
  long long y[3] = {x[0], x[1], x[2]};
  y[a] += d;
  return lin(c, map_index(c, 0, y[0]), map_index(c, 1, y[1]), map_index(c, 2, y[2]));
}

/* A38: the two one-sided values at position +1/2 from samples f[0..5] at -2..3
 * (lo from f[0..4], hi the mirror from f[5..1]), with the configured REC */
static void rec_pair(const orc_cfg* c, const double f[6], double* lo, double* hi) {
  double l[5], r[5];
  for (int m = 0; m < 5; m++) l[m] = f[m];
  for (int m = 0; m < 5; m++) r[m] = f[5 - m];
  *lo = orc_rec_left(l, c->rec);
  *hi = orc_rec_left(r, c->rec);
}

/* A39: UCT-HLL EMF E^cc at the edge owned by cell x.  p = cc+1, q = cc+2; W/E =
 * left/right along p, S/N = left/right along q.  E^cc = V^q b^p - V^p b^q (A43: V =
 * alpha v - beta, b = sqrt(gamma) B), the densitised flux along q of b^p and minus the
 * flux along p of b^q. */
static double uct_emf(const orc_cfg* c, const double* FS, const double* b3, int cc, const long long x[3]) {
  const long long N = ncells(c);
  const int p = (cc + 1) % 3, q = (cc + 2) % 3;
  const int comp[2] = {p, q};
  double f[6];
  /* p-face states (W = left, E = right) reconstructed along q: pS[side][k], pN[side][k] */
  double pS[2][2], pN[2][2];
  for (int side = 0; side < 2; side++)
    for (int k = 0; k < 2; k++) {
      for (int m = 0; m < 6; m++) f[m] = FS[(p * 8 + 3 * side + comp[k]) * N + lin_shift(c, x, q, m - 2)];
      rec_pair(c, f, &pS[side][k], &pN[side][k]);
    }
  /* q-face states (S = left, N = right) reconstructed along p: qW[side][k], qE[side][k] */
  double qW[2][2], qE[2][2];
  for (int side = 0; side < 2; side++)
    for (int k = 0; k < 2; k++) {
      for (int m = 0; m < 6; m++) f[m] = FS[(q * 8 + 3 * side + comp[k]) * N + lin_shift(c, x, p, m - 2)];
      rec_pair(c, f, &qW[side][k], &qE[side][k]);
    }
  /* staggered B^p along q, B^q along p */
  double bpS, bpN, bqW, bqE;
  for (int m = 0; m < 6; m++) f[m] = b3[p * N + lin_shift(c, x, q, m - 2)];
  rec_pair(c, f, &bpS, &bpN);
  for (int m = 0; m < 6; m++) f[m] = b3[q * N + lin_shift(c, x, p, m - 2)];
  rec_pair(c, f, &bqW, &bqE);
  /* A40: edge speeds = max over the two faces meeting at the edge */
  const long long id = lin(c, x[0], x[1], x[2]);
  const double app = fmax(FS[(p * 8 + 6) * N + id], FS[(p * 8 + 6) * N + lin_shift(c, x, q, 1)]);
  const double apm = fmax(FS[(p * 8 + 7) * N + id], FS[(p * 8 + 7) * N + lin_shift(c, x, q, 1)]);
  const double aqp = fmax(FS[(q * 8 + 6) * N + id], FS[(q * 8 + 6) * N + lin_shift(c, x, p, 1)]);
  const double aqm = fmax(FS[(q * 8 + 7) * N + id], FS[(q * 8 + 7) * N + lin_shift(c, x, p, 1)]);
  /* A38: quadrant velocities (v^p, v^q) = mean of the two double reconstructions */
  double vWS[2], vWN[2], vES[2], vEN[2];
  for (int k = 0; k < 2; k++) {
    vWS[k] = 0.5 * (pS[0][k] + qW[0][k]);
    vWN[k] = 0.5 * (pN[0][k] + qW[1][k]);
    vES[k] = 0.5 * (pS[1][k] + qE[0][k]);
    vEN[k] = 0.5 * (pN[1][k] + qE[1][k]);
  }
  const double EWS = vWS[1] * bpS - vWS[0] * bqW;
  const double EWN = vWN[1] * bpN - vWN[0] * bqW;
  const double EES = vES[1] * bpS - vES[0] * bqE;
  const double EEN = vEN[1] * bpN - vEN[0] * bqE;
  const double sp = app + apm, sq = aqp + aqm;
  if (!(sp > 0.0) || !(sq > 0.0)) /* unreachable for p > 0 (A4): central average */
    return 0.25 * (EWS + EWN + EES + EEN);
  return (app * aqp * EWS + app * aqm * EWN + apm * aqp * EES + apm * aqm * EEN) / (sp * sq)
       + app * apm * (bqE - bqW) / sp - aqp * aqm * (bpN - bpS) / sq;
}

/* A41: L(b^p) = -(Dh_q E^cc(+1/2) - Dh_q E^cc(-1/2)) / Delta_q
 *              + (Dh_cc E^q(+1/2) - Dh_cc E^q(-1/2)) / Delta_cc,  cc = p-1, q = p+1,
 * Dh_a = the DER operator along a (A5, never switched off by A31) */
static void uct_emf_induction(const orc_cfg* c, const double* FS, const double* b3, double* L8) {
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2], N = ncells(c);
  int nt = nthreads_of(c);
  double* E3 = (double*)malloc(sizeof(double) * 3 * N);
  if (!E3) return;
#pragma omp parallel for num_threads(nt) schedule(static)
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        const long long x[3] = {i, j, k};
        for (int cc = 0; cc < 3; cc++) E3[cc * N + lin(c, i, j, k)] = uct_emf(c, FS, b3, cc, x);
      }
#pragma omp parallel for num_threads(nt) schedule(static)
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        const long long x[3] = {i, j, k};
        for (int p = 0; p < 3; p++) {
          const int cc = (p + 2) % 3, q = (p + 1) % 3;
          double Ep[5], Em[5], Gp[5], Gm[5];
          for (int m = 0; m < 5; m++) {
            Ep[m] = E3[cc * N + lin_shift(c, x, q, m - 2)];
            Em[m] = E3[cc * N + lin_shift(c, x, q, m - 3)];
            Gp[m] = E3[q * N + lin_shift(c, x, cc, m - 2)];
            Gm[m] = E3[q * N + lin_shift(c, x, cc, m - 3)];
          }
          L8[(5 + p) * N + lin(c, i, j, k)] = -(orc_der(Ep, c->der) - orc_der(Em, c->der)) / dx_of(c, q)
                                            + (orc_der(Gp, c->der) - orc_der(Gm, c->der)) / dx_of(c, cc);
        }
      }
  free(E3);
}

/* UCT scope (A37): any metric; periodic or outflow axes.  On an outflow side every
 * staggered quantity (b, the face data, the EMFs) takes the ghost rule of A13 through
 * lin_shift: the nearest owned face / edge (zero gradient). */
static int uct_ok(const orc_cfg* c) { return c->divb == 2; }

/* A37: cell-centred field from the staggered one, 6-point midpoint interpolation
 * B^a(i) = (3 b_{i-5/2} - 25 b_{i-3/2} + 150 b_{i-1/2} + 150 b_{i+1/2} - 25 b_{i+3/2} + 3 b_{i+5/2}) / 256 */
int orc_uct_centre(const orc_cfg* c, const double* b3, double* Bc3) {
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2], N = ncells(c);
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        const long long x[3] = {i, j, k};
        for (int a = 0; a < 3; a++) {
          double f[6];
          for (int m = 0; m < 6; m++) f[m] = b3[a * N + lin_shift(c, x, a, m - 3)];
          Bc3[a * N + lin(c, i, j, k)] =
              (3.0 * f[0] - 25.0 * f[1] + 150.0 * f[2] + 150.0 * f[3] - 25.0 * f[4] + 3.0 * f[5]) / 256.0;
        }
      }
  return 0;
}

/* the divergence UCT preserves (A41): sum_a (Dh_a b^a(+1/2) - Dh_a b^a(-1/2)) / Delta_a */
int orc_uct_divh(const orc_cfg* c, const double* b3, double* out) {
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2], N = ncells(c);
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        const long long x[3] = {i, j, k};
        double d = 0.0;
        for (int a = 0; a < 3; a++) {
          double fp[5], fm[5];
          for (int m = 0; m < 5; m++) {
            fp[m] = b3[a * N + lin_shift(c, x, a, m - 2)];
            fm[m] = b3[a * N + lin_shift(c, x, a, m - 3)];
          }
          d += (orc_der(fp, c->der) - orc_der(fm, c->der)) / dx_of(c, a);
        }
        out[lin(c, i, j, k)] = d;
      }
  return 0;
}

/* state of a UCT run: the hydro prims of P8 and b3; B = I6(b3) / sqrt(gamma) at the centres */
int orc_set_prims_uct(const orc_cfg* c, const double* P8, const double* b3, double* U8, double* P5, long long* bad) {
  if (!uct_ok(c)) return -1;
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2], N = ncells(c);
  double* Q = (double*)malloc(sizeof(double) * 8 * N);
  double* Bc = (double*)malloc(sizeof(double) * 3 * N);
  if (!Q || !Bc) {
    free(Q);
    free(Bc);
    return -3;
  }
  memcpy(Q, P8, sizeof(double) * 5 * N);
  orc_uct_centre(c, b3, Bc);
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        const long long id = lin(c, i, j, k);
        double x[3] = {centre_of(c, 0, i), centre_of(c, 1, j), centre_of(c, 2, k)};
        orc_met m;
        orc_met_eval(c, x, &m);
        for (int a = 0; a < 3; a++) Q[(5 + a) * N + id] = Bc[a * N + id] / m.sqrtg;
      }
  int rc = orc_set_prims(c, Q, U8, P5, bad);
  /* U_B exactly I6(b) (the division and re-densitisation above may round) */
  if (!rc)
    for (long long e = 0; e < 3 * N; e++) U8[5 * N + e] = Bc[e];
  free(Q);
  free(Bc);
  return rc;
}

int orc_rhs_uct(const orc_cfg* c, const double* U8, const double* P5, const double* b3, double* L8) {
  if (!uct_ok(c)) return -1;
  return rhs_full(c, U8, P5, b3, L8);
}

int orc_stage_uct(const orc_cfg* c, int s, double dt, const double* Un, const double* Us, const double* Ps,
                  const double* bn, const double* bs, double* Uout, double* Pout, double* bout, orc_counts* cnt) {
  if (!uct_ok(c)) return -1;
  const long long N = ncells(c);
  double* L8 = (double*)malloc(sizeof(double) * 8 * N);
  double* Bc = (double*)malloc(sizeof(double) * 3 * N);
  if (!L8 || !Bc) {
    free(L8);
    free(Bc);
    return -3;
  }
  int rc = rhs_full(c, Us, Ps, bs, L8);
  if (rc) {
    free(L8);
    free(Bc);
    return rc;
  }
  /* the staggered field: literal RK forms (A7) per face */
  for (long long e = 0; e < 3 * N; e++) {
    const double Lb = L8[5 * N + e];
    if (s == 1)
      bout[e] = bn[e] + dt * Lb;
    else if (s == 2)
      bout[e] = 0.75 * bn[e] + 0.25 * (bs[e] + dt * Lb);
    else
      bout[e] = (1.0 / 3.0) * bn[e] + (2.0 / 3.0) * (bs[e] + dt * Lb);
  }
  orc_uct_centre(c, bout, Bc);
  long long nfl = 0, nfa = 0;
  int nt = nthreads_of(c);
  const long long n0 = c->n[0], n1 = c->n[1], n2 = c->n[2];
#pragma omp parallel for num_threads(nt) schedule(static) reduction(+ : nfl, nfa)
  for (long long k = 0; k < n2; k++)
    for (long long j = 0; j < n1; j++)
      for (long long i = 0; i < n0; i++) {
        const long long id = lin(c, i, j, k);
        double un[8], us[8], L[8], Uo[8], pp[5], Po[5];
        for (int q = 0; q < 8; q++) {
          un[q] = Un[q * N + id];
          us[q] = Us[q * N + id];
          L[q] = L8[q * N + id];
        }
        for (int q = 0; q < 5; q++) pp[q] = Ps[q * N + id];
        combine(s, dt, un, us, L, Uo);
        for (int a = 0; a < 3; a++) Uo[5 + a] = Bc[a * N + id]; /* A37: U_B = I6(b) */
        double x[3] = {centre_of(c, 0, i), centre_of(c, 1, j), centre_of(c, 2, k)};
        orc_met m;
        orc_met_eval(c, x, &m);
        orc_c2p_floors(c, &m, Uo, pp, Po, &nfl, &nfa);
        for (int q = 0; q < 8; q++) Uout[q * N + id] = Uo[q];
        for (int q = 0; q < 5; q++) Pout[q * N + id] = Po[q];
      }
  free(L8);
  free(Bc);
  if (cnt) {
    cnt->floor_events += nfl;
    cnt->c2p_failures += nfa;
  }
  return 0;
}

int orc_step_uct(const orc_cfg* c, double dt, double* U8, double* P5, double* b3, orc_counts* cnt) {
  if (!uct_ok(c)) return -1;
  const long long N = ncells(c);
  double* U1 = (double*)malloc(sizeof(double) * 8 * N);
  double* P1 = (double*)malloc(sizeof(double) * 5 * N);
  double* b1 = (double*)malloc(sizeof(double) * 3 * N);
  double* U2 = (double*)malloc(sizeof(double) * 8 * N);
  double* P2 = (double*)malloc(sizeof(double) * 5 * N);
  double* b2 = (double*)malloc(sizeof(double) * 3 * N);
  int rc = -3;
  if (U1 && P1 && b1 && U2 && P2 && b2) {
    rc = orc_stage_uct(c, 1, dt, U8, U8, P5, b3, b3, U1, P1, b1, cnt);
    if (!rc) rc = orc_stage_uct(c, 2, dt, U8, U1, P1, b3, b1, U2, P2, b2, cnt);
    if (!rc) rc = orc_stage_uct(c, 3, dt, U8, U2, P2, b3, b2, U8, P5, b3, cnt);
  }
  free(U1);
  free(P1);
  free(b1);
  free(U2);
  free(P2);
  free(b2);
  return rc;
}
