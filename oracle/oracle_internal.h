/* oracle_internal.h — ORACLE (test infrastructure only; see oracle.h). */
#ifndef ECHO_ORACLE_INTERNAL_H
#define ECHO_ORACLE_INTERNAL_H
#include "oracle.h"

typedef struct {
  double alpha, beta[3], g[3][3], gi[3][3], sqrtg;
} orc_met;

typedef struct {
  double dalpha[3], dbeta[3][3] /* [k][i] = d_k beta^i */, dg[3][3][3] /* [k][i][j] */;
} orc_metd;

/* every derived quantity of one primitive state in one metric (DESIGN A1) */
typedef struct {
  double W, v[3], vl[3], v2;    /* Lorentz factor, v^i, v_i, v^2 */
  double Bl[3], B2, vB;         /* B_i, B^2, v.B */
  double h, Z;                  /* specific enthalpy, Z = rho h W^2 */
  double D, S[3], Su[3], tau, U;/* D, S_i, S^i, tau, U = tau + D */
  double E[3], E2;              /* E^i = -eps^{ijk} v_j B_k, E^2 = B^2 v^2 - (v.B)^2 */
  double Wst[3][3];             /* stress W^{ij} */
} orc_aux;

void orc_met_eval(const orc_cfg* c, const double x[3], orc_met* m);
void orc_met_deriv_eval(const orc_cfg* c, const double x[3], orc_metd* d);

void orc_aux_eval(const orc_met* m, double gam, const double pr[8], orc_aux* q);
void orc_p2c(const orc_met* m, double gam, const double pr[8], double u[8]);
void orc_flux(const orc_met* m, double gam, const double pr[8], int dir, double f[8]);
void orc_speeds(const orc_met* m, double gam, const double pr[8], int dir, double* lm, double* lp);
void orc_hll(const orc_met* m, double gam, const double pl[8], const double prr[8], int dir, double F[8]);
void orc_sources(const orc_met* m, const orc_metd* d, double gam, const double pr[8], double s[8]);
int orc_c2p(const orc_cfg* c, const orc_met* m, const double u[8], const double guess[8],
            double pr_out[8], int* iters);
/* con2prim + floors of A9 applied to the densitised cons of one cell.
 * Ucell (8, densitised) may be rewritten; P5 prev in, P5 out.  Adds to cnt. */
void orc_c2p_floors(const orc_cfg* c, const orc_met* m, double Ucell[8], const double Pprev[5],
                    double Pout[5], long long* nfloor, long long* nfail);

#endif
