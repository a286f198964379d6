/*
 * oracle.h — CPU fp64 ORACLE for the ECHO-3DHPC time-step hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this code.
 * The product path (paper_1810_04597_b200/) never imports, links or executes
 * anything under oracle/, and this code shares no source, header, table or
 * helper with it.
 *
 * What it computes: one SSP-RK3 step of the 3+1 ideal-GRMHD finite-difference
 * scheme named by BASELINE.json:north_star — ghost fill, WENO5 reconstruction
 * of primitives, fast-speed bound + HLL flux, DER flux derivative, metric
 * sources, field-CD divergence-preserving B update (or, divb = 2, the staggered
 * field with upwind constrained transport, A37-A41), RK stage combine, per-cell
 * Newton con2prim with floors, CFL reduction.  The paper (PAPER.md:19,
 * "solve the equations of magneto-hydrodynamic in General Relativity, using
 * 3D finite-differences method and high-order reconstruction algorithms")
 * names the method but writes no formula; every formula here follows the
 * readings A1-A25 listed in DESIGN.md §3 (SURVEY.md §8(c) plus our additions).
 * Plain loops, fp64, compiled with -O2 -ffp-contract=off (no fast-math,
 * SPEC.md:191), OpenMP only over independent lines/cells so results are
 * bitwise independent of the thread count.
 *
 * Layouts (same as the public C-ABI, x1 fastest, no ghosts, row-major
 * [var][n3][n2][n1]):
 *   user prims  P8 : rho, v^1, v^2, v^3, p, B^1, B^2, B^3   (v contravariant)
 *   state prims P5 : rho, u~^1, u~^2, u~^3, p               (u~ = W v)
 *   conserved   U8 : sqrt(gamma) * (D, S_1, S_2, S_3, tau, B^1, B^2, B^3)
 * Parity status of every function: see DESIGN.md §4 (every function pinned; the
 * multi-dimensional blast / torus evolutions have no closed form and are covered
 * by the pins of their parts, 1-D exact relativistic Riemann solutions and the
 * torus-equilibrium convergence).
 */
#ifndef ECHO_ORACLE_H
#define ECHO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_NVAR = 8, ORC_NPRIM = 5, ORC_G = 5 };
enum { ORC_BC_PERIODIC = 0, ORC_BC_OUTFLOW = 1 };
enum { ORC_MINKOWSKI = 0, ORC_KERR_SCHILD = 1 };

typedef struct {
  int n[3];          /* owned cells per axis */
  double lo[3];      /* coordinate of the lower domain edge per axis */
  double hi[3];      /* coordinate of the upper domain edge per axis */
  int bc[3][2];      /* [axis][lower/upper] ORC_BC_* */
  int metric;        /* ORC_MINKOWSKI: Cartesian (x,y,z); ORC_KERR_SCHILD: (ln r, theta, phi) */
  double M, a;       /* black-hole mass and spin (KS only) */
  double gamma;      /* adiabatic index Gamma */
  double rho_floor, p_floor, w_max;
  int c2p_max_iter;  /* Newton cap (A8: 30) */
  double c2p_tol;    /* Newton tolerance on |dZ|/Z (A8: 1e-13) */
  int rec;           /* 0 WENO5 point-value form (A2), 1 WENO5 finite-volume form,
                        2 MP5 (Suresh & Huynh 1997, point values, A33),
                        3 WENO-Z (Borges et al. 2008, point values, A34),
                        4 MC2 (monotonized-central limited linear, A35),
                        5 PPM (Colella & Woodward 1984 on point values, A36),
                        6 characteristic-wise WENO5 of the hydro primitives (eigenvectors of
                          the flat-space relativistic-Euler Jacobian at the face, A44; B^i
                          component-wise; Minkowski only, not with divb = 2) */
  int der;           /* 6 DER6, 4 DER4, 2 plain difference (A5) */
  int divb;          /* 0 field-CD (A6), 1 none: plain flux difference for B,
                        2 UCT: staggered field + upwind constrained transport (A37-A41;
                        periodic or outflow axes (A42), any metric (A43);
                        the *_uct entry points) */
  double der_jump;   /* A31 DER switch: the DER correction at a face is dropped (H = F) when a face
                        of its 5-face stencil joins cells whose rho or p differ by more than
                        der_jump x the smaller value; <= 0 disables the switch */
  int nthreads;      /* OpenMP threads (<=0: library default) */
} orc_cfg;

typedef struct { long long floor_events, c2p_failures; } orc_counts;

/* ---------------- point-wise pieces (exposed for the pin tests) --------- */
/* metric at coordinates x: out[0]=alpha, out[1..3]=beta^i, out[4..12]=gamma_ij,
 * out[13..21]=gamma^ij, out[22]=sqrt(gamma).  Returns 0. */
int orc_metric(const orc_cfg* c, const double x[3], double out[23]);
/* coordinate derivatives at x: out[0..2]=d_k alpha, out[3+3k+i]=d_k beta^i,
 * out[12+9k+3i+j]=d_k gamma_ij.  Analytic (hand-derived) for KS. */
int orc_metric_deriv(const orc_cfg* c, const double x[3], double out[39]);
/* prims (rho,u~^i,p,B^i) -> non-densitised cons (D,S_i,tau,B^i) at x */
int orc_prim2cons_pt(const orc_cfg* c, const double x[3], const double pr[8], double u[8]);
/* non-densitised physical flux along axis dir (0,1,2) */
int orc_flux_pt(const orc_cfg* c, const double x[3], const double pr[8], int dir, double f[8]);
/* fast-speed bound lam[0]=lambda-, lam[1]=lambda+ along dir (A4) */
int orc_speeds_pt(const orc_cfg* c, const double x[3], const double pr[8], int dir, double lam[2]);
/* densitised HLL flux at a face located at x between states L and R */
int orc_hll_pt(const orc_cfg* c, const double x[3], const double pl[8], const double pr[8], int dir, double F[8]);
/* metric source terms s (non-densitised, 8 entries; D and B entries 0) at cell x */
int orc_sources_pt(const orc_cfg* c, const double x[3], const double pr[8], double s[8]);
/* WENO5 left-biased value at i+1/2 from u[0..4] = u_{i-2..i+2}; rec as orc_cfg */
double orc_weno5_left(const double u[5], int rec);
/* MP5 left-biased value at i+1/2 from u[0..4] = u_{i-2..i+2} (A33) */
double orc_mp5_left(const double u[5]);
/* WENO-Z left-biased value at i+1/2 from u[0..4] (A34) */
double orc_wenoz_left(const double u[5]);
/* MC2 left value at i+1/2 from u[0..4] (only u[1..3] enter; A35) */
double orc_mc2_left(const double u[5]);
/* PPM left state at i+1/2 (u_R of cell i) from u[0..4] (A36) */
double orc_ppm_left(const double u[5]);
/* rec = 6 (A44) at one face: st[8*m + v] = prims (rho, u~^i, p, B^i) of cells i-2+m, m = 0..5;
 * writes the hydro slots 0..4 of the left / right states qL, qR at face i+1/2 along axis a
 * (slots 5..7 zero).  Returns 0. */
int orc_charrec_face_pt(const orc_cfg* c, const double st[48], int a, double qL[8], double qR[8]);
/* DER correction at the centre face from F[0..4] = F_{i-3/2..i+5/2}; der = 6/4/2 */
double orc_der(const double F[5], int der);
/* con2prim at one cell: non-densitised cons u, guess prims (for Z0), result prims.
 * Returns 0 on convergence, 1 on failure.  *iters = Newton iterations used. */
int orc_c2p_pt(const orc_cfg* c, const double x[3], const double u[8], const double guess[8],
               double pr_out[8], int* iters);

/* ---------------- grid-level operations ------------------------------- */
/* user prims P8 -> state (U8 densitised, P5).  Returns 0, or -5 on the first
 * unphysical cell (rho<=0, p<=0 or v^2>=1), whose linear index goes in *bad. */
int orc_set_prims(const orc_cfg* c, const double* P8, double* U8, double* P5, long long* bad);
/* state -> user prims P8 */
int orc_get_prims(const orc_cfg* c, const double* U8, const double* P5, double* P8);
/* L(U) on every owned cell (8 vars, densitised, same layout as U8) */
int orc_rhs(const orc_cfg* c, const double* U8, const double* P5, double* L8);
/* L(U) at ncell cells idx[3*m+0..2] = (i,j,k); out[8*m+q] */
int orc_rhs_cells(const orc_cfg* c, const double* U8, const double* P5,
                  long long ncell, const long long* idx, double* out);
/* RK stage s (1,2,3) with inputs Un, Us (=Un for s=1), Ps (prims of Us).
 * Writes Uout (= U^1, U^2 or U^{n+1}) and Pout on every owned cell. */
int orc_stage(const orc_cfg* c, int s, double dt, const double* Un, const double* Us,
              const double* Ps, double* Uout, double* Pout, orc_counts* cnt);
/* same at sampled cells: Uout[8*m+q], Pout[5*m+q] */
int orc_stage_cells(const orc_cfg* c, int s, double dt, const double* Un, const double* Us,
                    const double* Ps, long long ncell, const long long* idx,
                    double* Uout, double* Pout, orc_counts* cnt);
/* one full SSP-RK3 step, in place on (U8, P5) */
int orc_step(const orc_cfg* c, double dt, double* U8, double* P5, orc_counts* cnt);
/* CFL: dt = cfl / max_cells sum_a max(|lam+_a|,|lam-_a|)/Delta_a.  -1 if all speeds are 0. */
int orc_max_dt(const orc_cfg* c, const double* U8, const double* P5, double cfl, double* dt);
/* con2prim + floors on every owned cell, P5 in: guess, out: result; U8 may be
 * rewritten where floors fire. */
int orc_con2prim(const orc_cfg* c, double* U8, double* P5, orc_counts* cnt);
/* max over owned cells of |sum_a D2_a(sqrt(gamma) B^a)| (SPEC.md:172 operator) */
double orc_divb(const orc_cfg* c, const double* U8);

/* ---------------- UCT (divb = 2; A37-A41) -------------------
 * b3 [3][n3][n2][n1]: sqrt(gamma) B^a at the face i_a + 1/2 of cell (i1,i2,i3).
 * The state's U8 slots 5..7 hold the cell-centred field I6(b3) (A37).
 * Return -1 unless divb = 2. */
/* UCT state: hydro prims from P8 (its B ignored), U_B = I6(b3), B = U_B / sqrt(gamma) */
int orc_set_prims_uct(const orc_cfg* c, const double* P8, const double* b3, double* U8, double* P5, long long* bad);
/* A37 centring: Bc3[a] = 6-point midpoint interpolation of b3[a] along a */
int orc_uct_centre(const orc_cfg* c, const double* b3, double* Bc3);
/* the preserved divergence sum_a delta_a Dh_a b^a at every cell (A41) */
int orc_uct_divh(const orc_cfg* c, const double* b3, double* out);
/* L on every owned cell: slots 0..4 hydro (as orc_rhs), slots 5..7 L(b^a) at the faces */
int orc_rhs_uct(const orc_cfg* c, const double* U8, const double* P5, const double* b3, double* L8);
/* RK stage s with the staggered field: bn, bs in, bout out (may alias bn at s = 3) */
int orc_stage_uct(const orc_cfg* c, int s, double dt, const double* Un, const double* Us, const double* Ps,
                  const double* bn, const double* bs, double* Uout, double* Pout, double* bout, orc_counts* cnt);
/* one SSP-RK3 step in place on (U8, P5, b3) */
int orc_step_uct(const orc_cfg* c, double dt, double* U8, double* P5, double* b3, orc_counts* cnt);

#ifdef __cplusplus
}
#endif
#endif
