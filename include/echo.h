/*
 * echo.h — C-ABI of the B200-native ECHO-3DHPC time-step library (libecho_b200.so).
 *
 * The paper (arXiv 1810.04597) studies the time step of ECHO-3DHPC, "a Fortran
 * application developed to solve the equations of magneto-hydrodynamic in
 * General Relativity, using 3D finite-differences method and high-order
 * reconstruction algorithms", timed per iteration on 512^3 and
 * 1024^3 grids (Table 1).  This library evaluates exactly that
 * step on one B200: per SSP-RK3 stage a ghost fill, per-axis WENO5
 * reconstruction + HLL flux + DER6 flux derivative, metric sources, a field-CD
 * divergence-preserving B update, the RK combine and a per-cell Newton
 * con2prim with floors; plus the CFL max-speed reduction.  The formulas are
 * DESIGN.md §2 and readings A1-A30 (the paper prints none).
 *
 * Conventions shared by every entry point
 *  - Arrays are fp64, row-major [var][n3][n2][n1] (x1 fastest), owned cells
 *    only (no ghost cells), N = n1*n2*n3 cells per variable.
 *      user prims  P8 : rho, v^1, v^2, v^3, p, B^1, B^2, B^3   (v contravariant
 *                       Eulerian 3-velocity, B non-densitised)       [A29]
 *      state prims P5 : rho, u~^1, u~^2, u~^3, p with u~ = W v
 *      conserved   U8 : sqrt(gamma) * (D, S_1, S_2, S_3, tau, B^1, B^2, B^3) [A10]
 *  - `on_device` = 1: the pointer is device memory (e.g. torch tensor
 *    data_ptr()); the copy is stream-ordered on the context stream and the call
 *    returns without synchronising.  `on_device` = 0: host memory; the call
 *    copies and synchronises before returning.
 *  - Ownership: the context owns every device allocation (made in
 *    echo_create, freed in echo_destroy).  Caller buffers are never retained.
 *  - Errors: every int-returning call returns ECHO_OK (0) or a negative
 *    echo_status; echo_last_error() then names the violated rule and, for
 *    unphysical states, the first bad cell and its values (SPEC.md:110 idea).
 *    Asynchronous kernel faults surface at the next synchronising call.
 *  - Threading: one control thread per context; several
 *    contexts may share a device.
 *  - There is no CPU fallback: every step runs in the sm_100a kernels of this
 *    library; a missing device is ECHO_E_CUDA at echo_create.
 */
#ifndef ECHO_B200_H
#define ECHO_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct echo_ctx echo_ctx;

typedef enum {
  ECHO_OK = 0,
  ECHO_E_ARG = -1,         /* invalid argument (rule named in echo_last_error) */
  ECHO_E_CUDA = -2,        /* CUDA runtime error (no device, launch failure, ...) */
  ECHO_E_OOM = -3,         /* device allocation failed */
  ECHO_E_ORDER = -4,       /* call out of order, e.g. echo_step before echo_set_prims */
  ECHO_E_UNPHYSICAL = -5,  /* rho <= 0, p <= 0 or v^2 >= 1 in echo_set_prims */
  ECHO_E_NONFINITE = -6    /* all CFL speeds zero / non-finite (echo_max_dt), or a NaN/Inf in the
                              state (echo_check_finite; debug mode ECHO_DEBUG_NANSCAN) */
} echo_status;

typedef enum { ECHO_BC_PERIODIC = 0, ECHO_BC_OUTFLOW = 1, ECHO_BC_HALO = 2 } echo_bc;  /* A13; HALO: slabs */

/* Ghost planes per side of a slab (z boundaries of kind ECHO_BC_HALO): kG = 5 for
 * WENO5 + DER6, plus one because the sweeps also evaluate the EMF on the first
 * ghost plane (the field-CD curl of the edge plane reads it). */
#define ECHO_HALO_PLANES 6
/* UCT (divb = 2) slabs store 8: the induction's DER along z reads the edge EMFs of 3 ghost
 * planes, whose z reconstructions read face data 5 planes in, whose HLL states read the
 * primitives 7 planes in */
#define ECHO_HALO_PLANES_UCT 8
typedef enum { ECHO_METRIC_MINKOWSKI = 0, ECHO_METRIC_KERR_SCHILD = 1 } echo_metric_kind;

/* Grid: n owned cells per axis (n >= 1; periodic n < 5 is allowed, ghosts wrap
 * modulo n [A12]); [lo, hi) coordinate extent per axis (lo < hi).  Minkowski
 * uses Cartesian (x, y, z); Kerr-Schild uses (ln r, theta, phi) [A14] and
 * requires sin(theta) != 0 at every centre and face of the ghost-extended range.
 * bc[a][0]/[1] = lower/upper boundary of axis a.  ECHO_BC_HALO (axis 2 only) makes the
 *   context one z-slab of a domain decomposition (the paper's MPI
 *   Cartesian decomposition): its ghost planes are stored and must be
 *   filled before every stage — from the neighbour slab (echo_halo_export on the
 *   neighbour, echo_halo_import here) or, on a physical outflow side of the slab,
 *   by echo_halo_fill; echo_step is then refused (use echo_stage).  n[2] >= 6.
 * rec: 0 = WENO5 point-value form (A2, default), 1 = WENO5 finite-volume form,
 *      2 = MP5 (Suresh & Huynh 1997 on point values, reading A33),
 *      3 = WENO-Z (Borges et al. 2008 weights on the point form, reading A34),
 *      4 = MC2, the monotonized-central limited linear reconstruction (reading A35),
 *      5 = PPM (Colella & Woodward 1984 constraints on point values, reading A36),
 *      6 = characteristic-wise WENO5 of the hydro primitives (reading A44: per face, the
 *          stencil's (rho, u~, p) projected on the left eigenvectors of the flat-space
 *          relativistic-Euler Jacobian at the mean of the two adjacent cells, WENO5 point form
 *          per characteristic field, projected back; B^i component-wise WENO5; SURVEY §8(f) f3
 *          "characteristic-wise reconstruction").  Minkowski only and not with divb = 2
 *          (ECHO_E_ARG at echo_create).
 * der: 6 = DER6 (A5, default), 4 = DER4, 2 = plain flux difference.
 * divb: 0 = field-CD constrained transport (A6, default), 1 = none, 2 = UCT: staggered
 *   field + upwind constrained transport (readings A37-A41; echo_set_face_field below).
 * der_jump: DER shock switch (A31): the DER correction at a face is dropped
 *   (H = F) when one of the 5 faces of its stencil joins two cells whose rho or
 *   p differ by more than der_jump x the smaller of the two; <= 0 disables it
 *   (default 0.5). */
typedef struct {
  int n[3];
  double lo[3], hi[3];
  int bc[3][2];
  int rec;
  int der;
  int divb;
  double der_jump;
  double dz;  /* > 0: the z cell size Delta_z itself instead of (hi[2] - lo[2]) / n[2] (z slabs take the
                 global grid's, so that every z difference of the slab is the single domain's bit for
                 bit; it must agree with hi - lo to 1e-12 relative); 0: derived */
} echo_grid;

/* Stationary background metric (A1, A14): Minkowski, or Kerr-Schild with mass M >= 0 and spin a
 * (M = 0 is flat space in oblate-spheroidal / spherical coordinates; used by the pins). */
typedef struct {
  int kind; /* echo_metric_kind */
  double M, a;
} echo_metric;

/* Ideal-gas EOS and con2prim controls (A8, A9): gamma > 1, floors > 0,
 * w_max > 1, c2p_max_iter >= 1, c2p_tol > 0. */
typedef struct {
  double gamma;
  double rho_floor, p_floor, w_max;
  int c2p_max_iter;
  double c2p_tol;
} echo_eos;

/* Event counters (A9: floors are applied and counted, never silent). */
typedef struct {
  unsigned long long floor_events; /* cells where a floor / W_max rescale fired */
  unsigned long long c2p_failures; /* cells where Newton failed (previous-stage fallback) */
  unsigned long long steps;        /* completed echo_step calls */
  unsigned long long stages;       /* completed RK stages (including those of echo_step) */
} echo_stats_t;

/* Create a context on the current CUDA device; allocates all device state
 * (about 32 fp64 fields of N cells).  Validation: see the struct comments;
 * violations give ECHO_E_ARG.  *out is NULL on failure. */
int echo_create(const echo_grid* grid, const echo_metric* metric, const echo_eos* eos, echo_ctx** out);

/* Free every device allocation of ctx (NULL is a no-op). */
void echo_destroy(echo_ctx* ctx);

/* Launch every kernel of ctx on `cuda_stream` (a cudaStream_t; NULL = legacy default stream). */
int echo_set_stream(echo_ctx* ctx, void* cuda_stream);

/* Set the state from user prims P8 (layout above): U^n = sqrt(gamma) prim2cons(P)
 * (DESIGN a0), P5 with u~ = v / sqrt(1 - v^2).  Rejects rho <= 0, p <= 0,
 * v^2 >= 1 (ECHO_E_UNPHYSICAL, first bad cell named). */
int echo_set_prims(echo_ctx* ctx, const double* p8, int on_device);

/* Current user prims P8 (B = U_B / sqrt(gamma), v = u~ / W). */
int echo_get_prims(echo_ctx* ctx, double* p8, int on_device);

/* UCT (grid.divb = 2; readings A37-A43; periodic or outflow axes (A42), any
 * metric (A43); z-slab boundaries with the copy exchange, ECHO_HALO_PLANES_UCT ghost planes whose
 * messages also carry b; the fused links are refused): the magnetic state is the staggered field
 * b3[a][n3][n2][n1] = sqrt(gamma) B^a at the centre of the face i_a + 1/2 of cell
 * (i1, i2, i3) (point values).  After echo_set_prims (which supplies the hydro
 * primitives; its B is replaced), echo_set_face_field sets b, the cell-centred field
 * U_B = I6(b) (6-point midpoint interpolation along a; B = U_B / sqrt(gamma)) and U.  Every step then
 * updates b by the UCT-HLL edge EMFs with the DER operator along the
 * differentiation direction, which keeps sum_a delta_a Dh_a b^a at roundoff.
 * Stepping a divb = 2 context before echo_set_face_field is ECHO_E_ORDER, as is
 * echo_set_cons (U_B must stay I6(b)).  echo_rhs returns L(b^a) at the faces in
 * slots 5..7.  echo_get_face_field returns the current b (same layout).  Host
 * buffers synchronise; device buffers are stream-ordered. */
int echo_set_face_field(echo_ctx* ctx, const double* b3, int on_device);
int echo_get_face_field(echo_ctx* ctx, double* b3, int on_device);

/* Replace U^n by u8 and recover P by con2prim + floors (guess: current P).
 * Requires a prior echo_set_prims (ECHO_E_ORDER). */
int echo_set_cons(echo_ctx* ctx, const double* u8, int on_device);

/* Current conserved state U8 (U^n after a step; U^s inside a step). */
int echo_get_cons(echo_ctx* ctx, double* u8, int on_device);

/* Raw stage state: U^n (8 fields), U^s (8 fields, meaningful after stage 1 or 2),
 * P5 (rho, u~^i, p).  Any pointer may be NULL.  Used by stage-level parity. */
int echo_get_state(echo_ctx* ctx, double* un8, double* us8, double* p5, int on_device);

/* L(U) of the current state (DESIGN §2 steps 1-4): 8 fields, layout of U8. */
int echo_rhs(echo_ctx* ctx, double* l8, int on_device);

/* con2prim + floors on the current conserved state (guess: current P);
 * adds this call's counts to *delta if non-NULL (synchronises). */
int echo_con2prim(echo_ctx* ctx, echo_stats_t* delta);

/* One SSP-RK3 stage s (1, 2 or 3) with time step dt > 0 (SPEC.md:154 forms, A7):
 * s=1: U^s = U^n + dt L(U^n); s=2: U^s = 0.75 U^n + 0.25 (U^s + dt L(U^s));
 * s=3: U^n = (1/3) U^n + (2/3)(U^s + dt L(U^s)); each followed by con2prim.
 * Stages must be issued in order 1, 2, 3 (ECHO_E_ORDER otherwise).  Asynchronous. */
int echo_stage(echo_ctx* ctx, int s, double dt);

/* The two halves of echo_stage(s, dt): the axis sweeps of stage s (L of the stage
 * input), then the K3 update (sources, curl, RK combine, con2prim; slab mode: the
 * fused ghost stores of echo_halo_link).  In order, without other stage calls between. */
int echo_stage_sweeps(echo_ctx* ctx, int s);
int echo_stage_update(echo_ctx* ctx, int s, double dt);
/* The sweeps of a slab stage in two parts, so that the halo exchange overlaps computation:
 * echo_stage_sweeps_interior(s) runs the x and y sweeps over the owned planes, which read no
 * ghost plane (call it right after echo_halo_export, while the messages are in flight);
 * echo_stage_sweeps_boundary(s) runs the x and y sweeps of the first ghost plane on each side
 * and the z sweep (call it after echo_halo_import / echo_halo_fill).  Together they equal
 * echo_stage_sweeps(s) bit for bit; echo_stage_update(s, dt) follows.  Slab contexts only,
 * not UCT (ECHO_E_ORDER). */
int echo_stage_sweeps_interior(echo_ctx* ctx, int s);
int echo_stage_sweeps_boundary(echo_ctx* ctx, int s);
/* UCT slabs (divb = 2 with halo boundaries): the cell update centres the NEW b^z of 3 faces
 * beyond the slab, which the neighbour's induction writes, so a stage is
 *   exchange (echo_halo_export / import / fill) -> echo_stage_sweeps(s)
 *   -> echo_stage_update_field(s, dt)   (the induction, A41)
 *   -> new-field exchange: echo_halo_export_field / echo_halo_import_field, or
 *      echo_halo_fill_field on a physical outflow side (echo_halo_field_doubles(ctx) doubles:
 *      the new b^z of the 3 owned planes next to the side)
 *   -> echo_stage_update_cells(s, dt)   (hydro RK, U_B = I6(b), con2prim, A37)
 * echo_stage and echo_stage_update are refused on such contexts (ECHO_E_ORDER). */
int echo_stage_update_field(echo_ctx* ctx, int s, double dt);
int echo_stage_update_cells(echo_ctx* ctx, int s, double dt);
long long echo_halo_field_doubles(const echo_ctx* ctx);
int echo_halo_export_field(echo_ctx* ctx, int side, double* buf, int on_device);
int echo_halo_import_field(echo_ctx* ctx, int side, const double* buf, int on_device);
int echo_halo_fill_field(echo_ctx* ctx, int side);

/* One full SSP-RK3 step (stages 1, 2, 3) with dt > 0.  Asynchronous. */
int echo_step(echo_ctx* ctx, double dt);

/* CFL (SPEC.md:163 form, A11): *dt_out = cfl / max_cells sum_a max(|lambda+_a|, |lambda-_a|)/Delta_a.
 * Synchronises (one 8-byte device-to-host copy).  ECHO_E_NONFINITE if the max is 0 or not finite. */
int echo_max_dt(echo_ctx* ctx, double cfl, double* dt_out);

/* nsteps x (echo_max_dt(cfl) + echo_step(dt)) with the time step computed on the device:
 * the same dt values bit for bit (dt = cfl / m in IEEE division, m the reduction fused
 * into the previous step's last update) and the same state, without a host round trip
 * per step.  The step (its dt kernel, 9 sweeps and 3 updates) is captured once into a
 * CUDA graph (re-captured when cfl changes) and replayed nsteps times; one
 * synchronisation at the end.  dt_log: host array of nsteps doubles receiving each
 * step's dt (may be NULL); *steps_done (may be NULL): steps completed.
 * ECHO_E_NONFINITE if the max speed became 0 or not finite before step *steps_done + 1:
 * the device skips every later update, so the state is that after *steps_done steps.
 * Not in slab mode (ECHO_E_ORDER), nor with a step in progress.  Synchronises. */
int echo_advance(echo_ctx* ctx, int nsteps, double cfl, double* dt_log, int* steps_done);

/* Accumulated counters (synchronises). */
int echo_stats(echo_ctx* ctx, echo_stats_t* out);

/* ---- z-slab domain decomposition (ECHO_BC_HALO) ----
 * A halo message holds what the neighbour's sweeps read of the ECHO_HALO_PLANES owned
 * planes next to one side — rho, u~^i, p and B^i of every cell (Minkowski: B from the
 * stage-input U) — echo_halo_doubles(ctx) doubles (0 without halo boundaries), an
 * internal layout that only echo_halo_import of a context with the same n[0], n[1] and
 * metric reads.  side 0 = lower z, 1 = upper z.
 *   echo_halo_export(ctx, 0, buf, dev): planes 0..5 (for the lower neighbour's side 1)
 *   echo_halo_import(ctx, 0, buf, dev): ghost planes -6..-1 from the lower neighbour
 *   echo_halo_fill(ctx, side): a physical outflow side: ghost planes = the edge plane
 * Call them between stages (after the previous stage / echo_set_prims, before
 * echo_stage), on the context stream; device buffers stay stream-ordered. */
long long echo_halo_doubles(const echo_ctx* ctx);
/* Fused exchange: link `side` of ctx to the slab `peer` (in this process; another
 * device needs peer access enabled).  From then on the update of each stage also
 * stores the new P and U of ctx's 6 planes next to `side` straight into peer's ghost
 * planes (and, on a physical outflow side, replicates the edge plane into ctx's own
 * ghost planes): no export/import is needed.  The caller orders, per stage,
 * echo_stage_sweeps on every slab before echo_stage_update on any (the update
 * overwrites ghost planes the neighbour's sweeps read).  peer = NULL unlinks. */
int echo_halo_link(echo_ctx* ctx, int side, echo_ctx* peer);
/* The same link to a slab owned by another process (one process per GPU): the
 * peer exports its arrays' CUDA IPC handles (echo_ipc_export: 3 x 64 bytes into
 * `handles`, its n[2] into *nz), this process maps them (echo_halo_link_ipc; the
 * peer's n[0], n[1] must equal ctx's; handles = NULL unlinks and unmaps).  Across
 * processes the stage ordering is the caller's: every rank's sweeps of stage s
 * complete before any neighbour's update of stage s, and every update before the
 * neighbours' next sweeps (slab.DistSlab: stream sync + barrier). */
int echo_ipc_export(echo_ctx* ctx, void* handles, int* nz);
/* Fill the ghost planes of `side` by reading the linked neighbour's 6 edge planes
 * (P and the stage-input U) through the link — the first stage's ghosts after
 * echo_set_prims; later stages get theirs from the neighbour's update. */
int echo_halo_pull(echo_ctx* ctx, int side);
int echo_halo_link_ipc(echo_ctx* ctx, int side, const void* handles, int peer_nz);
int echo_halo_export(echo_ctx* ctx, int side, double* buf, int on_device);
int echo_halo_import(echo_ctx* ctx, int side, const double* buf, int on_device);
int echo_halo_fill(echo_ctx* ctx, int side);

/* ---- failure detection (SURVEY.md §8(b) "Errors": ECHO_E_NONFINITE comes from a NaN scan
 * naming the first bad cell; §5 "Failure detection") ----
 * echo_check_finite: scan the current state, U (8 slots) and the state primitives (rho, u~^i,
 * p; + B^i in a curved metric) of every owned cell for NaN / Inf.  Synchronises.  ECHO_OK, or
 * ECHO_E_NONFINITE with echo_last_error naming the first bad value in linear cell order:
 * "U[q]" or "P[q]", its value and the cell (i,j,k).
 * echo_set_debug(ctx, ECHO_DEBUG_NANSCAN): from then on every RK stage ends with that scan
 * of its new state (one extra kernel per stage, stream-ordered).  echo_stage / echo_step then
 * synchronise after each stage and return ECHO_E_NONFINITE at the first stage that produced a
 * non-finite value; echo_advance halts on the device (later updates are skipped, the state is
 * that after the offending stage) and reports it at its end.  flags = 0 turns it off.  The
 * environment variable ECHO_DEBUG_NANSCAN=1 at echo_create sets the flag. */
enum { ECHO_DEBUG_NANSCAN = 1 };
/* Out-of-bounds write detection (compute-sanitizer is closed on this build's GPU pool): with the
 * environment variable ECHO_GUARD_BANDS=1 at echo_create (contexts without halo boundaries),
 * every state array (U^n, U^s, P, the accumulator(s); UCT: the staggered field, face data and
 * edge EMFs) gets 32 KB guard bands before and after, filled with 0xA5 bytes.
 * echo_check_guards verifies every band (synchronises): ECHO_OK, or ECHO_E_CUDA naming the array
 * and how far outside it the nearest overwritten double lies.  ECHO_E_ORDER without guards. */
int echo_check_guards(echo_ctx* ctx);
int echo_set_debug(echo_ctx* ctx, int flags);
int echo_check_finite(echo_ctx* ctx);

/* ---- checkpoint / restart (SURVEY.md §5 "Checkpoint/resume") ----
 * A checkpoint is the raw device state that the next step reads, taken at a step boundary: U^n,
 * the state primitives with their per-cell con2prim guess (and, in a curved metric, B) and, with
 * divb = 2, the staggered field b^n: echo_checkpoint_doubles(ctx) doubles in an internal record
 * layout that only echo_checkpoint_load of a context created with the same grid, metric and EOS
 * reads.  Loading it and stepping continues bit for bit as if the run had not stopped (same
 * states, same CFL dt), unlike a restart through echo_set_prims(echo_get_prims()), which
 * re-derives U from rounded primitives.  Save: ECHO_E_ORDER without a state or inside a step
 * (after echo_stage 1 or 2).  Slab contexts (ECHO_BC_HALO): echo_checkpoint_doubles = 0 and
 * ECHO_E_ORDER (checkpoint the whole domain instead).  Host buffers synchronise, device buffers
 * are stream-ordered.  The event counters are not part of the state. */
long long echo_checkpoint_doubles(const echo_ctx* ctx);
int echo_checkpoint_save(echo_ctx* ctx, double* buf, int on_device);
int echo_checkpoint_load(echo_ctx* ctx, const double* buf, int on_device);

/* Text of the last error of ctx ("" if none); NULL ctx gives the last echo_create error. */
const char* echo_last_error(const echo_ctx* ctx);

/* Kernel-time profiling on the context stream with CUDA events.
 * echo_profile(ctx, 1) starts recording (and clears the totals), 0 stops.
 * echo_profile_read(ctx, id, &ms, &launches) synchronises and returns the summed
 * device time and launch count of kernel class id (0 <= id < echo_kernel_classes()),
 * whose name is echo_kernel_name(id). */
int echo_profile(echo_ctx* ctx, int enable);
int echo_profile_read(echo_ctx* ctx, int id, double* ms, long long* launches);
int echo_kernel_classes(void);
const char* echo_kernel_name(int id);

/* Number of kernels this context has launched so far. */
long long echo_launch_count(const echo_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
