// echo_kernels.h — host-callable launchers of the sm_100a kernels (internal).
// Device state: every per-cell record has 8 variables, stored row-interleaved
// ([k][j][var][i], echo_dev.cuh rec_base):
//   P = rho, u~^1..3, p, B^1..3        (B non-densitised; slots 5..7 kept only in a curved
//                                      metric: in Minkowski B^i = U_B is read from U)
//   U = sqrt(g) (D, S_1..3, tau, B^1..3)
//   R = L_D, L_S1..3, L_tau, Omega_1..3 (field-CD) or L_B1..3 (divb none)
#pragma once
#include <cuda_runtime.h>

#include "echo_dev.cuh"

namespace echo {

// K2x/K2y/K2z: axis sweep (DESIGN §2 step 2): P -> R (x writes, y/z accumulate),
// a marching pipeline over whole lines (no tile-halo recomputation)
// P: stage-input primitives; UB: the array holding B^i in slots 5..7 (P in a curved metric,
// the stage-input U in Minkowski, where B^i = U_B)
// UCT (divb = 2): Bface = the stage-input staggered field (slot a = b^a), FSo = this axis's
// face-data array (uct.cu); NULL otherwise
// zr (x/y sweeps only; zn = 0: every plane of the sweep, incl. the slab's first ghost planes):
// sweep the planes zb .. zb + zn - 1 only (slab mode: the interior sweeps overlap the halo exchange)
struct PlaneRange {
  int zb = 0, zn = 0;
};
cudaError_t launch_march(int axis, bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P,
                         const double* UB, double* R, cudaStream_t st, const double* Bface = nullptr,
                         double* FSo = nullptr, PlaneRange zr = PlaneRange{});

// slab mode, fused ghost exchange: K3 also stores the new P and U of the owned planes
// next to a linked side straight into the neighbour slab's ghost planes (peer memory:
// the same device, or another GPU over NVLink), and replicates the edge plane into its
// own ghost planes on a physical outflow side.  dstP/dstU[side]: the neighbour's P /
// (same-role) U array shifted so that adding a cell's record offset gives the target
// ghost cell; NULL = not linked.
struct GhostLinks {
  double* dstP[2];
  double* dstU[2];
  int replicate[2];
  int on;
};

// K3 modes
enum UpdateMode { kModeStage = 0, kModeRhs = 1, kModeC2P = 2 };

// K3: sources + curl + RK combine + con2prim/floors (stage), or L(U) only into
// Lout[var][cell] (rhs), or con2prim/floors of Un only (c2p).  counters[0]
// floors, [1] failures.  cfl_out (may be NULL; zeroed by the caller): the CFL
// max-speed reduction (a9) of the new state, fused into the same pass.
cudaError_t launch_update(int mode, bool ks, const GridP& g, const EosP& e, const MetTables& mt, int s, double dt,
                          const double* R, const double* Un, const double* Us, double* Uout, double* P, double* Lout,
                          unsigned long long* counters, unsigned long long* cfl_out, cudaStream_t st,
                          const GhostLinks* links = nullptr, const double* dtp = nullptr);

// K3 of stage s (as launch_update kModeStage, reading the accumulator Rold) fused with the x
// sweep of the new state into the accumulator Rnew (fused.cu; not in slab or UCT mode:
// cudaErrorInvalidValue).  Bit-for-bit the same results as the two separate kernels.
cudaError_t launch_update_march(bool ks, const GridP& g, const EosP& e, const MetTables& mt, int s, double dt,
                                const double* dtp, const double* Rold, const double* Un, const double* Us, double* Uout,
                                double* P, unsigned long long* counters, unsigned long long* cfl_out, double* Rnew,
                                cudaStream_t st);

// device-driven time loop: dtp = adv = [dt, halt, steps done] (doubles); launch_update with
// dtp set reads dt from adv[0] and does nothing once adv[1] != 0.  k_cfl_dt sets
// adv[0] = cfl / m from the CFL reduction bits (halt on m <= 0 or non-finite) and appends
// it to log[steps done] while steps done < cap.
cudaError_t launch_cfl_dt(double cfl, const unsigned long long* maxbits, double* adv, double* log, long long cap,
                          cudaStream_t st);

// debug NaN/Inf scan of U (8 slots) and P (np slots) of the owned cells: first bad value's
// (cell id * 16 + slot, P slots 8..) atomicMin'd into *first (init LLONG_MAX); a hit sets adv[1] = 2
// when adv is given (device-driven loop: halts it)
cudaError_t launch_nanscan(const GridP& g, const double* U, const double* P, int np, long long* first, double* adv,
                           cudaStream_t st);

// a9: per-cell sum_a max|lambda_a|/Delta_a, max-reduced into *out (u64 bit pattern, zeroed by caller)
cudaError_t launch_max_speed(bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P,
                             const double* U, unsigned long long* out, cudaStream_t st);

// a0: user prims [8][cell] (rho, v, p, B) -> P, U; first unphysical cell into *bad (init LLONG_MAX)
cudaError_t launch_prim2cons(bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P8, double* P,
                             double* U, long long* bad, cudaStream_t st);

// P -> user prims [8][cell]
cudaError_t launch_get_prims(bool ks, const GridP& g, const MetTables& mt, const double* P, const double* U,
                             double* P8, cudaStream_t st);

// device records (first nq variables) <-> caller arrays [q][cell]
cudaError_t launch_layout(const GridP& g, const double* src, double* dst, int nq, bool to_soa, cudaStream_t st);

// ---- UCT (divb = 2, uct.cu; DESIGN A37-A41): Bst slots 0..2 b^n, 3..5 b^s; FS[a] face data
// of axis a; Ed slots 0..2 the edge EMFs
cudaError_t launch_uct_emf(const GridP& g, const double* const FS[3], const double* Bin, double* Ed, cudaStream_t st);
// mode 0: RK stage s of the face field (dt, or from dtp as launch_update); mode 1: L(b) into
// Lout[5 + a][cell]
cudaError_t launch_uct_induct(const GridP& g, int mode, int s, double dt, const double* dtp, const double* Ed,
                              double* Bst, double* Lout, cudaStream_t st);
// hydro RK combine (rhs from the sweeps in R, + KS sources), U_B = I6(b), con2prim + floors, CFL rate
cudaError_t launch_uct_cell(bool ks, const GridP& g, const EosP& e, const MetTables& mt, int s, double dt,
                            const double* dtp, const double* R, const double* Un, const double* Us, double* Uout,
                            double* P, const double* Bst, unsigned long long* counters, unsigned long long* cfl_out,
                            cudaStream_t st);
// U_B = I6(b^n) and U recomputed from the state's hydro primitives (echo_set_face_field;
// KS: also B = U_B / sqrt(g) into P)
cudaError_t launch_uct_centre_p2c(bool ks, const GridP& g, const EosP& e, const MetTables& mt, double* P, double* U,
                                  const double* Bst, cudaStream_t st);

}  // namespace echo
