// echo_kernels.h — host-callable launchers of the sm_100a kernels (internal).
#pragma once
#include <cuda_runtime.h>

#include "echo_dev.cuh"

namespace echo {

// K2x/K2y/K2z: axis sweep (DESIGN §2 step 2)
cudaError_t launch_sweep(int axis, bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P,
                         const double* U, double* R, double* Om, cudaStream_t st);

// K3 modes
enum UpdateMode { kModeStage = 0, kModeRhs = 1, kModeC2P = 2 };

// K3: sources + curl + RK combine + con2prim/floors (stage), or L(U) only (rhs),
// or con2prim/floors only (c2p).  counters[0] floors, [1] failures.
cudaError_t launch_update(int mode, bool ks, const GridP& g, const EosP& e, const MetTables& mt, int s, double dt,
                          const double* R, const double* Om, const double* Un, const double* Us, double* Uout,
                          double* P, double* Lout, unsigned long long* counters, cudaStream_t st);

// a9: per-cell sum_a max|lambda_a|/Delta_a, max-reduced into *out (u64 bit pattern, zeroed by caller)
cudaError_t launch_max_speed(bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P,
                             const double* U, unsigned long long* out, cudaStream_t st);

// a0: user prims (rho, v, p, B) -> P5 + U8; first unphysical cell into *bad (init LLONG_MAX)
cudaError_t launch_prim2cons(bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P8,
                             double* P5, double* U8, long long* bad, cudaStream_t st);

// state -> user prims
cudaError_t launch_get_prims(bool ks, const GridP& g, const MetTables& mt, const double* P5, const double* U8,
                             double* P8, cudaStream_t st);

}  // namespace echo
