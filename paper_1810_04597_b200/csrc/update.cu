// update.cu — per-cell kernels on the cell-interleaved state (64 B per cell):
// K3 (metric sources a6, field-CD curl a5, RK combine a7, con2prim + floors a8),
// the CFL max-speed reduction a9, the prim<->cons conversions of the API (a0)
// and the layout conversions between the C-ABI's [var][cell] arrays and the
// device's [cell][8] records.  One thread per cell, 16-byte vector loads;
// every counter is warp-aggregated before its single atomic.
#include <cuda_runtime.h>

#include <climits>

#include "cell_physics.cuh"
#include "echo_dev.cuh"
#include "echo_kernels.h"

namespace echo {

// -------------------------------------------------------------- K3 kernel
// MODE stage: U^{s+1} = RK(U^n, U^s, L) then con2prim/floors -> Uout, P (stage_cell).
// MODE rhs:   L(U) into Lout ([var][cell], the C-ABI layout).
// MODE c2p:   con2prim/floors of Un in place -> Un, P.
// block max of v (all threads of the block call it) -> one atomicMax on the u64 bit pattern
ECHO_D void block_max_atomic(double v, unsigned long long* out) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __shared__ double red[kCellThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double bm = red[0];
#pragma unroll
    for (int w = 1; w < kCellThreads / 32; w++) bm = fmax(bm, red[w]);
    atomicMax(out, (unsigned long long)__double_as_longlong(bm));  // non-negative doubles order as u64
  }
}

// Kerr-Schild: the metric records and the sources need more registers than 85 (at 3 CTAs/SM
// the curved-metric stage kernel spilled 180 B per thread): 2 CTAs/SM there (ECHO_KS_UPDATE_BPS)
#ifndef ECHO_KS_UPDATE_BPS
#define ECHO_KS_UPDATE_BPS 2
#endif
template <bool KS, int MODE, bool DIVB_NONE>
__global__ void __launch_bounds__(kCellThreads, KS ? ECHO_KS_UPDATE_BPS : 3)
k_update(const GridP g, const EosP e, const MetTables mt, const int s, const double dt, const double* __restrict__ R,
         const double* Un, const double* Us, double* Uout, double* P, double* __restrict__ Lout,
         unsigned long long* counters, unsigned long long* cfl_out, const GhostLinks gl, const double* dtp) {
  const long long N = g.N;
  double dtv = dt;
  if (dtp) {  // device-driven time loop (echo_advance): dt from k_cfl_dt; a halted loop skips the update
    if (dtp[1] != 0.0) return;  // uniform over the grid: no thread is left at the block barrier
    dtv = dtp[0];
  }
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = id < N;
  int ev = 0;
  double rate = 0.0;
  if (active) {
    int i, j, k;
    cell_ijk(g, id, i, j, k);
    if (MODE == kModeStage) {
      ev = stage_cell<KS, DIVB_NONE>(g, e, mt, s, dtv, R, Un, Us, Uout, P, i, j, k, cfl_out != nullptr, rate, &gl);
    } else {
      const auto m = MetAt<KS>::get(mt, i, j);
      const long long rb = rec_base(g, i, j, k), vs = g.vs;
      double Pp[8];
      if (KS) {
        ld8(P + rb, vs, Pp);
      } else {
#pragma unroll
        for (int v = 0; v < 5; v++) Pp[v] = P[rb + v * vs];
      }
      if (MODE == kModeRhs) {
        double L[8];
        cell_L<KS, DIVB_NONE>(g, e, mt, m, R, rb, i, j, k, Pp, L);
#pragma unroll
        for (int q = 0; q < 8; q++) Lout[q * N + id] = L[q];
      } else {  // c2p
        double Uo[8], Po[8];
        ld8(Un + rb, vs, Uo);
        ev = c2p_floors(m, e, Uo, guess_Z(m, e, Pp), [&](double* pv) {
#pragma unroll
          for (int v = 0; v < 5; v++) pv[v] = Pp[v];
        }, Po);
        const double isg = !KS ? 1.0 : frcp(m.sqrtg());
#pragma unroll
        for (int c = 0; c < 3; c++) Po[5 + c] = !KS ? Uo[5 + c] : Uo[5 + c] * isg;
        st8(Uout + rb, vs, Uo);
        st_prims<KS>(P + rb, vs, Po);
        if (!KS) P[rb + kSlotZ * vs] = guess_Z(m, e, Po);
        if (cfl_out) rate = cfl_rate(m, g, e, Po);
      }
    }
  }
  if (cfl_out) block_max_atomic(rate, cfl_out);
  if (MODE != kModeRhs) {
    unsigned fl = __reduce_add_sync(0xffffffffu, ev == 1 ? 1u : 0u);
    unsigned fa = __reduce_add_sync(0xffffffffu, ev == 2 ? 1u : 0u);
    if ((threadIdx.x & 31) == 0) {
      if (fl) atomicAdd(counters + 0, (unsigned long long)fl);
      if (fa) atomicAdd(counters + 1, (unsigned long long)fa);
    }
  }
}

template <bool KS, int MODE>
static cudaError_t upd2(const GridP& g, const EosP& e, const MetTables& mt, int s, double dt, const double* R,
                        const double* Un, const double* Us, double* Uout, double* P, double* Lout,
                        unsigned long long* cnt, unsigned long long* cfl, cudaStream_t st, const GhostLinks& gl,
                        const double* dtp) {
  unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  if (g.divb == 1)
    k_update<KS, MODE, true><<<blocks, kCellThreads, 0, st>>>(g, e, mt, s, dt, R, Un, Us, Uout, P, Lout, cnt, cfl, gl, dtp);
  else
    k_update<KS, MODE, false><<<blocks, kCellThreads, 0, st>>>(g, e, mt, s, dt, R, Un, Us, Uout, P, Lout, cnt, cfl, gl, dtp);
  return cudaGetLastError();
}

template <bool KS>
static cudaError_t upd1(int mode, const GridP& g, const EosP& e, const MetTables& mt, int s, double dt, const double* R,
                        const double* Un, const double* Us, double* Uout, double* P, double* Lout,
                        unsigned long long* cnt, unsigned long long* cfl, cudaStream_t st, const GhostLinks& gl,
                        const double* dtp) {
  if (mode == kModeRhs) return upd2<KS, kModeRhs>(g, e, mt, s, dt, R, Un, Us, Uout, P, Lout, cnt, nullptr, st, gl, nullptr);
  if (mode == kModeC2P) return upd2<KS, kModeC2P>(g, e, mt, s, dt, R, Un, Us, Uout, P, Lout, cnt, cfl, st, gl, nullptr);
  return upd2<KS, kModeStage>(g, e, mt, s, dt, R, Un, Us, Uout, P, Lout, cnt, cfl, st, gl, dtp);
}

cudaError_t launch_update(int mode, bool ks, const GridP& g, const EosP& e, const MetTables& mt, int s, double dt,
                          const double* R, const double* Un, const double* Us, double* Uout, double* P, double* Lout,
                          unsigned long long* counters, unsigned long long* cfl_out, cudaStream_t st,
                          const GhostLinks* links, const double* dtp) {
  GhostLinks none{};
  const GhostLinks& gl = links ? *links : none;
  if (ks) return upd1<true>(mode, g, e, mt, s, dt, R, Un, Us, Uout, P, Lout, counters, cfl_out, st, gl, dtp);
  return upd1<false>(mode, g, e, mt, s, dt, R, Un, Us, Uout, P, Lout, counters, cfl_out, st, gl, dtp);
}

// ------------------------------------------------------ CFL reduction (a9)
template <bool KS>
__global__ void __launch_bounds__(kCellThreads)
k_max_speed(const GridP g, const EosP e, const MetTables mt, const double* __restrict__ P, const double* __restrict__ U,
            unsigned long long* out) {
  const long long N = g.N;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double val = 0.0;
  if (id < N) {
    int i, j, k;
    cell_ijk(g, id, i, j, k);
    const auto m = MetAt<KS>::get(mt, i, j);
    double pr[8];
    const long long rb = rec_base(g, i, j, k);
    ld8(P + rb, g.vs, pr);
    if (!KS)
      for (int c = 0; c < 3; c++) pr[5 + c] = U[rb + (5 + c) * g.vs];  // B^i = U_B (Minkowski)
    val = cfl_rate(m, g, e, pr);
  }
  block_max_atomic(val, out);
}

cudaError_t launch_max_speed(bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P,
                             const double* U, unsigned long long* out, cudaStream_t st) {
  unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  if (ks) k_max_speed<true><<<blocks, kCellThreads, 0, st>>>(g, e, mt, P, U, out);
  else k_max_speed<false><<<blocks, kCellThreads, 0, st>>>(g, e, mt, P, U, out);
  return cudaGetLastError();
}

// ------------------------------------------- device-side time step (echo_advance)
// dt = cfl / m (IEEE division: the host's echo_max_dt value bit for bit) from the
// reduction the previous step's last update left in *maxbits; adv = [dt, halt, count].
// A zero or non-finite m sets halt, after which every update of the loop is skipped.
__global__ void k_cfl_dt(double cfl, const unsigned long long* __restrict__ maxbits, double* adv, double* log,
                         long long cap) {
  if (adv[1] != 0.0) return;
  const double m = __longlong_as_double((long long)*maxbits);
  if (!(m > 0.0) || !isfinite(m)) {
    adv[1] = 1.0;
    return;
  }
  const double dt = cfl / m;
  adv[0] = dt;
  const long long n = (long long)adv[2];
  if (n < cap) log[n] = dt;
  adv[2] = (double)(n + 1);
}

cudaError_t launch_cfl_dt(double cfl, const unsigned long long* maxbits, double* adv, double* log, long long cap,
                          cudaStream_t st) {
  k_cfl_dt<<<1, 1, 0, st>>>(cfl, maxbits, adv, log, cap);
  return cudaGetLastError();
}

// ------------------------------------------------ debug NaN / Inf scan (SURVEY §8(b) "Errors")
// first non-finite value of the state: U (8 slots) and the primitives P (slots 0..4; 0..7 in a
// curved metric) of every owned cell; *first = min over bad values of (linear cell id) * 16 + slot
// (slots 0..7 U, 8..15 P), init LLONG_MAX.  adv (device loop, may be NULL): a hit sets the halt
// flag adv[1] = 2, after which the loop's later updates do nothing (the state is kept for the report).
__global__ void __launch_bounds__(kCellThreads)
k_nanscan(const GridP g, const double* __restrict__ U, const double* __restrict__ P, int np, long long* first,
          double* adv) {
  const long long N = g.N;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long code = LLONG_MAX;
  if (id < N) {
    const long long rb = rec_base_id(g, id), vs = g.vs;
    for (int q = 15; q >= 0; q--) {  // the lowest bad slot wins
      if (q >= 8 && q - 8 >= np) continue;
      const double v = q < 8 ? U[rb + q * vs] : P[rb + (q - 8) * vs];
      if (!isfinite(v)) code = id * 16 + q;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long other = __shfl_xor_sync(0xffffffffu, code, o);
    code = other < code ? other : code;
  }
  if ((threadIdx.x & 31) == 0 && code != LLONG_MAX) {
    atomicMin((unsigned long long*)first, (unsigned long long)code);
    if (adv) adv[1] = 2.0;
  }
}

cudaError_t launch_nanscan(const GridP& g, const double* U, const double* P, int np, long long* first, double* adv,
                           cudaStream_t st) {
  unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  k_nanscan<<<blocks, kCellThreads, 0, st>>>(g, U, P, np, first, adv);
  return cudaGetLastError();
}

// ------------------------------------------------------------ a0 and back
// user prims [8][cell] (rho, v^i, p, B^i) -> P[cell][8] (rho, u~^i, p, B^i), Un[cell][8]
template <bool KS>
__global__ void __launch_bounds__(kCellThreads)
k_prim2cons(const GridP g, const EosP e, const MetTables mt, const double* __restrict__ P8, double* __restrict__ P,
            double* __restrict__ U, long long* bad) {
  const long long N = g.N;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= N) return;
  int i, j, k;
  cell_ijk(g, id, i, j, k);
  const auto m = MetAt<KS>::get(mt, i, j);
  double v[3] = {P8[1 * N + id], P8[2 * N + id], P8[3 * N + id]}, vl[3];
  m.lower(v, vl);
  const double v2 = v[0] * vl[0] + v[1] * vl[1] + v[2] * vl[2];
  const double rho = P8[id], p = P8[4 * N + id];
  if (!(rho > 0.0) || !(p > 0.0) || !(v2 < 1.0)) {
    atomicMin((unsigned long long*)bad, (unsigned long long)id);
    return;
  }
  const double W = 1.0 / sqrt(1.0 - v2);
  double pr[8] = {rho, W * v[0], W * v[1], W * v[2], p, P8[5 * N + id], P8[6 * N + id], P8[7 * N + id]};
  State s;
  make_state(m, e, pr, s);
  const double sg = m.sqrtg();
  double u[8] = {sg * s.D, sg * s.S[0], sg * s.S[1], sg * s.S[2], sg * s.tau, sg * pr[5], sg * pr[6], sg * pr[7]};
  st8(U + rec_base(g, i, j, k), g.vs, u);
  if (!KS) pr[kSlotZ] = guess_Z(m, e, pr);  // Minkowski: B lives in U; slot 5 holds the Newton guess
  st8(P + rec_base(g, i, j, k), g.vs, pr);
}

cudaError_t launch_prim2cons(bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P8, double* P,
                             double* U, long long* bad, cudaStream_t st) {
  unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  if (ks) k_prim2cons<true><<<blocks, kCellThreads, 0, st>>>(g, e, mt, P8, P, U, bad);
  else k_prim2cons<false><<<blocks, kCellThreads, 0, st>>>(g, e, mt, P8, P, U, bad);
  return cudaGetLastError();
}

// P[cell][8] -> user prims [8][cell] (v = u~ / W)
template <bool KS>
__global__ void __launch_bounds__(kCellThreads)
k_get_prims(const GridP g, const MetTables mt, const double* __restrict__ P, const double* __restrict__ U,
            double* __restrict__ P8) {
  const long long N = g.N;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= N) return;
  int i, j, k;
  cell_ijk(g, id, i, j, k);
  const auto m = MetAt<KS>::get(mt, i, j);
  double pr[8];
  const long long rb = rec_base(g, i, j, k);
  ld8(P + rb, g.vs, pr);
  if (!KS)
    for (int c = 0; c < 3; c++) pr[5 + c] = U[rb + (5 + c) * g.vs];  // B^i = U_B (Minkowski)
  double u[3] = {pr[1], pr[2], pr[3]}, ul[3];
  m.lower(u, ul);
  const double iW = frsqrt(1.0 + u[0] * ul[0] + u[1] * ul[1] + u[2] * ul[2]);
  P8[id] = pr[0];
#pragma unroll
  for (int c = 0; c < 3; c++) P8[(1 + c) * N + id] = u[c] * iW;
  P8[4 * N + id] = pr[4];
#pragma unroll
  for (int c = 0; c < 3; c++) P8[(5 + c) * N + id] = pr[5 + c];
}

cudaError_t launch_get_prims(bool ks, const GridP& g, const MetTables& mt, const double* P, const double* U,
                             double* P8, cudaStream_t st) {
  unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  if (ks) k_get_prims<true><<<blocks, kCellThreads, 0, st>>>(g, mt, P, U, P8);
  else k_get_prims<false><<<blocks, kCellThreads, 0, st>>>(g, mt, P, U, P8);
  return cudaGetLastError();
}

// ------------------------------------------------ layout conversions
// aos[cell][8] (first nq slots) <-> soa[q][cell]
__global__ void __launch_bounds__(kCellThreads)
k_layout(const GridP g, const double* __restrict__ src, double* __restrict__ dst, int nq, int to_soa) {
  const long long N = g.N;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= N) return;
  const long long rb = rec_base_id(g, id), vs = g.vs;
  if (to_soa) {
    for (int q = 0; q < nq; q++) dst[q * N + id] = src[rb + q * vs];
  } else {
    for (int q = 0; q < nq; q++) dst[rb + q * vs] = src[q * N + id];
  }
}

cudaError_t launch_layout(const GridP& g, const double* src, double* dst, int nq, bool to_soa, cudaStream_t st) {
  unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  k_layout<<<blocks, kCellThreads, 0, st>>>(g, src, dst, nq, to_soa ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace echo
