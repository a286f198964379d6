// update.cu — per-cell kernels: K3 (metric sources a6, field-CD curl a5, RK
// combine a7, con2prim + floors a8), the CFL max-speed reduction a9, and the
// prim<->cons conversions of the API (a0).  One thread per cell; every
// counter is warp-aggregated before its single atomic.
#include <cuda_runtime.h>

#include <climits>

#include "echo_dev.cuh"
#include "echo_kernels.h"

namespace echo {

constexpr int kCellThreads = 256;

ECHO_D void cell_ijk(const GridP& g, long long id, int& i, int& j, int& k) {
  long long r = id / g.n[0];
  i = (int)(id - r * g.n[0]);
  k = (int)(r / g.n[1]);
  j = (int)(r - (long long)k * g.n[1]);
}

template <bool KS>
struct MetAt;
template <>
struct MetAt<false> {
  using T = FlatMet;
  static ECHO_D T get(const MetTables&, int, int) { return FlatMet(); }
};
template <>
struct MetAt<true> {
  using T = GenMet;
  static ECHO_D T get(const MetTables& mt, int i, int j) { return load_met(cen_rec(mt, i, j)); }
};

// ----------------------------------------------------------- con2prim (A8)
// 1-D Newton in Z = rho h W^2 with the oracle's iteration rules (A8, A27, A28).
// u: non-densitised (D, S_i, tau, B^i); guess: (rho, u~^i, p); out: (rho, u~^i, p).
template <class M>
ECHO_D int c2p_newton(const M& m, const EosP& e, const double* u, const double* guess, double* out) {
  const double D = u[0], tau = u[4];
  const double S[3] = {u[1], u[2], u[3]};
  const double B[3] = {u[5], u[6], u[7]};
  const double Ut = tau + D;
  double Su[3], Bl[3];
  m.raise(S, Su);
  m.lower(B, Bl);
  const double S2 = S[0] * Su[0] + S[1] * Su[1] + S[2] * Su[2];
  const double B2 = B[0] * Bl[0] + B[1] * Bl[1] + B[2] * Bl[2];
  const double SB = S[0] * B[0] + S[1] * B[1] + S[2] * B[2];
  const double SB2 = SB * SB;
  double gu[3] = {guess[1], guess[2], guess[3]}, gl[3];
  m.lower(gu, gl);
  double Z = (guess[0] + e.gfac * guess[4]) * (1.0 + gu[0] * gl[0] + gu[1] * gl[1] + gu[2] * gl[2]);
  bool polish = false, ok = false;
  for (int it = 1; it <= e.maxit; it++) {
    const double iZ = frcp(Z);
    const double ZB = Z + B2;
    const double iZB = frcp(ZB);
    const double iZ2 = iZ * iZ, iZB2 = iZB * iZB;
    double v2 = (Z * Z * S2 + SB2 * (2.0 * Z + B2)) * iZ2 * iZB2;
    bool clamped = false;
    if (v2 > e.v2max) { v2 = e.v2max; clamped = true; }
    const double sq = fsqrt(1.0 - v2);
    const double p = e.gm * (Z * (1.0 - v2) - D * sq);
    const double f = Z - p + 0.5 * B2 * (1.0 + v2) - 0.5 * SB2 * iZ2 - Ut;
    const double dv2 = clamped ? 0.0 : -2.0 * iZB2 * iZB * (S2 + SB2 * (3.0 * Z * Z + 3.0 * Z * B2 + B2 * B2) * iZ2 * iZ);
    const double dp = e.gm * ((1.0 - v2) - Z * dv2 + D * dv2 * (0.5 * frcp(sq)));
    const double df = 1.0 - dp + 0.5 * B2 * dv2 + SB2 * iZ2 * iZ;
    double Zn = Z - f * frcp(df);
    if (!(Zn > 0.0)) Zn = 0.5 * Z;
    const double dZ = fabs(Zn - Z);
    Z = Zn;
    if (!isfinite(Z)) return 1;
    if (polish) { ok = true; break; }
    if (dZ <= e.tol * Z) {
      polish = true;
      if (it == e.maxit) ok = true;
    }
  }
  if (!ok) return 1;
  const double iZ = frcp(Z);
  const double ZB = Z + B2;
  const double iZB = frcp(ZB);
  double v2 = (Z * Z * S2 + SB2 * (2.0 * Z + B2)) * (iZ * iZ) * (iZB * iZB);
  if (v2 > e.v2max) v2 = e.v2max;
  const double sq = fsqrt(1.0 - v2);
  const double W = frcp(sq);
  out[0] = D * sq;
  out[4] = e.gm * (Z * (1.0 - v2) - D * sq);
  double vl[3], vu[3];
#pragma unroll
  for (int i = 0; i < 3; i++) vl[i] = (S[i] + SB * Bl[i] * iZ) * iZB;
  m.raise(vl, vu);
#pragma unroll
  for (int i = 0; i < 3; i++) out[1 + i] = W * vu[i];
  if (!isfinite(out[0]) || !isfinite(out[4])) return 1;
  return 0;
}

// A9 floors on the densitised cons Uc (8); Pprev (5) in, Pout (5) out.
// Returns 0 (nothing), 1 (floor event), 2 (failure).
template <class M>
ECHO_D int c2p_floors(const M& m, const EosP& e, double* Uc, const double* Pprev, double* Pout) {
  const double isg = 1.0 / m.sqrtg();
  double u[8];
#pragma unroll
  for (int q = 0; q < 8; q++) u[q] = M::kFlat ? Uc[q] : Uc[q] * isg;
  double pr[5];
  int status = c2p_newton(m, e, u, Pprev, pr);
  int ev = 0;
  if (status != 0) {
    double up[3] = {Pprev[1], Pprev[2], Pprev[3]}, ul[3];
    m.lower(up, ul);
    double Wp = sqrt(1.0 + up[0] * ul[0] + up[1] * ul[1] + up[2] * ul[2]);
    pr[1] = up[0]; pr[2] = up[1]; pr[3] = up[2];
    pr[0] = fmax(u[0] / Wp, e.rho_floor);
    pr[4] = fmax(Pprev[4], e.p_floor);
    ev = 2;
  } else {
    bool ch = false;
    if (pr[0] < e.rho_floor) { pr[0] = e.rho_floor; ch = true; }
    if (pr[4] < e.p_floor) { pr[4] = e.p_floor; ch = true; }
    double uu[3] = {pr[1], pr[2], pr[3]}, ul[3];
    m.lower(uu, ul);
    double Wu2 = 1.0 + uu[0] * ul[0] + uu[1] * ul[1] + uu[2] * ul[2];
    double Wu = sqrt(Wu2);
    if (Wu > e.w_max) {
      double sc = sqrt((e.w_max * e.w_max - 1.0) / (Wu * Wu - 1.0));
      pr[1] *= sc; pr[2] *= sc; pr[3] *= sc;
      ch = true;
    }
    ev = ch ? 1 : 0;
  }
  if (ev) {
    double p8[8] = {pr[0], pr[1], pr[2], pr[3], pr[4], u[5], u[6], u[7]};
    State s;
    make_state(m, e, p8, s);
    const double sg = m.sqrtg();
    Uc[0] = sg * s.D;
    Uc[1] = sg * s.S[0];
    Uc[2] = sg * s.S[1];
    Uc[3] = sg * s.S[2];
    Uc[4] = sg * s.tau;
  }
#pragma unroll
  for (int q = 0; q < 5; q++) Pout[q] = pr[q];
  return ev;
}

// ----------------------------------------------------- metric sources (a6)
// s(S_i) = 1/2 alpha W^{jk} d_i gamma_jk + S_j d_i beta^j - U d_i alpha
// s(tau) = 1/2 W^{ik} beta^j d_j gamma_ik + W_i^j d_j beta^i - S^j d_j alpha
// with W^{jk} = (Z+B^2) v^j v^k - (v.B)(B^j v^k + v^j B^k) - B^j B^k / W^2 + p_tot gamma^{jk};
// only d/dx1, d/dx2 are non-zero (stationary, axisymmetric metric).
ECHO_D void add_sources(const GenMet& m, const double* __restrict__ dr, const EosP& e, const double* pr, double* L) {
  State s;
  make_state(m, e, pr, s);
  const double ZB = s.tau + s.D + s.ptot;  // Z + B^2
  const double Ut = s.tau + s.D;
  double Wt[6];
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = a; b < 3; b++)
      Wt[sidx(a, b)] = ZB * s.v[a] * s.v[b] - s.vB * (s.B[a] * s.v[b] + s.v[a] * s.B[b]) - s.B[a] * s.B[b] * s.W2i +
                       s.ptot * m.gi[sidx(a, b)];
  double Su[3];
  m.raise(s.S, Su);
  // derivative records: dalpha[2], dbeta[2][3], dg[2][6]
  double dA[2], dB[2][3], dG[2][6];
#pragma unroll
  for (int k = 0; k < 2; k++) {
    dA[k] = __ldg(dr + k);
#pragma unroll
    for (int i = 0; i < 3; i++) dB[k][i] = __ldg(dr + 2 + 3 * k + i);
#pragma unroll
    for (int i = 0; i < 6; i++) dG[k][i] = __ldg(dr + 8 + 6 * k + i);
  }
  auto contract = [&](const double* dg) {  // W^{jk} dg_jk over the symmetric storage
    return Wt[0] * dg[0] + Wt[3] * dg[3] + Wt[5] * dg[5] + 2.0 * (Wt[1] * dg[1] + Wt[2] * dg[2] + Wt[4] * dg[4]);
  };
  const double sg = m.sqrtg();
  double e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll
  for (int k = 0; k < 2; k++) {
    double wdg = contract(dG[k]);
    double sdb = s.S[0] * dB[k][0] + s.S[1] * dB[k][1] + s.S[2] * dB[k][2];
    L[1 + k] += sg * (0.5 * m.a * wdg + sdb - Ut * dA[k]);
    e1 += 0.5 * m.b[k] * wdg;
    e3 += Su[k] * dA[k];
    // W_i^k d_k beta^i = sum_i gamma_il W^{lk} d_k beta^i
#pragma unroll
    for (int i = 0; i < 3; i++) {
      double Wik = m.g[sidx(i, 0)] * Wt[sidx(0, k)] + m.g[sidx(i, 1)] * Wt[sidx(1, k)] + m.g[sidx(i, 2)] * Wt[sidx(2, k)];
      e2 += Wik * dB[k][i];
    }
  }
  L[4] += sg * (e1 + e2 - e3);
}

// -------------------------------------------------------------- K3 kernel
template <bool KS, int MODE, bool DIVB_NONE>
__global__ void __launch_bounds__(kCellThreads, 3)
k_update(const GridP g, const EosP e, const MetTables mt, const int s, const double dt, const double* __restrict__ R,
         const double* __restrict__ Om, const double* Un, const double* Us, double* Uout, double* P,
         double* __restrict__ Lout, unsigned long long* counters) {
  const long long N = g.N;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = id < N;
  int ev = 0;
  if (active) {
    int i, j, k;
    cell_ijk(g, id, i, j, k);
    const auto m = MetAt<KS>::get(mt, i, j);
    double Pp[5];
#pragma unroll
    for (int q = 0; q < 5; q++) Pp[q] = P[q * N + id];
    double L[8];
    if (MODE != kModeC2P) {
#pragma unroll
      for (int q = 0; q < 5; q++) L[q] = R[q * N + id];
      if (KS) {
        double pr[8] = {Pp[0], Pp[1], Pp[2], Pp[3], Pp[4], 0.0, 0.0, 0.0};
        const double isg = 1.0 / m.sqrtg();
#pragma unroll
        for (int c = 0; c < 3; c++) pr[5 + c] = Us[(5 + c) * N + id] * isg;
        if constexpr (KS) add_sources(m, der_rec(mt, i, j), e, pr, L);
      }
      if (DIVB_NONE) {
#pragma unroll
        for (int c = 0; c < 3; c++) L[5 + c] = R[(5 + c) * N + id];
      } else {
        // L(sqrt(g) B^c) = -D_{c+1} Omega_{c+2} + D_{c+2} Omega_{c+1}   (A6, A26)
        const int ci[3] = {i, j, k};
        auto nb = [&](int ax, int d) {
          int cc[3] = {ci[0], ci[1], ci[2]};
          cc[ax] = map_index(cc[ax] + d, g.n[ax], g.bc[ax][0], g.bc[ax][1]);
          return ((long long)cc[2] * g.n[1] + cc[1]) * g.n[0] + cc[0];
        };
#pragma unroll
        for (int c = 0; c < 3; c++) {
          const int a1 = (c + 1) % 3, a2 = (c + 2) % 3;
          const double* Ok = Om + a2 * N;
          const double* Oj = Om + a1 * N;
          L[5 + c] = -(Ok[nb(a1, 1)] - Ok[nb(a1, -1)]) * (0.5 * g.idx[a1]) +
                     (Oj[nb(a2, 1)] - Oj[nb(a2, -1)]) * (0.5 * g.idx[a2]);
        }
      }
    }
    if (MODE == kModeRhs) {
#pragma unroll
      for (int q = 0; q < 8; q++) Lout[q * N + id] = L[q];
    } else {
      double Uo[8];
      if (MODE == kModeStage) {
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const double un = Un[q * N + id];
          if (s == 1) Uo[q] = un + dt * L[q];
          else if (s == 2) Uo[q] = 0.75 * un + 0.25 * (Us[q * N + id] + dt * L[q]);
          else Uo[q] = (1.0 / 3.0) * un + (2.0 / 3.0) * (Us[q * N + id] + dt * L[q]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; q++) Uo[q] = Un[q * N + id];
      }
      double Po[5];
      ev = c2p_floors(m, e, Uo, Pp, Po);
#pragma unroll
      for (int q = 0; q < 8; q++) Uout[q * N + id] = Uo[q];
#pragma unroll
      for (int q = 0; q < 5; q++) P[q * N + id] = Po[q];
    }
  }
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
                        const double* Om, const double* Un, const double* Us, double* Uout, double* P, double* Lout,
                        unsigned long long* cnt, cudaStream_t st) {
  unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  if (g.divb == 1)
    k_update<KS, MODE, true><<<blocks, kCellThreads, 0, st>>>(g, e, mt, s, dt, R, Om, Un, Us, Uout, P, Lout, cnt);
  else
    k_update<KS, MODE, false><<<blocks, kCellThreads, 0, st>>>(g, e, mt, s, dt, R, Om, Un, Us, Uout, P, Lout, cnt);
  return cudaGetLastError();
}

template <bool KS>
static cudaError_t upd1(int mode, const GridP& g, const EosP& e, const MetTables& mt, int s, double dt, const double* R,
                        const double* Om, const double* Un, const double* Us, double* Uout, double* P, double* Lout,
                        unsigned long long* cnt, cudaStream_t st) {
  if (mode == kModeRhs) return upd2<KS, kModeRhs>(g, e, mt, s, dt, R, Om, Un, Us, Uout, P, Lout, cnt, st);
  if (mode == kModeC2P) return upd2<KS, kModeC2P>(g, e, mt, s, dt, R, Om, Un, Us, Uout, P, Lout, cnt, st);
  return upd2<KS, kModeStage>(g, e, mt, s, dt, R, Om, Un, Us, Uout, P, Lout, cnt, st);
}

cudaError_t launch_update(int mode, bool ks, const GridP& g, const EosP& e, const MetTables& mt, int s, double dt,
                          const double* R, const double* Om, const double* Un, const double* Us, double* Uout,
                          double* P, double* Lout, unsigned long long* counters, cudaStream_t st) {
  if (ks) return upd1<true>(mode, g, e, mt, s, dt, R, Om, Un, Us, Uout, P, Lout, counters, st);
  return upd1<false>(mode, g, e, mt, s, dt, R, Om, Un, Us, Uout, P, Lout, counters, st);
}

// ------------------------------------------------------ CFL reduction (a9)
template <bool KS>
__global__ void __launch_bounds__(kCellThreads)
k_max_speed(const GridP g, const EosP e, const MetTables mt, const double* __restrict__ P,
            const double* __restrict__ U, unsigned long long* out) {
  const long long N = g.N;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double val = 0.0;
  if (id < N) {
    int i, j, k;
    cell_ijk(g, id, i, j, k);
    const auto m = MetAt<KS>::get(mt, i, j);
    double pr[8];
#pragma unroll
    for (int q = 0; q < 5; q++) pr[q] = P[q * N + id];
    const double isg = 1.0 / m.sqrtg();
#pragma unroll
    for (int c = 0; c < 3; c++) pr[5 + c] = KS ? U[(5 + c) * N + id] * isg : U[(5 + c) * N + id];
    State s;
    make_state(m, e, pr, s);
#pragma unroll
    for (int a = 0; a < 3; a++) {
      double lm, lp;
      speeds(m, e, pr, s, a, lm, lp);
      val += fmax(fabs(lp), fabs(lm)) * g.idx[a];
    }
    if (!(val == val)) val = __longlong_as_double(0x7ff0000000000000LL);  // NaN -> +inf (flagged on host)
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) val = fmax(val, __shfl_xor_sync(0xffffffffu, val, o));
  __shared__ double red[kCellThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = val;
  __syncthreads();
  if (threadIdx.x == 0) {
    double bm = red[0];
#pragma unroll
    for (int w = 1; w < kCellThreads / 32; w++) bm = fmax(bm, red[w]);
    atomicMax(out, (unsigned long long)__double_as_longlong(bm));  // non-negative doubles order as u64
  }
}

cudaError_t launch_max_speed(bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P,
                             const double* U, unsigned long long* out, cudaStream_t st) {
  unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  if (ks) k_max_speed<true><<<blocks, kCellThreads, 0, st>>>(g, e, mt, P, U, out);
  else k_max_speed<false><<<blocks, kCellThreads, 0, st>>>(g, e, mt, P, U, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------ a0 and back
template <bool KS>
__global__ void __launch_bounds__(kCellThreads)
k_prim2cons(const GridP g, const EosP e, const MetTables mt, const double* __restrict__ P8, double* __restrict__ P5,
            double* __restrict__ U8, long long* bad) {
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
  U8[0 * N + id] = sg * s.D;
#pragma unroll
  for (int c = 0; c < 3; c++) U8[(1 + c) * N + id] = sg * s.S[c];
  U8[4 * N + id] = sg * s.tau;
#pragma unroll
  for (int c = 0; c < 3; c++) U8[(5 + c) * N + id] = sg * pr[5 + c];
#pragma unroll
  for (int q = 0; q < 5; q++) P5[q * N + id] = pr[q];
}

cudaError_t launch_prim2cons(bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P8,
                             double* P5, double* U8, long long* bad, cudaStream_t st) {
  unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  if (ks) k_prim2cons<true><<<blocks, kCellThreads, 0, st>>>(g, e, mt, P8, P5, U8, bad);
  else k_prim2cons<false><<<blocks, kCellThreads, 0, st>>>(g, e, mt, P8, P5, U8, bad);
  return cudaGetLastError();
}

template <bool KS>
__global__ void __launch_bounds__(kCellThreads)
k_get_prims(const GridP g, const MetTables mt, const double* __restrict__ P5, const double* __restrict__ U8,
            double* __restrict__ P8) {
  const long long N = g.N;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= N) return;
  int i, j, k;
  cell_ijk(g, id, i, j, k);
  const auto m = MetAt<KS>::get(mt, i, j);
  double u[3] = {P5[1 * N + id], P5[2 * N + id], P5[3 * N + id]}, ul[3];
  m.lower(u, ul);
  const double iW = rsqrt(1.0 + u[0] * ul[0] + u[1] * ul[1] + u[2] * ul[2]);
  P8[id] = P5[id];
#pragma unroll
  for (int c = 0; c < 3; c++) P8[(1 + c) * N + id] = u[c] * iW;
  P8[4 * N + id] = P5[4 * N + id];
  const double isg = 1.0 / m.sqrtg();
#pragma unroll
  for (int c = 0; c < 3; c++) P8[(5 + c) * N + id] = KS ? U8[(5 + c) * N + id] * isg : U8[(5 + c) * N + id];
}

cudaError_t launch_get_prims(bool ks, const GridP& g, const MetTables& mt, const double* P5, const double* U8,
                             double* P8, cudaStream_t st) {
  unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  if (ks) k_get_prims<true><<<blocks, kCellThreads, 0, st>>>(g, mt, P5, U8, P8);
  else k_get_prims<false><<<blocks, kCellThreads, 0, st>>>(g, mt, P5, U8, P8);
  return cudaGetLastError();
}

}  // namespace echo
