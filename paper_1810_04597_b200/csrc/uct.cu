// uct.cu — the staggered-field update of divb = 2 (UCT; DESIGN.md
// readings A37-A43): periodic or outflow axes (A42: on an outflow side the staggered
// quantities take the nearest owned face / edge, as the cell ghosts do, A13), any metric
// (A43: the face data carry V = alpha v - beta, so the EMF step needs no metric).
//
// State: Bst record array, slots 0..2 = b^n, 3..5 = b^s, where b^a = sqrt(gamma) B^a at
// the face i_a + 1/2 owned by cell i.  The sweeps (march.cu, DM = 2) take the normal
// field of every face from the stage-input b and leave per owned face, in FS[a] (one
// record array per axis), the face data of the EMF step: v^1..3 of the left and of the
// right HLL state (V = alpha v - beta), a+ = S_R, a- = -S_L.  Then per stage:
//   k_uct_emf     E^c at the edge (i_p + 1/2, i_q + 1/2, i_c) owned by each cell, (c, p, q)
//                 cyclic: 4 quadrant states from double reconstructions of the face data
//                 (A38) combined by the UCT-HLL formula (A39, A40)          -> Ed slots 0..2
//   k_uct_induct  L(b^p) = -delta_q Dh_q E^c + delta_c Dh_c E^q (A41) and the literal RK
//                 form of stage s per face (or L(b) alone for echo_rhs)     -> Bst
//   k_uct_cell    hydro RK combine from the sweeps' rhs (+ KS sources), U_B = I6(b) (A37),
//                 con2prim + floors, the CFL rate of the new state           -> U, P
// One thread per cell; neighbours through the ghost index map (L1/L2).
#include <cuda_runtime.h>

#include "cell_physics.cuh"
#include "echo_dev.cuh"
#include "echo_kernels.h"

namespace echo {
namespace {

ECHO_D long long rec_shift(const GridP& g, const int x[3], int a, int d) {
  int y[3] = {x[0], x[1], x[2]};
  y[a] = map_index(y[a] + d, g.n[a], g.bc[a][0], g.bc[a][1]);  // A13 / A42: wrap or nearest owned
  return rec_base(g, y[0], y[1], y[2]);
}

// the two one-sided values at +1/2 from samples f[0..5] at -2..3 (A38): lo from f[0..4],
// hi the mirror from f[5..1] (rec_both of the cells at 0 and +1; the unused halves are dead code)
template <int REC>
ECHO_D void rec_pair(const double f[6], double& lo, double& hi) {
  if constexpr (REC == 0) {  // WENO5 point form: one face each (no shared second normalisation)
    lo = weno5_one(f[0], f[1], f[2], f[3], f[4]);
    hi = weno5_one(f[5], f[4], f[3], f[2], f[1]);
  } else {
    double dead0, dead1;
    rec_both<REC>(f[0], f[1], f[2], f[3], f[4], lo, dead0);
    rec_both<REC>(f[1], f[2], f[3], f[4], f[5], dead1, hi);
  }
}

// A38 quadrant velocities (V^p, V^q) = the mean of the two double reconstructions, A39
// quadrant EMFs E = V^q b^p - V^p b^q and the UCT-HLL combination.  pS/pN[side][k]: the p-face
// state side (0 W, 1 E) component k (0 p, 1 q) at the edge from below / above along q;
// qW/qE[side][k]: the q-face state side (0 S, 1 N) from the W / E side along p.
ECHO_D double emf_combine(const double pS[2][2], const double pN[2][2], const double qW[2][2], const double qE[2][2],
                          double bpS, double bpN, double bqW, double bqE, double app, double apm, double aqp,
                          double aqm) {
  double v[4][2];
#pragma unroll
  for (int k = 0; k < 2; k++) {
    v[0][k] = 0.5 * (pS[0][k] + qW[0][k]);  // WS
    v[1][k] = 0.5 * (pN[0][k] + qW[1][k]);  // WN
    v[2][k] = 0.5 * (pS[1][k] + qE[0][k]);  // ES
    v[3][k] = 0.5 * (pN[1][k] + qE[1][k]);  // EN
  }
  const double EWS = v[0][1] * bpS - v[0][0] * bqW;
  const double EWN = v[1][1] * bpN - v[1][0] * bqW;
  const double EES = v[2][1] * bpS - v[2][0] * bqE;
  const double EEN = v[3][1] * bpN - v[3][0] * bqE;
  const double sp = app + apm, sq = aqp + aqm;
  if (sp > 0.0 && sq > 0.0) {
    const double isp = frcp(sp), isq = frcp(sq);  // (MUFU seed + refinement, A32)
    return (app * (aqp * EWS + aqm * EWN) + apm * (aqp * EES + aqm * EEN)) * (isp * isq) +
           app * apm * (bqE - bqW) * isp - aqp * aqm * (bpN - bpS) * isq;
  }
  return 0.25 * (EWS + EWN + EES + EEN);  // unreachable for p > 0 (A4): central average
}

// E^CC at the edge owned by cell x (one component per thread: the three are independent,
// and a thread holding all three needs ~170 registers, one CTA per SM)
template <int REC, int CC>
ECHO_D double uct_emf_one(const GridP& g, const double* const FS[3], const double* __restrict__ Bin, const int x[3],
                          long long rb) {
  constexpr int p = (CC + 1) % 3, q = (CC + 2) % 3;
  const int comp[2] = {p, q};
  const long long vs = g.vs;
  double f[6];
  long long oq[6], op[6];
#pragma unroll
  for (int m = 0; m < 6; m++) {
    oq[m] = rec_shift(g, x, q, m - 2);
    op[m] = rec_shift(g, x, p, m - 2);
  }
  // p-face states (W: slots 0..2, E: 3..5) along q -> S, N; q-face states (S, N) along p -> W, E
  double pS[2][2], pN[2][2], qW[2][2], qE[2][2];
#pragma unroll
  for (int side = 0; side < 2; side++)
#pragma unroll
    for (int k = 0; k < 2; k++) {
#pragma unroll
      for (int m = 0; m < 6; m++) f[m] = __ldg(FS[p] + oq[m] + (3 * side + comp[k]) * vs);
      rec_pair<REC>(f, pS[side][k], pN[side][k]);
#pragma unroll
      for (int m = 0; m < 6; m++) f[m] = __ldg(FS[q] + op[m] + (3 * side + comp[k]) * vs);
      rec_pair<REC>(f, qW[side][k], qE[side][k]);
    }
  double bpS, bpN, bqW, bqE;
#pragma unroll
  for (int m = 0; m < 6; m++) f[m] = __ldg(Bin + oq[m] + p * vs);
  rec_pair<REC>(f, bpS, bpN);
#pragma unroll
  for (int m = 0; m < 6; m++) f[m] = __ldg(Bin + op[m] + q * vs);
  rec_pair<REC>(f, bqW, bqE);
  // A40: max over the two faces meeting at the edge (oq[3] = +1 along q, op[3] = +1 along p)
  const double app = fmax(__ldg(FS[p] + rb + 6 * vs), __ldg(FS[p] + oq[3] + 6 * vs));
  const double apm = fmax(__ldg(FS[p] + rb + 7 * vs), __ldg(FS[p] + oq[3] + 7 * vs));
  const double aqp = fmax(__ldg(FS[q] + rb + 6 * vs), __ldg(FS[q] + op[3] + 6 * vs));
  const double aqm = fmax(__ldg(FS[q] + rb + 7 * vs), __ldg(FS[q] + op[3] + 7 * vs));
  return emf_combine(pS, pN, qW, qE, bpS, bpN, bqW, bqE, app, apm, aqp, aqm);
}

// grid (cells / kCellThreads, 3): blockIdx.y = the EMF component
// -DECHO_EMF_BPS=n: the E^z kernel compiled for n CTAs per SM (default: ptxas's own budget)
#ifdef ECHO_EMF_BPS
#define ECHO_EMF_BOUNDS __launch_bounds__(kCellThreads, ECHO_EMF_BPS)
#else
#define ECHO_EMF_BOUNDS __launch_bounds__(kCellThreads)
#endif
template <int REC>
__global__ void ECHO_EMF_BOUNDS
k_uct_emf(const GridP g, const double* __restrict__ FSx, const double* __restrict__ FSy,
          const double* __restrict__ FSz, const double* __restrict__ Bin, double* __restrict__ Ed, int cc0) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= g.N) return;
  int x[3];
  cell_ijk(g, id, x[0], x[1], x[2]);
  const double* FS[3] = {FSx, FSy, FSz};
  const long long rb = rec_base(g, x[0], x[1], x[2]);
  const int cc = blockIdx.y + cc0;
  double E;
  if (cc == 0) E = uct_emf_one<REC, 0>(g, FS, Bin, x, rb);
  else if (cc == 1) E = uct_emf_one<REC, 1>(g, FS, Bin, x, rb);
  else E = uct_emf_one<REC, 2>(g, FS, Bin, x, rb);
  Ed[rb + cc * g.vs] = E;
}

// E^x (CC = 0: q = z) and E^y (CC = 1: p = z) marching along z: one thread per (i, j)
// column and z segment keeps the samples along z of the face data and b that these two
// components reconstruct along z in 6-entry register windows (one new load per stream and
// step instead of six from planes far apart); the in-plane samples (z-face data and b^z along
// y or x) are loaded per step.  Same arithmetic as uct_emf_one.
constexpr int kZSeg = 16;  // planes per thread
#ifndef ECHO_ZSEG_IC
#define ECHO_ZSEG_IC 16  // planes per thread of the induction and cell-update marches
#endif
constexpr int kZSegIC = ECHO_ZSEG_IC;
#ifndef ECHO_INDUCT_BPS
#define ECHO_INDUCT_BPS 8  // CTAs per SM the induction march is compiled for (64 registers;
                           // 0: ptxas's own budget; profiles/r02_uct_ic_ab)
#endif
#if ECHO_INDUCT_BPS > 0
#define ECHO_INDUCT_BOUNDS __launch_bounds__(128, ECHO_INDUCT_BPS)
#else
#define ECHO_INDUCT_BOUNDS __launch_bounds__(128)
#endif
#ifndef ECHO_UCT_CELL_BPS
#define ECHO_UCT_CELL_BPS 6  // CTAs per SM of the flat-metric cell-update march (80 registers)
#endif
#ifndef ECHO_EMF_ZM_BPS
#define ECHO_EMF_ZM_BPS 3  // (168 registers, 52-104 B of spills; 2 CTAs/SM: variant "emf2" below)
#endif
template <int REC, int CC>
__global__ void __launch_bounds__(128, ECHO_EMF_ZM_BPS)
k_uct_emf_zm(const GridP g, const double* __restrict__ FSx, const double* __restrict__ FSy,
             const double* __restrict__ FSz, const double* __restrict__ Bin, double* __restrict__ Ed, const int kzb,
             const int kze) {
  constexpr int p = (CC + 1) % 3, q = (CC + 2) % 3;
  constexpr bool ZQ = (q == 2);   // CC 0: z is q; CC 1: z is p
  constexpr int ip = ZQ ? p : q;  // the in-plane direction of the other pairs (y for CC 0, x for CC 1)
  const double* __restrict__ Fz = (CC == 0) ? FSy : FSx;  // face data reconstructed along z
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= g.n[0]) return;
  // planes kzb .. kze - 1: the owned ones, and in slab mode (stored ghost planes) 3 more below and
  // 2 above, whose EMFs the induction's DER along z reads
  const int k0 = kzb + blockIdx.z * kZSeg;
  const int k1 = min(k0 + kZSeg, kze);
  const long long vs = g.vs;
  // along-z windows: 4 face-data streams (slot 3 side + comp), b (slot bz), speeds (slots 6, 7) at k, k+1
  const int comp[2] = {p, q};
  const int bz = ZQ ? p : q;
  double wv[4][6], wb[6], ws[2][2];
  {
    int x[3] = {i, j, k0};
#pragma unroll
    for (int m = 0; m < 6; m++) {
      const long long o = rec_shift(g, x, 2, m - 2);
#pragma unroll
      for (int s2 = 0; s2 < 4; s2++) wv[s2][m] = __ldg(Fz + o + (3 * (s2 >> 1) + comp[s2 & 1]) * vs);
      wb[m] = __ldg(Bin + o + bz * vs);
    }
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const long long o = rec_shift(g, x, 2, h);
      ws[0][h] = __ldg(Fz + o + 6 * vs);
      ws[1][h] = __ldg(Fz + o + 7 * vs);
    }
  }
  for (int k = k0; k < k1; k++) {
    const int x[3] = {i, j, k};
    const long long rb = rec_base(g, i, j, k);
    // pairs along z from the windows
    double zlo[2][2], zhi[2][2];
#pragma unroll
    for (int s2 = 0; s2 < 4; s2++) rec_pair<REC>(wv[s2], zlo[s2 >> 1][s2 & 1], zhi[s2 >> 1][s2 & 1]);
    double bzlo, bzhi;
    rec_pair<REC>(wb, bzlo, bzhi);
    const double az_p = fmax(ws[0][0], ws[0][1]), az_m = fmax(ws[1][0], ws[1][1]);
    // in-plane pairs: z-face data and b^z along ip
    long long oi[6];
#pragma unroll
    for (int m = 0; m < 6; m++) oi[m] = rec_shift(g, x, ip, m - 2);
    double ilo[2][2], ihi[2][2], f[6];
#pragma unroll
    for (int side = 0; side < 2; side++)
#pragma unroll
      for (int kk = 0; kk < 2; kk++) {
#pragma unroll
        for (int m = 0; m < 6; m++) f[m] = __ldg(FSz + oi[m] + (3 * side + comp[kk]) * vs);
        rec_pair<REC>(f, ilo[side][kk], ihi[side][kk]);
      }
    double bilo, bihi;
#pragma unroll
    for (int m = 0; m < 6; m++) f[m] = __ldg(Bin + oi[m] + 2 * vs);
    rec_pair<REC>(f, bilo, bihi);
    const double ai_p = fmax(__ldg(FSz + rb + 6 * vs), __ldg(FSz + oi[3] + 6 * vs));
    const double ai_m = fmax(__ldg(FSz + rb + 7 * vs), __ldg(FSz + oi[3] + 7 * vs));
    double E;
    if constexpr (ZQ)  // z-pairs: p-face (y-face) states along q = z; in-plane: q-face (z-face) states along p = y
      E = emf_combine(zlo, zhi, ilo, ihi, bzlo, bzhi, bilo, bihi, az_p, az_m, ai_p, ai_m);
    else               // z-pairs: q-face (x-face) states along p = z; in-plane: p-face (z-face) states along q = x
      E = emf_combine(ilo, ihi, zlo, zhi, bilo, bihi, bzlo, bzhi, ai_p, ai_m, az_p, az_m);
    Ed[rb + CC * vs] = E;
    if (k + 1 < k1) {  // slide the windows by one plane
      const long long o = rec_shift(g, x, 2, 4);
#pragma unroll
      for (int s2 = 0; s2 < 4; s2++) {
#pragma unroll
        for (int m = 0; m < 5; m++) wv[s2][m] = wv[s2][m + 1];
        wv[s2][5] = __ldg(Fz + o + (3 * (s2 >> 1) + comp[s2 & 1]) * vs);
      }
#pragma unroll
      for (int m = 0; m < 5; m++) wb[m] = wb[m + 1];
      wb[5] = __ldg(Bin + o + bz * vs);
      const long long o2 = rec_shift(g, x, 2, 2);
      ws[0][0] = ws[0][1];
      ws[1][0] = ws[1][1];
      ws[0][1] = __ldg(Fz + o2 + 6 * vs);
      ws[1][1] = __ldg(Fz + o2 + 7 * vs);
    }
  }
}

// A41 induction of the three faces owned by a cell; MODE 0: RK stage s into Bst (dt from
// dtp when set; halted loop: nothing), MODE 1: L(b) into Lout[5 + a][cell] (echo_rhs)
template <int DER>
__global__ void __launch_bounds__(kCellThreads)
k_uct_induct(const GridP g, int mode, int s, double dt, const double* dtp, const double* __restrict__ Ed,
             double* Bst, double* __restrict__ Lout) {
  if (dtp) {
    if (dtp[1] != 0.0) return;
    dt = dtp[0];
  }
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= g.N) return;
  int x[3];
  cell_ijk(g, id, x[0], x[1], x[2]);
  const long long vs = g.vs;
  const long long rb = rec_base(g, x[0], x[1], x[2]);
#pragma unroll
  for (int p = 0; p < 3; p++) {
    const int cc = (p + 2) % 3, q = (p + 1) % 3;
    double Eq[6], Ec[6];  // E^cc along q, E^q along cc: samples -3..2
#pragma unroll
    for (int m = 0; m < 6; m++) {
      Eq[m] = __ldg(Ed + rec_shift(g, x, q, m - 3) + cc * vs);
      Ec[m] = __ldg(Ed + rec_shift(g, x, cc, m - 3) + q * vs);
    }
    const double Lb = -(der5<DER>(Eq[1], Eq[2], Eq[3], Eq[4], Eq[5]) - der5<DER>(Eq[0], Eq[1], Eq[2], Eq[3], Eq[4])) *
                          g.idx[q] +
                      (der5<DER>(Ec[1], Ec[2], Ec[3], Ec[4], Ec[5]) - der5<DER>(Ec[0], Ec[1], Ec[2], Ec[3], Ec[4])) *
                          g.idx[cc];
    if (mode == 1) {
      Lout[(5 + p) * g.N + id] = Lb;
      continue;
    }
    const double bn = Bst[rb + p * vs];
    double bo;
    if (s == 1) {
      bo = bn + dt * Lb;
      Bst[rb + (3 + p) * vs] = bo;
    } else if (s == 2) {
      bo = 0.75 * bn + 0.25 * (Bst[rb + (3 + p) * vs] + dt * Lb);
      Bst[rb + (3 + p) * vs] = bo;
    } else {
      bo = (1.0 / 3.0) * bn + (2.0 / 3.0) * (Bst[rb + (3 + p) * vs] + dt * Lb);
      Bst[rb + p * vs] = bo;
    }
  }
}

// The same induction marching along z: one thread per (i, j) column and kZSeg planes keeps
// the two along-z EMF streams (E^y for b^x, E^x for b^y) in 6-entry register windows.
template <int DER>
__global__ void ECHO_INDUCT_BOUNDS
k_uct_induct_zm(const GridP g, int mode, int s, double dt, const double* dtp, const double* __restrict__ Ed,
                double* Bst, double* __restrict__ Lout) {
  if (dtp) {
    if (dtp[1] != 0.0) return;
    dt = dtp[0];
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= g.n[0]) return;
  const int k0 = blockIdx.z * kZSegIC;
  const int k1 = min(k0 + kZSegIC, g.n[2]);
  const long long vs = g.vs;
  double wy[6], wx[6];  // E^y and E^x at (i, j, k-3 .. k+2)
  {
    const int x[3] = {i, j, k0};
#pragma unroll
    for (int m = 0; m < 6; m++) {
      const long long o = rec_shift(g, x, 2, m - 3);
      wy[m] = __ldg(Ed + o + 1 * vs);
      wx[m] = __ldg(Ed + o + 0 * vs);
    }
  }
  for (int k = k0; k < k1; k++) {
    const int x[3] = {i, j, k};
    const long long rb = rec_base(g, i, j, k);
    const long long id = ((long long)k * g.n[1] + j) * g.n[0] + i;
    double Lb[3];
#pragma unroll
    for (int p = 0; p < 3; p++) {
      const int cc = (p + 2) % 3, q = (p + 1) % 3;
      double Eq[6], Ec[6];  // E^cc along q, E^q along cc: samples -3..2
#pragma unroll
      for (int m = 0; m < 6; m++) {
        if (q == 2) Eq[m] = wx[m];  // p = y: E^x along z
        else Eq[m] = __ldg(Ed + rec_shift(g, x, q, m - 3) + cc * vs);
        if (cc == 2) Ec[m] = wy[m];  // p = x: E^y along z
        else Ec[m] = __ldg(Ed + rec_shift(g, x, cc, m - 3) + q * vs);
      }
      Lb[p] = -(der5<DER>(Eq[1], Eq[2], Eq[3], Eq[4], Eq[5]) - der5<DER>(Eq[0], Eq[1], Eq[2], Eq[3], Eq[4])) * g.idx[q] +
              (der5<DER>(Ec[1], Ec[2], Ec[3], Ec[4], Ec[5]) - der5<DER>(Ec[0], Ec[1], Ec[2], Ec[3], Ec[4])) * g.idx[cc];
    }
#pragma unroll
    for (int p = 0; p < 3; p++) {
      if (mode == 1) {
        Lout[(5 + p) * g.N + id] = Lb[p];
        continue;
      }
      const double bn = Bst[rb + p * vs];
      if (s == 1) {
        Bst[rb + (3 + p) * vs] = bn + dt * Lb[p];
      } else if (s == 2) {
        Bst[rb + (3 + p) * vs] = 0.75 * bn + 0.25 * (Bst[rb + (3 + p) * vs] + dt * Lb[p]);
      } else {
        Bst[rb + p * vs] = (1.0 / 3.0) * bn + (2.0 / 3.0) * (Bst[rb + (3 + p) * vs] + dt * Lb[p]);
      }
    }
    if (k + 1 < k1) {  // slide: the next plane's window ends at k + 3
      const long long o = rec_shift(g, x, 2, 3);
#pragma unroll
      for (int m = 0; m < 5; m++) {
        wy[m] = wy[m + 1];
        wx[m] = wx[m + 1];
      }
      wy[5] = __ldg(Ed + o + 1 * vs);
      wx[5] = __ldg(Ed + o + 0 * vs);
    }
  }
}

// A37: I6 of the face field at slot offset `slot` of Bst, per component, at cell x
ECHO_D void centre_field(const GridP& g, const double* __restrict__ Bst, int slot, const int x[3], double Bc[3]) {
  const long long vs = g.vs;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    double f[6];
#pragma unroll
    for (int m = 0; m < 6; m++) f[m] = Bst[rec_shift(g, x, a, m - 3) + (slot + a) * vs];
    Bc[a] = fma(3.0, f[0] + f[5], fma(-25.0, f[1] + f[4], 150.0 * (f[2] + f[3]))) * (1.0 / 256.0);
  }
}

// one cell of the UCT update (Bc = I6 of the field this stage wrote): hydro RK combine
// (+ KS sources), U_B = Bc, con2prim + floors; returns the A9 event code
template <bool KS>
ECHO_D int uct_cell_body(const GridP& g, const EosP& e, const MetTables& mt, int s, double dt,
                         const double* __restrict__ R, const double* Un, const double* Us, double* Uout, double* P,
                         const int x[3], const double Bc[3], bool want_rate, double& rate) {
  const long long rb = rec_base(g, x[0], x[1], x[2]), vs = g.vs;
  const auto m = MetAt<KS>::get(mt, x[0], x[1]);
  double Pp[8], Uo[8], L[8];
  double Z0;
  if (KS) {
    ld8(P + rb, vs, Pp);  // B for the sources
    Z0 = guess_Z(m, e, Pp);
  } else {
    Z0 = P[rb + kSlotZ * vs];  // the stored Newton guess
  }
#pragma unroll
  for (int q = 0; q < 5; q++) L[q] = R[rb + q * vs];
  if constexpr (KS) add_sources(m, der_rec(mt, x[0], x[1]), e, Pp, L);  // a6
#pragma unroll
  for (int q = 0; q < 5; q++) Uo[q] = Un[rb + q * vs];  // hydro only: U_B comes from b
  if (s == 1) {
#pragma unroll
    for (int q = 0; q < 5; q++) Uo[q] = Uo[q] + dt * L[q];
  } else {
    const double c0 = (s == 2) ? 0.75 : (1.0 / 3.0), c1 = (s == 2) ? 0.25 : (2.0 / 3.0);
#pragma unroll
    for (int q = 0; q < 5; q++) Uo[q] = c0 * Uo[q] + c1 * (Us[rb + q * vs] + dt * L[q]);
  }
#pragma unroll
  for (int a = 0; a < 3; a++) Uo[5 + a] = Bc[a];
  double Po[8];
  const int ev = c2p_floors(m, e, Uo, Z0, [&](double* pv) {
#pragma unroll
    for (int v = 0; v < 5; v++) pv[v] = KS ? Pp[v] : P[rb + v * vs];
  }, Po);
  const double isg = !KS ? 1.0 : frcp(m.sqrtg());
#pragma unroll
  for (int a = 0; a < 3; a++) Po[5 + a] = Uo[5 + a] * isg;
  st8(Uout + rb, vs, Uo);
  st_prims<KS>(P + rb, vs, Po);
  if (!KS) P[rb + kSlotZ * vs] = guess_Z(m, e, Po);
  if (want_rate) rate = fmax(rate, cfl_rate(m, g, e, Po));
  return ev;
}

// block-level max of the CFL rate -> one atomic; warp-aggregated event counters
ECHO_D void uct_reduce(double rate, int nfl, int nfa, unsigned long long* counters, unsigned long long* cfl_out) {
  if (cfl_out) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rate = fmax(rate, __shfl_xor_sync(0xffffffffu, rate, o));
    __shared__ double red[32];
    const int nw = (blockDim.x + 31) >> 5;
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = rate;
    __syncthreads();
    if (threadIdx.x == 0) {
      double bm = red[0];
      for (int w = 1; w < nw; w++) bm = fmax(bm, red[w]);
      atomicMax(cfl_out, (unsigned long long)__double_as_longlong(bm));
    }
  }
  const unsigned fl = __reduce_add_sync(0xffffffffu, (unsigned)nfl);
  const unsigned fa = __reduce_add_sync(0xffffffffu, (unsigned)nfa);
  if ((threadIdx.x & 31) == 0) {
    if (fl) atomicAdd(counters + 0, (unsigned long long)fl);
    if (fa) atomicAdd(counters + 1, (unsigned long long)fa);
  }
}

template <bool KS>
__global__ void __launch_bounds__(kCellThreads, KS ? 2 : 3)  // KS: spill-free at 128 registers
k_uct_cell(const GridP g, const EosP e, const MetTables mt, int s, double dt, const double* dtp,
           const double* __restrict__ R, const double* Un, const double* Us, double* Uout, double* P,
           const double* __restrict__ Bst, unsigned long long* counters, unsigned long long* cfl_out) {
  if (dtp) {
    if (dtp[1] != 0.0) return;  // uniform over the grid (no thread left at a block barrier)
    dt = dtp[0];
  }
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int ev = 0;
  double rate = 0.0;
  if (id < g.N) {
    int x[3];
    cell_ijk(g, id, x[0], x[1], x[2]);
    double Bc[3];
    centre_field(g, Bst, s == 3 ? 0 : 3, x, Bc);  // the field this stage just wrote
    ev = uct_cell_body<KS>(g, e, mt, s, dt, R, Un, Us, Uout, P, x, Bc, cfl_out != nullptr, rate);
  }
  uct_reduce(rate, ev == 1, ev == 2, counters, cfl_out);
}

// the same marching along z (one thread per (i, j) column and kZSeg planes): the centring's
// b^z samples along z come from a 6-entry register window
template <bool KS>
__global__ void __launch_bounds__(128, KS ? 4 : ECHO_UCT_CELL_BPS)  // KS: spill-free at 128 registers
k_uct_cell_zm(const GridP g, const EosP e, const MetTables mt, int s, double dt, const double* dtp,
              const double* __restrict__ R, const double* Un, const double* Us, double* Uout, double* P,
              const double* __restrict__ Bst, unsigned long long* counters, unsigned long long* cfl_out) {
  if (dtp) {
    if (dtp[1] != 0.0) return;  // uniform over the grid
    dt = dtp[0];
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k0 = blockIdx.z * kZSegIC;
  const int k1 = min(k0 + kZSegIC, g.n[2]);
  const int slot = s == 3 ? 0 : 3;
  const long long vs = g.vs;
  int nfl = 0, nfa = 0;
  double rate = 0.0;
  if (i < g.n[0]) {
    double wz[6];  // b^z at faces k-3 .. k+2 (owned by cells k-3 .. k+2)
    {
      const int x[3] = {i, j, k0};
#pragma unroll
      for (int m = 0; m < 6; m++) wz[m] = Bst[rec_shift(g, x, 2, m - 3) + (slot + 2) * vs];
    }
    for (int k = k0; k < k1; k++) {
      const int x[3] = {i, j, k};
      double Bc[3];
#pragma unroll
      for (int a = 0; a < 2; a++) {
        double f[6];
#pragma unroll
        for (int m = 0; m < 6; m++) f[m] = Bst[rec_shift(g, x, a, m - 3) + (slot + a) * vs];
        Bc[a] = fma(3.0, f[0] + f[5], fma(-25.0, f[1] + f[4], 150.0 * (f[2] + f[3]))) * (1.0 / 256.0);
      }
      Bc[2] = fma(3.0, wz[0] + wz[5], fma(-25.0, wz[1] + wz[4], 150.0 * (wz[2] + wz[3]))) * (1.0 / 256.0);
      const int ev = uct_cell_body<KS>(g, e, mt, s, dt, R, Un, Us, Uout, P, x, Bc, cfl_out != nullptr, rate);
      nfl += ev == 1;
      nfa += ev == 2;
      if (k + 1 < k1) {
#pragma unroll
        for (int m = 0; m < 5; m++) wz[m] = wz[m + 1];
        wz[5] = Bst[rec_shift(g, x, 2, 3) + (slot + 2) * vs];
      }
    }
  }
  uct_reduce(rate, nfl, nfa, counters, cfl_out);
}

// set: U_B = I6(b^n) and U from the state's hydro primitives (a0 with the new field)
template <bool KS>
__global__ void __launch_bounds__(kCellThreads)
k_uct_centre_p2c(const GridP g, const EosP e, const MetTables mt, double* __restrict__ P, double* __restrict__ U,
                 const double* __restrict__ Bst) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= g.N) return;
  int x[3];
  cell_ijk(g, id, x[0], x[1], x[2]);
  const long long rb = rec_base(g, x[0], x[1], x[2]), vs = g.vs;
  const auto m = MetAt<KS>::get(mt, x[0], x[1]);
  double pr[8], Bc[3];
#pragma unroll
  for (int v = 0; v < 5; v++) pr[v] = P[rb + v * vs];
  centre_field(g, Bst, 0, x, Bc);
  const double sg = m.sqrtg(), isg = !KS ? 1.0 : 1.0 / sg;
#pragma unroll
  for (int a = 0; a < 3; a++) pr[5 + a] = Bc[a] * isg;
  State st;
  make_state(m, e, pr, st);
  double u[8] = {sg * st.D, sg * st.S[0], sg * st.S[1], sg * st.S[2], sg * st.tau, Bc[0], Bc[1], Bc[2]};
  st8(U + rb, vs, u);
  if (KS) st8(P + rb, vs, pr);
}

#ifndef ECHO_EMF_ZMARCH
#define ECHO_EMF_ZMARCH 1
#endif
template <int REC>
cudaError_t emf_rec(const GridP& g, const double* const FS[3], const double* Bin, double* Ed, cudaStream_t st) {
  if (ECHO_EMF_ZMARCH) {  // E^x, E^y marching along z; E^z one thread per edge
    const int kzb = g.zhalo ? -3 : 0, kze = g.n[2] + (g.zhalo ? 2 : 0);
    const dim3 zb((unsigned)((g.n[0] + 127) / 128), (unsigned)g.n[1], (unsigned)((kze - kzb + kZSeg - 1) / kZSeg));
    k_uct_emf_zm<REC, 0><<<zb, 128, 0, st>>>(g, FS[0], FS[1], FS[2], Bin, Ed, kzb, kze);
    k_uct_emf_zm<REC, 1><<<zb, 128, 0, st>>>(g, FS[0], FS[1], FS[2], Bin, Ed, kzb, kze);
    const dim3 blocks((unsigned)((g.N + kCellThreads - 1) / kCellThreads), 1);
    k_uct_emf<REC><<<blocks, kCellThreads, 0, st>>>(g, FS[0], FS[1], FS[2], Bin, Ed, 2);
  } else {
    if (g.zhalo) return cudaErrorInvalidValue;  // slab mode needs the z-march (ghost-plane EMFs)
    const dim3 blocks((unsigned)((g.N + kCellThreads - 1) / kCellThreads), 3);
    k_uct_emf<REC><<<blocks, kCellThreads, 0, st>>>(g, FS[0], FS[1], FS[2], Bin, Ed, 0);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_uct_emf(const GridP& g, const double* const FS[3], const double* Bin, double* Ed, cudaStream_t st) {
  switch (g.rec) {
    case 1: return emf_rec<1>(g, FS, Bin, Ed, st);
    case 2: return emf_rec<2>(g, FS, Bin, Ed, st);
    case 3: return emf_rec<3>(g, FS, Bin, Ed, st);
    case 4: return emf_rec<4>(g, FS, Bin, Ed, st);
    case 5: return emf_rec<5>(g, FS, Bin, Ed, st);
    default: return emf_rec<0>(g, FS, Bin, Ed, st);
  }
}

#ifndef ECHO_INDUCT_ZMARCH
#define ECHO_INDUCT_ZMARCH 1
#endif
cudaError_t launch_uct_induct(const GridP& g, int mode, int s, double dt, const double* dtp, const double* Ed,
                              double* Bst, double* Lout, cudaStream_t st) {
  if (ECHO_INDUCT_ZMARCH) {
    const dim3 zb((unsigned)((g.n[0] + 127) / 128), (unsigned)g.n[1], (unsigned)((g.n[2] + kZSegIC - 1) / kZSegIC));
    if (g.der == 4) k_uct_induct_zm<4><<<zb, 128, 0, st>>>(g, mode, s, dt, dtp, Ed, Bst, Lout);
    else if (g.der == 2) k_uct_induct_zm<2><<<zb, 128, 0, st>>>(g, mode, s, dt, dtp, Ed, Bst, Lout);
    else k_uct_induct_zm<6><<<zb, 128, 0, st>>>(g, mode, s, dt, dtp, Ed, Bst, Lout);
    return cudaGetLastError();
  }
  const unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  if (g.der == 4) k_uct_induct<4><<<blocks, kCellThreads, 0, st>>>(g, mode, s, dt, dtp, Ed, Bst, Lout);
  else if (g.der == 2) k_uct_induct<2><<<blocks, kCellThreads, 0, st>>>(g, mode, s, dt, dtp, Ed, Bst, Lout);
  else k_uct_induct<6><<<blocks, kCellThreads, 0, st>>>(g, mode, s, dt, dtp, Ed, Bst, Lout);
  return cudaGetLastError();
}

#ifndef ECHO_CELL_ZMARCH
#define ECHO_CELL_ZMARCH 1
#endif
cudaError_t launch_uct_cell(bool ks, const GridP& g, const EosP& e, const MetTables& mt, int s, double dt,
                            const double* dtp, const double* R, const double* Un, const double* Us, double* Uout,
                            double* P, const double* Bst, unsigned long long* counters, unsigned long long* cfl_out,
                            cudaStream_t st) {
  if (ECHO_CELL_ZMARCH) {
    const dim3 zb((unsigned)((g.n[0] + 127) / 128), (unsigned)g.n[1], (unsigned)((g.n[2] + kZSegIC - 1) / kZSegIC));
    if (ks)
      k_uct_cell_zm<true><<<zb, 128, 0, st>>>(g, e, mt, s, dt, dtp, R, Un, Us, Uout, P, Bst, counters, cfl_out);
    else
      k_uct_cell_zm<false><<<zb, 128, 0, st>>>(g, e, mt, s, dt, dtp, R, Un, Us, Uout, P, Bst, counters, cfl_out);
    return cudaGetLastError();
  }
  const unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  if (ks)
    k_uct_cell<true><<<blocks, kCellThreads, 0, st>>>(g, e, mt, s, dt, dtp, R, Un, Us, Uout, P, Bst, counters, cfl_out);
  else
    k_uct_cell<false><<<blocks, kCellThreads, 0, st>>>(g, e, mt, s, dt, dtp, R, Un, Us, Uout, P, Bst, counters, cfl_out);
  return cudaGetLastError();
}

cudaError_t launch_uct_centre_p2c(bool ks, const GridP& g, const EosP& e, const MetTables& mt, double* P, double* U,
                                  const double* Bst, cudaStream_t st) {
  const unsigned blocks = (unsigned)((g.N + kCellThreads - 1) / kCellThreads);
  if (ks) k_uct_centre_p2c<true><<<blocks, kCellThreads, 0, st>>>(g, e, mt, P, U, Bst);
  else k_uct_centre_p2c<false><<<blocks, kCellThreads, 0, st>>>(g, e, mt, P, U, Bst);
  return cudaGetLastError();
}

}  // namespace echo
