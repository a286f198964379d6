#pragma once
// march_pair.cuh — the x sweep (K2x, DESIGN.md §2 step 2, rows a1-a5) with two cells per lane.
//
// The same marching pipeline as march_impl.cuh's x sweep (one warp per line, warp barriers only,
// every reconstruction / face flux / DER value computed once per line), but each lane owns two
// consecutive slots of a 64-cell chunk: lane i handles slots 2i and 2i+1 in every phase.
//   A  WENO5 (rec) of cells B+3+2i and B+4+2i: their stencils B+1+2i .. B+6+2i are six ring
//      entries, read as two 8-byte and two 16-byte shared loads per variable (10 8-byte loads
//      for the two cells in the one-cell mapping); the A31 flags of faces B+3+2i, B+4+2i
//   D1 DER at faces X0+2i and X0+2i+1 (X0 = B - 64) from the six faces X0+2i-2 .. X0+2i+3:
//      three 16-byte loads per component (ten 8-byte loads)
//   D2 cells X0+2i (left face from lane i-1 by one shuffle) and X0+2i+1 (both faces in-lane);
//      the two results leave as one 16-byte store per rhs/EMF slot
//   B  HLL at faces B+2+2i (left state from lane i-1) and B+3+2i (both states in-lane): half
//      the shuffles, and two independent face computations per lane
// Primitive pairs arrive by 16-byte cp.async (even cell, 16-byte aligned: vs and pitch are even)
// except where the ghost index map (a1) breaks contiguity.  Same operations per cell and face in
// the same order as the one-cell mapping: results are bitwise identical to it.
#include "march_impl.cuh"

namespace echo {
namespace march {

#ifndef ECHO_X_PAIR
#define ECHO_X_PAIR 0  // 1: the x sweep with two cells per lane (opt-in: measured slower)
#endif
#ifndef ECHO_X2_NL
#define ECHO_X2_NL 4   // lines (warps) per CTA
#endif
#ifndef ECHO_X2_BPS
#define ECHO_X2_BPS 4  // CTAs per SM (4 x 4 warps: 128 registers)
#endif

struct GeoX2 {
  static constexpr int NL = ECHO_X2_NL;
  static constexpr int CH = 64;      // cells per chunk (2 per lane)
  static constexpr int THREADS = NL * 32;
  static constexpr int BPS = ECHO_X2_BPS;
  static constexpr int C_FIRST = -1;  // its A phase reaches the ghost cell -3
  static constexpr int B_FIRST = C_FIRST * CH;
  // primitive ring: live [B + CH + 1, B + 2 CH + 5] at a prefetch, the first window [-6, 70): 76
  static constexpr int RING = 80;
  // face-flux ring: B(c) writes faces B+2 .. B+CH+1 while D1(c+1) still needs B-2 ..: CH + 4
  static constexpr int RINGF = 80;
  static constexpr int RR = 256;     // A31 face-flag byte ring (>= 2 CH + 5)
  static constexpr int VP = NL * RING;
  static constexpr int VF = NL * RINGF;
  static constexpr int OFF_P = 0;
  static constexpr int OFF_F = OFF_P + 8 * VP;
  static constexpr int OFF_E = OFF_F + 7 * VF;   // left states qL at the warp edge [2][8][NL]
  static constexpr int OFF_HE = OFF_E + 2 * 8 * NL;  // DER values H at the warp edge [2][7][NL]
  static constexpr int TOTAL = OFF_HE + 2 * 7 * NL;
  static constexpr size_t SMEM = sizeof(double) * TOTAL + NL * RR;
  static_assert(RING % 2 == 0 && RINGF % 2 == 0 && (VP % 2) == 0 && (VF % 2) == 0, "16-byte pairs");
  static ECHO_HD int wrap(int p) { return p >= RING ? p - RING : (p < 0 ? p + RING : p); }
  static ECHO_HD int wrapf(int p) { return p >= RINGF ? p - RINGF : (p < 0 ? p + RINGF : p); }
  static ECHO_HD int ring(int x) { return ((x % RING) + RING) % RING; }
  static ECHO_HD int ringf(int x) { return ((x % RINGF) + RINGF) % RINGF; }
};

ECHO_D void lds2(const double* p, double& a, double& b) {
  const double2 v = *reinterpret_cast<const double2*>(p);
  a = v.x;
  b = v.y;
}
ECHO_D void sts2(double* p, double a, double b) { *reinterpret_cast<double2*>(p) = make_double2(a, b); }

// cp.async of the primitives of cells x, x+1 (x even) of line t (record base lb) into ring slot
// pair `pos` (even)
ECHO_D void load_pair_x(const GridP& g, const LineGeom& lg, long long lb, int x, int pos,
                        const double* __restrict__ P, const double* __restrict__ UB, unsigned sp) {
  const long long vs = g.vs;
  const unsigned s = sp + 8u * pos;
  if (x >= 0 && x + 1 < lg.na) {  // contiguous, 16-byte aligned (x even, vs and pitch even)
#pragma unroll
    for (int v = 0; v < 8; v++) cp_async16(s + 8u * v * GeoX2::VP, (v < 5 ? P : UB) + lb + x + v * vs);
  } else {
    const long long a0 = lb + map_index(x, lg.na, g.bc[0][0], g.bc[0][1]);
    const long long a1 = lb + map_index(x + 1, lg.na, g.bc[0][0], g.bc[0][1]);
#pragma unroll
    for (int v = 0; v < 8; v++) {
      const double* base = (v < 5 ? P : UB) + v * vs;
      cp_async8(s + 8u * v * GeoX2::VP, base + a0);
      cp_async8(s + 8u * (v * GeoX2::VP + 1), base + a1);
    }
  }
}

// the first window [-6, 70) of a line (38 pairs: lanes 0..31, then lanes 0..5 once more)
ECHO_D void load_window_x2(const GridP& g, const LineGeom& lg, long long unit, int t, int lane,
                           const double* __restrict__ P, const double* __restrict__ UB, unsigned sp) {
  const int t0 = (int)(unit % lg.tt_groups) * GeoX2::NL;
  const int zz = (int)(unit / lg.tt_groups) + lg.zoff;
  const long long lb = base_of<0>(g, 0, min(t0 + t, lg.nt - 1), zz);
  for (int x = -6 + 2 * lane; x < 70; x += 64) load_pair_x(g, lg, lb, x, GeoX2::ring(x), P, UB, sp);
}

template <bool KS, int DER, int REC, int DM>
ECHO_D void march_unit_x2(const GridP& g, const EosP& e, const MetTables& mt, const LineGeom& lg, const long long unit,
                          const long long next, const double* __restrict__ P, const double* __restrict__ UB, double* R,
                          const double* __restrict__ Bface, double* __restrict__ FSo, double* smem) {
  using GE = GeoX2;
  constexpr bool DN = DM == 1;
  constexpr bool UCT = DM == 2;
  constexpr int CH = GE::CH, RR = GE::RR;
  const int t = threadIdx.x >> 5;      // line in the group (one warp per line)
  const int lane = threadIdx.x & 31;
  const int s0 = 2 * lane;             // this lane's first slot
  const double idxa = g.idx[0];
  const long long vs = g.vs;
  unsigned char* rough = reinterpret_cast<unsigned char*>(smem + GE::TOTAL) + t * RR;
  double* const sP = smem + GE::OFF_P + t * GE::RING;   // + v VP + position
  double* const sF = smem + GE::OFF_F + t * GE::RINGF;  // + q VF + position
  const unsigned spP = (unsigned)__cvta_generic_to_shared(sP);

  const int t0 = (int)(unit % lg.tt_groups) * GE::NL;
  const int zz = (int)(unit / lg.tt_groups) + lg.zoff;
  const bool line_ok = t0 + t < lg.nt;
  const int tt = min(t0 + t, lg.nt - 1);
  const long long lb = base_of<0>(g, 0, tt, zz);
  int rb = GE::ring(GE::B_FIRST);
  int rbf = GE::ringf(GE::B_FIRST);
  for (int c = GE::C_FIRST; c <= lg.nchunks; c++, rb = GE::wrap(rb + CH), rbf = GE::wrapf(rbf + CH)) {
    const int B = c * CH;
    const int par = c & 1;
    const bool ab = c < lg.nchunks;
    const bool d2 = c >= 1;
    const int X0 = B - CH;
    cp_async_wait0();
    __syncwarp();  // (0) primitives of chunk c landed; F, flags and edges of chunk c-1 visible

    // ---- A: WENO of cells xr0 = B+3+2i and xr1 = xr0+1 (a2), the A31 flags of faces xr0, xr1 ----
    double qL0[8], qR0[8], qL1[8], qR1[8];
    const int xr0 = B + 3 + s0;
    if (!(ab && xr0 + 1 >= -3)) {  // the prologue needs cells -3..2 only
#pragma unroll
      for (int v = 0; v < 8; v++) qL0[v] = qR0[v] = qL1[v] = qR1[v] = 0.0;
    } else {
      bool rg0 = false, rg1 = false;
      const int p2 = GE::wrap(rb + 2 + s0);  // even: cells xr0-1, xr0
      const int p1 = GE::wrap(p2 - 1), p4 = GE::wrap(p2 + 2), p6 = GE::wrap(p2 + 4);
#pragma unroll
      for (int v = 0; v < 8; v++) {
        const double* r = sP + v * GE::VP;
        double u1, u2, u3, u4, u5, u6;  // cells xr0-2 .. xr0+3
        u1 = r[p1];
        lds2(r + p2, u2, u3);
        lds2(r + p4, u4, u5);
        u6 = r[p6];
        rec_both<REC>(u1, u2, u3, u4, u5, qL0[v], qR0[v]);
        rec_both<REC>(u2, u3, u4, u5, u6, qL1[v], qR1[v]);
        if (v == 0 || v == 4) {
          if (!(qL0[v] > 0.0)) qL0[v] = u3;  // A25 positivity fallback
          if (!(qR0[v] > 0.0)) qR0[v] = u3;
          if (!(qL1[v] > 0.0)) qL1[v] = u4;
          if (!(qR1[v] > 0.0)) qR1[v] = u4;
          const double lo0 = u3 < u4 ? u3 : u4, lo1 = u4 < u5 ? u4 : u5;
          rg0 |= fabs(u4 - u3) > g.der_jump * lo0;  // face xr0 joins cells xr0, xr0+1
          rg1 |= fabs(u5 - u4) > g.der_jump * lo1;
        }
      }
      rough[xr0 & (RR - 1)] = rg0;
      rough[(xr0 + 1) & (RR - 1)] = rg1;
      if (lane == 31) {  // the left state of cell B+CH+2 for slot 0 of the next chunk
        double* ed = smem + GE::OFF_E + ((c + 1) & 1) * 8 * GE::NL + t;
#pragma unroll
        for (int v = 0; v < 8; v++) ed[v * GE::NL] = qL1[v];
      }
    }

    // ---- D1: DER (a4) at faces f0 = X0+2i and f0+1 (faces f0-2 .. f0+3) ----
    double H0[7], H1[7];
    if (d2 || (c == 0 && lane == 31)) {  // c = 0: the face -1/2 (lane 31's second), carried to D(1)
      const int f0 = X0 + s0;
      bool plain0 = false, plain1 = false;
#pragma unroll
      for (int m = 0; m < 6; m++) {
        const bool r = rough[(f0 - 2 + m) & (RR - 1)] != 0;
        if (m < 5) plain0 |= r;
        if (m > 0) plain1 |= r;
      }
      const int fa = GE::wrapf(rbf - CH + s0 - 2);  // even
      const int fb = GE::wrapf(fa + 2), fc = GE::wrapf(fa + 4);
#pragma unroll
      for (int q = 0; q < 7; q++) {
        const double* Fq = sF + q * GE::VF;
        double Fm2, Fm1, F0, Fp1, Fp2, Fp3;
        lds2(Fq + fa, Fm2, Fm1);
        lds2(Fq + fb, F0, Fp1);
        lds2(Fq + fc, Fp2, Fp3);
        const double h0 = der5<DER>(Fm2, Fm1, F0, Fp1, Fp2);
        const double h1 = der5<DER>(Fm1, F0, Fp1, Fp2, Fp3);
        H0[q] = plain0 ? F0 : h0;
        H1[q] = plain1 ? Fp1 : h1;
      }
      if (lane == 31) {  // H at face X0+CH-1 for slot 0 of the next chunk
        double* ed = smem + GE::OFF_HE + ((c + 1) & 1) * 7 * GE::NL + t;
#pragma unroll
        for (int q = 0; q < 7; q++) ed[q * GE::NL] = H1[q];
      }
    } else {
#pragma unroll
      for (int q = 0; q < 7; q++) H0[q] = H1[q] = 0.0;
    }
    __syncwarp();  // (1) A and D1 done: primitives of chunk c dead, edges published

    // prefetch: chunk c+1's cells [B+CH+4, B+2CH+6) (33 pairs), or the next line group's window
    if (c <= GE::C_FIRST || c >= lg.nchunks) {
    } else if (c + 1 < lg.nchunks) {
      const int x = B + CH + 4 + s0;
      load_pair_x(g, lg, lb, x, GE::wrap(rb + CH + 4 + s0 - GE::RING), P, UB, spP);
      if (lane == 0) load_pair_x(g, lg, lb, B + 2 * CH + 4, GE::wrap(rb + 2 * CH + 4 - GE::RING), P, UB, spP);
    } else if (next >= 0 && next < lg.nunits) {
      load_window_x2(g, lg, next, t, lane, P, UB, spP);
    }
    cp_async_commit();

    // ---- D2: cells X0+2i, X0+2i+1: flux differences into the rhs, field-CD EMF (a5) ----
    if (d2) {
      double Hm[7];
#pragma unroll
      for (int q = 0; q < 7; q++) Hm[q] = __shfl_up_sync(0xffffffffu, H1[q], 1);
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 7; q++) Hm[q] = smem[GE::OFF_HE + par * 7 * GE::NL + q * GE::NL + t];
      }
      const int x0 = X0 + s0;
      if (line_ok && x0 < lg.na) {
        const bool both = x0 + 1 < lg.na;
        double* dst = R + lb + x0;
#pragma unroll
        for (int q = 0; q < 7; q++) {
          if (UCT && q >= 5) continue;
          // the face fluxes carry 1/Delta_x (hll_face scale): the difference needs no multiply
          double a, b;
          if (q < 5 || DN) {
            a = Hm[q] - H0[q];
            b = H0[q] - H1[q];
          } else {
            const double ha = (0.25 * g.dx[0]) * (H0[q] + Hm[q]);
            const double hb = (0.25 * g.dx[0]) * (H1[q] + H0[q]);
            a = (q == 5) ? -ha : ha;
            b = (q == 5) ? -hb : hb;
          }
          double* d = dst + out_slot<0, DN>(q) * vs;
          if (both) sts2(d, a, b);
          else d[0] = a;
        }
      }
    }

    // ---- B: faces xf0 = B+2+2i (left state: lane i-1's cell B+2+2i) and xf1 = xf0+1 (a3) ----
    const int xf0 = B + 2 + s0;
    if (ab) {  // (warp-uniform: the shuffles need every lane)
      double pl[8];
#pragma unroll
      for (int v = 0; v < 8; v++) pl[v] = __shfl_up_sync(0xffffffffu, qL1[v], 1);
      if (lane == 0) {
#pragma unroll
        for (int v = 0; v < 8; v++) pl[v] = smem[GE::OFF_E + par * 8 * GE::NL + v * GE::NL + t];
      }
      if (xf0 + 1 >= -3) {
      double Fa[7], Fb[7];
      auto face = [&](int xf, double* ql, double* qr, double* F) {
        auto face_hll = [&](const auto& mf) {
          if constexpr (UCT) {
            // A37: both states take the staggered normal field of face xf + 1/2 (owned by cell xf)
            const long long fo = lb + (long long)map_index(xf, lg.na, g.bc[0][0], g.bc[0][1]);
            const double bnv = Bface[fo] * (KS ? frcp(mf.sqrtg()) : 1.0);
            ql[5] = bnv;
            qr[5] = bnv;
            double fsv[8];
            hll_face(mf, e, ql, qr, 0, F, fsv, idxa);
            if (xf >= 0 && xf < lg.na && line_ok) {
#pragma unroll
              for (int m = 0; m < 8; m++) FSo[lb + xf + m * vs] = fsv[m];
            }
          } else {
            hll_face(mf, e, ql, qr, 0, F, nullptr, idxa);
          }
        };
        if constexpr (KS) {
          const int af = max(-kG, min(xf + 1, lg.na + kG));  // face af - 1/2
          face_hll(load_met(f0_rec(mt, af, tt)));
        } else {
          face_hll(FlatMet());
        }
      };
      face(xf0, pl, qR0, Fa);
      face(xf0 + 1, qL0, qR1, Fb);
      const int fp = GE::wrapf(rbf + 2 + s0);  // even
#pragma unroll
      for (int q = 0; q < 7; q++) sts2(sF + q * GE::VF + fp, Fa[q], Fb[q]);
      }
    }
  }
}

template <bool KS, int DER, int REC, int DM>
__global__ void __launch_bounds__(GeoX2::THREADS, GeoX2::BPS)
k_march_x2(const GridP g, const EosP e, const MetTables mt, const LineGeom lg, const double* __restrict__ P,
           const double* __restrict__ UB, double* R, const double* __restrict__ Bface, double* __restrict__ FSo) {
  extern __shared__ __align__(16) double smem_x2[];
  const int t = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned spP = (unsigned)__cvta_generic_to_shared(smem_x2 + GeoX2::OFF_P + t * GeoX2::RING);
  long long unit = blockIdx.x;
  if (unit < lg.nunits) load_window_x2(g, lg, unit, t, lane, P, UB, spP);
  cp_async_commit();
  for (; unit < lg.nunits; unit += gridDim.x)
    march_unit_x2<KS, DER, REC, DM>(g, e, mt, lg, unit, unit + gridDim.x, P, UB, R, Bface, FSo, smem_x2);
  cp_async_wait0();
}

}  // namespace march
}  // namespace echo
