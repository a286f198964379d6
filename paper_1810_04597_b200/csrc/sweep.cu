// sweep.cu — the axis-sweep kernels K2x/K2y/K2z (DESIGN.md §2 step 2, rows a1-a5).
//
// One CTA owns a tile of NL lines x TA cells along the sweep axis.  The tile's
// primitives (8 fields, TA + 2*5 cells per line) are read from HBM once per
// sweep with coalesced loads into shared memory; the ghost fill (a1) happens
// in that load as an index map (periodic wrap mod n / outflow clamp), so no
// padded arrays and no separate ghost pass exist.  Then, all from shared memory:
//   A  WENO5 per (cell, variable): both faces of the cell, shared beta_k (a2)
//   B  one thread per face: states, speeds, HLL (a3), densitised
//   C1 DER6 per (face, component) (a4)
//   C2 per (cell, component): rhs -= dH/Delta, field-CD EMF contributions (a5)
// Each interface flux is computed by exactly one thread in a fixed operation
// order, so results are bitwise run-to-run deterministic.
#include <cuda_runtime.h>

#include "echo_dev.cuh"
#include "echo_kernels.h"

namespace echo {

constexpr int TA = 64;         // cells along the axis per tile
constexpr int NL = 4;          // lines per tile
constexpr int LEN_P = TA + 10; // primitive stencil per line
constexpr int LEN_Q = TA + 6;  // reconstructed cells per line
constexpr int NF = TA + 5;     // faces per line
constexpr int NH = TA + 1;     // DER faces per line
constexpr int kSweepThreads = NF * NL;  // 276: one face per thread in phase B
constexpr int SZ_P = 8 * NL * LEN_P;
constexpr int SZ_Q = 16 * NL * LEN_Q;
static_assert(7 * NL * NF <= SZ_P, "F must fit in the primitive tile");
static_assert(7 * NL * NH <= SZ_Q, "H must fit in the state tile");
constexpr size_t kSweepSmem = sizeof(double) * (SZ_P + SZ_Q);

template <int AX, int LEN>
ECHO_D int soff(int t, int a) {  // conflict-free layout: the coalesced index is fastest
  return AX == 0 ? t * LEN + a : a * NL + t;
}
template <int AX, int LEN>
ECHO_D void split(int r, int& t, int& a) {
  if (AX == 0) { t = r / LEN; a = r - t * LEN; }
  else { a = r / NL; t = r - a * NL; }
}

// first axis that writes a given B/Omega component (the others accumulate)
ECHO_HD int first_axis(int comp) { return comp == 0 ? 1 : 0; }

template <int AX, bool KS, int DER, int REC, bool DIVB_NONE>
__global__ void __launch_bounds__(kSweepThreads, 2)
k_sweep(const GridP g, const EosP e, const MetTables mt, const double* __restrict__ P,
        const double* __restrict__ U, double* __restrict__ R, double* __restrict__ Om) {
  extern __shared__ double smem[];
  double* sP = smem;         // [8][...LEN_P], later F [7][...NF]
  double* sQ = smem + SZ_P;  // [16][...LEN_Q] (L: 0-7, R: 8-15), later H [7][...NH]
  const int tid = threadIdx.x;
  const long long N = g.N;
  const int na = g.n[AX];
  // tile origin
  const int a0 = (AX == 0 ? blockIdx.x : blockIdx.y) * TA;
  const int t0 = (AX == 0 ? blockIdx.y : blockIdx.x) * NL;
  const int TAX = (AX == 0) ? 1 : 0;  // array axis of the transverse (line) index
  const int nt = g.n[TAX];
  const int zz = blockIdx.z;          // the remaining axis index
  // (along a, transverse t) -> (i, j, k)
  auto cell = [&](int a, int t, int& i, int& j, int& k) {
    if (AX == 0) { i = a; j = t; k = zz; }
    else if (AX == 1) { i = t; j = a; k = zz; }
    else { i = t; j = zz; k = a; }
  };
  const int bclo = g.bc[AX][0], bchi = g.bc[AX][1];

  // ---- load: 8 primitives with the ghost rule as an index map (a1) ----
  for (int it = tid; it < SZ_P; it += kSweepThreads) {
    int v = it / (NL * LEN_P);
    int r = it - v * (NL * LEN_P);
    int t, m;
    split<AX, LEN_P>(r, t, m);
    int ag = map_index(a0 - kG + m, na, bclo, bchi);
    int tg = min(t0 + t, nt - 1);
    int i, j, k;
    cell(ag, tg, i, j, k);
    long long id = ((long long)k * g.n[1] + j) * g.n[0] + i;
    double val;
    if (v < 5) {
      val = __ldg(P + v * N + id);
    } else {
      val = __ldg(U + v * N + id);
      if (KS) val = val / __ldg(cen_rec(mt, i, j) + 16);
    }
    sP[v * (NL * LEN_P) + soff<AX, LEN_P>(t, m)] = val;
  }
  __syncthreads();

  // ---- A: WENO5, both faces of each cell, per variable (a2) ----
  for (int it = tid; it < 8 * NL * LEN_Q; it += kSweepThreads) {
    int v = it / (NL * LEN_Q);
    int r = it - v * (NL * LEN_Q);
    int t, c;
    split<AX, LEN_Q>(r, t, c);
    const double* row = sP + v * (NL * LEN_P);
    double um2 = row[soff<AX, LEN_P>(t, c)];
    double um1 = row[soff<AX, LEN_P>(t, c + 1)];
    double u0 = row[soff<AX, LEN_P>(t, c + 2)];
    double up1 = row[soff<AX, LEN_P>(t, c + 3)];
    double up2 = row[soff<AX, LEN_P>(t, c + 4)];
    double qL, qR;
    weno5_both<REC>(um2, um1, u0, up1, up2, qL, qR);
    if (v == 0 || v == 4) {  // A25 positivity fallback
      if (!(qL > 0.0)) qL = u0;
      if (!(qR > 0.0)) qR = u0;
    }
    sQ[v * (NL * LEN_Q) + soff<AX, LEN_Q>(t, c)] = qL;
    sQ[(8 + v) * (NL * LEN_Q) + soff<AX, LEN_Q>(t, c)] = qR;
  }
  __syncthreads();

  // ---- B: one face per thread: states, speeds, HLL (a3) ----
  {
    int t, fa;
    split<AX, NF>(tid, t, fa);
    double pl[8], pr[8];
#pragma unroll
    for (int v = 0; v < 8; v++) {
      pl[v] = sQ[v * (NL * LEN_Q) + soff<AX, LEN_Q>(t, fa)];
      pr[v] = sQ[(8 + v) * (NL * LEN_Q) + soff<AX, LEN_Q>(t, fa + 1)];
    }
    double F[7];
    auto hll = [&](const auto& m) {
      State sl, sr;
      make_state(m, e, pl, sl);
      make_state(m, e, pr, sr);
      double uL[7], fL[7], uR[7], fR[7];
      cons_flux(m, sl, AX, uL, fL);
      cons_flux(m, sr, AX, uR, fR);
      double lmL, lpL, lmR, lpR;
      speeds(m, e, pl, sl, AX, lmL, lpL);
      speeds(m, e, pr, sr, AX, lmR, lpR);
      double sL = fmin(0.0, fmin(lmL, lmR));
      double sR = fmax(0.0, fmax(lpL, lpR));
      double den = sR - sL;
      if (den > 0.0) {
        double inv = m.sqrtg() / den;
        double ss = sL * sR;
#pragma unroll
        for (int q = 0; q < 7; q++) F[q] = (sR * fL[q] - sL * fR[q] + ss * (uR[q] - uL[q])) * inv;
      } else {
#pragma unroll
        for (int q = 0; q < 7; q++) F[q] = 0.5 * (fL[q] + fR[q]) * m.sqrtg();
      }
    };
    if (KS) {
      int af = a0 - 3 + fa + 1;  // face af - 1/2
      af = max(-kG, min(af, na + kG));
      int tg = min(t0 + t, nt - 1);
      const double* rec;
      if (AX == 0) rec = f0_rec(mt, af, tg);
      else if (AX == 1) rec = f1_rec(mt, tg, af);
      else rec = cen_rec(mt, tg, zz);
      hll(load_met(rec));
    } else {
      hll(FlatMet());
    }
    // sP is free since phase A (synchronised above); phase B reads only sQ
#pragma unroll
    for (int q = 0; q < 7; q++) sP[q * (NL * NF) + soff<AX, NF>(t, fa)] = F[q];
  }
  __syncthreads();

  // ---- C1: DER flux derivative at faces a0-1/2 .. a0+TA-1/2 (a4) ----
  for (int it = tid; it < 7 * NL * NH; it += kSweepThreads) {
    int q = it / (NL * NH);
    int r = it - q * (NL * NH);
    int t, h;
    split<AX, NH>(r, t, h);
    const double* Fq = sP + q * (NL * NF);
    double Hv = der5<DER>(Fq[soff<AX, NF>(t, h)], Fq[soff<AX, NF>(t, h + 1)], Fq[soff<AX, NF>(t, h + 2)],
                          Fq[soff<AX, NF>(t, h + 3)], Fq[soff<AX, NF>(t, h + 4)]);
    sQ[q * (NL * NH) + soff<AX, NH>(t, h)] = Hv;
  }
  __syncthreads();

  // ---- C2: flux differences into rhs; field-CD EMF (a5) ----
  const double idxa = g.idx[AX];
  for (int it = tid; it < 7 * NL * TA; it += kSweepThreads) {
    int q = it / (NL * TA);
    int r = it - q * (NL * TA);
    int t, c;
    split<AX, TA>(r, t, c);
    int a = a0 + c, tg = t0 + t;
    if (a >= na || tg >= nt) continue;
    int i, j, k;
    cell(a, tg, i, j, k);
    long long id = ((long long)k * g.n[1] + j) * g.n[0] + i;
    const double* Hq = sQ + q * (NL * NH);
    double Hp = Hq[soff<AX, NH>(t, c + 1)], Hm = Hq[soff<AX, NH>(t, c)];
    if (q < 5) {
      double d = -(Hp - Hm) * idxa;
      double* dst = R + q * N + id;
      *dst = (AX == 0) ? d : (*dst + d);
    } else {
      const int b1 = (AX + 1) % 3, b2 = (AX + 2) % 3;
      const int bc = (q == 5) ? b1 : b2;  // which B component this flux transports
      if (DIVB_NONE) {
        double d = -(Hp - Hm) * idxa;
        double* dst = R + (5 + bc) * N + id;
        *dst = (first_axis(bc) == AX) ? d : (*dst + d);
      } else {
        double hs = 0.25 * (Hp + Hm);
        if (q == 5) {  // flux of B^{a+1} -> -1/4 into Omega_{a+2}
          double* dst = Om + b2 * N + id;
          *dst = (first_axis(b2) == AX) ? -hs : (*dst - hs);
        } else {       // flux of B^{a+2} -> +1/4 into Omega_{a+1}
          double* dst = Om + b1 * N + id;
          *dst = (first_axis(b1) == AX) ? hs : (*dst + hs);
        }
      }
    }
  }
}

template <int AX, bool KS, int DER, int REC, bool DN>
static cudaError_t launch_one(const GridP& g, const EosP& e, const MetTables& mt, const double* P, const double* U,
                              double* R, double* Om, cudaStream_t st) {
  auto kern = k_sweep<AX, KS, DER, REC, DN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    if (err != cudaSuccess) return err;
    attr = true;
  }
  dim3 grid;
  if (AX == 0) grid = dim3((g.n[0] + TA - 1) / TA, (g.n[1] + NL - 1) / NL, g.n[2]);
  else if (AX == 1) grid = dim3((g.n[0] + NL - 1) / NL, (g.n[1] + TA - 1) / TA, g.n[2]);
  else grid = dim3((g.n[0] + NL - 1) / NL, (g.n[2] + TA - 1) / TA, g.n[1]);
  kern<<<grid, kSweepThreads, kSweepSmem, st>>>(g, e, mt, P, U, R, Om);
  return cudaGetLastError();
}

template <int AX, bool KS, int DER, int REC>
static cudaError_t launch_dn(const GridP& g, const EosP& e, const MetTables& mt, const double* P, const double* U,
                             double* R, double* Om, cudaStream_t st) {
  if (g.divb == 1) return launch_one<AX, KS, DER, REC, true>(g, e, mt, P, U, R, Om, st);
  return launch_one<AX, KS, DER, REC, false>(g, e, mt, P, U, R, Om, st);
}

template <int AX, bool KS, int DER>
static cudaError_t launch_rec(const GridP& g, const EosP& e, const MetTables& mt, const double* P, const double* U,
                              double* R, double* Om, cudaStream_t st) {
  if (g.rec == 1) return launch_dn<AX, KS, DER, 1>(g, e, mt, P, U, R, Om, st);
  return launch_dn<AX, KS, DER, 0>(g, e, mt, P, U, R, Om, st);
}

template <int AX, bool KS>
static cudaError_t launch_der(const GridP& g, const EosP& e, const MetTables& mt, const double* P, const double* U,
                              double* R, double* Om, cudaStream_t st) {
  if (g.der == 4) return launch_rec<AX, KS, 4>(g, e, mt, P, U, R, Om, st);
  if (g.der == 2) return launch_rec<AX, KS, 2>(g, e, mt, P, U, R, Om, st);
  return launch_rec<AX, KS, 6>(g, e, mt, P, U, R, Om, st);
}

cudaError_t launch_sweep(int axis, bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P,
                         const double* U, double* R, double* Om, cudaStream_t st) {
  if (ks) {
    if (axis == 0) return launch_der<0, true>(g, e, mt, P, U, R, Om, st);
    if (axis == 1) return launch_der<1, true>(g, e, mt, P, U, R, Om, st);
    return launch_der<2, true>(g, e, mt, P, U, R, Om, st);
  }
  if (axis == 0) return launch_der<0, false>(g, e, mt, P, U, R, Om, st);
  if (axis == 1) return launch_der<1, false>(g, e, mt, P, U, R, Om, st);
  return launch_der<2, false>(g, e, mt, P, U, R, Om, st);
}

}  // namespace echo
