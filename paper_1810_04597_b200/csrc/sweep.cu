// sweep.cu — the axis-sweep kernels K2x/K2y/K2z (DESIGN.md §2 step 2, rows a1-a5).
//
// Device records are row-interleaved ([k][j][var][i], echo_dev.cuh):
// P = (rho, u~^i, p, B^i), R = (L_D, L_S, L_tau, Omega^i).
//
// A persistent CTA walks over tiles of NL lines x TA = 58 cells along the sweep
// axis (x sweep: NL = 4 lines, 256 threads, 2 CTAs/SM; y/z sweeps: NL = 8
// consecutive x-lines = 64 B per row, 512 threads, 1 CTA/SM).  Every thread owns
// one (line, position) slot x in [0, 64) of its line in every phase, so no
// per-item index division exists and one address computation serves all 8
// variables / 7 flux components.  The next tile's primitives (TA + 2*5 cells
// per line) and the rhs/EMF values it will accumulate into are prefetched with
// cp.async into a second shared-memory buffer while the current tile is
// computed.  The ghost fill (a1) is an index map inside those loads (periodic
// wrap mod n / outflow clamp): no padded arrays, no ghost pass.  Per tile:
//   A  WENO5 of the 8 variables of cell x: both faces, shared beta_k (a2)
//   B  face x: states, speeds, HLL (a3), densitised
//   C1 DER6 of the 7 flux components at face x, with the A31 shock switch (a4)
//   C2 cell x: rhs -= dH/Delta, field-CD EMF contributions (a5)
// Each interface flux is computed by exactly one thread in a fixed operation
// order, so results are bitwise run-to-run deterministic.
#include <cuda_runtime.h>

#include "echo_dev.cuh"
#include "echo_kernels.h"

namespace echo {

constexpr int TA = 58;         // owned cells per line per tile
constexpr int SLOT = 64;       // slots per line: thread = (line, slot)
constexpr int LEN_P = TA + 10; // primitive stencil per line (68)
constexpr int LEN_Q = TA + 6;  // reconstructed cells per line (64 = SLOT)
constexpr int NF = TA + 5;     // faces per line (63)
constexpr int NH = TA + 1;     // DER faces per line (59)
static_assert(LEN_Q == SLOT, "one reconstructed cell per thread");

template <int AX>
struct Geo {
  static constexpr int NL = (AX == 0) ? 4 : 8;  // lines per tile (y/z: 8 x-lines = 64 B rows)
  static constexpr int LOG_NL = (AX == 0) ? 2 : 3;
  static constexpr int THREADS = NL * SLOT;
  static constexpr int BPS = (AX == 0) ? 3 : 1;  // CTAs per SM
  static constexpr int VP = NL * LEN_P;  // variable stride in the primitive buffer
  static constexpr int VQ = NL * LEN_Q;  // variable stride in the state buffer
  static constexpr int VF = NL * NF;     // component stride of F
  static constexpr int VH = NL * NH;     // component stride of H
  static constexpr int VA = NL * TA;     // component stride of the accumulation buffer
  static constexpr int SZ_P = 8 * VP;    // one primitive buffer (later reused for F)
  static constexpr int SZ_Q = 16 * VQ;   // L/R states (later reused for H)
  static constexpr int SZ_A = (AX == 0) ? 0 : 7 * VA;  // one rhs/EMF accumulation buffer
  static constexpr int OFF_P0 = 0, OFF_P1 = SZ_P, OFF_Q = 2 * SZ_P, OFF_A0 = OFF_Q + SZ_Q, OFF_A1 = OFF_A0 + SZ_A;
  static constexpr size_t SMEM = sizeof(double) * (OFF_A1 + SZ_A);
  static_assert(7 * VF <= SZ_P, "F must fit in the primitive tile");
  static_assert(7 * VH <= SZ_Q, "H must fit in the state tile");
};

// conflict-free layout: for the x sweep the along-axis index is fastest, for
// y/z the line (x) index is fastest — matching the coalesced global direction
template <int AX, int LEN>
ECHO_HD int soff(int t, int a) {
  return AX == 0 ? t * LEN + a : a * Geo<AX>::NL + t;
}

// first axis that writes a given B/Omega component (the others accumulate)
ECHO_HD int first_axis(int comp) { return comp == 0 ? 1 : 0; }

// does sweep AX accumulate into (rather than overwrite) its output component q?
template <int AX, bool DN>
ECHO_HD bool accumulates(int q) {
  if (q < 5) return AX != 0;
  const int b1 = (AX + 1) % 3, b2 = (AX + 2) % 3;
  if (DN) return first_axis(q == 5 ? b1 : b2) != AX;
  return first_axis(q == 5 ? b2 : b1) != AX;  // q=5 -> Omega_{a+2}, q=6 -> Omega_{a+1}
}
// variable slot of R holding output component q of sweep AX
template <int AX, bool DN>
ECHO_HD int out_slot(int q) {
  if (q < 5) return q;
  const int b1 = (AX + 1) % 3, b2 = (AX + 2) % 3;
  if (DN) return 5 + (q == 5 ? b1 : b2);  // L(B^{a+1}), L(B^{a+2})
  return 5 + (q == 5 ? b2 : b1);          // Omega_{a+2}, Omega_{a+1}
}

ECHO_D void cp_async8(unsigned saddr, const double* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gsrc));
}
ECHO_D void cp_async16(unsigned saddr, const double* gsrc) {  // L2 only (no L1 allocation)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gsrc));
}
ECHO_D void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
ECHO_D void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

struct TileGeom {
  int na, nt, ta_tiles, tt_tiles, nz;
  int vec16;  // n1 even and 16-B aligned bases: x pairs of every variable row are 16-B aligned
  long long ntiles;
};

template <int AX>
ECHO_D void tile_origin(const TileGeom& tg, long long tile, int& a0, int& t0, int& zz) {
  // AX = 0: x tiles fastest; AX = 1, 2: transverse (x) tiles fastest -> neighbouring CTAs share rows
  constexpr int NL = Geo<AX>::NL;
  long long r;
  if (AX == 0) {
    a0 = (int)(tile % tg.ta_tiles) * TA;
    r = tile / tg.ta_tiles;
    t0 = (int)(r % tg.tt_tiles) * NL;
    zz = (int)(r / tg.tt_tiles);
  } else {
    t0 = (int)(tile % tg.tt_tiles) * NL;
    r = tile / tg.tt_tiles;
    a0 = (int)(r % tg.ta_tiles) * TA;
    zz = (int)(r / tg.ta_tiles);
  }
}

// record base (var 0) of the cell at along-axis a, line t, remaining index zz
template <int AX>
ECHO_D long long base_of(const GridP& g, int a, int t, int zz) {
  if (AX == 0) return rec_base(g, a, t, zz);
  if (AX == 1) return rec_base(g, t, a, zz);
  return rec_base(g, t, zz, a);
}

// cp.async loads of one tile: primitives (+ old rhs/EMF values to accumulate into)
template <int AX, bool DN>
ECHO_D void issue_tile_loads(const GridP& g, const TileGeom& tg, long long tile, int t, int x,
                             const double* __restrict__ P, const double* R, unsigned sP, unsigned sA) {
  using GE = Geo<AX>;
  int a0, t0, zz;
  tile_origin<AX>(tg, tile, a0, t0, zz);
  const int tt = min(t0 + t, tg.nt - 1);
  const long long vs = g.n[0];  // variable stride inside a row
  // y/z sweeps: the lines of a tile are consecutive x; when they are all in
  // range and 16-B aligned, even lines fetch 16 B (two lines) with one L2-only
  // cp.async and odd lines issue nothing
  const bool vec = (AX != 0) && tg.vec16 && (t0 + GE::NL <= tg.nt);
  if (vec && (t & 1)) return;
#pragma unroll
  for (int pass = 0; pass < 2; pass++) {
    const int m = x + pass * SLOT;
    if (pass == 1 && m >= LEN_P) break;
    const int ag = map_index(a0 - kG + m, tg.na, g.bc[AX][0], g.bc[AX][1]);
    const double* src = P + base_of<AX>(g, ag, tt, zz);
    const unsigned s = sP + 8u * soff<AX, LEN_P>(t, m);
#pragma unroll
    for (int v = 0; v < 8; v++) {
      if (vec) cp_async16(s + 8u * v * GE::VP, src + v * vs);
      else cp_async8(s + 8u * v * GE::VP, src + v * vs);
    }
  }
  if (AX != 0 && x < TA) {
    const int a = min(a0 + x, tg.na - 1);
    const double* src = R + base_of<AX>(g, a, tt, zz);
    const unsigned s = sA + 8u * soff<AX, TA>(t, x);
#pragma unroll
    for (int q = 0; q < 7; q++) {
      if (!accumulates<AX, DN>(q)) continue;
      if (vec) cp_async16(s + 8u * q * GE::VA, src + out_slot<AX, DN>(q) * vs);
      else cp_async8(s + 8u * q * GE::VA, src + out_slot<AX, DN>(q) * vs);
    }
  }
}

template <int AX, bool KS, int DER, int REC, bool DN>
__global__ void __launch_bounds__(Geo<AX>::THREADS, Geo<AX>::BPS)
k_sweep(const GridP g, const EosP e, const MetTables mt, const TileGeom tg, const double* __restrict__ P,
        double* R) {
  using GE = Geo<AX>;
  extern __shared__ double smem[];
  __shared__ unsigned char sRough[GE::THREADS];  // A31 flag of face x of line t
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  const int tid = threadIdx.x;
  const int t = (AX == 0) ? (tid >> 6) : (tid & (GE::NL - 1));  // line
  const int x = (AX == 0) ? (tid & 63) : (tid >> GE::LOG_NL);    // slot along the line
  const double idxa = g.idx[AX];

  long long tile = blockIdx.x;
  if (tile < tg.ntiles)
    issue_tile_loads<AX, DN>(g, tg, tile, t, x, P, R, sbase + 8u * GE::OFF_P0, sbase + 8u * GE::OFF_A0);
  cp_async_commit();
  for (int iter = 0; tile < tg.ntiles; iter++, tile += gridDim.x) {
    const int cur = iter & 1;
    const int offP = cur ? GE::OFF_P1 : GE::OFF_P0;
    const int offA = cur ? GE::OFF_A1 : GE::OFF_A0;
    const long long nxt = tile + gridDim.x;
    if (nxt < tg.ntiles)
      issue_tile_loads<AX, DN>(g, tg, nxt, t, x, P, R, sbase + 8u * (cur ? GE::OFF_P0 : GE::OFF_P1),
                               sbase + 8u * (cur ? GE::OFF_A0 : GE::OFF_A1));
    cp_async_commit();
    cp_async_wait1();
    __syncthreads();

    int a0, t0, zz;
    tile_origin<AX>(tg, tile, a0, t0, zz);
    const int tt = min(t0 + t, tg.nt - 1);

    // ---- A: WENO5 of the 8 variables of reconstructed cell x (a2) ----
    {
      const double* row = smem + offP;
      bool rough = false;
#pragma unroll 4
      for (int v = 0; v < 8; v++) {
        const double* r = row + v * GE::VP;
        double u[5];
#pragma unroll
        for (int m = 0; m < 5; m++) u[m] = r[soff<AX, LEN_P>(t, x + m)];
        double qL, qR;
        weno5_both<REC>(u[0], u[1], u[2], u[3], u[4], qL, qR);
        if (v == 0 || v == 4) {
          if (!(qL > 0.0)) qL = u[2];  // A25 positivity fallback
          if (!(qR > 0.0)) qR = u[2];
          // A31: face x joins cells x and x+1; a jump in rho or p switches DER off nearby
          rough |= g.der_jump > 0.0 && fabs(u[3] - u[2]) > g.der_jump * fmin(u[2], u[3]);
        }
        smem[GE::OFF_Q + v * GE::VQ + soff<AX, LEN_Q>(t, x)] = qL;
        smem[GE::OFF_Q + (8 + v) * GE::VQ + soff<AX, LEN_Q>(t, x)] = qR;
      }
      sRough[t * SLOT + x] = rough;
    }
    __syncthreads();

    // ---- B: face x (between reconstructed cells x and x+1): HLL (a3) ----
    if (x < NF) {
      double pl[8], pr[8];
#pragma unroll
      for (int v = 0; v < 8; v++) {
        pl[v] = smem[GE::OFF_Q + v * GE::VQ + soff<AX, LEN_Q>(t, x)];
        pr[v] = smem[GE::OFF_Q + (8 + v) * GE::VQ + soff<AX, LEN_Q>(t, x + 1)];
      }
      double F[7];
      if (KS) {
        int af = a0 - 3 + x + 1;  // face af - 1/2
        af = max(-kG, min(af, tg.na + kG));
        const double* rec;
        if (AX == 0) rec = f0_rec(mt, af, tt);
        else if (AX == 1) rec = f1_rec(mt, tt, af);
        else rec = cen_rec(mt, tt, zz);
        hll_face(load_met(rec), e, pl, pr, AX, F);
      } else {
        hll_face(FlatMet(), e, pl, pr, AX, F);
      }
      // the primitive buffer of this tile is free since phase A: it takes F
#pragma unroll
      for (int q = 0; q < 7; q++) smem[offP + q * GE::VF + soff<AX, NF>(t, x)] = F[q];
    }
    __syncthreads();

    // ---- C1: DER flux derivative at face x: faces a0-1/2 .. a0+TA-1/2 (a4) ----
    if (x < NH) {
      const unsigned char* rf = sRough + t * SLOT + x;
      const bool plain = rf[0] | rf[1] | rf[2] | rf[3] | rf[4];  // A31: stencil crosses a jump
#pragma unroll
      for (int q = 0; q < 7; q++) {
        const double* Fq = smem + offP + q * GE::VF;
        double Hv = plain ? Fq[soff<AX, NF>(t, x + 2)]
                          : der5<DER>(Fq[soff<AX, NF>(t, x)], Fq[soff<AX, NF>(t, x + 1)], Fq[soff<AX, NF>(t, x + 2)],
                                      Fq[soff<AX, NF>(t, x + 3)], Fq[soff<AX, NF>(t, x + 4)]);
        smem[GE::OFF_Q + q * GE::VH + soff<AX, NH>(t, x)] = Hv;
      }
    }
    __syncthreads();

    // ---- C2: cell x: flux differences into rhs; field-CD EMF (a5) ----
    if (x < TA && a0 + x < tg.na && t0 + t < tg.nt) {
      double* dst = R + base_of<AX>(g, a0 + x, t0 + t, zz);
      const long long vs = g.n[0];
#pragma unroll
      for (int q = 0; q < 7; q++) {
        const double* Hq = smem + GE::OFF_Q + q * GE::VH;
        const double Hp = Hq[soff<AX, NH>(t, x + 1)], Hm = Hq[soff<AX, NH>(t, x)];
        double d;
        if (q < 5 || DN) {
          d = -(Hp - Hm) * idxa;
        } else {
          const double hs = 0.25 * (Hp + Hm);
          d = (q == 5) ? -hs : hs;  // flux of B^{a+1} -> -1/4 Omega_{a+2}; of B^{a+2} -> +1/4 Omega_{a+1}
        }
        dst[out_slot<AX, DN>(q) * vs] =
            accumulates<AX, DN>(q) ? (smem[offA + q * GE::VA + soff<AX, TA>(t, x)] + d) : d;
      }
    }
    __syncthreads();  // buffers of this tile are refilled by the next iteration's prefetch
  }
}

template <int AX, bool KS, int DER, int REC, bool DN>
static cudaError_t launch_one(const GridP& g, const EosP& e, const MetTables& mt, const double* P, double* R,
                              cudaStream_t st) {
  using GE = Geo<AX>;
  auto kern = k_sweep<AX, KS, DER, REC, DN>;
  static int grid_cap = 0;
  if (!grid_cap) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GE::SMEM);
    if (err != cudaSuccess) return err;
    int dev, sms, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, GE::THREADS, GE::SMEM);
    grid_cap = sms * (per > 0 ? per : 1);
  }
  TileGeom tg;
  tg.na = g.n[AX];
  tg.nt = g.n[AX == 0 ? 1 : 0];
  tg.ta_tiles = (tg.na + TA - 1) / TA;
  tg.tt_tiles = (tg.nt + GE::NL - 1) / GE::NL;
  tg.nz = (AX == 2) ? g.n[1] : g.n[2];
  tg.vec16 = (g.n[0] % 2 == 0) && ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(R)) % 16 == 0);
  tg.ntiles = (long long)tg.ta_tiles * tg.tt_tiles * tg.nz;
  unsigned blocks = (unsigned)(tg.ntiles < grid_cap ? tg.ntiles : grid_cap);
  kern<<<blocks, GE::THREADS, GE::SMEM, st>>>(g, e, mt, tg, P, R);
  return cudaGetLastError();
}

template <int AX, bool KS, int DER, int REC>
static cudaError_t launch_dn(const GridP& g, const EosP& e, const MetTables& mt, const double* P, double* R,
                             cudaStream_t st) {
  if (g.divb == 1) return launch_one<AX, KS, DER, REC, true>(g, e, mt, P, R, st);
  return launch_one<AX, KS, DER, REC, false>(g, e, mt, P, R, st);
}

template <int AX, bool KS, int DER>
static cudaError_t launch_rec(const GridP& g, const EosP& e, const MetTables& mt, const double* P, double* R,
                              cudaStream_t st) {
  if (g.rec == 1) return launch_dn<AX, KS, DER, 1>(g, e, mt, P, R, st);
  return launch_dn<AX, KS, DER, 0>(g, e, mt, P, R, st);
}

template <int AX, bool KS>
static cudaError_t launch_der(const GridP& g, const EosP& e, const MetTables& mt, const double* P, double* R,
                              cudaStream_t st) {
  if (g.der == 4) return launch_rec<AX, KS, 4>(g, e, mt, P, R, st);
  if (g.der == 2) return launch_rec<AX, KS, 2>(g, e, mt, P, R, st);
  return launch_rec<AX, KS, 6>(g, e, mt, P, R, st);
}

cudaError_t launch_sweep(int axis, bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P,
                         double* R, cudaStream_t st) {
  if (ks) {
    if (axis == 0) return launch_der<0, true>(g, e, mt, P, R, st);
    if (axis == 1) return launch_der<1, true>(g, e, mt, P, R, st);
    return launch_der<2, true>(g, e, mt, P, R, st);
  }
  if (axis == 0) return launch_der<0, false>(g, e, mt, P, R, st);
  if (axis == 1) return launch_der<1, false>(g, e, mt, P, R, st);
  return launch_der<2, false>(g, e, mt, P, R, st);
}

}  // namespace echo
