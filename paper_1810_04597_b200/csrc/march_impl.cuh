#pragma once
// march_impl.cuh — the axis-sweep kernels K2x/K2y/K2z as a marching pipeline
// (DESIGN.md §2 step 2, rows a1-a5; §7).
//
// A persistent CTA owns a group of NL lines and marches along them in chunks of
// CH cells: x sweep 4 lines x 32 cells, 128 threads (one warp per line), 6 CTAs/SM;
// y/z sweeps 8 consecutive x-lines (64-byte rows) x 4 cells = one warp per CTA,
// 12 CTAs/SM.  In both every exchange of the march stays inside a warp, so the
// chunk barriers are warp barriers and the warps run decoupled.  Thread i
// of a line handles, in chunk c (base B = CH c):
//   A  WENO5 (or MP5) of reconstructed cell B+3+i (8 variables, both faces; a2)
//      and the A31 jump flag of face B+3+i
//   D1 DER6 (a4) at the right face of cell B-CH+i of the previous chunk (its
//      5-face stencil ends at face B+1, written by B(c-1)); edge lanes publish it
//   -- barrier (1): primitives of chunk c dead, edges visible; prefetch chunk c+1 --
//   D2 the left face from lane i-1 (shuffle / edge buffer), the flux difference
//      into the rhs and the field-CD EMF (a5) of cell B-CH+i
//   B  HLL flux at face B+2+i (a3): the left state comes from lane i-1 (warp
//      shuffle; the first slot from the previous chunk through an edge buffer)
//   -- barrier (0) of chunk c+1 --
// so every reconstruction, every face flux and every DER value is computed
// exactly once per line (no tile halo), and a chunk needs two barriers.  The
// first chunk starts at C_FIRST = -ceil(6/CH) so that A reaches the ghost cell
// -3; one epilogue chunk (D only) finishes the line.  Primitives stream through a
// ring of >= CH + 10 cells in shared memory: the next chunk's CH cells (or the
// next line group's first window) are prefetched with cp.async as soon as phase A
// has consumed the current ones; the ghost fill (a1) is the index map of those
// loads (slab mode: stored ghost planes).  Results are bitwise deterministic
// (fixed per-lane operation order).
#include <cuda_runtime.h>

#include <atomic>

#include "echo_dev.cuh"
#include "echo_kernels.h"

namespace echo {
namespace march {

// Line-group geometry per sweep axis: NL lines x CH cells per chunk
// (THREADS = NL CH), BPS CTAs per SM.  Overridable at build time for tuning
// runs (-DECHO_YZ_NL=8 -DECHO_YZ_CH=32 -DECHO_YZ_BPS=2, likewise ECHO_X_*).
#ifndef ECHO_PDL
#define ECHO_PDL 0  // programmatic dependent launch of the y and z sweeps (-DECHO_PDL=1; no gain measured)
#endif
#ifndef ECHO_ACC_REGS
#define ECHO_ACC_REGS 1  // y/z: the old accumulator values by plain loads into registers (not cp.async to smem)
#endif
#ifndef ECHO_EDGE_SELECT
#define ECHO_EDGE_SELECT 0  // y/z: the edge-buffer values loaded by every lane and selected (branch free)
#endif
#ifndef ECHO_BALLOT_FLAGS
#define ECHO_BALLOT_FLAGS 1  // A31 flags as warp ballots + a per-line bit history (warp-local kernels)
#endif
#ifndef ECHO_X_NL
#define ECHO_X_NL 4
#define ECHO_X_CH 32
#define ECHO_X_BPS 6
#endif
// -DECHO_YZ_LINE_MAJOR: the y/z sweeps take the x sweep's thread mapping (one warp per
// line, lanes = consecutive cells along it; NL lines adjacent in x share their 32-byte
// sectors through L1) instead of lanes alternating between 8 adjacent x-lines
#ifdef ECHO_YZ_LINE_MAJOR
#ifndef ECHO_YZ_NL
#define ECHO_YZ_NL 4
#define ECHO_YZ_CH 32
#define ECHO_YZ_BPS 6
#endif
#endif
#ifndef ECHO_YZ_NL
#define ECHO_YZ_NL 8
#define ECHO_YZ_CH 4
#define ECHO_YZ_BPS 12
#endif
// -DECHO_YZ_TRANS=1: the field-CD / divb-none y/z sweeps (not UCT's) take the x sweep's thread
// mapping (one warp per line, 32 cells per chunk) over NL = 8 x-adjacent lines, and every global
// access is transposed through shared memory: the ring is filled by lanes running over the 8
// lines (64-byte rows), and the rhs contributions of a chunk are written to a shared buffer
// that the next chunk adds to the accumulator with the same transposed mapping (CTA barriers)
#ifndef ECHO_YZ_TRANS
#define ECHO_YZ_TRANS 0
#endif
#ifndef ECHO_YZT_NL
#define ECHO_YZT_NL 8
#define ECHO_YZT_BPS 3
#endif
struct GeomSpec {
  int nl, ch, bps;
};
constexpr GeomSpec kGeomX{ECHO_X_NL, ECHO_X_CH, ECHO_X_BPS};
constexpr GeomSpec kGeomYZ{ECHO_YZ_NL, ECHO_YZ_CH, ECHO_YZ_BPS};
constexpr GeomSpec kGeomYZT{ECHO_YZT_NL, 32, ECHO_YZT_BPS};

constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }
constexpr bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }
// the smallest stride >= n that is r mod 16 doubles (r = 16 / lines): a half-warp's transposed
// accesses (NL lines x 16/NL positions) and 16 consecutive positions of one line (the march's
// reads) both hit distinct bank pairs
constexpr int pad16(int n, int r) { return n + ((16 + r - n % 16) % 16); }

#ifdef ECHO_YZ_LINE_MAJOR
constexpr bool kYzLineMajor = true;
#else
constexpr bool kYzLineMajor = false;
#endif

// V = 1: the transposed y/z geometry (ECHO_YZ_TRANS)
template <int AX, int V = 0>
struct Geo {
  static constexpr bool TRANS = V == 1;
  static_assert(!TRANS || AX != 0, "the transposed geometry is the y/z sweeps'");
  static constexpr GeomSpec S = TRANS ? kGeomYZT : (AX == 0) ? kGeomX : kGeomYZ;
  // line-major thread mapping (slot fastest): the x sweep, and y/z with ECHO_YZ_LINE_MAJOR or TRANS
  static constexpr bool LM = (AX == 0) || kYzLineMajor || TRANS;
  static constexpr int NL = S.nl;
  static constexpr int CH = S.ch;                             // cells per chunk = threads per line
  static constexpr int LOG_NL = ilog2(NL);
  static constexpr int LOG_CH = ilog2(CH);
  // ring length for primitives and face fluxes: >= CH + 10 live entries (a power of two when cheap;
  // -DECHO_TIGHT_RINGS: exactly the live length, less shared memory per CTA for more CTAs per SM)
#ifdef ECHO_TIGHT_RINGS
  static constexpr bool TIGHT = AX != 0;  // y/z only (the x rings stay powers of two)
#else
  static constexpr bool TIGHT = false;
#endif
  // TRANS: multiples of 16 (a line's 16 consecutive positions stay on distinct bank pairs across
  // the wrap) that fit 3 CTAs of 8 lines per SM
  static constexpr int RING = TRANS ? (CH + 10 + 15) / 16 * 16
                            : TIGHT ? CH + 10
                                    : (CH + 10 <= 16) ? 16 : (CH + 10 <= 32) ? 32 : (CH + 10 <= 64) ? 64 : CH + 16;
  // face-flux ring: B(c) writes faces B+2..B+CH+1 while faces B-2..B+1 are still needed by D(c+1)
  static constexpr int RINGF = TRANS ? (CH + 4 + 15) / 16 * 16
                             : TIGHT ? CH + 4
                                     : (CH + 4 <= 8) ? 8 : (CH + 4 <= 32) ? 32 : (CH + 4 <= 64) ? 64 : CH + 16;
  // line strides of the primitive ring and of the rhs-contribution buffer (TRANS: both are
  // written or read transposed, so padded to 2 mod 16)
  static constexpr int LSP = TRANS ? pad16(RING, 16 / NL) : RING;
  static constexpr int LSD = TRANS ? pad16(CH, 16 / NL) : CH;
  // first chunk: its A phase reaches down to the ghost cell -3 (WENO of cells -3.. for faces -3..)
  static constexpr int C_FIRST = -((6 + CH - 1) / CH);
  static constexpr int B_FIRST = C_FIRST * CH;
  // ring length (bytes per line) of the A31 face flags: written in A for faces B+3..B+CH+2 while D
  // reads faces B-CH-2..B+1 in the same barrier interval -> >= 2 CH + 5
  static constexpr int RR = (2 * CH + 5 <= 16) ? 16 : (2 * CH + 5 <= 64) ? 64 : (2 * CH + 5 <= 128) ? 128 : 256;
  static constexpr int THREADS = NL * CH;
  static constexpr int BPS = S.bps;
  static constexpr int DELTA = LM ? 1 : NL;                   // lane distance between slots i and i+1
  static constexpr int SLOTS_PER_WARP = 32 / DELTA;           // consecutive slots inside one warp
  static constexpr int NEDGE = CH / SLOTS_PER_WARP;           // warp-edge slots per line
  static constexpr int VP = NL * LSP;                         // variable stride, primitive ring
  static constexpr int VF = NL * RINGF;                       // component stride, F ring
  static constexpr int VA = NL * CH;                          // component stride, accumulation buffer
  static constexpr int VE = NL * NEDGE;                       // variable stride, edge buffers
  static constexpr int VD = NL * LSD;                         // component stride, TRANS rhs contributions
  static constexpr int OFF_P = 0;
  static constexpr int OFF_F = OFF_P + 8 * VP;
  static constexpr int OFF_A = OFF_F + 7 * VF;
  // the y/z accumulation buffer (none with ECHO_ACC_REGS: the old values are held in registers)
  static constexpr int OFF_D = OFF_A + ((AX == 0 || ECHO_ACC_REGS || TRANS) ? 0 : 7 * VA);
  static constexpr int OFF_E = OFF_D + (TRANS ? 7 * VD : 0);  // left states qL at warp edges [2][8]
  static constexpr int OFF_HE = OFF_E + 2 * 8 * VE;                 // DER fluxes H at warp edges [2][7]
  static constexpr int TOTAL = OFF_HE + 2 * 7 * VE;
  static constexpr size_t SMEM = sizeof(double) * TOTAL + NL * RR;  // + A31 flag ring (bytes)
  // x sweep with one warp per line: every exchange of the march (ring, edges, flags, loads) stays
  // inside the warp, so the chunk barriers are warp barriers and the warps run decoupled
  // (likewise any one-warp CTA, e.g. y/z: 8 lines x 4 cells)
  static constexpr bool WARP_LOCAL = !TRANS && ((LM && CH == 32) || THREADS == 32);
  static_assert(is_pow2(NL) && is_pow2(CH), "NL and CH must be powers of two");
  static_assert(CH >= 4 && THREADS <= 1024 && THREADS >= 32 && (LM ? CH >= 32 : NL <= 32),
                "unsupported line geometry");
  static_assert(AX != 0 || NL * CH <= 1024, "x geometry");
  static_assert(!TRANS || (CH == 32 && ECHO_ACC_REGS), "TRANS: 32-cell chunks, accumulator in registers");
  // shared-memory offsets: primitive ring, face-flux ring, accumulation / contribution buffers
  // (conflict-free: slot/position fastest for line-major mappings, line fastest otherwise)
  static ECHO_HD int pofs(int t, int pos) { return LM ? t * LSP + pos : pos * NL + t; }
  static ECHO_HD int fofs(int t, int pos) { return LM ? t * RINGF + pos : pos * NL + t; }
  static ECHO_HD int aofs(int t, int i) { return LM ? t * CH + i : i * NL + t; }
  static ECHO_HD int dofs(int t, int i) { return t * LSD + i; }
  // a ring position of cell/face x (x may be negative)
  static ECHO_HD int ring(int x) {
    if constexpr (is_pow2(RING)) return x & (RING - 1);
    else return ((x % RING) + RING) % RING;
  }
  // ring position rb + d for a chunk base position rb in [0, RING) and -RING <= d < RING
  static ECHO_HD int wrap(int p) {
    if constexpr (is_pow2(RING)) return p & (RING - 1);
    else return p >= RING ? p - RING : (p < 0 ? p + RING : p);
  }
};

template <int AX, class GE = Geo<AX>>
ECHO_HD int ringf(int x) {
  constexpr int RF = GE::RINGF;
  if constexpr (is_pow2(RF)) return x & (RF - 1);
  else return ((x % RF) + RF) % RF;
}
template <int AX, class GE = Geo<AX>>
ECHO_HD int wrapf(int p) {
  constexpr int RF = GE::RINGF;
  if constexpr (is_pow2(RF)) return p & (RF - 1);
  else return p >= RF ? p - RF : (p < 0 ? p + RF : p);
}

// the sweep geometry of axis AX and divergence treatment DM (UCT keeps the lane-over-lines y/z
// geometry: its face-data stores are per lane)
template <int AX, int DM>
struct GeoSel {
  using type = Geo<AX, (AX != 0 && DM != 2 && ECHO_YZ_TRANS) ? 1 : 0>;
};

ECHO_HD int first_axis(int comp) { return comp == 0 ? 1 : 0; }
template <int AX, bool DN>
ECHO_HD bool accumulates(int q) {
  if (q < 5) return AX != 0;
  const int b1 = (AX + 1) % 3, b2 = (AX + 2) % 3;
  if (DN) return first_axis(q == 5 ? b1 : b2) != AX;
  return first_axis(q == 5 ? b2 : b1) != AX;
}
template <int AX, bool DN>
ECHO_HD int out_slot(int q) {
  if (q < 5) return q;
  const int b1 = (AX + 1) % 3, b2 = (AX + 2) % 3;
  if (DN) return 5 + (q == 5 ? b1 : b2);
  return 5 + (q == 5 ? b2 : b1);
}

ECHO_D void cp_async8(unsigned saddr, const double* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gsrc));
}
ECHO_D void cp_async16(unsigned saddr, const double* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gsrc));
}
ECHO_D void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
ECHO_D void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }
ECHO_D void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

struct LineGeom {
  int na, nt, tt_groups, nz, nchunks;
  int vec16;
  // slab mode (stored z ghost planes): the x/y sweeps also run on the planes zoff = -1 and nz;
  // the z sweep's lines cover cells coff = -1 .. n3 and read every ghost as a stored plane
  int zoff, coff, stored;
  long long nunits;
};

template <int AX, class GE = Geo<AX>>
ECHO_D void unit_origin(const LineGeom& lg, long long unit, int& t0, int& zz) {
  t0 = (int)(unit % lg.tt_groups) * GE::NL;
  zz = (int)(unit / lg.tt_groups) + lg.zoff;
}

template <int AX>
ECHO_D long long base_of(const GridP& g, int a, int t, int zz) {
  if (AX == 0) return rec_base(g, a, t, zz);
  if (AX == 1) return rec_base(g, t, a, zz);
  return rec_base(g, t, zz, a);
}

// element stride along the sweep axis in the record layout
template <int AX>
ECHO_D long long axis_stride(const GridP& g) {
  return AX == 0 ? 1LL : (AX == 1 ? g.pitch : (long long)g.n[1] * g.pitch);
}

// cp.async of the primitives of cell x of line t (line record base lb) into the ring
template <int AX, class GE = Geo<AX>>
ECHO_D void load_cells(const GridP& g, const LineGeom& lg, long long lb, int t, int x, bool vec,
                       const double* __restrict__ P, const double* __restrict__ UB, unsigned sbase) {
  // slab z sweep: ghosts are stored planes (-kZH .. n + kZH - 1); the clamp only touches the
  // cells past the line end that the last chunk's window over-fetches (never used)
  const int ag = lg.stored ? min(max(x + lg.coff, -g.zhalo), g.n[AX] + g.zhalo - 1)
                           : map_index(x, lg.na, g.bc[AX][0], g.bc[AX][1]);
  const long long off = lb + ag * axis_stride<AX>(g);
  const long long vs = g.vs;
  const unsigned s = sbase + 8u * (GE::OFF_P + GE::pofs(t, GE::ring(x)));
#pragma unroll
  for (int v = 0; v < 8; v++) {
    const double* src = (v < 5 ? P : UB) + off + v * vs;
    if (vec) cp_async16(s + 8u * v * GE::VP, src);
    else cp_async8(s + 8u * v * GE::VP, src);
  }
}

// record base of line t of a unit (cell 0 along the sweep axis)
template <int AX>
ECHO_D long long line_base(const GridP& g, const LineGeom& lg, int t0, int zz, int t) {
  return base_of<AX>(g, 0, min(t0 + t, lg.nt - 1), zz);
}

// the first window [-5, CH + 5) of a line group (cells -5..4 feed the prologue chunk); (t, i): the
// loading thread's line and slot (TRANS: its transposed pair)
template <int AX, class GE = Geo<AX>>
ECHO_D void load_window(const GridP& g, const LineGeom& lg, long long unit, int t, int i,
                        const double* __restrict__ P, const double* __restrict__ UB, unsigned sbase) {
  int t0, zz;
  unit_origin<AX, GE>(lg, unit, t0, zz);
  const bool vec = !GE::LM && lg.vec16 && (t0 + GE::NL <= lg.nt);
  if (vec && (t & 1)) return;
  const long long lb = line_base<AX>(g, lg, t0, zz, t);
#pragma unroll
  for (int x = -kG + i; x <= GE::B_FIRST + 2 * GE::CH + 4; x += GE::CH) load_cells<AX, GE>(g, lg, lb, t, x, vec, P, UB, sbase);
}

// TRANS: R (cell X0p + iT of line tT) = old value accT + the contribution in the shared buffer
template <int AX, class GE, bool DN>
ECHO_D void store_contrib(const GridP& g, const LineGeom& lg, double* R, long long lbT, bool lineT_ok, int tT, int iT,
                          int X0p, const double (&accT)[7], const double* smem) {
  if (!(X0p + iT < lg.na && lineT_ok)) return;
  const long long vs = g.vs;
  const double idxa = g.idx[AX];
  double* dst = R + lbT + (long long)(X0p + iT + lg.coff) * axis_stride<AX>(g);
#pragma unroll
  for (int q = 0; q < 7; q++) {
    const double dq = smem[GE::OFF_D + q * GE::VD + GE::dofs(tT, iT)];
    double v;
    if (q < 5 || DN) v = accumulates<AX, DN>(q) ? fma(dq, idxa, accT[q]) : dq * idxa;
    else v = accumulates<AX, DN>(q) ? accT[q] + dq : dq;
    dst[out_slot<AX, DN>(q) * vs] = v;
  }
}

// DM: divergence treatment 0 field-CD (EMF Omega into R slots 5..7), 1 none (B flux
// differences), 2 UCT (uct.cu: the normal field of each face from the staggered Bface,
// the face data of the EMF step into FSo, hydro only into R)
// One unit (line group) of the march: chunks C_FIRST .. nchunks of the unit's NL lines.  The
// unit's first window must already be in flight (load_window + commit); in its last chunk the
// march prefetches the first window of `next` (when 0 <= next < nunits; -1: none).
template <int AX, bool KS, int DER, int REC, int DM>
ECHO_D void march_unit(const GridP& g, const EosP& e, const MetTables& mt, const LineGeom& lg, const long long unit,
                       const long long next, const double* __restrict__ P, const double* __restrict__ UB, double* R,
                       const double* __restrict__ Bface, double* __restrict__ FSo, double* smem, bool& dep_waited) {
  using GE = typename GeoSel<AX, DM>::type;
  constexpr bool TR = GE::TRANS;
  constexpr bool DN = DM == 1;
  constexpr bool UCT = DM == 2;
  constexpr int CH = GE::CH, RING = GE::RING, RINGF = GE::RINGF, RR = GE::RR;
  // A31 flags as ballots: warp-local kernels whose chunk of a line lies in one warp
  constexpr bool kBallot = ECHO_BALLOT_FLAGS && (GE::LM ? CH == 32 : (GE::WARP_LOCAL && CH * GE::NL == 32));
  unsigned char* rough = reinterpret_cast<unsigned char*>(smem + GE::TOTAL);  // [NL][RR] face flags
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  const int tid = threadIdx.x;
  const int t = GE::LM ? (tid >> GE::LOG_CH) : (tid & (GE::NL - 1));  // line in the group
  const int i = GE::LM ? (tid & (CH - 1)) : (tid >> GE::LOG_NL);      // slot along the line
  const bool edge_in = (i % GE::SLOTS_PER_WARP) == 0;                            // left neighbour in another warp/chunk
  const bool edge_out = (i % GE::SLOTS_PER_WARP) == GE::SLOTS_PER_WARP - 1;       // right neighbour in another warp/chunk
  const int eslot_out = ((i + 1) & (CH - 1)) / GE::SLOTS_PER_WARP;               // edge slot this thread publishes
  const int eslot_in = i / GE::SLOTS_PER_WARP;                                   // edge slot this thread reads
  const double idxa = g.idx[AX];
  const double kFluxScale = AX == 0 ? idxa : 1.0;
  const long long vs = g.vs;
  // TRANS: the transposed pair (line, slot) of this thread for every global access
  const int tT = TR ? (tid & (GE::NL - 1)) : t;
  const int iT = TR ? (tid >> GE::LOG_NL) : i;

  {
    int t0, zz;
    unit_origin<AX, GE>(lg, unit, t0, zz);
    const bool line_ok = t0 + t < lg.nt;
    const long long lb = line_base<AX>(g, lg, t0, zz, t);
    const long long as = axis_stride<AX>(g);
    const int tt = min(t0 + t, lg.nt - 1);
    const bool vec = !GE::LM && lg.vec16 && (t0 + GE::NL <= lg.nt);
    const long long lbT = TR ? line_base<AX>(g, lg, t0, zz, tT) : lb;  // (TRANS) line tT's record base
    const bool lineT_ok = t0 + tT < lg.nt;
    unsigned long long fhist = 0ull;  // A31 flags of this line's faces, newest chunk in the top CH bits
    int rb = GE::ring(GE::B_FIRST);  // primitive-ring position of the chunk base B
    int rbf = ringf<AX, GE>(GE::B_FIRST);  // face-flux-ring position of B
    double accT[7];  // (TRANS) the old rhs/EMF values of cell (tT, X0 + iT), added by the next chunk
    // (TRANS) store_contrib: the rhs contributions of the previous chunk's output cells X0p + slot
    // (written to the shared buffer by their lanes in D2) added to the accumulator, transposed
    for (int c = GE::C_FIRST; c <= lg.nchunks; c++, rb = GE::wrap(rb + CH), rbf = wrapf<AX, GE>(rbf + CH)) {
      const int B = c * CH;
      const int par = c & 1;
      const bool ab = c < lg.nchunks;       // A and B phases
      const bool d2 = c >= 1;               // D: outputs cells X0 + i of chunk c-1
      const int X0 = B - CH;
      cp_async_wait0();
      if constexpr (GE::WARP_LOCAL) __syncwarp();
      else __syncthreads();  // (0) primitives of chunk c landed; F, flags and edges of chunk c-1 visible
      double acc[7];  // ECHO_ACC_REGS: the old rhs/EMF values of the output cell, in registers
      if constexpr (TR) {
        if (c >= 2) store_contrib<AX, GE, DN>(g, lg, R, lbT, lineT_ok, tT, iT, X0 - CH, accT, smem);  // chunk c-1's
      }
      if (AX != 0 && d2) {  // old rhs/EMF values of the output cells (accumulated in D)
        if (!dep_waited) {  // the previous sweep's R (uniform: every thread reaches it at the same chunk)
          asm volatile("griddepcontrol.wait;" ::: "memory");
          dep_waited = true;
        }
        if constexpr (TR) {  // plain loads (transposed pair), added when the next chunk stores
          const int a = min(X0 + iT, lg.na - 1) + lg.coff;
          const double* src = R + lbT + (long long)a * as;
#pragma unroll
          for (int q = 0; q < 7; q++) accT[q] = !accumulates<AX, DN>(q) ? 0.0 : src[out_slot<AX, DN>(q) * vs];
        } else if constexpr (ECHO_ACC_REGS) {  // plain loads issued now, consumed in D2 (latency behind A, D1)
          const int a = min(X0 + i, lg.na - 1) + lg.coff;
          const double* src = R + lb + a * as;
#pragma unroll
          for (int q = 0; q < 7; q++)
            acc[q] = (!accumulates<AX, DN>(q) || (UCT && q >= 5)) ? 0.0 : src[out_slot<AX, DN>(q) * vs];
        } else if (!(vec && (t & 1))) {
          const int a = min(X0 + i, lg.na - 1) + lg.coff;
          const double* src = R + lb + a * as;
          const unsigned s = sbase + 8u * (GE::OFF_A + GE::aofs(t, i));
#pragma unroll
          for (int q = 0; q < 7; q++) {
            if (!accumulates<AX, DN>(q) || (UCT && q >= 5)) continue;
            if (vec) cp_async16(s + 8u * q * GE::VA, src + out_slot<AX, DN>(q) * vs);
            else cp_async8(s + 8u * q * GE::VA, src + out_slot<AX, DN>(q) * vs);
          }
        }
      }
      cp_async_commit();

      // ---- A: WENO5 of reconstructed cell xr = B+3+i (a2) and the A31 flag of face xr ----
      const int rr = GE::wrap(rb + 3 + i);  // ring position of xr
      double qL[8], qR[8];
      bool rgh = false;
      // inactive lanes' values are shuffled but never used; the x sweep zero-fills them all the
      // same (without it ptxas spills at 80 registers), the y/z sweeps skip the fill
      if (!(ab && B + 3 + i >= -3)) {  // the prologue needs cells -3..2 only
        if constexpr (GE::LM) {
#pragma unroll
          for (int v = 0; v < 8; v++) qL[v] = qR[v] = 0.0;
        }
      } else {
        int pos[5];
#pragma unroll
        for (int m = 0; m < 5; m++) pos[m] = GE::pofs(t, GE::wrap(rr - 2 + m));
        constexpr bool CHAR = REC == 6;  // A44: the hydro states per face from the characteristic fields
#pragma unroll
        for (int v = 0; v < 8; v++) {
          const double* r = smem + GE::OFF_P + v * GE::VP;
          double u[5];
#pragma unroll
          for (int m = 0; m < 5; m++) u[m] = r[pos[m]];
          if (!CHAR || v >= 5) rec_both<CHAR ? 0 : REC>(u[0], u[1], u[2], u[3], u[4], qL[v], qR[v]);
          if (v == 0 || v == 4) {
            if constexpr (!CHAR) {
              if (!(qL[v] > 0.0)) qL[v] = u[2];  // A25 positivity fallback
              if (!(qR[v] > 0.0)) qR[v] = u[2];
            }
            // face xr joins cells xr and xr+1 (der_jump = +inf when the switch is off: never fires)
            const double lo = u[2] < u[3] ? u[2] : u[3];
            rgh |= fabs(u[3] - u[2]) > g.der_jump * lo;
          }
        }
        if constexpr (CHAR) {
          // face xf = xr - 1 (between cells xr-1 and xr): stencil cells xr-3 .. xr+2 in the sweep frame;
          // its left state goes to qL (used by this lane in B, no shuffle), its right state to qR
          double q6[6][5];
          constexpr int cmp[3] = {1 + AX, 1 + (AX + 1) % 3, 1 + (AX + 2) % 3};
#pragma unroll
          for (int m = 0; m < 6; m++) {
            const int ps = GE::pofs(t, GE::wrap(rr - 3 + m));
            q6[m][0] = smem[GE::OFF_P + 0 * GE::VP + ps];
#pragma unroll
            for (int d = 0; d < 3; d++) q6[m][1 + d] = smem[GE::OFF_P + cmp[d] * GE::VP + ps];
            q6[m][4] = smem[GE::OFF_P + 4 * GE::VP + ps];
          }
          double fL[5], fR[5];
          char_face(e, q6, fL, fR);
          qL[0] = fL[0];
          qR[0] = fR[0];
          qL[4] = fL[4];
          qR[4] = fR[4];
#pragma unroll
          for (int d = 0; d < 3; d++) {
            qL[cmp[d]] = fL[1 + d];
            qR[cmp[d]] = fR[1 + d];
          }
          // A25: a non-positive rho or p takes the value of the cell the state was reconstructed in
          if (!(qL[0] > 0.0)) qL[0] = q6[2][0];
          if (!(qL[4] > 0.0)) qL[4] = q6[2][4];
          if (!(qR[0] > 0.0)) qR[0] = q6[3][0];
          if (!(qR[4] > 0.0)) qR[4] = q6[3][4];
        }
        if constexpr (!kBallot) rough[t * RR + ((B + 3 + i) & (RR - 1))] = rgh;
        if (edge_out) {  // publish the left state of cell xr for the slot to the right
          const int dpar = (i == CH - 1) ? ((c + 1) & 1) : par;
#pragma unroll
          for (int v = 0; v < 8; v++) smem[GE::OFF_E + dpar * 8 * GE::VE + v * GE::VE + eslot_out * GE::NL + t] = qL[v];
        }
      }

      unsigned fm = 0u;  // this chunk's CH flags of line t
      if constexpr (kBallot) {
        const unsigned b = __ballot_sync(0xffffffffu, rgh);
        if constexpr (GE::LM) {
          fm = b;  // lane = slot
        } else if constexpr (GE::NL == 8 && CH == 4) {
          fm = (((b >> t) & 0x01010101u) * 0x10204080u) >> 28;  // lanes i*8 + t, i = 0..3
        } else {  // lanes i*NL + t, i = 0..CH-1
#pragma unroll
          for (int i2 = 0; i2 < CH; i2++) fm |= ((b >> (i2 * GE::NL + t)) & 1u) << i2;
        }
      }
      // ---- D1: DER flux (a4) at the right face X0+i+1/2 of cell X0+i (faces X0+i-2..X0+i+2) ----
      double H[7];
      if (d2 || (c == 0 && i == CH - 1)) {  // c = 0: the left face -1/2 of cell 0, carried to D(1)
        bool plain = false;
#pragma unroll
        for (int m = 0; m < 5; m++)
          if constexpr (!kBallot) plain |= rough[t * RR + ((X0 + i - 2 + m) & (RR - 1))] != 0;  // A31
        if constexpr (kBallot) {  // faces X0+i-2+m: bits 59-CH+i+m of the line's history (chunk c-1 on top)
          plain = ((fhist >> (59 - CH + i)) & 0x1Full) != 0;
        }
        int fpos[5];
#pragma unroll
        for (int m = 0; m < 5; m++) fpos[m] = GE::fofs(t, wrapf<AX, GE>(rbf - CH + i - 2 + m));
#pragma unroll
        for (int q = 0; q < 7; q++) {
          const double* Fq = smem + GE::OFF_F + q * GE::VF;
          const double F0 = Fq[fpos[2]];
          const double h = der5<DER>(Fq[fpos[0]], Fq[fpos[1]], F0, Fq[fpos[3]], Fq[fpos[4]]);
          H[q] = plain ? F0 : h;  // select, no branch
        }
        if (edge_out) {  // publish H for the slot to the right (slot CH-1: for slot 0 of the next chunk)
          const int dpar = (i == CH - 1) ? ((c + 1) & 1) : par;
#pragma unroll
          for (int q = 0; q < 7; q++) smem[GE::OFF_HE + dpar * 7 * GE::VE + q * GE::VE + eslot_out * GE::NL + t] = H[q];
        }
      } else if constexpr (GE::LM) {
#pragma unroll
        for (int q = 0; q < 7; q++) H[q] = 0.0;
      }
      cp_async_wait0();  // the old rhs/EMF values of this thread's copies
      if constexpr (kBallot) fhist = (fhist >> CH) | ((unsigned long long)fm << (64 - CH));
      if constexpr (GE::WARP_LOCAL) __syncwarp();
      else __syncthreads();  // (1) A and D1 done: primitives of chunk c dead, edges published, A buffer landed

      {  // prefetch: the next chunk's CH new cells, or the next line group's first window
         // (the prologue's window already holds chunk 0's cells)
        if (c <= GE::C_FIRST || c >= lg.nchunks) {  // (the window holds the first two chunks)
        } else if (c + 1 < lg.nchunks) {
          if (!(vec && (t & 1))) load_cells<AX, GE>(g, lg, lbT, tT, B + CH + kG + iT, vec, P, UB, sbase);
        } else if (next >= 0 && next < lg.nunits) {
          load_window<AX, GE>(g, lg, next, tT, iT, P, UB, sbase);
        }
        cp_async_commit();
      }

      // ---- D2: cell X0+i: flux differences into rhs; field-CD EMF (a5) ----
      if (d2) {
        double Hm[7];
#pragma unroll
        for (int q = 0; q < 7; q++) Hm[q] = __shfl_up_sync(0xffffffffu, H[q], GE::DELTA);
        // edge lanes take the value from the edge buffer: every lane loads (branch free, so the
        // shared loads can be scheduled early), the edge lanes select it
        if constexpr (ECHO_EDGE_SELECT && !GE::LM) {
#pragma unroll
          for (int q = 0; q < 7; q++) {
            const double eh = smem[GE::OFF_HE + par * 7 * GE::VE + q * GE::VE + eslot_in * GE::NL + t];
            Hm[q] = edge_in ? eh : Hm[q];
          }
        } else if (edge_in) {
#pragma unroll
          for (int q = 0; q < 7; q++) Hm[q] = smem[GE::OFF_HE + par * 7 * GE::VE + q * GE::VE + eslot_in * GE::NL + t];
        }
        if constexpr (TR) {  // the contributions to the shared buffer; the next chunk adds them (transposed)
          if (X0 + i < lg.na && line_ok) {
#pragma unroll
            for (int q = 0; q < 7; q++) {
              double d;
              if (q < 5 || DN) d = Hm[q] - H[q];  // (times 1/Delta in store_contrib)
              else {
                const double hs = 0.25 * (H[q] + Hm[q]);
                d = (q == 5) ? -hs : hs;
              }
              smem[GE::OFF_D + q * GE::VD + GE::dofs(t, i)] = d;
            }
          }
        } else if (X0 + i < lg.na && line_ok) {
          double* dst = R + lb + (X0 + i + lg.coff) * as;
#pragma unroll
          for (int q = 0; q < 7; q++) {
            if (UCT && q >= 5) continue;
            // x: the face fluxes carry the factor 1/Delta_a (hll_face scale), so H are DER values of
            // F / Delta_a and the difference needs no multiply; y/z keep F (their multiply fuses with
            // the accumulation into an FMA)
            double d;
            if (q < 5 || DN) {
              d = AX == 0 ? Hm[q] - H[q] : -(H[q] - Hm[q]) * idxa;
            } else {
              const double hs = (AX == 0 ? 0.25 * g.dx[AX] : 0.25) * (H[q] + Hm[q]);
              d = (q == 5) ? -hs : hs;
            }
            dst[out_slot<AX, DN>(q) * vs] =
                accumulates<AX, DN>(q) ? ((ECHO_ACC_REGS ? acc[q] : smem[GE::OFF_A + q * GE::VA + GE::aofs(t, i)]) + d) : d;
          }
        }
      }

      // ---- B: face xf = B+2+i between reconstructed cells xf and xf+1 (a3) ----
      if (ab) {
        double pl[8];
        constexpr int V0 = REC == 6 ? 5 : 0;  // A44: the hydro left state of this face is the lane's own
#pragma unroll
        for (int v = V0; v < 8; v++) pl[v] = __shfl_up_sync(0xffffffffu, qL[v], GE::DELTA);
        if constexpr (ECHO_EDGE_SELECT && !GE::LM) {
#pragma unroll
          for (int v = V0; v < 8; v++) {  // (branch free, as for H above)
            const double ee = smem[GE::OFF_E + par * 8 * GE::VE + v * GE::VE + eslot_in * GE::NL + t];
            pl[v] = edge_in ? ee : pl[v];
          }
        } else if (edge_in) {
#pragma unroll
          for (int v = V0; v < 8; v++) pl[v] = smem[GE::OFF_E + par * 8 * GE::VE + v * GE::VE + eslot_in * GE::NL + t];
        }
#pragma unroll
        for (int v = 0; v < V0; v++) pl[v] = qL[v];
        const int xf = B + 2 + i;
        if (xf >= -3) {
          double F[7];
          // the face metric (KS: 2-D tables; Minkowski: flat)
          auto face_hll = [&](const auto& mf) {
            if constexpr (UCT) {
              // A37: both states take the staggered normal field of face xf + 1/2 (owned by
              // cell xf; A42 ghost rule), b = sqrt(g) B
              // (slab z sweep: the line's cell xf is the slab's cell xf + coff, ghosts stored)
              const long long fo = lb + (long long)(lg.stored ? xf + lg.coff : map_index(xf, lg.na, g.bc[AX][0], g.bc[AX][1])) * as;
              const double bnv = Bface[fo + AX * vs] * (KS ? frcp(mf.sqrtg()) : 1.0);
              pl[5 + AX] = bnv;
              qR[5 + AX] = bnv;
              double fsv[8];
              hll_face(mf, e, pl, qR, AX, F, fsv, kFluxScale);
              if (xf >= 0 && xf < lg.na && line_ok) {
#pragma unroll
                for (int m = 0; m < 8; m++) FSo[lb + (long long)(xf + lg.coff) * as + m * vs] = fsv[m];
              }
            } else {
              hll_face(mf, e, pl, qR, AX, F, nullptr, kFluxScale);
            }
          };
          if (KS) {
            const int af = max(-kG, min(xf + 1, lg.na + kG));  // face af - 1/2
            const double* rec;
            if (AX == 0) rec = f0_rec(mt, af, tt);
            else if (AX == 1) rec = f1_rec(mt, tt, af);
            else rec = cen_rec(mt, tt, zz);
            face_hll(load_met(rec));
          } else {
            face_hll(FlatMet());
          }
          const int fp = GE::fofs(t, wrapf<AX, GE>(rbf + 2 + i));
#pragma unroll
          for (int q = 0; q < 7; q++) smem[GE::OFF_F + q * GE::VF + fp] = F[q];
        }
      }
    }
    if constexpr (TR) {  // the last chunk's contributions (its D2 ran in the epilogue chunk)
      __syncthreads();
      store_contrib<AX, GE, DN>(g, lg, R, lbT, lineT_ok, tT, iT, (lg.nchunks - 1) * CH, accT, smem);
    }
  }
}

// CTAs per SM of a sweep: about half for rec = 6 (its per-face eigen-projection needs ~2x the registers;
// ECHO_REC6_X_BPS / ECHO_REC6_YZ_BPS);
// the Kerr-Schild x sweep (face metric records) spilled 164 B at the x sweep's 80 registers: 4 CTAs (128)
#ifndef ECHO_KSX_BPS
#define ECHO_KSX_BPS 4
#endif
// (and the UCT x sweep, which also writes the face data, spilled 56 B at 80: 5 CTAs)
#ifndef ECHO_UCTX_BPS
#define ECHO_UCTX_BPS 5
#endif
#ifndef ECHO_REC6_X_BPS
#define ECHO_REC6_X_BPS 3
#endif
#ifndef ECHO_REC6_YZ_BPS
#define ECHO_REC6_YZ_BPS 10  // 164 registers (6: 240): 120.2-120.3 vs 123.6-123.7 ms/step with rec 6 (profiles/r02_rec6_ab)
#endif
template <int AX, bool KS, int REC, int DM>
constexpr int sweep_bps() {
  using GE = typename GeoSel<AX, DM>::type;
  return REC == 6 ? (AX == 0 ? ECHO_REC6_X_BPS : ECHO_REC6_YZ_BPS)
                  : ((KS && AX == 0) ? ECHO_KSX_BPS : ((DM == 2 && AX == 0) ? ECHO_UCTX_BPS : GE::BPS));
}

template <int AX, bool KS, int DER, int REC, int DM>
__global__ void __launch_bounds__(GeoSel<AX, DM>::type::THREADS, (sweep_bps<AX, KS, REC, DM>()))
k_march(const GridP g, const EosP e, const MetTables mt, const LineGeom lg, const double* __restrict__ P,
        const double* __restrict__ UB, double* R, const double* __restrict__ Bface, double* __restrict__ FSo) {
  using GE = typename GeoSel<AX, DM>::type;
  extern __shared__ double smem[];
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  const int tid = threadIdx.x;
  // the first window's loads: the thread's own (line, slot), or its transposed pair (TRANS)
  const int t = (GE::LM && !GE::TRANS) ? (tid >> GE::LOG_CH) : (tid & (GE::NL - 1));
  const int i = (GE::LM && !GE::TRANS) ? (tid & (GE::CH - 1)) : (tid >> GE::LOG_NL);
  // programmatic dependent launch (ECHO_PDL): the next sweep's CTAs may start as this grid's
  // CTAs retire, and run their first chunks (which read only P and U) over its tail; a y/z
  // sweep waits for the previous sweep's grid before its first access to R
  if constexpr (ECHO_PDL && AX != 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  bool dep_waited = !(ECHO_PDL && AX != 0);
  long long unit = blockIdx.x;
  if (unit < lg.nunits) load_window<AX, GE>(g, lg, unit, t, i, P, UB, sbase);
  cp_async_commit();
  for (; unit < lg.nunits; unit += gridDim.x)
    march_unit<AX, KS, DER, REC, DM>(g, e, mt, lg, unit, unit + gridDim.x, P, UB, R, Bface, FSo, smem, dep_waited);
  cp_async_wait0();
}

// -DECHO_YZ_MAXNREG=n: the y/z sweeps compiled with a register cap of n (__maxnreg__, which cannot be
// combined with __launch_bounds__) instead of the CTAs-per-SM bound, e.g. 152 registers = 13 one-warp
// CTAs per SM, a budget between the 12 (168) and 14 (128) that launch bounds can express
#ifdef ECHO_YZ_MAXNREG
template <int AX, bool KS, int DER, int REC, int DM>
__global__ void __maxnreg__(ECHO_YZ_MAXNREG)
k_march_mr(const GridP g, const EosP e, const MetTables mt, const LineGeom lg, const double* __restrict__ P,
           const double* __restrict__ UB, double* R, const double* __restrict__ Bface, double* __restrict__ FSo) {
  using GE = typename GeoSel<AX, DM>::type;
  extern __shared__ double smem[];
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  const int tid = threadIdx.x;
  const int t = (GE::LM && !GE::TRANS) ? (tid >> GE::LOG_CH) : (tid & (GE::NL - 1));
  const int i = (GE::LM && !GE::TRANS) ? (tid & (GE::CH - 1)) : (tid >> GE::LOG_NL);
  bool dep_waited = true;
  long long unit = blockIdx.x;
  if (unit < lg.nunits) load_window<AX, GE>(g, lg, unit, t, i, P, UB, sbase);
  cp_async_commit();
  for (; unit < lg.nunits; unit += gridDim.x)
    march_unit<AX, KS, DER, REC, DM>(g, e, mt, lg, unit, unit + gridDim.x, P, UB, R, Bface, FSo, smem, dep_waited);
  cp_async_wait0();
}
#endif

// line-group geometry of a sweep launch (the slab extension included)
template <int AX, class GE = Geo<AX>>
inline LineGeom make_line_geom(const GridP& g, const double* P, const double* R, const PlaneRange& zr = PlaneRange{}) {
  LineGeom lg;
  lg.na = g.n[AX];
  lg.nt = g.n[AX == 0 ? 1 : 0];
  lg.tt_groups = (lg.nt + GE::NL - 1) / GE::NL;
  lg.nz = (AX == 2) ? g.n[1] : g.n[2];
  lg.zoff = 0;
  lg.coff = 0;
  lg.stored = 0;
  if (g.zhalo) {
    // field-CD: the owned planes and the first ghost plane on each side (the x/y sweeps' EMF there
    // feeds the curl); UCT: 5 ghost planes on each side (the face data the edge EMFs of 3 ghost
    // planes reconstruct along z)
    const int ext = g.divb == 2 ? 5 : 1;
    if (AX == 2) {
      lg.na += 2 * ext;
      lg.coff = -ext;
      lg.stored = 1;
    } else {
      lg.nz += 2 * ext;
      lg.zoff = -ext;
    }
  }
  if (AX != 2 && zr.zn > 0) {  // x/y sweeps over planes zb .. zb + zn - 1 only (slab overlap, echo.h)
    lg.zoff = zr.zb;
    lg.nz = zr.zn;
  }
  lg.nchunks = (lg.na + GE::CH - 1) / GE::CH;  // (after the slab extension of na)
  lg.vec16 = (g.n[0] % 2 == 0) && ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(R)) % 16 == 0);
  lg.nunits = (long long)lg.tt_groups * lg.nz;
  return lg;
}
inline LineGeom x_line_geom(const GridP& g, const double* R, const double* P) { return make_line_geom<0>(g, P, R); }

}  // namespace march
}  // namespace echo
