// fused.cu — the update K3 of RK stage s fused with the x sweep of the state it produces
// (DESIGN.md §7 "update + x sweep"): one persistent kernel over the x sweep's line groups
// (NL = 4 rows of one z plane).  For each unit a CTA first runs K3 (rows a5-a9: curl, metric
// sources, RK combine, con2prim + floors, CFL rate) on the unit's 4 x n1 cells, then, after a
// block barrier, marches the x sweep (rows a1-a4, march_impl.cuh) over the same 4 rows of the
// new state.  K3 is bound by HBM and the sweep by the FP64 pipe: interleaved in one grid, the
// CTAs of an SM are at any time in different phases, so the two bottlenecks overlap instead
// of adding up, and the sweep's loads of the rows K3 has just written are mostly L2 hits.
//
// Hazard: K3 at row j reads the field-CD EMF Omega of rows j +- 1 and planes k +- 1 from the
// accumulator R of stage s, while the x sweep of the next stage writes its accumulator; the two
// are different buffers (api.cu double-buffers R).  Every other access is to the unit's own
// cells.  Results are bit-for-bit those of K3 followed by the x sweep (the same per-cell code).
#include <cuda_runtime.h>

#include <atomic>

#include "cell_physics.cuh"
#include "march_impl.cuh"

namespace echo {
namespace march {

// K3 of stage s on line t (one row of n1 cells: consecutive lanes on consecutive x, coalesced)
// of a unit, by the 32 lanes of the warp that sweeps that line
template <bool KS, int DM>
ECHO_D void k3_line(const GridP& g, const EosP& e, const MetTables& mt, const LineGeom& lg, long long unit, int t,
                    int lane, int s, double dt, const double* __restrict__ Rold, const double* Un, const double* Us,
                    double* Uout, double* P, bool want_rate, double& rate, unsigned& nfl, unsigned& nfa) {
  int t0, zz;
  unit_origin<0>(lg, unit, t0, zz);
  if (t0 + t >= lg.nt) return;
  for (int i = lane; i < g.n[0]; i += 32) {
    const int ev = stage_cell<KS, DM == 1>(g, e, mt, s, dt, Rold, Un, Us, Uout, P, i, t0 + t, zz, want_rate, rate);
    nfl += ev == 1;
    nfa += ev == 2;
  }
}

// Warps are independent: warp t runs K3 on line t of a unit, then (after __syncwarp: its lanes'
// stores are visible to its own loads) the x sweep of that line, unit after unit.  The work of
// every unit is the same, so warps that start together would stay in phase (all in K3, HBM
// bound, then all sweeping, FP64 bound).  Half of the warps on each scheduler therefore run one
// K3 ahead: K3(u0), K3(u1), sweep(u0), K3(u2), sweep(u1), ... -- they are sweeping while the
// others wait on memory, and vice versa.
template <bool KS, int DER, int REC, int DM>
__global__ void __launch_bounds__(Geo<0>::THREADS, Geo<0>::BPS)
k_update_march(const GridP g, const EosP e, const MetTables mt, const LineGeom lg, const int s, const double dt,
               const double* __restrict__ dtp, const double* __restrict__ Rold, const double* Un, const double* Us,
               double* Uout, double* P, unsigned long long* counters, unsigned long long* cfl_out, double* Rnew,
               const int nsm) {
  using GE = Geo<0>;
  extern __shared__ double smem[];
  double dtv = dt;
  if (dtp) {  // device-driven loop: dt from k_cfl_dt; a halted loop does nothing (uniform over the grid)
    if (dtp[1] != 0.0) return;
    dtv = dtp[0];
  }
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  const int tid = threadIdx.x;
  const int t = tid >> GE::LOG_CH;  // the warp's line
  const int i = tid & (GE::CH - 1);
  const double* UB = KS ? P : Uout;  // B^i of the new state (Minkowski: U_B)
  const bool want = cfl_out != nullptr;
  unsigned nfl = 0, nfa = 0;
  double rate = 0.0;
  bool dep_waited = true;
  // warps of one scheduler (t mod 4) in consecutive CTAs of an SM alternate the lag
  const bool ahead = ((t + (int)(blockIdx.x / nsm)) & 1) != 0;
  const long long step = gridDim.x;
  long long u = blockIdx.x;
  if (ahead && u < lg.nunits) k3_line<KS, DM>(g, e, mt, lg, u, t, i, s, dtv, Rold, Un, Us, Uout, P, want, rate, nfl, nfa);
  for (; u < lg.nunits; u += step) {
    const long long k3u = ahead ? u + step : u;  // the unit whose K3 runs in this iteration
    if (k3u < lg.nunits) k3_line<KS, DM>(g, e, mt, lg, k3u, t, i, s, dtv, Rold, Un, Us, Uout, P, want, rate, nfl, nfa);
    __syncwarp();  // the line's new P and U are visible to the warp's loads
    load_window<0>(g, lg, u, t, i, P, UB, sbase);
    cp_async_commit();
    march_unit<0, KS, DER, REC, DM>(g, e, mt, lg, u, -1, P, UB, Rnew, nullptr, nullptr, smem, dep_waited);
    cp_async_wait0();
  }
  // ---- the CFL max-rate reduction (a9, stage 3) and the A9 counters: one atomic each per CTA / warp
  if (cfl_out) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rate = fmax(rate, __shfl_xor_sync(0xffffffffu, rate, o));
    __syncthreads();  // the ring is free: every warp finished its march
    if ((tid & 31) == 0) smem[tid >> 5] = rate;
    __syncthreads();
    if (tid == 0) {
      double bm = smem[0];
      for (int w = 1; w < GE::THREADS / 32; w++) bm = fmax(bm, smem[w]);
      atomicMax(cfl_out, (unsigned long long)__double_as_longlong(bm));
    }
  }
  nfl = __reduce_add_sync(0xffffffffu, nfl);
  nfa = __reduce_add_sync(0xffffffffu, nfa);
  if ((tid & 31) == 0) {
    if (nfl) atomicAdd(counters + 0, (unsigned long long)nfl);
    if (nfa) atomicAdd(counters + 1, (unsigned long long)nfa);
  }
}

template <bool KS, int DER, int REC, int DM>
static cudaError_t launch_um(const GridP& g, const EosP& e, const MetTables& mt, int s, double dt, const double* dtp,
                             const double* Rold, const double* Un, const double* Us, double* Uout, double* P,
                             unsigned long long* counters, unsigned long long* cfl_out, double* Rnew, cudaStream_t st) {
  using GE = Geo<0>;
  auto kern = k_update_march<KS, DER, REC, DM>;
  constexpr int kMaxDev = 64;
  static std::atomic<int> grid_caps[kMaxDev];
  int dev = 0;
  cudaGetDevice(&dev);
  int grid_cap = dev < kMaxDev ? grid_caps[dev].load(std::memory_order_relaxed) : 0;
  if (!grid_cap) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GE::SMEM);
    if (err != cudaSuccess) return err;
    int sms, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, GE::THREADS, GE::SMEM);
    grid_cap = sms * (per > 0 ? per : 1);
    if (dev < kMaxDev) grid_caps[dev].store(grid_cap, std::memory_order_relaxed);
  }
  LineGeom lg = x_line_geom(g, Rnew, P);
  const unsigned blocks = (unsigned)(lg.nunits < grid_cap ? lg.nunits : grid_cap);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  kern<<<blocks, GE::THREADS, GE::SMEM, st>>>(g, e, mt, lg, s, dt, dtp, Rold, Un, Us, Uout, P, counters, cfl_out, Rnew,
                                               sms);
  return cudaGetLastError();
}

template <bool KS, int DER, int REC>
static cudaError_t um_dm(const GridP& g, const EosP& e, const MetTables& mt, int s, double dt, const double* dtp,
                         const double* Rold, const double* Un, const double* Us, double* Uout, double* P,
                         unsigned long long* cnt, unsigned long long* cfl, double* Rnew, cudaStream_t st) {
  if (g.divb == 1) return launch_um<KS, DER, REC, 1>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, cnt, cfl, Rnew, st);
  return launch_um<KS, DER, REC, 0>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, cnt, cfl, Rnew, st);
}
template <bool KS, int DER>
static cudaError_t um_rec(const GridP& g, const EosP& e, const MetTables& mt, int s, double dt, const double* dtp,
                          const double* Rold, const double* Un, const double* Us, double* Uout, double* P,
                          unsigned long long* cnt, unsigned long long* cfl, double* Rnew, cudaStream_t st) {
  switch (g.rec) {
    case 6: return cudaErrorInvalidValue;  // (the fused kernel keeps the x sweep's register budget)
    case 1: return um_dm<KS, DER, 1>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, cnt, cfl, Rnew, st);
    case 2: return um_dm<KS, DER, 2>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, cnt, cfl, Rnew, st);
    case 3: return um_dm<KS, DER, 3>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, cnt, cfl, Rnew, st);
    case 4: return um_dm<KS, DER, 4>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, cnt, cfl, Rnew, st);
    case 5: return um_dm<KS, DER, 5>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, cnt, cfl, Rnew, st);
    default: return um_dm<KS, DER, 0>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, cnt, cfl, Rnew, st);
  }
}
template <bool KS>
static cudaError_t um_der(const GridP& g, const EosP& e, const MetTables& mt, int s, double dt, const double* dtp,
                          const double* Rold, const double* Un, const double* Us, double* Uout, double* P,
                          unsigned long long* cnt, unsigned long long* cfl, double* Rnew, cudaStream_t st) {
  if (g.der == 4) return um_rec<KS, 4>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, cnt, cfl, Rnew, st);
  if (g.der == 2) return um_rec<KS, 2>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, cnt, cfl, Rnew, st);
  return um_rec<KS, 6>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, cnt, cfl, Rnew, st);
}

}  // namespace march

cudaError_t launch_update_march(bool ks, const GridP& g, const EosP& e, const MetTables& mt, int s, double dt,
                                const double* dtp, const double* Rold, const double* Un, const double* Us, double* Uout,
                                double* P, unsigned long long* counters, unsigned long long* cfl_out, double* Rnew,
                                cudaStream_t st) {
  // slabs, UCT and the curved metric keep the separate kernels (Kerr-Schild: the fused kernel
  // spills at the x sweep's 80-register budget, ptxas 584 B)
  if (g.zhalo || g.divb == 2 || ks) return cudaErrorInvalidValue;
  (void)mt;
  return march::um_der<false>(g, e, mt, s, dt, dtp, Rold, Un, Us, Uout, P, counters, cfl_out, Rnew, st);
}

}  // namespace echo
