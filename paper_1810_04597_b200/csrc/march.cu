// march.cu — launchers of the axis-sweep kernels K2x/K2y/K2z (march_impl.cuh).
#include "march_pair.cuh"

namespace echo {
namespace march {

// the x sweep with two cells per lane (march_pair.cuh); its own per-device grid cap
template <bool KS, int DER, int REC, int DM>
static cudaError_t launch_x2(const GridP& g, const EosP& e, const MetTables& mt, const double* P, const double* UB,
                             double* R, const double* Bface, double* FSo, cudaStream_t st, const PlaneRange& zr) {
  auto kern = k_march_x2<KS, DER, REC, DM>;
  constexpr int kMaxDev = 64;
  static std::atomic<int> grid_caps[kMaxDev];
  int dev = 0;
  cudaGetDevice(&dev);
  int grid_cap = dev < kMaxDev ? grid_caps[dev].load(std::memory_order_relaxed) : 0;
  if (!grid_cap) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GeoX2::SMEM);
    if (err != cudaSuccess) return err;
    int sms, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, GeoX2::THREADS, GeoX2::SMEM);
    grid_cap = sms * (per > 0 ? per : 1);
    if (dev < kMaxDev) grid_caps[dev].store(grid_cap, std::memory_order_relaxed);
  }
  const LineGeom lg = make_line_geom<0, GeoX2>(g, P, R, zr);
  const unsigned blocks = (unsigned)(lg.nunits < grid_cap ? lg.nunits : grid_cap);
  kern<<<blocks, GeoX2::THREADS, GeoX2::SMEM, st>>>(g, e, mt, lg, P, UB, R, Bface, FSo);
  return cudaGetLastError();
}

template <int AX, bool KS, int DER, int REC, int DM>
static cudaError_t launch_one(const GridP& g, const EosP& e, const MetTables& mt, const double* P, const double* UB,
                              double* R, const double* Bface, double* FSo, cudaStream_t st,
                              const PlaneRange& zr) {
  using GE = typename GeoSel<AX, DM>::type;
  if constexpr (AX == 0 && REC != 6 && ECHO_X_PAIR) {  // 16-byte pairs need 16-byte aligned fields
    if ((((uintptr_t)P) | ((uintptr_t)UB) | ((uintptr_t)R)) % 16 == 0)
      return launch_x2<KS, DER, REC, DM>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  }
  auto kern = k_march<AX, KS, DER, REC, DM>;
#ifdef ECHO_YZ_MAXNREG
  if constexpr (AX != 0 && REC != 6 && !ECHO_PDL) kern = k_march_mr<AX, KS, DER, REC, DM>;
#endif
  // per device (the attribute and the occupancy are per-device properties); the cache is
  // written at most once per device, racing writers store the same value
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
  const LineGeom lg = make_line_geom<AX, GE>(g, P, R, zr);
  unsigned blocks = (unsigned)(lg.nunits < grid_cap ? lg.nunits : grid_cap);
  if (ECHO_PDL && AX != 0) {  // y/z: may start over the previous sweep's tail (griddepcontrol)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(GE::THREADS);
    cfg.dynamicSmemBytes = GE::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, g, e, mt, lg, P, UB, R, Bface, FSo);
  }
  kern<<<blocks, GE::THREADS, GE::SMEM, st>>>(g, e, mt, lg, P, UB, R, Bface, FSo);
  return cudaGetLastError();
}

template <int AX, bool KS, int DER, int REC>
static cudaError_t launch_dn(const GridP& g, const EosP& e, const MetTables& mt, const double* P, const double* UB, double* R,
                             const double* Bface, double* FSo, cudaStream_t st,
                              const PlaneRange& zr) {
  if constexpr (REC == 6) {  // A44: not with UCT (echo_create refuses it)
    if (g.divb == 2) return cudaErrorInvalidValue;
  } else {
    if (g.divb == 2) return launch_one<AX, KS, DER, REC, 2>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  }
  if (g.divb == 1) return launch_one<AX, KS, DER, REC, 1>(g, e, mt, P, UB, R, nullptr, nullptr, st, zr);
  return launch_one<AX, KS, DER, REC, 0>(g, e, mt, P, UB, R, nullptr, nullptr, st, zr);
}
template <int AX, bool KS, int DER>
static cudaError_t launch_rec(const GridP& g, const EosP& e, const MetTables& mt, const double* P, const double* UB, double* R,
                              const double* Bface, double* FSo, cudaStream_t st,
                              const PlaneRange& zr) {
  if (g.rec == 6) {  // A44: flat metric only (echo_create refuses Kerr-Schild)
    if constexpr (KS) return cudaErrorInvalidValue;
    else return launch_dn<AX, KS, DER, 6>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  }
  if (g.rec == 5) return launch_dn<AX, KS, DER, 5>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  if (g.rec == 4) return launch_dn<AX, KS, DER, 4>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  if (g.rec == 3) return launch_dn<AX, KS, DER, 3>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  if (g.rec == 2) return launch_dn<AX, KS, DER, 2>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  if (g.rec == 1) return launch_dn<AX, KS, DER, 1>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  return launch_dn<AX, KS, DER, 0>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
}
template <int AX, bool KS>
static cudaError_t launch_der(const GridP& g, const EosP& e, const MetTables& mt, const double* P, const double* UB, double* R,
                              const double* Bface, double* FSo, cudaStream_t st,
                              const PlaneRange& zr) {
  if (g.der == 4) return launch_rec<AX, KS, 4>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  if (g.der == 2) return launch_rec<AX, KS, 2>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  return launch_rec<AX, KS, 6>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
}

}  // namespace march

cudaError_t launch_march(int axis, bool ks, const GridP& g, const EosP& e, const MetTables& mt, const double* P,
                         const double* UB, double* R, cudaStream_t st, const double* Bface, double* FSo,
                         PlaneRange zr) {
  using namespace march;
  if (ks) {
    if (axis == 0) return launch_der<0, true>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
    if (axis == 1) return launch_der<1, true>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
    return launch_der<2, true>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  }
  if (axis == 0) return launch_der<0, false>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  if (axis == 1) return launch_der<1, false>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
  return launch_der<2, false>(g, e, mt, P, UB, R, Bface, FSo, st, zr);
}

}  // namespace echo
