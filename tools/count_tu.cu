// count_tu.cu — instantiates only the Minkowski WENO5/DER6/field-CD sweeps (and the fused
// update + x sweep) so an arithmetic rewrite can be compiled and its FP64 SASS counted in
// seconds: nvcc -cubin ... tools/count_tu.cu && tools/fp64_count.sh <cubin>
#include "../paper_1810_04597_b200/csrc/march_impl.cuh"

namespace echo {
namespace march {
template __global__ void k_march<0, false, 6, 0, 0>(const GridP, const EosP, const MetTables, const LineGeom,
                                                    const double*, const double*, double*, const double*, double*);
template __global__ void k_march<1, false, 6, 0, 0>(const GridP, const EosP, const MetTables, const LineGeom,
                                                    const double*, const double*, double*, const double*, double*);
template __global__ void k_march<2, false, 6, 0, 0>(const GridP, const EosP, const MetTables, const LineGeom,
                                                    const double*, const double*, double*, const double*, double*);
}  // namespace march
}  // namespace echo
namespace echo {
namespace march {
template __global__ void k_march<0, false, 6, 6, 0>(const GridP, const EosP, const MetTables, const LineGeom,
                                                    const double*, const double*, double*, const double*, double*);
template __global__ void k_march<1, false, 6, 6, 0>(const GridP, const EosP, const MetTables, const LineGeom,
                                                    const double*, const double*, double*, const double*, double*);
}  // namespace march
}  // namespace echo
