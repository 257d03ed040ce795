// lscan_inst_f64.cu — kernel instantiations for double (see lscan_inst.cuh)
#include "lscan_inst.cuh"

namespace lscan {
const DtypeKernels &kernels_f64() {
    static const DtypeKernels k = make_kernels<double>();
    return k;
}
}  // namespace lscan
