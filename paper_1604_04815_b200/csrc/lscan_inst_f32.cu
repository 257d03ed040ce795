// lscan_inst_f32.cu — kernel instantiations for float (see lscan_inst.cuh)
#include "lscan_inst.cuh"

namespace lscan {
const DtypeKernels &kernels_f32() {
    static const DtypeKernels k = make_kernels<float>();
    return k;
}
}  // namespace lscan
