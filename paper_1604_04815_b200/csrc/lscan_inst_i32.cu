// lscan_inst_i32.cu — kernel instantiations for int32_t (see lscan_inst.cuh)
#include "lscan_inst.cuh"

namespace lscan {
const DtypeKernels &kernels_i32() {
    static const DtypeKernels k = make_kernels<int32_t>();
    return k;
}
}  // namespace lscan
