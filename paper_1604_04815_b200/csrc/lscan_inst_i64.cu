// lscan_inst_i64.cu — kernel instantiations for int64_t (see lscan_inst.cuh)
#include "lscan_inst.cuh"

namespace lscan {
const DtypeKernels &kernels_i64() {
    static const DtypeKernels k = make_kernels<int64_t>();
    return k;
}
}  // namespace lscan
