// inst_i32.cu -- explicit instantiation of the launchers/kernels for int32_t.
#include "launch.cuh"

namespace mm {
MM_DEFINE_INST(int32_t)
}  // namespace mm
