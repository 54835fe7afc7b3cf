// inst_i8.cu -- explicit instantiation of the launchers/kernels for int8_t.
#include "launch.cuh"

namespace mm {
MM_DEFINE_INST(int8_t)
}  // namespace mm
