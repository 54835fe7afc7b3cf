// inst_i16.cu -- explicit instantiation of the launchers/kernels for int16_t.
#include "launch.cuh"

namespace mm {
MM_DEFINE_INST(int16_t)
}  // namespace mm
