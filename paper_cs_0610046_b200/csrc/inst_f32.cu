// inst_f32.cu -- explicit instantiation of the launchers/kernels for float.
#include "launch.cuh"

namespace mm {
MM_DEFINE_INST(float)
}  // namespace mm
