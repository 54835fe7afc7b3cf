// inst_f64.cu -- explicit instantiation of the launchers/kernels for double.
#include "launch.cuh"

namespace mm {
MM_DEFINE_INST(double)
}  // namespace mm
