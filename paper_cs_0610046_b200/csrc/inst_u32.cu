// inst_u32.cu -- explicit instantiation of the launchers/kernels for uint32_t.
#include "launch.cuh"

namespace mm {
MM_DEFINE_INST(uint32_t)
}  // namespace mm
