// inst_u16.cu -- explicit instantiation of the launchers/kernels for uint16_t.
#include "launch.cuh"

namespace mm {
MM_DEFINE_INST(uint16_t)
}  // namespace mm
