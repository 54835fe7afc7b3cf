// inst_u8.cu -- explicit instantiation of the launchers/kernels for uint8_t.
#include "launch.cuh"

namespace mm {
MM_DEFINE_INST(uint8_t)
}  // namespace mm
