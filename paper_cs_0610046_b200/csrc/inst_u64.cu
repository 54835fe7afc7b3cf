// inst_u64.cu -- explicit instantiation of the launchers/kernels for uint64_t.
#include "launch.cuh"

namespace mm {
MM_DEFINE_INST(uint64_t)
}  // namespace mm
