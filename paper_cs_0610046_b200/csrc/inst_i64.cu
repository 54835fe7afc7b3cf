// inst_i64.cu -- explicit instantiation of the launchers/kernels for int64_t.
#include "launch.cuh"

namespace mm {
MM_DEFINE_INST(int64_t)
}  // namespace mm
