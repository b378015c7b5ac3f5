// Assembly kernels for dimension 3, kernel family 3 (rbg_kernel_family, include/rbg.h).
#include "rbg_asm.cuh"

namespace rbg {
RBG_ASM_DEFINE(3, 3)
}  // namespace rbg
