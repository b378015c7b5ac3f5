// Assembly kernels for dimension 2, kernel family 2 (rbg_kernel_family, include/rbg.h).
#include "rbg_asm.cuh"

namespace rbg {
RBG_ASM_DEFINE(2, 2)
}  // namespace rbg
