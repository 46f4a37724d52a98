// Instantiates the hot-path kernels for OP_EASGD (one translation unit per op so the three
// compile in parallel; the kernel templates live in tc_kernels.cuh).
#include "tc_kernels.cuh"

namespace tc {
const void* kernel_ptr_easgd(int algo, int p) { return kernel_ptr<OP_EASGD>(algo, p); }
}  // namespace tc
