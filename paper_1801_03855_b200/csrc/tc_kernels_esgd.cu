// Instantiates the hot-path kernels for OP_ESGD (NEXT row f2: elastic averaging fused with the
// SGD step in one pass).  Only the TMA kernels implement it: k_local_tma at p = 1 and the TMA
// two-shot otherwise (the runtime selects nothing else for this op).
#include "tc_kernels.cuh"

namespace tc {
const void* kernel_ptr_esgd(int algo, int p) {
  if (algo == ALGO_LOCAL) return (const void*)k_local_tma<OP_ESGD>;
  if (algo != ALGO_TWOSHOT_TMA) return nullptr;
  switch (p) {
    case 2: return (const void*)k_twoshot_tma<OP_ESGD, 2>;
    case 3: return (const void*)k_twoshot_tma<OP_ESGD, 3>;
    case 4: return (const void*)k_twoshot_tma<OP_ESGD, 4>;
    case 5: return (const void*)k_twoshot_tma<OP_ESGD, 5>;
    case 6: return (const void*)k_twoshot_tma<OP_ESGD, 6>;
    case 7: return (const void*)k_twoshot_tma<OP_ESGD, 7>;
    case 8: return (const void*)k_twoshot_tma<OP_ESGD, 8>;
  }
  return nullptr;
}
}  // namespace tc
