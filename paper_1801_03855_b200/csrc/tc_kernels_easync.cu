// Instantiates the asynchronous-server elastic update (NEXT row f2: every chunk's owner applies
// the clients' Elastic1/Elastic2 pairs in a recorded arrival order).  Only the
// TMA two-shot implements it (p = 1 is tc_easgd_update's local path: one arrival).
#include "tc_kernels.cuh"

namespace tc {
const void* kernel_ptr_easync(int algo, int p) {
  if (algo != ALGO_TWOSHOT_TMA) return nullptr;
  switch (p) {
    case 2: return (const void*)k_twoshot_tma<OP_EASYNC, 2>;
    case 3: return (const void*)k_twoshot_tma<OP_EASYNC, 3>;
    case 4: return (const void*)k_twoshot_tma<OP_EASYNC, 4>;
    case 5: return (const void*)k_twoshot_tma<OP_EASYNC, 5>;
    case 6: return (const void*)k_twoshot_tma<OP_EASYNC, 6>;
    case 7: return (const void*)k_twoshot_tma<OP_EASYNC, 7>;
    case 8: return (const void*)k_twoshot_tma<OP_EASYNC, 8>;
  }
  return nullptr;
}
}  // namespace tc
