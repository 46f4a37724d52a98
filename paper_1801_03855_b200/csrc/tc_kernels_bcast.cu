// Instantiates the tensor broadcast (P:183 weight initialisation, P:205-213 KVStore.pull):
// scatter from the root (each owner copies its chunk of the root's tensors), then the TMA
// two-shot's allgather; or, for groups in multicast-bound memory, the root's multicast stores
// through the switch (k_nvls_bcast).
#include "tc_kernels.cuh"

namespace tc {
const void* kernel_ptr_bcast(int algo, int p) {
  if (algo == ALGO_NVLS) {
    switch (p) {
      case 2: return (const void*)k_nvls_bcast<2>;
      case 3: return (const void*)k_nvls_bcast<3>;
      case 4: return (const void*)k_nvls_bcast<4>;
      case 5: return (const void*)k_nvls_bcast<5>;
      case 6: return (const void*)k_nvls_bcast<6>;
      case 7: return (const void*)k_nvls_bcast<7>;
      case 8: return (const void*)k_nvls_bcast<8>;
    }
    return nullptr;
  }
  if (algo != ALGO_TWOSHOT_TMA) return nullptr;
  switch (p) {
    case 2: return (const void*)k_twoshot_tma<OP_BCAST, 2>;
    case 3: return (const void*)k_twoshot_tma<OP_BCAST, 3>;
    case 4: return (const void*)k_twoshot_tma<OP_BCAST, 4>;
    case 5: return (const void*)k_twoshot_tma<OP_BCAST, 5>;
    case 6: return (const void*)k_twoshot_tma<OP_BCAST, 6>;
    case 7: return (const void*)k_twoshot_tma<OP_BCAST, 7>;
    case 8: return (const void*)k_twoshot_tma<OP_BCAST, 8>;
  }
  return nullptr;
}
}  // namespace tc
