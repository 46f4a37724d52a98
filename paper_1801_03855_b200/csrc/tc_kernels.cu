// Kernel selection and launch (the kernels themselves: tc_kernels.cuh, instantiated per op in
// tc_kernels_{allreduce,sgd,easgd}.cu).
#include "tc_internal.h"

namespace tc {
const void* kernel_ptr_allreduce(int algo, int p, int variant);
const void* kernel_ptr_sgd(int algo, int p, int variant);
const void* kernel_ptr_easgd(int algo, int p, int variant);

namespace {
const void* select_kernel(int op, int algo, int p, int variant) {
  switch (op) {
    case OP_ALLREDUCE: return kernel_ptr_allreduce(algo, p, variant);
    case OP_SGD: return kernel_ptr_sgd(algo, p, variant);
    case OP_EASGD: return kernel_ptr_easgd(algo, p, variant);
  }
  return nullptr;
}

}  // namespace

int max_ctas_per_sm(int op, int algo, int p, int threads, int variant) {
  const void* k = select_kernel(op, algo, p, variant);
  if (!k) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, threads, 0) != cudaSuccess) return 0;
  return n;
}

cudaError_t launch_hot(int op, int algo, const KParams& kp, int ctas, int threads, int nlocal,
                       bool cooperative, cudaStream_t stream, int variant) {
  const void* k = select_kernel(op, algo, kp.p, variant);
  if (!k) return cudaErrorInvalidValue;
  KParams arg = kp;
  void* args[] = {&arg};
  dim3 grid(ctas, nlocal), block(threads);
  if (cooperative) return cudaLaunchCooperativeKernel(k, grid, block, args, 0, stream);
  return cudaLaunchKernel(k, grid, block, args, 0, stream);
}

}  // namespace tc
