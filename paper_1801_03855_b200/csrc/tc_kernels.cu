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

// The p = 1 TMA stream (variant 0 of ALGO_LOCAL) runs kTmaThreads threads with kTmaSmem bytes
// of dynamic shared memory.
bool is_tma(int algo, int variant) { return algo == ALGO_LOCAL && variant == 0; }

cudaError_t prepare(const void* k, int algo, int variant) {
  if (!is_tma(algo, variant)) return cudaSuccess;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
}

}  // namespace

int max_ctas_per_sm(int op, int algo, int p, int threads, int variant) {
  const void* k = select_kernel(op, algo, p, variant);
  if (!k || prepare(k, algo, variant) != cudaSuccess) return 0;
  int n = 0;
  const bool tma = is_tma(algo, variant);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, tma ? kTmaThreads : threads,
                                                    tma ? kTmaSmem : 0) != cudaSuccess)
    return 0;
  return n;
}

cudaError_t launch_hot(int op, int algo, const KParams& kp, int ctas, int threads, int nlocal,
                       bool cooperative, cudaStream_t stream, int variant) {
  const void* k = select_kernel(op, algo, kp.p, variant);
  if (!k) return cudaErrorInvalidValue;
  cudaError_t e = prepare(k, algo, variant);
  if (e != cudaSuccess) return e;
  KParams arg = kp;
  void* args[] = {&arg};
  const bool tma = is_tma(algo, variant);
  dim3 grid(ctas, nlocal), block(tma ? kTmaThreads : threads);
  const size_t smem = tma ? kTmaSmem : 0;
  if (cooperative) return cudaLaunchCooperativeKernel(k, grid, block, args, smem, stream);
  return cudaLaunchKernel(k, grid, block, args, smem, stream);
}

}  // namespace tc
