// Kernel selection and launch (the kernels themselves: tc_kernels.cuh, instantiated per op in
// tc_kernels_{allreduce,sgd,easgd}.cu).
#include "tc_internal.h"

namespace tc {
const void* kernel_ptr_allreduce(int algo, int p);
const void* kernel_ptr_sgd(int algo, int p);
const void* kernel_ptr_easgd(int algo, int p);
const void* kernel_ptr_esgd(int algo, int p);
const void* kernel_ptr_bcast(int algo, int p);
const void* kernel_ptr_easync(int algo, int p);

namespace {
const void* select_kernel(int op, int algo, int p) {
  switch (op) {
    case OP_ALLREDUCE: return kernel_ptr_allreduce(algo, p);
    case OP_SGD: return kernel_ptr_sgd(algo, p);
    case OP_EASGD: return kernel_ptr_easgd(algo, p);
    case OP_ESGD: return kernel_ptr_esgd(algo, p);
    case OP_BCAST: return kernel_ptr_bcast(algo, p);
    case OP_EASYNC: return kernel_ptr_easync(algo, p);
  }
  return nullptr;
}

// TMA kernels run fixed thread counts with dynamic shared memory: the p = 1 stream (ALGO_LOCAL)
// and the TMA two-shot.
struct Shape {
  int threads;
  int smem;
};
Shape shape_of(int op, int algo, int p, int threads) {
  if (algo == ALGO_LOCAL) return {kTmaThreads, local_smem(op)};
  if (algo == ALGO_TWOSHOT_TMA) return {kT2Threads, t2_smem(op, p)};
  // NVLS: the allreduce takes the comm's thread count (>= 2 warps), the other ops 512
  if (algo == ALGO_NVLS) return {op == OP_ALLREDUCE ? threads : kNvlsThreads, 0};
  return {threads, 0};
}

cudaError_t prepare(const void* k, const Shape& sh) {
  if (sh.smem == 0) return cudaSuccess;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sh.smem);
}

}  // namespace

int max_ctas_per_sm(int op, int algo, int p, int threads) {
  const void* k = select_kernel(op, algo, p);
  const Shape sh = shape_of(op, algo, p, threads);
  if (!k || prepare(k, sh) != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, sh.threads, sh.smem) != cudaSuccess)
    return 0;
  return n;
}

int launch_threads(int op, int algo, int p, int threads) {
  return shape_of(op, algo, p, threads).threads;
}

cudaError_t launch_hot(int op, int algo, const KParams& kp, int ctas, int threads, int nlocal,
                       bool cooperative, cudaStream_t stream) {
  const void* k = select_kernel(op, algo, kp.p);
  if (!k) return cudaErrorInvalidValue;
  const Shape sh = shape_of(op, algo, kp.p, threads);
  cudaError_t e = prepare(k, sh);
  if (e != cudaSuccess) return e;
  KParams arg = kp;
  void* args[] = {&arg};
  dim3 grid(ctas, nlocal), block(sh.threads);
  const size_t smem = sh.smem;
  if (cooperative) return cudaLaunchCooperativeKernel(k, grid, block, args, smem, stream);
  return cudaLaunchKernel(k, grid, block, args, smem, stream);
}

}  // namespace tc
