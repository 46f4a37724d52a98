// NVLink / NVSwitch data-path probe for B200 (design evidence, not product code).
//
// Kernels launched from tools/nvl_probe.py (one process per GPU, torch symmetric memory for the
// multicast and peer pointers).  Each measures the ceiling of one way to move an allreduce's
// bytes, so the product kernels can be designed against measured numbers:
//   mm_ar     : NVLS allreduce of this rank's owner range: multimem.ld_reduce + multimem.st
//   mm_ld     : multimem.ld_reduce only (result stored to local memory)
//   mm_st     : multimem.st only (source: local memory)
//   tma_push  : cp.async.bulk shared -> peer global (stores over NVLink from the TMA engine),
//               every peer 1/(p-1) of the bytes, in one kernel
//   tma_pull  : cp.async.bulk peer global -> shared (loads over NVLink), every peer
//   st_push   : 16-B st.global from registers into every peer (SM stores)
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
//        -o tools/bin/libnvl_probe.so tools/nvl_probe.cu
#include <cuda_runtime.h>
#include <cstdint>

namespace {

__device__ __forceinline__ float4 mm_ldr(const float* p, int weak) {
  float4 v;
  if (weak)
    asm volatile("multimem.ld_reduce.weak.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  else
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mm_st(float* p, float4 v, int weak) {
  if (weak)
    asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  else
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// MODE 0: ld_reduce + st (allreduce), 1: ld_reduce -> local, 2: local -> st
template <int U, int MODE>
__global__ void mm_kernel(float* mc, float* local, long lo, long hi, int weak) {
  const long stride = (long)gridDim.x * blockDim.x * U;
  for (long i = lo + (long)blockIdx.x * blockDim.x * U + threadIdx.x; i < hi; i += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long j = i + (long)u * blockDim.x;
      if (j < hi) {
        if (MODE == 2) v[u] = reinterpret_cast<const float4*>(local)[j];
        else v[u] = mm_ldr(mc + 4 * j, weak);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long j = i + (long)u * blockDim.x;
      if (j < hi) {
        if (MODE == 1) reinterpret_cast<float4*>(local)[j] = v[u];
        else mm_st(mc + 4 * j, v[u], weak);
      }
    }
  }
}

struct Peers { float* p[8]; };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Block b serves peer j = b % np.  Each block streams its share of the peer's part in tiles of
// `tile` bytes out of shared memory with bulk stores, at most `depth` groups in flight.
__global__ void tma_push_kernel(Peers peers, int np, long part_bytes, int tile, int depth,
                                int rank) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int j = blockIdx.x % np;
  const int bpp = gridDim.x / np;
  const int bi = blockIdx.x / np;
  if (bi >= bpp) return;
  // destination: the peer's buffer, region of this rank (so pushes never overlap)
  unsigned char* dst = (unsigned char*)peers.p[j] + (long)rank * part_bytes;
  const long ntiles = part_bytes / tile;
  if (threadIdx.x == 0) {
    int inflight = 0;
    for (long t = bi; t < ntiles; t += bpp) {
      const int slot = (int)(t / bpp) % depth;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                       dst + t * tile),
                   "r"(smem_u32(sm + (long)slot * tile)), "r"(tile)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (++inflight >= depth) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(7) : "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra W_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

// Block b pulls from peer j = b % np into a ring of `depth` shared-memory tiles (nothing consumes
// the data: the ceiling of the TMA pull).
__global__ void tma_pull_kernel(Peers peers, int np, long part_bytes, int tile, int depth,
                                int rank) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[16];
  const int j = blockIdx.x % np;
  const int bpp = gridDim.x / np;
  const int bi = blockIdx.x / np;
  if (bi >= bpp || threadIdx.x != 0) return;
  for (int s = 0; s < depth; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const unsigned char* src = (const unsigned char*)peers.p[j] + (long)rank * part_bytes;
  const long ntiles = part_bytes / tile;
  long k = 0;
  for (long t = bi; t < ntiles; t += bpp, ++k) {
    const int s = (int)(k % depth);
    if (k >= depth) mbar_wait(&full[s], (uint32_t)((k / depth - 1) & 1));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                 "r"(tile) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(sm + (long)s * tile)), "l"(src + t * tile), "r"(tile),
        "r"(smem_u32(&full[s]))
        : "memory");
  }
  for (long q = (k > depth ? k - depth : 0); q < k; ++q)
    mbar_wait(&full[q % depth], (uint32_t)((q / depth) & 1));
}

// SM stores: block b writes its share of peer j's region with 16-B stores, U per thread in flight.
template <int U>
__global__ void st_push_kernel(Peers peers, int np, long part_bytes, int rank) {
  const int j = blockIdx.x % np;
  const int bpp = gridDim.x / np;
  const int bi = blockIdx.x / np;
  if (bi >= bpp) return;
  float4* dst = (float4*)((unsigned char*)peers.p[j] + (long)rank * part_bytes);
  const long n = part_bytes / 16;
  const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
  for (long i = (long)bi * blockDim.x * U + threadIdx.x; i < n; i += (long)bpp * blockDim.x * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long q = i + (long)u * blockDim.x;
      if (q < n) dst[q] = v;
    }
  }
}

}  // namespace

extern "C" {

int probe_mm(int mode, float* mc, float* local, long lo4, long hi4, int ctas, int threads,
             int unroll, int weak, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
#define L(U, M) mm_kernel<U, M><<<ctas, threads, 0, s>>>(mc, local, lo4, hi4, weak)
#define LM(U)                   \
  if (mode == 0) L(U, 0);       \
  else if (mode == 1) L(U, 1);  \
  else L(U, 2);
  switch (unroll) {
    case 1: LM(1); break;
    case 2: LM(2); break;
    case 4: LM(4); break;
    case 8: LM(8); break;
    default: return -1;
  }
#undef LM
#undef L
  return (int)cudaGetLastError();
}

int probe_tma(int push, float** peers, int np, long part_bytes, int tile, int depth, int ctas,
              int rank, void* stream) {
  Peers P{};
  for (int i = 0; i < np && i < 8; ++i) P.p[i] = peers[i];
  const int smem = tile * depth;
  if (push) {
    cudaFuncSetAttribute(tma_push_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tma_push_kernel<<<ctas, 32, smem, (cudaStream_t)stream>>>(P, np, part_bytes, tile, depth, rank);
  } else {
    cudaFuncSetAttribute(tma_pull_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tma_pull_kernel<<<ctas, 32, smem, (cudaStream_t)stream>>>(P, np, part_bytes, tile, depth, rank);
  }
  return (int)cudaGetLastError();
}

int probe_st_push(float** peers, int np, long part_bytes, int ctas, int threads, int rank,
                  void* stream) {
  Peers P{};
  for (int i = 0; i < np && i < 8; ++i) P.p[i] = peers[i];
  st_push_kernel<4><<<ctas, threads, 0, (cudaStream_t)stream>>>(P, np, part_bytes, rank);
  return (int)cudaGetLastError();
}

}  // extern "C"
