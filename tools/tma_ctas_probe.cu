// Per-CTA TMA throughput at low CTA counts (design evidence for k_twoshot_tma, not product code).
//
// Every GPU pulls a peer's buffer (ring pattern, all GPUs concurrently) with G CTAs:
//   tma-load : W producer warps per CTA, each lane 0 keeping its own ring of NS/W stages of CH
//              bytes full with cp.async.bulk global->shared (data discarded): the load ceiling;
//   tma-copy : the same, then cp.async.bulk shared->global into local memory;
//   ldg      : 1024 threads per CTA, ld.global.cg 16 B x U in flight per thread, stored locally.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tma_ctas_probe tools/tma_ctas_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void wait_parity(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
               "@!P bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(par) : "memory");
}

// W warps, each with its own ring of NSW stages; chunks dealt round-robin over (CTA, warp).
template <int CH, int NSW, int W, bool STORE>
__global__ void tma_pull(const char* __restrict__ src, char* __restrict__ dst, size_t nbytes) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[W * NSW];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0) return;
  uint64_t* mb = bar + w * NSW;
  char* ring = sm + (size_t)w * NSW * CH;
  for (int s = 0; s < NSW; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mb[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t nch = nbytes / CH, lanes = (size_t)gridDim.x * W, me = (size_t)blockIdx.x * W + w;
  const size_t mine = nch > me ? (nch - me + lanes - 1) / lanes : 0;
  auto issue = [&](size_t k) {
    const int s = (int)(k % NSW);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mb[s])), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(ring + (size_t)s * CH)), "l"(src + (me + k * lanes) * CH), "r"(CH),
                 "r"(smem_u32(&mb[s])) : "memory");
  };
  for (size_t k = 0; k < mine && k < NSW; ++k) issue(k);
  for (size_t k = 0; k < mine; ++k) {
    const int s = (int)(k % NSW);
    wait_parity(&mb[s], (uint32_t)((k / NSW) & 1));
    if (STORE) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + (me + k * lanes) * CH),
                   "r"(smem_u32(ring + (size_t)s * CH)), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    if (k + NSW < mine) issue(k + NSW);
  }
  if (STORE) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int U>
__global__ void __launch_bounds__(1024) ldg_pull(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (; i < n; i += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < n) asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(src + j));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < n) dst[j] = v[u];
    }
  }
}

int main(int argc, char** argv) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need >= 2 GPUs\n"); return 0; }
  const size_t bytes = (size_t)256 << 20;
  std::vector<char*> a(n), b(n);
  std::vector<cudaStream_t> st(n);
  std::vector<cudaEvent_t> e0(n), e1(n);
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    for (int q = 0; q < n; ++q)
      if (q != d) { int ok = 0; CK(cudaDeviceCanAccessPeer(&ok, d, q)); if (ok) CK(cudaDeviceEnablePeerAccess(q, 0)); }
    CK(cudaMalloc(&a[d], bytes));
    CK(cudaMalloc(&b[d], bytes));
    CK(cudaMemset(a[d], 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  auto run = [&](const char* name, auto launch) {
    for (int rep = 0; rep < 2; ++rep) {
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d])); }
      for (int it = 0; it < 3; ++it)
        for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); launch(d); }
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e1[d], st[d])); }
      float worst = 0;
      for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d)); CK(cudaEventSynchronize(e1[d]));
        float ms = 0; CK(cudaEventElapsedTime(&ms, e0[d], e1[d])); if (ms > worst) worst = ms;
      }
      CK(cudaGetLastError());
      if (rep == 1) printf("%-44s %8.1f GB/s per GPU\n", name, bytes * 3.0 / (worst / 1e3) / 1e9);
    }
  };
  char name[128];
  auto tma = [&](const char* what, auto kern, int ch, int nsw, int w) {
    const int smem = ch * nsw * w;
    for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); }
    for (int g : {8, 16, 32, 64, 148}) {
      snprintf(name, sizeof name, "%s CH=%dK NS=%dx%d G=%d", what, ch / 1024, w, nsw, g);
      run(name, [&](int d) { int q = (d + 1) % n; kern<<<g, 32 * w, smem, st[d]>>>(a[q], b[d], bytes); });
    }
  };
  tma("tma-load", tma_pull<4096, 32, 1, false>, 4096, 32, 1);
  tma("tma-load", tma_pull<16384, 8, 1, false>, 16384, 8, 1);
  tma("tma-load", tma_pull<32768, 5, 1, false>, 32768, 5, 1);
  tma("tma-load", tma_pull<16384, 2, 4, false>, 16384, 2, 4);
  tma("tma-load", tma_pull<4096, 8, 4, false>, 4096, 8, 4);
  tma("tma-copy", tma_pull<16384, 8, 1, true>, 16384, 8, 1);
  tma("tma-copy", tma_pull<32768, 5, 1, true>, 32768, 5, 1);
  for (int g : {8, 16, 32, 64, 148}) {
    snprintf(name, sizeof name, "ldg.cg 1024 thr U=8 G=%d", g);
    run(name, [&](int d) { int q = (d + 1) % n; ldg_pull<8><<<g, 1024, 0, st[d]>>>((const float4*)a[q], (float4*)b[d], bytes / 16); });
  }
  printf("done\n");
  return 0;
}
