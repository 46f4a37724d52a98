// NVLink peer-access probe for B200 (design evidence for libtc's kernels, not product code).
//
// One process drives all visible GPUs with peer access enabled.  For each kernel shape it
// measures, with CUDA events on every device and the max over devices:
//   pull : every GPU copies a peer's buffer into its own memory (loads cross NVLink)
//   push : every GPU copies its own buffer into a peer's memory (stores cross NVLink)
// in the "ring" pattern (GPU i with GPU i+1 mod n, all concurrently: every GPU both sends and
// receives, as in an allreduce), plus cudaMemcpyPeerAsync for reference.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o p2p_probe tools/p2p_probe.cu
//   ./p2p_probe [MB]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)

template <int U, int MODE>
__global__ void copy_kernel(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (; i < n; i += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < n) {
        const float* p = (const float*)(src + j);
        if (MODE == 0) {
          v[u] = src[j];
        } else if (MODE == 1) {
          asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(p));
        } else if (MODE == 2) {
          asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(p));
        } else {
          asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(p));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < n) dst[j] = v[u];
    }
  }
}

// All-peer pattern in ONE kernel: block b works for peer j = b % np (np = n-1 peers); every GPU
// moves 1/np of the buffer to/from each peer concurrently (the reduce-scatter traffic shape).
struct Peers { float4* p[8]; };
template <int U, bool PUSH>
__global__ void allpeer_kernel(Peers peers, float4* local, size_t part, int np) {
  const int j = blockIdx.x % np;
  const int bpp = gridDim.x / np;
  const int bj = blockIdx.x / np;
  float4* remote = peers.p[j] + (size_t)j * part;
  float4* mine = local + (size_t)j * part;
  size_t i = (size_t)bj * blockDim.x * U + threadIdx.x;
  const size_t stride = (size_t)bpp * blockDim.x * U;
  for (; i < part; i += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t k = i + (size_t)u * blockDim.x;
      if (k < part) {
        const float* src = (const float*)(PUSH ? mine + k : remote + k);
        asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(src));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t k = i + (size_t)u * blockDim.x;
      if (k < part) { if (PUSH) remote[k] = v[u]; else mine[k] = v[u]; }
    }
  }
}

// TMA bulk-copy engine: ONE thread per CTA streams CH-byte chunks global -> smem -> global with
// cp.async.bulk (NS stages).  Chunks are taken round-robin by CTA.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
template <int CH, int NS>
__global__ void __launch_bounds__(32) tma_copy(const char* __restrict__ src, char* __restrict__ dst,
                                               size_t nbytes) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long bar[NS];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NS; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const size_t nch = nbytes / CH;
  // my chunks: c = blockIdx.x + k * gridDim.x
  size_t mine = nch > blockIdx.x ? (nch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto chunk = [&](size_t k) { return (size_t)blockIdx.x + k * gridDim.x; };
  auto issue = [&](size_t k) {
    const int s = (int)(k % NS);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                 "r"(CH));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sm + (size_t)s * CH)),
        "l"(src + chunk(k) * CH), "r"(CH), "r"(smem_u32(&bar[s]))
        : "memory");
  };
  for (size_t k = 0; k < mine && k < NS; ++k) issue(k);
  for (size_t k = 0; k < mine; ++k) {
    const int s = (int)(k % NS);
    const uint32_t parity = (uint32_t)((k / NS) & 1);
    asm volatile(
        "{\n.reg .pred P;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(&bar[s])),
        "r"(parity)
        : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                     dst + chunk(k) * CH),
                 "r"(smem_u32(sm + (size_t)s * CH)), "r"(CH)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    if (k + NS < mine) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue(k + NS);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Local fused-SGD stream on flat buffers (3 reads, 2 writes per element): LDG version.
__device__ __forceinline__ float4 ldna(const float4* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void sgd4(float4 g, float4& w, float4& d) {
  float* gp = &g.x; float* wp = &w.x; float* dp = &d.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float t = __fadd_rn(__fmul_rn(0.01f, gp[i]), __fmul_rn(1e-4f, wp[i]));
    dp[i] = __fsub_rn(__fmul_rn(0.9f, dp[i]), __fmul_rn(0.1f, t));
    wp[i] = __fadd_rn(wp[i], dp[i]);
  }
}
template <int U>
__global__ void sgd_ldg(const float4* __restrict__ g, float4* __restrict__ w, float4* __restrict__ d,
                        size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (; i < n; i += stride) {
    float4 a[U], b[U], c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < n) { a[u] = ldna(g + j); b[u] = ldna(w + j); c[u] = ldna(d + j); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < n) { sgd4(a[u], b[u], c[u]); w[j] = b[u]; d[j] = c[u]; }
    }
  }
}
// Same, but every CTA streams its own contiguous 1/gridDim range (no grid-stride locality).
template <int U>
__global__ void sgd_ldg_ranges(const float4* __restrict__ g, float4* __restrict__ w,
                               float4* __restrict__ d, size_t n) {
  const size_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
  for (size_t i = lo + threadIdx.x; i < hi; i += (size_t)blockDim.x * U) {
    float4 a[U], b[U], c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < hi) { a[u] = ldna(g + j); b[u] = ldna(w + j); c[u] = ldna(d + j); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < hi) { sgd4(a[u], b[u], c[u]); w[j] = b[u]; d[j] = c[u]; }
    }
  }
}
// TMA version: warp 0 lane 0 produces (bulk loads of g, w, d tiles into NS stages), the other
// warps consume from shared memory and store with STG.
template <int TILE, int NS>
__global__ void __launch_bounds__(32 * 9) sgd_tma(const float4* __restrict__ g, float4* __restrict__ w,
                                                  float4* __restrict__ d, size_t n) {
  extern __shared__ __align__(128) float4 sm4[];
  __shared__ __align__(8) unsigned long long full[NS], empty[NS];
  const int warp = threadIdx.x >> 5, lane_id = threadIdx.x & 31;
  const int ncons = blockDim.x - 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(ncons));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t ntiles = (n + TILE - 1) / TILE;
  auto wait = [](unsigned long long* b, uint32_t parity) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
                 "@!P bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
  };
  if (warp == 0) {
    if (lane_id != 0) return;
    size_t k = 0;
    for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
      const int s = (int)(k % NS);
      if (k >= NS) wait(&empty[s], (uint32_t)(((k / NS) - 1) & 1));
      const size_t lo = tile * TILE;
      const uint32_t cnt = (uint32_t)(n - lo < TILE ? n - lo : TILE);
      const uint32_t bytes = cnt * 16;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(3 * bytes));
      const float4* src[3] = {g + lo, w + lo, d + lo};
      for (int o = 0; o < 3; ++o)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(sm4 + ((size_t)s * 3 + o) * TILE)), "l"(src[o]), "r"(bytes),
                     "r"(smem_u32(&full[s])) : "memory");
    }
    return;
  }
  size_t k = 0;
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    const int s = (int)(k % NS);
    wait(&full[s], (uint32_t)((k / NS) & 1));
    const size_t lo = tile * TILE;
    const int cnt = (int)(n - lo < TILE ? n - lo : TILE);
    const float4* sg = sm4 + ((size_t)s * 3 + 0) * TILE;
    const float4* sw = sm4 + ((size_t)s * 3 + 1) * TILE;
    const float4* sd = sm4 + ((size_t)s * 3 + 2) * TILE;
    for (int i = threadIdx.x - 32; i < cnt; i += ncons) {
      float4 a = sg[i], b = sw[i], c = sd[i];
      sgd4(a, b, c);
      w[lo + i] = b;
      d[lo + i] = c;
    }
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
  }
}

typedef void (*KFn)(const float4*, float4*, size_t);

template <int U, int MODE> KFn kfn() { return copy_kernel<U, MODE>; }

int main(int argc, char** argv) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need >= 2 GPUs\n"); return 0; }
  size_t mb = argc > 1 ? atol(argv[1]) : 256;
  size_t bytes = mb << 20, nvec = bytes / 16;
  std::vector<float4*> a(n), b(n);
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
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  printf("GPUs %d, SMs %d, buffer %zu MB per GPU, ring pattern (all GPUs concurrently)\n", n, sms, mb);

  auto run = [&](const char* name, auto launch) {
    for (int rep = 0; rep < 2; ++rep) {  // rep 0 = warmup
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d])); }
      const int iters = 5;
      for (int it = 0; it < iters; ++it)
        for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); launch(d); }
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e1[d], st[d])); }
      float worst = 0;
      for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        if (ms > worst) worst = ms;
      }
      CK(cudaGetLastError());
      if (rep == 1) printf("%-48s %8.1f GB/s per GPU per direction\n", name, bytes * 5.0 / (worst / 1e3) / 1e9);
    }
  };

  struct Shape { int ctas_per_sm, threads; };
  Shape shapes[] = {{1, 512}, {2, 512}, {4, 256}, {8, 256}, {2, 1024}, {16, 128}};
  const char* modes[] = {"ld", "ld.L1::no_allocate", "ld.cg", "ld.nc.na"};
  KFn fns[4][4] = {{kfn<1,0>(), kfn<2,0>(), kfn<4,0>(), kfn<8,0>()},
                   {kfn<1,1>(), kfn<2,1>(), kfn<4,1>(), kfn<8,1>()},
                   {kfn<1,2>(), kfn<2,2>(), kfn<4,2>(), kfn<8,2>()},
                   {kfn<1,3>(), kfn<2,3>(), kfn<4,3>(), kfn<8,3>()}};
  int unr[4] = {1, 2, 4, 8};
  char name[128];
  for (int m = 0; m < 4; ++m)
    for (auto s : shapes)
      for (int ui = 0; ui < 4; ++ui) {
        if (m != 1 && !(s.ctas_per_sm == 2 && s.threads == 512)) continue;  // flavours at one shape
        int grid = sms * s.ctas_per_sm;
        KFn f = fns[m][ui];
        snprintf(name, sizeof name, "pull %s %dx%d U=%d", modes[m], grid, s.threads, unr[ui]);
        run(name, [&](int d) { int q = (d + 1) % n;
          f<<<grid, s.threads, 0, st[d]>>>(a[q], b[d], nvec); });
      }
  for (auto s : shapes)
    for (int ui = 0; ui < 4; ++ui) {
      int grid = sms * s.ctas_per_sm;
      KFn f = fns[1][ui];
      snprintf(name, sizeof name, "push %dx%d U=%d", grid, s.threads, unr[ui]);
      run(name, [&](int d) { int q = (d + 1) % n;
        f<<<grid, s.threads, 0, st[d]>>>(a[d], b[q], nvec); });
    }
  {
    int grid = sms * 2;
    KFn f = fns[1][2];
    snprintf(name, sizeof name, "local HBM copy %dx512 U=4", grid);
    run(name, [&](int d) { f<<<grid, 512, 0, st[d]>>>(a[d], b[d], nvec); });
  }
  {
    // fused SGD stream (3 reads + 2 writes per element) over 3 flat buffers of bytes/3 each
    size_t n3 = nvec / 3;
    double sgd_bytes = 5.0 * n3 * 16;
    auto runs = [&](const char* nm, auto launch) {
      for (int rep = 0; rep < 2; ++rep) {
        for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
        CK(cudaSetDevice(0));
        CK(cudaEventRecord(e0[0], st[0]));
        for (int it = 0; it < 5; ++it) launch(0);
        CK(cudaEventRecord(e1[0], st[0]));
        CK(cudaEventSynchronize(e1[0]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0[0], e1[0]));
        CK(cudaGetLastError());
        if (rep) printf("%-48s %8.1f GB/s HBM (5 x %zu MB)\n", nm, sgd_bytes * 5 / (ms / 1e3) / 1e9, n3 * 16 >> 20);
      }
    };
    float4* G = a[0]; float4* Wt = a[0] + n3; float4* D = a[0] + 2 * n3;
    runs("sgd LDG 148x512 U=4", [&](int) { sgd_ldg<4><<<sms, 512, 0, st[0]>>>(G, Wt, D, n3); });
    runs("sgd LDG 296x512 U=2", [&](int) { sgd_ldg<2><<<2 * sms, 512, 0, st[0]>>>(G, Wt, D, n3); });
    runs("sgd LDG 296x512 U=4", [&](int) { sgd_ldg<4><<<2 * sms, 512, 0, st[0]>>>(G, Wt, D, n3); });
    runs("sgd LDG 592x256 U=4", [&](int) { sgd_ldg<4><<<4 * sms, 256, 0, st[0]>>>(G, Wt, D, n3); });
    runs("sgd LDG ranges 148x512 U=4", [&](int) { sgd_ldg_ranges<4><<<sms, 512, 0, st[0]>>>(G, Wt, D, n3); });
    runs("sgd LDG ranges 296x512 U=2", [&](int) { sgd_ldg_ranges<2><<<2 * sms, 512, 0, st[0]>>>(G, Wt, D, n3); });
    CK(cudaFuncSetAttribute(sgd_tma<512, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 512 * 16 * 3 * 4));
    CK(cudaFuncSetAttribute(sgd_tma<256, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 16 * 3 * 8));
    CK(cudaFuncSetAttribute(sgd_tma<1024, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 * 16 * 3 * 4));
    runs("sgd TMA tile=8K NS=4 148x288", [&](int) { sgd_tma<512, 4><<<sms, 288, 512 * 16 * 3 * 4, st[0]>>>(G, Wt, D, n3); });
    runs("sgd TMA tile=4K NS=8 148x288", [&](int) { sgd_tma<256, 8><<<sms, 288, 256 * 16 * 3 * 8, st[0]>>>(G, Wt, D, n3); });
    runs("sgd TMA tile=16K NS=4 148x288", [&](int) { sgd_tma<1024, 4><<<sms, 288, 1024 * 16 * 3 * 4, st[0]>>>(G, Wt, D, n3); });
    runs("sgd TMA tile=8K NS=4 296x288", [&](int) { sgd_tma<512, 4><<<2 * sms, 288, 512 * 16 * 3 * 4, st[0]>>>(G, Wt, D, n3); });
  }
  run("cudaMemcpyPeerAsync pull", [&](int d) { int q = (d + 1) % n;
    CK(cudaMemcpyPeerAsync(b[d], d, a[q], q, bytes, st[d])); });
  {
    // TMA bulk copies: local, pull (src = peer), push (dst = peer)
    auto tma = [&](const char* what, int mode, auto kern, int ch, int ns, int cps) {
      int smem = ch * ns;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      snprintf(name, sizeof name, "TMA %s CH=%dK NS=%d ctas=%d", what, ch / 1024, ns, sms * cps);
      run(name, [&](int d) {
        int q = (d + 1) % n;
        const char* s = (const char*)(mode == 1 ? a[q] : a[d]);
        char* t = (char*)(mode == 2 ? b[q] : b[d]);
        kern<<<sms * cps, 32, smem, st[d]>>>(s, t, bytes);
      });
    };
    for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); }
    for (int mode = 0; mode < 3; ++mode) {
      const char* w = mode == 0 ? "local" : mode == 1 ? "pull" : "push";
      for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaFuncSetAttribute(tma_copy<16384, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8));
        CK(cudaFuncSetAttribute(tma_copy<32768, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 6));
        CK(cudaFuncSetAttribute(tma_copy<8192, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8));
        CK(cudaFuncSetAttribute(tma_copy<16384, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 4));
      }
      CK(cudaSetDevice(0));
      tma(w, mode, tma_copy<16384, 8>, 16384, 8, 1);
      tma(w, mode, tma_copy<32768, 6>, 32768, 6, 1);
      tma(w, mode, tma_copy<8192, 8>, 8192, 8, 2);
      tma(w, mode, tma_copy<16384, 4>, 16384, 4, 3);
    }
  }
  for (int push = 0; push < 2; ++push)
    for (int cps : {1, 2, 4}) {
      int grid = sms * cps;
      grid -= grid % (n - 1);
      size_t part = nvec / (n - 1);
      snprintf(name, sizeof name, "all-peer %s one kernel %dx512 U=4", push ? "push" : "pull", grid);
      run(name, [&](int d) {
        Peers pp{};
        for (int j = 0; j < n - 1; ++j) pp.p[j] = (push ? b : a)[(d + 1 + j) % n];
        if (push) allpeer_kernel<4, true><<<grid, 512, 0, st[d]>>>(pp, a[d], part, n - 1);
        else allpeer_kernel<4, false><<<grid, 512, 0, st[d]>>>(pp, b[d], part, n - 1);
      });
    }
  if (n > 2) {
    // all-to-all pull: GPU d reads 1/(n-1) of the buffer from every peer concurrently
    int grid = sms * 2;
    KFn f = fns[1][2];
    size_t part = nvec / (n - 1);
    run("pull all-peers 2x512 U=4 (1/(n-1) from each)", [&](int d) {
      for (int j = 1; j < n; ++j) { int q = (d + j) % n;
        f<<<grid / (n - 1), 512, 0, st[d]>>>(a[q] + (j - 1) * part, b[d] + (j - 1) * part, part); }
    });
  }
  printf("done\n");
  return 0;
}
