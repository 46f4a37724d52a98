// Hot-path kernels of libtc for sm_100a (B200): the tensor allreduce of PAPER.md §6
// (reduce-scatter + allgather), fused with the SGD step (Eq. 1) or the elastic
// averaging update (Eqs. elastic1/elastic2).
//
// Design:
//  * One kernel per call.  Each rank runs `B` CTAs; CTA b of every rank handles the same
//    sub-range b of every owner chunk, so the three cross-GPU barriers are per-CTA-pair flag
//    exchanges (no grid-wide sync): thread k of CTA b stores the epoch into peer k's flag word
//    [barrier][my rank][b] with st.release.sys and spins on its own word with ld.acquire.sys.
//  * Two-shot (A3+A4): ENTRY barrier -> reduce-scatter of the owned chunk (each slot pulls the
//    16-B vectors of all p ranks over NVLink, sums them in float64 in rank order 0..p-1, rounds
//    once, writes in place, and applies the epilogue) -> MID barrier -> allgather of the other
//    p-1 chunks from their owners (rotated start so every GPU serves one reader at a time),
//    each followed by the epilogue -> EXIT barrier (owners' chunks stay readable until every
//    peer has pulled them).
//  * One-shot (A5, small groups): copy the local group into a parity-selected staging buffer,
//    ENTRY barrier, every rank reduces all slots from all p staging buffers.  No exit barrier:
//    a staging half is rewritten two calls later, after the next call's ENTRY barrier proved
//    every peer finished this one.
//  * Local (p = 1): the epilogue as a single HBM stream.
//  * Arithmetic: float64 accumulation in canonical rank order (R3/R4), explicit _rn fp32 ops for
//    the SGD/elastic epilogues (no FMA contraction, R5), so GPU == CPU oracle bit for bit.
#include <cuda_runtime.h>
#include <cstdint>

#include "tc_internal.h"

namespace tc {
namespace {

// ------------------------------------------------------------------ memory primitives
__device__ __forceinline__ float4 ld16(const float* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st16(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float ld4(const float* p) {
  float v;
  asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st4(float* p, float v) {
  asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float& lane(float4& v, int i) { return (&v.x)[i]; }

// ------------------------------------------------------------------ barrier (A2)
__device__ __forceinline__ size_t flag_index(int bar, int src, int cta) {
  return ((size_t)bar * kMaxRanks + src) * kMaxCtas + cta;
}

// Per-CTA-pair barrier across the p ranks.  Returns false (CTA must stop) on timeout.
__device__ bool cta_barrier(const KParams& kp, int r, int bar) {
  __syncthreads();  // every thread's prior stores of this CTA precede the release below
  const int k = threadIdx.x;
  bool ok = true;
  if (k < kp.p && k != r) {
    st_release_sys(kp.flags[k] + flag_index(bar, r, blockIdx.x), kp.epoch);
    const uint32_t* mine = kp.flags[r] + flag_index(bar, k, blockIdx.x);
    if ((int32_t)(ld_acquire_sys(mine) - kp.epoch) < 0) {
      const unsigned long long t0 = globaltimer();
      while ((int32_t)(ld_acquire_sys(mine) - kp.epoch) < 0) {
        if (globaltimer() - t0 > kp.timeout_ns) {
          atomicCAS_system(kp.err, 0, (int)TC_ERR_TIMEOUT);
          ok = false;
          break;
        }
      }
    }
  }
  return __syncthreads_and(ok) != 0;
}

// ------------------------------------------------------------------ element arithmetic
// PH_RS: reduce from P sources (reduce-scatter / one-shot / local);  PH_AG: copy from owner.
enum Phase { PH_RS = 0, PH_AG = 1 };

// Which local operands a (op, phase) reads: A = primary (x/g), B = w or center, C = dw.
template <int OP, int PH> struct Needs {
  static constexpr bool loadA = (OP == OP_EASGD && PH == PH_AG);
  static constexpr bool loadB = (OP == OP_SGD) || (OP == OP_EASGD);
  static constexpr bool loadC = (OP == OP_SGD);
  static constexpr bool storeB = (OP == OP_SGD) || (OP == OP_EASGD);
  static constexpr bool storeC = (OP == OP_SGD);
};

// SGD epilogue (A6), fp32 mirror of the oracle: t = R(R(rs*G)+R(wd*w)); dw' = R(R(mu*dw)-R(lr*t));
// w' = R(w+dw').
__device__ __forceinline__ void sgd1(const KParams& kp, float G, float& w, float& dw) {
  const float t = __fadd_rn(__fmul_rn(kp.rescale, G), __fmul_rn(kp.wd, w));
  dw = __fsub_rn(__fmul_rn(kp.mu, dw), __fmul_rn(kp.lr, t));
  w = __fadd_rn(w, dw);
}

// One element.  in[k]: source values (P of them for PH_RS, in[0] = owner's value for PH_AG).
// la/lb/lc: local operands; outputs written back into la/lb/lc.
template <int OP, int PH, int P>
__device__ __forceinline__ void elem(const KParams& kp, int r, const float* in, float& la,
                                     float& lb, float& lc) {
  if constexpr (OP == OP_ALLREDUCE) {
    if constexpr (PH == PH_RS) {
      double acc = (double)in[0];
#pragma unroll
      for (int k = 1; k < P; ++k) acc = __dadd_rn(acc, (double)in[k]);
      la = __double2float_rn(__dmul_rn(acc, (double)kp.scale));
    } else {
      la = in[0];
    }
  } else if constexpr (OP == OP_SGD) {
    float G;
    if constexpr (PH == PH_RS) {
      double acc = (double)in[0];
#pragma unroll
      for (int k = 1; k < P; ++k) acc = __dadd_rn(acc, (double)in[k]);
      G = __double2float_rn(acc);
    } else {
      G = in[0];
    }
    la = G;  // the reduced gradient is written back (R15)
    sgd1(kp, G, lb, lc);
  } else {  // OP_EASGD: la = x_r, lb = center
    if constexpr (PH == PH_RS) {
      const float xc = lb;
      float s = 0.f, xr = in[0];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const float d = __fsub_rn(in[k], xc);
        s = (k == 0) ? d : __fadd_rn(s, d);
        if (k == r) xr = in[k];
      }
      const float dr = __fsub_rn(xr, xc);
      la = __fsub_rn(xr, __fmul_rn(kp.alpha, dr));
      lb = __fadd_rn(xc, __fmul_rn(kp.alpha, s));
    } else {
      const float dr = __fsub_rn(la, lb);  // uses this rank's (old) center replica
      la = __fsub_rn(la, __fmul_rn(kp.alpha, dr));
      lb = in[0];  // the owner's new center
    }
  }
}

// ------------------------------------------------------------------ segment processing
struct Seg {
  const float* src[kMaxRanks];  // P sources (element 0 of this tensor in each source)
  float* a;
  float* b;
  float* c;
};

// Local slots [s0, s1) of one tensor, full 16-B vectors, U slots per thread in flight.
template <int OP, int PH, int P, int U>
__device__ __forceinline__ void seg_vec(const KParams& kp, int r, const Seg& sg, int s0, int s1) {
  using N = Needs<OP, PH>;
  constexpr int NS = (PH == PH_RS) ? P : 1;
  const int nthr = blockDim.x;
  for (int s = s0 + (int)threadIdx.x; s < s1; s += nthr * U) {
    float4 in[U][NS];
    float4 va[U], vb[U], vc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int ss = s + u * nthr;
      if (ss < s1) {
        const size_t e = (size_t)ss * 4;
#pragma unroll
        for (int k = 0; k < NS; ++k) in[u][k] = ld16(sg.src[k] + e);
        if constexpr (N::loadA) va[u] = ld16(sg.a + e);
        if constexpr (N::loadB) vb[u] = ld16(sg.b + e);
        if constexpr (N::loadC) vc[u] = ld16(sg.c + e);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int ss = s + u * nthr;
      if (ss < s1) {
        const size_t e = (size_t)ss * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float x[NS];
#pragma unroll
          for (int k = 0; k < NS; ++k) x[k] = lane(in[u][k], i);
          float la = N::loadA ? lane(va[u], i) : 0.f;
          float lb = N::loadB ? lane(vb[u], i) : 0.f;
          float lc = N::loadC ? lane(vc[u], i) : 0.f;
          elem<OP, PH, P>(kp, r, x, la, lb, lc);
          lane(va[u], i) = la;
          if constexpr (N::storeB) lane(vb[u], i) = lb;
          if constexpr (N::storeC) lane(vc[u], i) = lc;
        }
        st16(sg.a + e, va[u]);
        if constexpr (N::storeB) st16(sg.b + e, vb[u]);
        if constexpr (N::storeC) st16(sg.c + e, vc[u]);
      }
    }
  }
}

// Elements [e0, e1) one at a time (unaligned tensors and partial last slots).
template <int OP, int PH, int P>
__device__ __forceinline__ void seg_scalar(const KParams& kp, int r, const Seg& sg, int64_t e0,
                                           int64_t e1) {
  using N = Needs<OP, PH>;
  constexpr int NS = (PH == PH_RS) ? P : 1;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    float x[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) x[k] = ld4(sg.src[k] + e);
    float la = N::loadA ? ld4(sg.a + e) : 0.f;
    float lb = N::loadB ? ld4(sg.b + e) : 0.f;
    float lc = N::loadC ? ld4(sg.c + e) : 0.f;
    elem<OP, PH, P>(kp, r, x, la, lb, lc);
    st4(sg.a + e, la);
    if constexpr (N::storeB) st4(sg.b + e, lb);
    if constexpr (N::storeC) st4(sg.c + e, lc);
  }
}

// Source selection for a segment.
enum SrcKind { SRC_TENSORS = 0, SRC_STAGE = 1, SRC_OWNER = 2 };

// Walk global slots [lo, hi) of the flat space, tensor by tensor (uniform control flow).
template <int OP, int PH, int P, int U, int SRC>
__device__ void walk(const KParams& kp, int r, int q, int lo, int hi) {
  if (lo >= hi) return;
  // first tensor t with prefix[t] <= lo < prefix[t+1]
  int a = 0, b = kp.T;  // invariant prefix[a] <= lo < prefix[b]
  while (b - a > 1) {
    const int m = (a + b) >> 1;
    if (__ldg(kp.prefix + m) <= lo) a = m; else b = m;
  }
  int t = a;
  const int T = kp.T;
  while (lo < hi) {
    int t_lo = __ldg(kp.prefix + t), t_hi = __ldg(kp.prefix + t + 1);
    while (t_hi <= lo) {  // skip empty tensors
      ++t;
      t_lo = t_hi;
      t_hi = __ldg(kp.prefix + t + 1);
    }
    const int seg_hi = hi < t_hi ? hi : t_hi;
    Seg sg;
    const size_t mine = (size_t)r * T + t;
    sg.a = kp.a[mine];
    sg.b = (Needs<OP, PH>::loadB || Needs<OP, PH>::storeB) ? kp.b[mine] : nullptr;
    sg.c = (Needs<OP, PH>::loadC || Needs<OP, PH>::storeC) ? kp.c[mine] : nullptr;
    if constexpr (SRC == SRC_TENSORS) {
      // sources: every rank's tensor t of the primary group (EASGD: x_k; others: x_k / g_k)
#pragma unroll
      for (int k = 0; k < P; ++k) sg.src[k] = kp.a[(size_t)k * T + t];
    } else if constexpr (SRC == SRC_STAGE) {
#pragma unroll
      for (int k = 0; k < P; ++k) sg.src[k] = kp.stage[k] + kp.stage_off + (size_t)t_lo * 4;
    } else {  // SRC_OWNER: allgather from owner q; EASGD gathers the center, else primary
      sg.src[0] = (OP == OP_EASGD) ? kp.b[(size_t)q * T + t] : kp.a[(size_t)q * T + t];
    }
    const int64_t n = __ldg(kp.numel + t);
    const int s0 = lo - t_lo, s1 = seg_hi - t_lo;  // local slots
    const int full = (int)(n >> 2);                // complete 16-B slots of tensor t
    const bool vec = __ldg(kp.vec_ok + t) && (!kp.vec_ok_b || __ldg(kp.vec_ok_b + t)) &&
                     (!kp.vec_ok_c || __ldg(kp.vec_ok_c + t));
    if (vec) {
      const int v1 = s1 < full ? s1 : full;
      if (s0 < v1) seg_vec<OP, PH, P, U>(kp, r, sg, s0, v1);
      if (s1 > full) seg_scalar<OP, PH, P>(kp, r, sg, (int64_t)full * 4, n);
    } else {
      const int64_t e1 = (int64_t)s1 * 4 < n ? (int64_t)s1 * 4 : n;
      seg_scalar<OP, PH, P>(kp, r, sg, (int64_t)s0 * 4, e1);
    }
    lo = seg_hi;
    ++t;
  }
}

// Copy local primary-group slots [lo, hi) into this rank's staging half (flat slot layout).
__device__ void stage_copy(const KParams& kp, int r, int lo, int hi) {
  if (lo >= hi) return;
  int a = 0, b = kp.T;
  while (b - a > 1) {
    const int m = (a + b) >> 1;
    if (__ldg(kp.prefix + m) <= lo) a = m; else b = m;
  }
  int t = a;
  float* dst = kp.stage[r] + kp.stage_off;
  while (lo < hi) {
    int t_lo = __ldg(kp.prefix + t), t_hi = __ldg(kp.prefix + t + 1);
    while (t_hi <= lo) {
      ++t;
      t_lo = t_hi;
      t_hi = __ldg(kp.prefix + t + 1);
    }
    const int seg_hi = hi < t_hi ? hi : t_hi;
    const float* src = kp.a[(size_t)r * kp.T + t];
    float* d = dst + (size_t)t_lo * 4;
    const int64_t n = __ldg(kp.numel + t);
    const int s0 = lo - t_lo, s1 = seg_hi - t_lo, full = (int)(n >> 2);
    if (__ldg(kp.vec_ok + t)) {
      const int v1 = s1 < full ? s1 : full;
      for (int s = s0 + (int)threadIdx.x; s < v1; s += blockDim.x)
        st16(d + (size_t)s * 4, ld16(src + (size_t)s * 4));
      if (s1 > full)
        for (int64_t e = (int64_t)full * 4 + threadIdx.x; e < n; e += blockDim.x)
          st4(d + e, ld4(src + e));
    } else {
      const int64_t e1 = (int64_t)s1 * 4 < n ? (int64_t)s1 * 4 : n;
      for (int64_t e = (int64_t)s0 * 4 + threadIdx.x; e < e1; e += blockDim.x)
        st4(d + e, ld4(src + e));
    }
    lo = seg_hi;
    ++t;
  }
}

__device__ __forceinline__ void sub_range(int64_t lo, int64_t hi, int b, int B, int& out_lo,
                                          int& out_hi) {
  const int64_t len = hi - lo;
  out_lo = (int)(lo + len * b / B);
  out_hi = (int)(lo + len * (b + 1) / B);
}

__host__ __device__ constexpr int kUnroll(int P) { return P <= 2 ? 4 : (P <= 4 ? 2 : 1); }

// ------------------------------------------------------------------ kernels
template <int OP, int P>
__global__ void __launch_bounds__(512) k_twoshot(KParams kp) {
  const int r = kp.rank0 + (int)blockIdx.y;
  if (r == kp.absent_rank) return;
  const int b = blockIdx.x, B = gridDim.x;
  const int64_t M = kp.M;
  if (!cta_barrier(kp, r, BAR_ENTRY)) return;
  int lo, hi;
  sub_range(M * r / P, M * (r + 1) / P, b, B, lo, hi);
  walk<OP, PH_RS, P, kUnroll(P), SRC_TENSORS>(kp, r, r, lo, hi);
  if (!cta_barrier(kp, r, BAR_MID)) return;
#pragma unroll 1
  for (int j = 1; j < P; ++j) {
    const int q = (r + j) % P;
    sub_range(M * q / P, M * (q + 1) / P, b, B, lo, hi);
    walk<OP, PH_AG, P, 4, SRC_OWNER>(kp, r, q, lo, hi);
  }
  cta_barrier(kp, r, BAR_EXIT);
}

template <int OP, int P>
__global__ void __launch_bounds__(512) k_oneshot(KParams kp) {
  const int r = kp.rank0 + (int)blockIdx.y;
  if (r == kp.absent_rank) return;
  const int b = blockIdx.x, B = gridDim.x;
  int lo, hi;
  sub_range(0, kp.M, b, B, lo, hi);
  stage_copy(kp, r, lo, hi);
  if (!cta_barrier(kp, r, BAR_ENTRY)) return;
  walk<OP, PH_RS, P, kUnroll(P), SRC_STAGE>(kp, r, r, lo, hi);
}

template <int OP>
__global__ void __launch_bounds__(512) k_local(KParams kp) {
  const int r = kp.rank0 + (int)blockIdx.y;
  int lo, hi;
  sub_range(0, kp.M, blockIdx.x, gridDim.x, lo, hi);
  walk<OP, PH_RS, 1, 4, SRC_TENSORS>(kp, r, r, lo, hi);
}

template <int OP>
const void* kernel_ptr(int algo, int p) {
  if (algo == ALGO_LOCAL) return (const void*)k_local<OP>;
#define TC_CASE(PP)                                                       \
  case PP:                                                                \
    return algo == ALGO_TWOSHOT ? (const void*)k_twoshot<OP, PP>          \
                                : (const void*)k_oneshot<OP, PP>;
  switch (p) {
    TC_CASE(2) TC_CASE(3) TC_CASE(4) TC_CASE(5) TC_CASE(6) TC_CASE(7) TC_CASE(8)
    default: return nullptr;
  }
#undef TC_CASE
}

const void* select_kernel(int op, int algo, int p) {
  switch (op) {
    case OP_ALLREDUCE: return kernel_ptr<OP_ALLREDUCE>(algo, p);
    case OP_SGD: return kernel_ptr<OP_SGD>(algo, p);
    case OP_EASGD: return kernel_ptr<OP_EASGD>(algo, p);
  }
  return nullptr;
}

}  // namespace

int max_ctas_per_sm(int op, int algo, int p, int threads) {
  const void* k = select_kernel(op, algo, p);
  if (!k) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, threads, 0) != cudaSuccess) return 0;
  return n;
}

cudaError_t launch_hot(int op, int algo, const KParams& kp, int ctas, int threads, int nlocal,
                       bool cooperative, cudaStream_t stream) {
  const void* k = select_kernel(op, algo, kp.p);
  if (!k) return cudaErrorInvalidValue;
  KParams arg = kp;
  void* args[] = {&arg};
  dim3 grid(ctas, nlocal), block(threads);
  if (cooperative) return cudaLaunchCooperativeKernel(k, grid, block, args, 0, stream);
  return cudaLaunchKernel(k, grid, block, args, 0, stream);
}

}  // namespace tc
