// Hot-path kernels of libtc for sm_100a (B200): the tensor allreduce of PAPER.md §6
// (reduce-scatter + allgather), fused with the SGD step (Eq. 1) or the elastic
// averaging update (Eqs. elastic1/elastic2).
//
// Design:
//  * One kernel per call.  Each rank runs B CTAs; CTA b of every rank owns the same sub-range b
//    of every owner chunk, so cross-GPU synchronisation is per-CTA-pair flag exchange (no grid
//    sync): the epoch is stored into the peer's flag word [barrier][my rank][b] with
//    st.release.sys and awaited on the local word with ld.acquire.sys (timeout -> sticky error).
//  * Inside a CTA, warps take 32*U-slot pieces of the sub-range round-robin and every lane
//    resolves its slot's tensor (cached binary search over the slot prefix), so a sub-range
//    holding many tiny tensors (ResNet-50's BN vectors) is spread over all warps.
//  * Two-shot, pull (A2-A4): ENTRY barrier -> reduce-scatter: each owned slot pulls the 16-B
//    vectors of all p ranks over NVLink, sums them in float64 in rank order 0..p-1, rounds once,
//    applies the epilogue, writes in place and into a parity-selected staging chunk -> MID
//    barrier -> allgather: pull every other owner's staged chunk (rotated start), epilogue.
//    No exit barrier: peers read only staging, which is rewritten two calls later, after the
//    next call's first barrier proved every peer finished this one.
//  * Two-shot, push: every rank first STORES its contribution to each owner's receive scratch
//    (stores beat loads over NVLink), signalling per owner; the owner reduces from local HBM in
//    the same canonical order, then the staged pull allgather as above.  No entry barrier.
//  * One-shot (A5, small groups): copy the group into a parity-selected staging buffer, ENTRY
//    barrier, every rank reduces all slots from all p staging buffers.
//  * Local (p = 1): the epilogue as a single HBM stream.
//  * Arithmetic: float64 accumulation in canonical rank order (R3/R4) and explicit _rn fp32
//    ops for the SGD/elastic epilogues (no FMA contraction, R5): GPU == CPU oracle bit for bit.
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

// Phase timestamp (diagnostics only; kp.prof == nullptr in production).
__device__ __forceinline__ void stamp(const KParams& kp, int i) {
  if (kp.prof != nullptr && threadIdx.x == 0)
    kp.prof[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + i] = globaltimer();
}

// ------------------------------------------------------------------ flags (A2)
__device__ __forceinline__ size_t flag_index(int bar, int src, int cta) {
  return ((size_t)bar * kMaxRanks + src) * kMaxCtas + cta;
}

// Thread 0: tell rank `to` that this CTA (rank r) passed point `bar`.  Caller has synced.
__device__ __forceinline__ void signal_one(const KParams& kp, int bar, int r, int to) {
  st_release_sys(kp.flags[to] + flag_index(bar, r, blockIdx.x), kp.epoch);
}

// Whole CTA: publish arrival at `bar` to every peer (if do_signal), then wait for every
// peer's arrival.  Returns false (CTA must stop) on timeout.
__device__ bool barrier_all(const KParams& kp, int r, int bar, bool do_signal) {
  __syncthreads();  // every thread's prior stores of this CTA precede the release below
  const int k = threadIdx.x;
  bool ok = true;
  if (k < kp.p && k != r) {
    if (do_signal) st_release_sys(kp.flags[k] + flag_index(bar, r, blockIdx.x), kp.epoch);
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
enum Phase { PH_RS = 0, PH_AG = 1 };

// Local operands of (op, phase): A = primary (x / g), B = w or center, C = dw.
template <int OP, int PH, int P> struct Needs {
  static constexpr bool loadA = (OP == OP_EASGD && PH == PH_AG);
  static constexpr bool loadB = (OP == OP_SGD) || (OP == OP_EASGD);
  static constexpr bool loadC = (OP == OP_SGD);
  // p = 1 SGD: the reduced gradient is the gradient itself -- not stored back.
  static constexpr bool storeA = !(OP == OP_SGD && PH == PH_RS && P == 1);
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

// One element.  in[k]: P source values (PH_RS) or the owner's value in[0] (PH_AG).
// la/lb/lc: local operands in, results out.
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
      const float dr = __fsub_rn(la, lb);  // this rank's (old) center replica
      la = __fsub_rn(la, __fmul_rn(kp.alpha, dr));
      lb = in[0];  // the owner's new center
    }
  }
}

// ------------------------------------------------------------------ slot addressing
// One lane's slot: flat slot s of tensor t, element offset e, cnt valid elements (1..4).
struct SlotRef {
  int s, t, cnt;
  int64_t e;
  bool vec;  // full 16-B slot and the tensor is 16-B aligned in every group of the call
};

struct TensorCache {
  int t, lo, hi;
  int64_t n;
  bool vec;
};

__device__ __forceinline__ void resolve(const KParams& kp, TensorCache& c, int s, SlotRef& ref) {
  if (s < c.lo || s >= c.hi) {
    // largest t with prefix[t] <= s (then prefix[t+1] > s: empty tensors are skipped)
    int a = (c.t >= 0 && s >= c.hi) ? c.t + 1 : 0, b = kp.T;
    while (b - a > 1) {
      const int m = (a + b) >> 1;
      if (__ldg(kp.prefix + m) <= s) a = m; else b = m;
    }
    c.t = a;
    c.lo = __ldg(kp.prefix + a);
    c.hi = __ldg(kp.prefix + a + 1);
    c.n = __ldg(kp.numel + a);
    c.vec = __ldg(kp.vec_ok + a) && (!kp.vec_ok_b || __ldg(kp.vec_ok_b + a)) &&
            (!kp.vec_ok_c || __ldg(kp.vec_ok_c + a));
  }
  ref.s = s;
  ref.t = c.t;
  ref.e = (int64_t)(s - c.lo) * 4;
  const int64_t rem = c.n - ref.e;
  ref.cnt = rem >= 4 ? 4 : (int)rem;
  ref.vec = c.vec && ref.cnt == 4;
}

// Tensor-structured operand: tensor ref.t of `rank` in pointer table `tab` ([p][T]).
__device__ __forceinline__ float4 ldT(const KParams& kp, float* const* tab, int rank,
                                      const SlotRef& ref) {
  const float* base = tab[(size_t)rank * kp.T + ref.t] + ref.e;
  if (ref.vec) return ld16(base);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  v.x = ld4(base);
  if (ref.cnt > 1) v.y = ld4(base + 1);
  if (ref.cnt > 2) v.z = ld4(base + 2);
  if (ref.cnt > 3) v.w = ld4(base + 3);
  return v;
}
__device__ __forceinline__ void stT(const KParams& kp, float* const* tab, int rank,
                                    const SlotRef& ref, float4 v) {
  float* base = tab[(size_t)rank * kp.T + ref.t] + ref.e;
  if (ref.vec) {
    st16(base, v);
    return;
  }
  st4(base, v.x);
  if (ref.cnt > 1) st4(base + 1, v.y);
  if (ref.cnt > 2) st4(base + 2, v.z);
  if (ref.cnt > 3) st4(base + 3, v.w);
}

// Staging / scratch regions of the per-rank arena (flat, slot-indexed relative to a chunk).
__device__ __forceinline__ float* arena_stage(const KParams& kp, int rank, int parity) {
  return kp.arena[rank] + (size_t)parity * kp.chunk_cap * 4;
}
__device__ __forceinline__ float* arena_scratch(const KParams& kp, int rank, int src) {
  return kp.arena[rank] + (size_t)(2 + src) * kp.chunk_cap * 4;
}

// Warps take 32*U-slot pieces of [lo, hi) round-robin; each lane handles U slots 32 apart.
// Body: struct with `State`, load(ref, st) (issue every load) and finish(ref, st).
template <int U, class Body>
__device__ __forceinline__ void slot_loop(const KParams& kp, int lo, int hi, Body& body) {
  const int lane_id = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  constexpr int CH = 32 * U;
  TensorCache tcache{-1, 0, 0, 0, false};
  for (int base = lo + warp * CH; base < hi; base += nw * CH) {
    SlotRef ref[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int s = base + lane_id + 32 * u;
      if (s < hi) resolve(kp, tcache, s, ref[u]); else ref[u].cnt = 0;
    }
    typename Body::State st[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ref[u].cnt) body.load(ref[u], st[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ref[u].cnt) body.finish(ref[u], st[u]);
  }
}

// ------------------------------------------------------------------ phase bodies
enum SrcKind {
  SRC_TENSORS = 0,   // every rank's primary tensor (pull reduce-scatter, local path)
  SRC_SCRATCH = 1,   // own primary tensor for k == r, else own receive scratch of rank k (push)
  SRC_ONESHOT = 2,   // every rank's one-shot staging buffer (flat over the whole group)
};

// Reduce P sources, apply the epilogue to this rank's operands; optionally also write the
// reduced primary value into this rank's staging chunk (for the staged allgather).
template <int OP, int P, int SRC, bool STAGE_OUT>
struct ReduceBody {
  using N = Needs<OP, PH_RS, P>;
  const KParams& kp;
  int r;
  int origin;         // first slot of the chunk (flat offsets of staging / scratch)
  float* stage_out;   // this rank's staging chunk (STAGE_OUT)
  struct State {
    float4 x[P];
    float4 b, c;
  };
  __device__ __forceinline__ void load(const SlotRef& ref, State& st) const {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      if constexpr (SRC == SRC_TENSORS) {
        st.x[k] = ldT(kp, kp.a, k, ref);
      } else if constexpr (SRC == SRC_SCRATCH) {
        st.x[k] = (k == r) ? ldT(kp, kp.a, r, ref)
                           : ld16(arena_scratch(kp, r, k) + (size_t)(ref.s - origin) * 4);
      } else {
        st.x[k] = ld16(kp.stage[k] + kp.stage_off + (size_t)ref.s * 4);
      }
    }
    if constexpr (N::loadB) st.b = ldT(kp, kp.b, r, ref);
    if constexpr (N::loadC) st.c = ldT(kp, kp.c, r, ref);
  }
  __device__ __forceinline__ void finish(const SlotRef& ref, State& st) const {
    float4 oa;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float in[P];
#pragma unroll
      for (int k = 0; k < P; ++k) in[k] = lane(st.x[k], i);
      float la = 0.f;
      float lb = N::loadB ? lane(st.b, i) : 0.f;
      float lc = N::loadC ? lane(st.c, i) : 0.f;
      elem<OP, PH_RS, P>(kp, r, in, la, lb, lc);
      lane(oa, i) = la;
      if constexpr (N::storeB) lane(st.b, i) = lb;
      if constexpr (N::storeC) lane(st.c, i) = lc;
    }
    if constexpr (N::storeA) stT(kp, kp.a, r, ref, oa);
    if constexpr (N::storeB) stT(kp, kp.b, r, ref, st.b);
    if constexpr (N::storeC) stT(kp, kp.c, r, ref, st.c);
    if constexpr (STAGE_OUT) {
      // EASGD gathers the owner's new center, the other ops the reduced primary value
      st16(stage_out + (size_t)(ref.s - origin) * 4, OP == OP_EASGD ? st.b : oa);
    }
  }
};

// Allgather: take owner q's staged value, apply the epilogue to this rank's operands.
template <int OP>
struct GatherBody {
  using N = Needs<OP, PH_AG, 2>;
  const KParams& kp;
  int r;
  int origin;
  const float* src;   // owner's staging chunk
  struct State {
    float4 x, a, b, c;
  };
  __device__ __forceinline__ void load(const SlotRef& ref, State& st) const {
    st.x = ld16(src + (size_t)(ref.s - origin) * 4);
    if constexpr (N::loadA) st.a = ldT(kp, kp.a, r, ref);
    if constexpr (N::loadB) st.b = ldT(kp, kp.b, r, ref);
    if constexpr (N::loadC) st.c = ldT(kp, kp.c, r, ref);
  }
  __device__ __forceinline__ void finish(const SlotRef& ref, State& st) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float in[1] = {lane(st.x, i)};
      float la = N::loadA ? lane(st.a, i) : 0.f;
      float lb = N::loadB ? lane(st.b, i) : 0.f;
      float lc = N::loadC ? lane(st.c, i) : 0.f;
      elem<OP, PH_AG, 2>(kp, r, in, la, lb, lc);
      lane(st.a, i) = la;
      if constexpr (N::storeB) lane(st.b, i) = lb;
      if constexpr (N::storeC) lane(st.c, i) = lc;
    }
    stT(kp, kp.a, r, ref, st.a);
    if constexpr (N::storeB) stT(kp, kp.b, r, ref, st.b);
    if constexpr (N::storeC) stT(kp, kp.c, r, ref, st.c);
  }
};

// Copy this rank's primary tensors into a flat destination (push to an owner's scratch, or
// the one-shot staging buffer).
struct CopyOutBody {
  const KParams& kp;
  int r;
  int origin;
  float* dst;
  struct State {
    float4 x;
  };
  __device__ __forceinline__ void load(const SlotRef& ref, State& st) const {
    st.x = ldT(kp, kp.a, r, ref);
  }
  __device__ __forceinline__ void finish(const SlotRef& ref, State& st) const {
    st16(dst + (size_t)(ref.s - origin) * 4, st.x);
  }
};

__device__ __forceinline__ void sub_range(int64_t lo, int64_t hi, int b, int B, int& out_lo,
                                          int& out_hi) {
  const int64_t len = hi - lo;
  out_lo = (int)(lo + len * b / B);
  out_hi = (int)(lo + len * (b + 1) / B);
}

__host__ __device__ constexpr int unroll_for(int nsrc) {
  return nsrc <= 2 ? 4 : (nsrc <= 4 ? 2 : 1);
}

// Staged allgather of every other owner's chunk (rotated start: owner r+1 first).
template <int OP, int P>
__device__ __forceinline__ void gather_all(const KParams& kp, int r, int b, int B, int par) {
  const int64_t M = kp.M;
#pragma unroll 1
  for (int j = 1; j < P; ++j) {
    const int q = (r + j) % P;
    int lo, hi;
    sub_range(M * q / P, M * (q + 1) / P, b, B, lo, hi);
    GatherBody<OP> body{kp, r, (int)(M * q / P), arena_stage(kp, q, par)};
    slot_loop<4>(kp, lo, hi, body);
  }
}

// ------------------------------------------------------------------ kernels
template <int OP, int P>
__global__ void __launch_bounds__(512) k_twoshot_pull(KParams kp) {
  const int r = kp.rank0 + (int)blockIdx.y;
  if (r == kp.absent_rank) return;
  const int b = blockIdx.x, B = gridDim.x, par = (int)(kp.epoch & 1u);
  const int64_t M = kp.M;
  stamp(kp, 0);
  if (!barrier_all(kp, r, BAR_ENTRY, true)) return;
  stamp(kp, 1);
  int lo, hi;
  const int origin = (int)(M * r / P);
  sub_range(M * r / P, M * (r + 1) / P, b, B, lo, hi);
  {
    ReduceBody<OP, P, SRC_TENSORS, true> body{kp, r, origin, arena_stage(kp, r, par)};
    slot_loop<unroll_for(P)>(kp, lo, hi, body);
  }
  stamp(kp, 2);
  if (!barrier_all(kp, r, BAR_MID, true)) return;
  stamp(kp, 3);
  gather_all<OP, P>(kp, r, b, B, par);
  stamp(kp, 4);
  stamp(kp, 5);
}

template <int OP, int P>
__global__ void __launch_bounds__(512) k_twoshot_push(KParams kp) {
  const int r = kp.rank0 + (int)blockIdx.y;
  if (r == kp.absent_rank) return;
  const int b = blockIdx.x, B = gridDim.x, par = (int)(kp.epoch & 1u);
  const int64_t M = kp.M;
  stamp(kp, 0);
  // push my contribution of sub-range b of every other chunk into its owner's scratch
#pragma unroll 1
  for (int j = 1; j < P; ++j) {
    const int q = (r + j) % P;
    int lo, hi;
    sub_range(M * q / P, M * (q + 1) / P, b, B, lo, hi);
    CopyOutBody body{kp, r, (int)(M * q / P), arena_scratch(kp, q, r)};
    slot_loop<4>(kp, lo, hi, body);
    __syncthreads();
    if (threadIdx.x == 0) signal_one(kp, BAR_ENTRY, r, q);
  }
  stamp(kp, 1);
  if (!barrier_all(kp, r, BAR_ENTRY, false)) return;  // every peer's push has landed
  int lo, hi;
  const int origin = (int)(M * r / P);
  sub_range(M * r / P, M * (r + 1) / P, b, B, lo, hi);
  {
    ReduceBody<OP, P, SRC_SCRATCH, true> body{kp, r, origin, arena_stage(kp, r, par)};
    slot_loop<unroll_for(P)>(kp, lo, hi, body);
  }
  stamp(kp, 2);
  if (!barrier_all(kp, r, BAR_MID, true)) return;
  stamp(kp, 3);
  gather_all<OP, P>(kp, r, b, B, par);
  stamp(kp, 4);
  stamp(kp, 5);
}

template <int OP, int P>
__global__ void __launch_bounds__(512) k_oneshot(KParams kp) {
  const int r = kp.rank0 + (int)blockIdx.y;
  if (r == kp.absent_rank) return;
  int lo, hi;
  sub_range(0, kp.M, blockIdx.x, gridDim.x, lo, hi);
  stamp(kp, 0);
  {
    CopyOutBody body{kp, r, 0, kp.stage[r] + kp.stage_off};
    slot_loop<4>(kp, lo, hi, body);
  }
  if (!barrier_all(kp, r, BAR_ENTRY, true)) return;
  stamp(kp, 1);
  ReduceBody<OP, P, SRC_ONESHOT, false> body{kp, r, 0, nullptr};
  slot_loop<unroll_for(P)>(kp, lo, hi, body);
  stamp(kp, 5);
}

template <int OP, int MINB, int U>
__global__ void __launch_bounds__(512, MINB) k_local(KParams kp) {
  const int r = kp.rank0 + (int)blockIdx.y;
  int lo, hi;
  sub_range(0, kp.M, blockIdx.x, gridDim.x, lo, hi);
  ReduceBody<OP, 1, SRC_TENSORS, false> body{kp, r, 0, nullptr};
  slot_loop<U>(kp, lo, hi, body);
}

template <int OP>
const void* kernel_ptr(int algo, int p, int variant) {
  if (algo == ALGO_LOCAL) {
    switch (variant) {
      case 1: return (const void*)k_local<OP, 2, 2>;
      case 2: return (const void*)k_local<OP, 2, 4>;
      case 3: return (const void*)k_local<OP, 1, 8>;
      case 4: return (const void*)k_local<OP, 3, 2>;
      default: return (const void*)k_local<OP, 1, 4>;
    }
  }
#define TC_CASE(PP)                                                        \
  case PP:                                                                 \
    return algo == ALGO_TWOSHOT ? (const void*)k_twoshot_pull<OP, PP>      \
         : algo == ALGO_TWOSHOT_PUSH ? (const void*)k_twoshot_push<OP, PP> \
                                     : (const void*)k_oneshot<OP, PP>;
  switch (p) {
    TC_CASE(2) TC_CASE(3) TC_CASE(4) TC_CASE(5) TC_CASE(6) TC_CASE(7) TC_CASE(8)
    default: return nullptr;
  }
#undef TC_CASE
}

const void* select_kernel(int op, int algo, int p, int variant) {
  switch (op) {
    case OP_ALLREDUCE: return kernel_ptr<OP_ALLREDUCE>(algo, p, variant);
    case OP_SGD: return kernel_ptr<OP_SGD>(algo, p, variant);
    case OP_EASGD: return kernel_ptr<OP_EASGD>(algo, p, variant);
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
