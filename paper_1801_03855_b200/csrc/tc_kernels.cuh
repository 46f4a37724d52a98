#pragma once
// Hot-path kernels of libtc for sm_100a (B200): the tensor allreduce of PAPER.md §6
// (reduce-scatter + allgather), fused with the SGD step (Eq. 1) or the elastic
// averaging update (Eqs. elastic1/elastic2).
//
// Design:
//  * One kernel per call.  Each rank runs B CTAs; CTA b of every rank owns the same pieces
//    of every owner chunk, so cross-GPU synchronisation is per-CTA-pair flag exchange (no grid
//    sync): the epoch is stored into the peer's flag word [barrier][my rank][b] with
//    st.release.sys and awaited on the local word with ld.acquire.sys (timeout -> sticky error).
//  * Every range is cut into 128-slot pieces dealt round-robin to CTAs, then warps: the GPU
//    streams one contiguous window at a time (DRAM locality) and ranges holding many tiny
//    tensors (ResNet-50's BN vectors) are spread over all warps.  Each lane resolves its slot's
//    tensor from a per-128-slot-block tensor table and caches the tensor's pointers.
//  * Two-shot, pull (A2-A4): ENTRY barrier -> reduce-scatter: each owned slot pulls the 16-B
//    vectors of all p ranks over NVLink, sums them in float64 in rank order 0..p-1, rounds once,
//    applies the epilogue, writes in place and into a parity-selected staging chunk -> MID
//    barrier -> allgather: pull every other owner's staged chunk (rotated start), epilogue.
//    No exit barrier: peers read only staging, which is rewritten two calls later, after the
//    next call's first barrier proved every peer finished this one.
//  * Two-shot, TMA (the default for large groups): the same phases with the data moved by
//    cp.async.bulk into a shared-memory stage ring (producer warp + consumer warps).
//  * One-shot (A5, small groups): copy the group into a parity-selected staging buffer, ENTRY
//    barrier, every rank reduces all slots from all p staging buffers.  Low-latency (LL): every
//    element to every peer as an 8-B {value, epoch} word, no barrier.
//  * NVLS: the switch reduces and multicasts the owner chunk (tolerance contract), the SGD
//    epilogue consuming published rounds; the switch broadcast.
//  * Async-server EASGD: the owner applies the clients' arrivals in order, storing every
//    client's new chunk into its tensor.
//  * Local (p = 1): the epilogue as a single HBM stream (TMA).
//  * Arithmetic: float64 accumulation in canonical rank order (R3/R4) and explicit _rn fp32
//    ops for the SGD/elastic epilogues (no FMA contraction, R5): GPU == CPU oracle bit for bit.
#include <cuda_runtime.h>
#include <cstdint>

#include "tc_internal.h"

namespace tc {
namespace {

// ------------------------------------------------------------------ memory primitives
// Load flavour (measured, bench.py ResNet-50, TC_LD_MODE builds): .cg (L2 only) pulls peer
// memory 4-7% faster than .L1::no_allocate (p = 2 step 223 vs 239 us, p = 4 301 vs 314 us;
// tools/p2p_probe: 664 vs 637 GB/s) and is neutral on the local HBM stream.
#ifndef TC_LD_MODE
#define TC_LD_MODE 1
#endif
#if TC_LD_MODE == 1
#define TC_LD_Q "ld.global.cg"
#elif TC_LD_MODE == 2
#define TC_LD_Q "ld.global"
#else
#define TC_LD_Q "ld.global.L1::no_allocate"
#endif
__device__ __forceinline__ float4 ld16(const float* p) {
  float4 v;
  asm volatile(TC_LD_Q ".v4.f32 {%0,%1,%2,%3}, [%4];"
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
  asm volatile(TC_LD_Q ".f32 %0, [%1];" : "=f"(v) : "l"(p));
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
__device__ __forceinline__ float lane_of(const float4& v, int i) { return (&v.x)[i]; }

// Phase timestamp (diagnostics only; kp.prof == nullptr in production).
__device__ __forceinline__ void stamp(const KParams& kp, int i, int tid = 0) {
  if (kp.prof != nullptr && (int)threadIdx.x == tid)
    kp.prof[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + i] = globaltimer();
}

// ------------------------------------------------------------------ call epoch (device side)
// Every collective call on a comm gets the next epoch: the kernel reads its rank's counter at
// start and the last CTA to finish advances it, so no host state enters the kernel arguments and
// calls can be captured in a CUDA graph and replayed.  Flags compare against the epoch.
__shared__ uint32_t s_epoch;

__device__ __forceinline__ uint32_t ep() { return s_epoch; }
// one-shot staging half used by this call (floats)
__device__ __forceinline__ size_t stage_off() {
  return (size_t)(s_epoch & 1u) * (kStageCapacity / sizeof(float));
}

__device__ __forceinline__ void call_begin(const KParams& kp, int r) {
  if (threadIdx.x == 0) s_epoch = *(volatile uint32_t*)&kp.state[r].epoch + 1u;
  __syncthreads();
}

__device__ __forceinline__ void call_end(const KParams& kp, int r) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    DevState* st = kp.state + r;
    if (atomicAdd(&st->done, 1u) == gridDim.x - 1) {
      st->done = 0;
      __threadfence();
      *(volatile uint32_t*)&st->epoch = s_epoch;
    }
  }
}

// ------------------------------------------------------------------ flags (A2)
__device__ __forceinline__ size_t flag_index(int bar, int src, int cta) {
  return ((size_t)bar * kMaxRanks + src) * kMaxCtas + cta;
}

// Thread 0: tell rank `to` that this CTA (rank r) passed point `bar`.  Caller has synced.
__device__ __forceinline__ void signal_one(const KParams& kp, int bar, int r, int to) {
  st_release_sys(kp.flags[to] + flag_index(bar, r, blockIdx.x), ep());
}

// Whole CTA: publish arrival at `bar` to every peer (if do_signal), then wait for every
// peer's arrival.  Returns false (CTA must stop) on timeout.
__device__ bool barrier_all(const KParams& kp, int r, int bar, bool do_signal) {
  __syncthreads();  // every thread's prior stores of this CTA precede the release below
  const int k = threadIdx.x;
  bool ok = true;
  if (k < kp.p && k != r) {
    if (do_signal) st_release_sys(kp.flags[k] + flag_index(bar, r, blockIdx.x), ep());
    const uint32_t* mine = kp.flags[r] + flag_index(bar, k, blockIdx.x);
    if ((int32_t)(ld_acquire_sys(mine) - ep()) < 0) {
      const unsigned long long t0 = globaltimer();
      while ((int32_t)(ld_acquire_sys(mine) - ep()) < 0) {
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

// Whole CTA: publish arrival at `bar` to every peer without waiting.
__device__ __forceinline__ void signal_all(const KParams& kp, int r, int bar) {
  __syncthreads();
  const int k = threadIdx.x;
  if (k < kp.p && k != r) st_release_sys(kp.flags[k] + flag_index(bar, r, blockIdx.x), ep());
}

// ------------------------------------------------------------------ element arithmetic
enum Phase { PH_RS = 0, PH_AG = 1 };

// Local operands of (op, phase): A = primary (x / g), B = w or center, C = dw.
template <int OP, int PH, int P> struct Needs {
  static constexpr bool EL = (OP == OP_EASGD) || (OP == OP_ESGD);  // elastic: a = x, b = center
  // async EASGD: the owner updates every client's x (stored straight into the client's tensor)
  // and the center in the reduce-scatter; the allgather only brings the center
  static constexpr bool AS = OP == OP_EASYNC;
  static constexpr bool loadA = EL && PH == PH_AG;
  static constexpr bool loadB = (OP == OP_SGD) || EL || (AS && PH == PH_RS);
  static constexpr bool loadC = (OP == OP_SGD) || (OP == OP_ESGD);
  static constexpr bool loadD = (OP == OP_ESGD);  // the rank's own (unreduced) gradient
  // p = 1 SGD: the reduced gradient is the gradient itself -- not stored back.
  static constexpr bool storeA = !(OP == OP_SGD && PH == PH_RS && P == 1) && !AS;
  static constexpr bool storeB = (OP == OP_SGD) || EL || AS;
  static constexpr bool stageB = EL || AS;  // the staged (gathered) value is the new center
  static constexpr bool storeC = (OP == OP_SGD) || (OP == OP_ESGD);
};

// p = 1 TMA stream: operands per stage from the kernels' needs (must match local_ops()).
template <int OP>
__host__ __device__ constexpr int local_na() {
  using N = Needs<OP, PH_RS, 1>;
  return 1 + (N::loadB ? 1 : 0) + (N::loadC ? 1 : 0) + (N::loadD ? 1 : 0);
}

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
  if constexpr (OP == OP_BCAST) {
    la = in[0];  // the root's value (reduce-scatter: the root's copy; allgather: the owner's)
  } else if constexpr (OP == OP_ALLREDUCE) {
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
  } else if constexpr (OP == OP_EASYNC) {
    if constexpr (PH == PH_AG) lb = in[0];  // the owner's final center (RS: easync1)
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

// NEXT row f2, asynchronous server: the owner of a chunk is its server shard and applies the
// clients' arrivals in kp.order (oracle.easgd_async, reading R20): per arrival i, with the
// center as the earlier arrivals left it, d = R(x_i - xc); xc = R(xc + R(a d)) (Eq. elastic1);
// x_i' = R(x_i - R(a d)) (Eq. elastic2).  in[k]: client k's x; out[k]: its new x.
template <int P>
__device__ __forceinline__ void easync1(const KParams& kp, const float* in, float* out,
                                        float& xc) {
#pragma unroll
  for (int k = 0; k < P; ++k) out[k] = in[k];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const int i = kp.order[j];
    float xi = in[0];
#pragma unroll
    for (int k = 1; k < P; ++k)
      if (k == i) xi = in[k];
    const float ad = __fmul_rn(kp.alpha, __fsub_rn(xi, xc));
    xc = __fadd_rn(xc, ad);
    const float xo = __fsub_rn(xi, ad);
#pragma unroll
    for (int k = 0; k < P; ++k)
      if (k == i) out[k] = xo;
  }
}

// NEXT row f2: the elastic update (as OP_EASGD) followed in the same pass by the SGD-momentum
// update of the elastically moved parameters with this rank's own gradient ld (one GPU per
// client; Fig. code-snippet-4 order: Elastic2 then SGD.Update).  fp32 mirror of
// oracle.esgd_step: xe = R(x - R(a d)), then sgd1 on (G = ld, w = xe).  Other ops: elem().
template <int OP, int PH, int P>
__device__ __forceinline__ void elem4(const KParams& kp, int r, const float* in, float& la,
                                      float& lb, float& lc, float ld) {
  if constexpr (OP == OP_ESGD) {
    float xe;
    if constexpr (PH == PH_RS) {
      const float xc = lb;
      float s = 0.f, xr = in[0];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const float d = __fsub_rn(in[k], xc);
        s = (k == 0) ? d : __fadd_rn(s, d);
        if (k == r) xr = in[k];
      }
      xe = __fsub_rn(xr, __fmul_rn(kp.alpha, __fsub_rn(xr, xc)));
      lb = __fadd_rn(xc, __fmul_rn(kp.alpha, s));
    } else {
      xe = __fsub_rn(la, __fmul_rn(kp.alpha, __fsub_rn(la, lb)));
      lb = in[0];  // the owner's new center
    }
    sgd1(kp, ld, xe, lc);
    la = xe;
  } else {
    elem<OP, PH, P>(kp, r, in, la, lb, lc);
  }
}

// ------------------------------------------------------------------ slot addressing
// One lane's slot: flat slot s, element offset e inside its tensor, cnt valid elements (1..4).
struct SlotRef {
  int s, cnt;      // flat slot; number of valid elements (0 = inactive lane)
  int lo_i, hi_i;  // valid element lanes [lo_i, hi_i) of the slot
  int64_t e;       // element index of lane 0 inside its tensor (negative for a shifted head)
  bool vec;        // full 16-B slot, 16-B aligned in every group of the call
};

// Per-lane cache of the current tensor and the NP tensor pointers the phase body needs, so the
// steady state issues no pointer-table loads (refreshed only when a lane crosses a tensor).
template <int NP>
struct TensorCache {
  int t, lo, hi, shift;
  int64_t n;
  bool vec;
  float* ptr[NP];
};

// A tensor whose pointers sit m elements past a 16-B boundary on every rank (views of a flat
// bucket with odd sizes) is laid out with its slot grid shifted by m: slot 0 holds elements
// [0, 4-m), later slots are 16-B aligned, so it keeps the vector path.
template <class Body>
__device__ __forceinline__ void resolve(const KParams& kp, const Body& body,
                                        TensorCache<Body::NP>& c, int s, SlotRef& ref) {
  if (s < c.lo || s >= c.hi) {
    // the slot's tensor lies between the tensors holding the first slots of its 128-slot block
    // and of the next block: binary search there (largest t with prefix[t] <= s)
    const int blk = s >> kPieceShift;
    int t = __ldg(kp.block_t + blk);
    if (__ldg(kp.prefix + t + 1) <= s) {
      int b = __ldg(kp.block_t + blk + 1) + 1;  // prefix[b] > s
      while (b - t > 1) {
        const int m = (t + b) >> 1;
        if (__ldg(kp.prefix + m) <= s) t = m; else b = m;
      }
    }
    c.t = t;
    c.lo = __ldg(kp.prefix + t);
    c.hi = __ldg(kp.prefix + t + 1);
    c.n = __ldg(kp.numel + t);
    c.shift = __ldg(kp.shift + t);
    c.vec = __ldg(kp.vec_ok + t) &&
            (!kp.vec_ok_b || (__ldg(kp.vec_ok_b + t) && __ldg(kp.shift_b + t) == c.shift)) &&
            (!kp.vec_ok_c || (__ldg(kp.vec_ok_c + t) && __ldg(kp.shift_c + t) == c.shift));
    body.bind(t, c.ptr);
  }
  ref.s = s;
  ref.e = (int64_t)(s - c.lo) * 4 - c.shift;
  ref.lo_i = ref.e < 0 ? (int)(-ref.e) : 0;
  const int64_t rem = c.n - ref.e;
  ref.hi_i = rem >= 4 ? 4 : (int)rem;
  ref.cnt = ref.hi_i - ref.lo_i;
  ref.vec = c.vec && ref.cnt == 4;
}

// Tensor-structured operand at element ref.e of a tensor base pointer.
template <bool VEC>
__device__ __forceinline__ float4 ldv(const float* base, const SlotRef& ref) {
  base += ref.e;
  if constexpr (VEC) {
    return ld16(base);
  } else {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i >= ref.lo_i && i < ref.hi_i) lane(v, i) = ld4(base + i);
    return v;
  }
}
template <bool VEC>
__device__ __forceinline__ void stv(float* base, const SlotRef& ref, float4 v) {
  base += ref.e;
  if constexpr (VEC) {
    st16(base, v);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i >= ref.lo_i && i < ref.hi_i) st4(base + i, lane(v, i));
  }
}

// Staging regions of the per-rank arena (flat, slot-indexed relative to a chunk).
__device__ __forceinline__ float* arena_stage(const KParams& kp, int rank, int parity) {
  return kp.arena[rank] + (size_t)parity * kp.chunk_cap * 4;
}

// [lo, hi) is cut into pieces of kPiece slots dealt round-robin to the CTAs of the grid (then
// to the warps of a CTA), so at any moment the whole GPU streams one contiguous window of memory
// (DRAM page locality: +40% over per-CTA contiguous ranges, tools/p2p_probe.cu).  The piece ->
// CTA map depends only on (lo, hi, gridDim), so CTA b of every rank touches the same pieces of a
// chunk -- the pairing the per-CTA flags rely on.  A lane handles U slots 32 apart per step.
// Body: NP cached pointers filled by bind(t, ptr); load<VEC>(ref, ptr, st) issues every load
// of a slot; finish<VEC>(ref, st) computes and stores.  All U slots' loads precede the first
// finish.
template <int U, class Body>
__device__ __forceinline__ void slot_loop(const KParams& kp, int lo, int hi, const Body& body) {
  static_assert(kPiece % (32 * U) == 0, "piece must be a multiple of a warp step");
  const int lane_id = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int npieces = (hi - lo + kPiece - 1) / kPiece;
  TensorCache<Body::NP> tc;
  tc.t = -1;
  tc.lo = tc.hi = 0;
  for (int c = blockIdx.x + gridDim.x * warp; c < npieces; c += gridDim.x * nw) {
    const int pbase = lo + c * kPiece;
    const int pend = min(hi, pbase + kPiece);
#pragma unroll 1
    for (int step = pbase; step < pend; step += 32 * U) {
      SlotRef ref[U];
      typename Body::State st[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = step + lane_id + 32 * u;
        if (s < pend) {
          resolve(kp, body, tc, s, ref[u]);
          if (ref[u].vec) body.template load<true>(ref[u], tc.ptr, st[u]);
          else body.template load<false>(ref[u], tc.ptr, st[u]);
        } else {
          ref[u].cnt = 0;
          ref[u].vec = false;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (ref[u].vec) body.template finish<true>(ref[u], st[u]);
        else if (ref[u].cnt) body.template finish<false>(ref[u], st[u]);
      }
    }
  }
}

// Small groups: one slot per thread, threads of the grid in order (consecutive threads,
// consecutive slots), so every slot's tensor lookup runs in parallel instead of a warp walking
// a piece of many tiny tensors serially.
template <class Body>
__device__ __forceinline__ void slot_loop_flat(const KParams& kp, int lo, int hi,
                                               const Body& body) {
  TensorCache<Body::NP> tc;
  tc.t = -1;
  tc.lo = tc.hi = 0;
  const int stride = gridDim.x * blockDim.x;
  for (int s = lo + blockIdx.x * blockDim.x + threadIdx.x; s < hi; s += stride) {
    SlotRef ref;
    typename Body::State st;
    resolve(kp, body, tc, s, ref);
    if (ref.vec) {
      body.template load<true>(ref, tc.ptr, st);
      body.template finish<true>(ref, st);
    } else {
      body.template load<false>(ref, tc.ptr, st);
      body.template finish<false>(ref, st);
    }
  }
}

// ------------------------------------------------------------------ phase bodies
enum SrcKind {
  SRC_TENSORS = 0,   // every rank's primary tensor (pull reduce-scatter, local path)
  SRC_ONESHOT = 2,   // every rank's one-shot staging buffer (flat over the whole group)
};

// Reduce P sources, apply the epilogue to this rank's operands; optionally also write the
// reduced primary value into this rank's staging chunk (for the staged allgather).
// Cached pointers: [0..2] = this rank's a, b, c tensors, then (SRC_TENSORS) P source tensors.
template <int OP, int P, int SRC, bool STAGE_OUT>
struct ReduceBody {
  using N = Needs<OP, PH_RS, P>;
  static constexpr int NP = 3 + (SRC == SRC_TENSORS ? P : 0);
  const KParams& kp;
  int r;
  int origin;         // first slot of the chunk (flat offset of staging)
  float* stage_out;   // this rank's staging chunk (STAGE_OUT)
  struct State {
    float4 x[P];
    float4 b, c;
    float *pa, *pb, *pc;
  };
  __device__ __forceinline__ void bind(int t, float** ptr) const {
    const size_t mine = (size_t)r * kp.T + t;
    ptr[0] = kp.a[mine];
    ptr[1] = (N::loadB || N::storeB) ? kp.b[mine] : nullptr;
    ptr[2] = (N::loadC || N::storeC) ? kp.c[mine] : nullptr;
    if constexpr (SRC == SRC_TENSORS) {
      // P == 1 (local paths): the single source is this rank's own tensor
#pragma unroll
      for (int k = 0; k < P; ++k) ptr[3 + k] = kp.a[(size_t)(P == 1 ? r : k) * kp.T + t];
    }
  }
  template <bool VEC>
  __device__ __forceinline__ void load(const SlotRef& ref, float* const* ptr, State& st) const {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      if constexpr (SRC == SRC_TENSORS) {
        st.x[k] = ldv<VEC>(ptr[3 + k], ref);
      } else {
        st.x[k] = ld16(kp.stage[k] + stage_off() + (size_t)ref.s * 4);
      }
    }
    if constexpr (N::loadB) st.b = ldv<VEC>(ptr[1], ref);
    if constexpr (N::loadC) st.c = ldv<VEC>(ptr[2], ref);
    st.pa = ptr[0];
    st.pb = ptr[1];
    st.pc = ptr[2];
  }
  template <bool VEC>
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
    if constexpr (N::storeA) stv<VEC>(st.pa, ref, oa);
    if constexpr (N::storeB) stv<VEC>(st.pb, ref, st.b);
    if constexpr (N::storeC) stv<VEC>(st.pc, ref, st.c);
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
  static constexpr int NP = 3;
  const KParams& kp;
  int r;
  int origin;
  const float* src;   // owner's staging chunk
  struct State {
    float4 x, a, b, c;
    float *pa, *pb, *pc;
  };
  __device__ __forceinline__ void bind(int t, float** ptr) const {
    const size_t mine = (size_t)r * kp.T + t;
    ptr[0] = kp.a[mine];
    ptr[1] = (N::loadB || N::storeB) ? kp.b[mine] : nullptr;
    ptr[2] = (N::loadC || N::storeC) ? kp.c[mine] : nullptr;
  }
  template <bool VEC>
  __device__ __forceinline__ void load(const SlotRef& ref, float* const* ptr, State& st) const {
    st.x = ld16(src + (size_t)(ref.s - origin) * 4);
    if constexpr (N::loadA) st.a = ldv<VEC>(ptr[0], ref);
    if constexpr (N::loadB) st.b = ldv<VEC>(ptr[1], ref);
    if constexpr (N::loadC) st.c = ldv<VEC>(ptr[2], ref);
    st.pa = ptr[0];
    st.pb = ptr[1];
    st.pc = ptr[2];
  }
  template <bool VEC>
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
    stv<VEC>(st.pa, ref, st.a);
    if constexpr (N::storeB) stv<VEC>(st.pb, ref, st.b);
    if constexpr (N::storeC) stv<VEC>(st.pc, ref, st.c);
  }
};

// Copy this rank's primary tensors into a flat destination (the one-shot staging buffer).
struct CopyOutBody {
  static constexpr int NP = 1;
  const KParams& kp;
  int r;
  int origin;
  float* dst;
  struct State {
    float4 x;
  };
  __device__ __forceinline__ void bind(int t, float** ptr) const {
    ptr[0] = kp.a[(size_t)r * kp.T + t];
  }
  template <bool VEC>
  __device__ __forceinline__ void load(const SlotRef& ref, float* const* ptr, State& st) const {
    st.x = ldv<VEC>(ptr[0], ref);
  }
  template <bool VEC>
  __device__ __forceinline__ void finish(const SlotRef& ref, State& st) const {
    st16(dst + (size_t)(ref.s - origin) * 4, st.x);
  }
};

// Slots per lane per step: enough independent 16-B loads in flight within the register budget
// of MINB resident 512-thread CTAs per SM.
__host__ __device__ constexpr int unroll_for(int nsrc, int minb) {
  return minb >= 2 ? (nsrc <= 2 ? 2 : 1) : (nsrc <= 2 ? 4 : (nsrc <= 4 ? 2 : 1));
}

// Whole CTA: wait until rank q's CTA has passed `bar`.  Returns false on timeout.
__device__ bool wait_one(const KParams& kp, int r, int q, int bar) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    int ok = 1;
    const uint32_t* mine = kp.flags[r] + flag_index(bar, q, blockIdx.x);
    if ((int32_t)(ld_acquire_sys(mine) - ep()) < 0) {
      const unsigned long long t0 = globaltimer();
      while ((int32_t)(ld_acquire_sys(mine) - ep()) < 0) {
        if (globaltimer() - t0 > kp.timeout_ns) {
          atomicCAS_system(kp.err, 0, (int)TC_ERR_TIMEOUT);
          ok = 0;
          break;
        }
      }
    }
    s_ok = ok;
  }
  __syncthreads();
  const int ok = s_ok;
  __syncthreads();
  return ok != 0;
}

// Staged allgather: once every peer's CTA has staged its chunk (one barrier, so all CTAs start
// together), pull the other owners' chunks r+1, r+2, ... in turn.  At each step the ranks read
// from a permutation of the owners, the NVLink pattern B200 serves fastest.  Measured at p = 4
// (ResNet-50): barrier + rank rotation 117 us; per-owner waits (CTAs drift apart and the steps
// mix) 131-156 us; owners mixed per CTA 134-154 us; "whichever owner is ready first" 155-182 us.
template <int OP, int P, int MINB>
__device__ __forceinline__ bool gather_all(const KParams& kp, int r, int par) {
  const int64_t M = kp.M;
  if (!barrier_all(kp, r, BAR_MID, true)) return false;
#pragma unroll 1
  for (int j = 0; j < P - 1; ++j) {
    const int q = (r + 1 + j) % P;
    const int lo = (int)(M * q / P), hi = (int)(M * (q + 1) / P);
    GatherBody<OP> body{kp, r, lo, arena_stage(kp, q, par)};
    slot_loop<unroll_for(1, MINB)>(kp, lo, hi, body);
  }
  return true;
}

// ------------------------------------------------------------------ low-latency (LL)
// Rank r's words for peer k live in k's LL buffer [parity][source r][4*slot + lane]: 8 bytes =
// {epoch, value bits}.  8-byte stores are single-copy atomic, so a reader that sees the current
// epoch in a word also sees that word's value -- no separate flag, no barrier.  The parity half
// a call writes was last read two calls ago, which every peer finished before this call began.
__device__ __forceinline__ unsigned long long* ll_buf(const KParams& kp, int rank, int par,
                                                      int src) {
  return reinterpret_cast<unsigned long long*>(kp.stage[rank] + 2 * (kStageCapacity / sizeof(float))) +
         ((size_t)par * kp.p + src) * (size_t)kp.ll_cap;
}
__device__ __forceinline__ void st_ll(unsigned long long* p, float a, float b, uint32_t e) {
  const unsigned long long x = ((unsigned long long)e << 32) | __float_as_uint(a);
  const unsigned long long y = ((unsigned long long)e << 32) | __float_as_uint(b);
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(x), "l"(y) : "memory");
}
__device__ __forceinline__ void ld_ll(const unsigned long long* p, unsigned long long& x,
                                      unsigned long long& y) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(p) : "memory");
}

template <int OP, int P>
struct LLBody {
  using N = Needs<OP, PH_RS, P>;
  static constexpr int NP = 3;
  const KParams& kp;
  int r;
  int par;
  struct State {
    float4 own, b, c;
    float *pa, *pb, *pc;
  };
  __device__ __forceinline__ void bind(int t, float** ptr) const {
    const size_t mine = (size_t)r * kp.T + t;
    ptr[0] = kp.a[mine];
    ptr[1] = (N::loadB || N::storeB) ? kp.b[mine] : nullptr;
    ptr[2] = (N::loadC || N::storeC) ? kp.c[mine] : nullptr;
  }
  // Issue the local loads and push this slot to every peer.
  template <bool VEC>
  __device__ __forceinline__ void load(const SlotRef& ref, float* const* ptr, State& st) const {
    st.own = ldv<VEC>(ptr[0], ref);
    if constexpr (N::loadB) st.b = ldv<VEC>(ptr[1], ref);
    if constexpr (N::loadC) st.c = ldv<VEC>(ptr[2], ref);
    st.pa = ptr[0];
    st.pb = ptr[1];
    st.pc = ptr[2];
    const uint32_t e = ep();
#pragma unroll
    for (int k = 0; k < P; ++k) {
      if (k == r) continue;
      unsigned long long* dst = ll_buf(kp, k, par, r) + 4 * (size_t)ref.s;
      st_ll(dst, st.own.x, st.own.y, e);
      st_ll(dst + 2, st.own.z, st.own.w, e);
    }
  }
  // Wait for every peer's words of this slot, reduce in rank order, apply the epilogue.
  template <bool VEC>
  __device__ __forceinline__ void finish(const SlotRef& ref, State& st) const {
    const uint32_t e = ep();
    float4 in[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      if (k == r) {
        in[k] = st.own;
        continue;
      }
      const unsigned long long* src = ll_buf(kp, r, par, k) + 4 * (size_t)ref.s;
      unsigned long long x0, x1, x2, x3;
      unsigned long long t0 = 0;
      while (true) {
        ld_ll(src, x0, x1);
        ld_ll(src + 2, x2, x3);
        if ((uint32_t)(x0 >> 32) == e && (uint32_t)(x1 >> 32) == e && (uint32_t)(x2 >> 32) == e &&
            (uint32_t)(x3 >> 32) == e)
          break;
        if (t0 == 0) t0 = globaltimer();
        else if (globaltimer() - t0 > kp.timeout_ns) {
          atomicCAS_system(kp.err, 0, (int)TC_ERR_TIMEOUT);
          break;
        }
      }
      in[k] = make_float4(__uint_as_float((uint32_t)x0), __uint_as_float((uint32_t)x1),
                          __uint_as_float((uint32_t)x2), __uint_as_float((uint32_t)x3));
    }
    float4 oa;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float v[P];
#pragma unroll
      for (int k = 0; k < P; ++k) v[k] = lane(in[k], i);
      float la = 0.f;
      float lb = N::loadB ? lane(st.b, i) : 0.f;
      float lc = N::loadC ? lane(st.c, i) : 0.f;
      elem<OP, PH_RS, P>(kp, r, v, la, lb, lc);
      lane(oa, i) = la;
      if constexpr (N::storeB) lane(st.b, i) = lb;
      if constexpr (N::storeC) lane(st.c, i) = lc;
    }
    if constexpr (N::storeA) stv<VEC>(st.pa, ref, oa);
    if constexpr (N::storeB) stv<VEC>(st.pb, ref, st.b);
    if constexpr (N::storeC) stv<VEC>(st.pc, ref, st.c);
  }
};

// ------------------------------------------------------------------ kernels
template <int OP, int P, int MINB>
__global__ void __launch_bounds__(512, MINB) k_twoshot_pull(KParams kp) {
  const int r = kp.rank0 + (int)blockIdx.y;
  if (r == kp.absent_rank) return;
  call_begin(kp, r);
  const int par = (int)(ep() & 1u);
  const int64_t M = kp.M;
  stamp(kp, 0);
  if (!barrier_all(kp, r, BAR_ENTRY, true)) return;
  stamp(kp, 1);
  const int lo = (int)(M * r / P), hi = (int)(M * (r + 1) / P);
  {
    ReduceBody<OP, P, SRC_TENSORS, true> body{kp, r, lo, arena_stage(kp, r, par)};
    slot_loop<unroll_for(P, MINB)>(kp, lo, hi, body);
  }
  stamp(kp, 2);
  stamp(kp, 3);
  if (!gather_all<OP, P, MINB>(kp, r, par)) return;
  stamp(kp, 4);
  call_end(kp, r);
  stamp(kp, 5);
}

template <int OP, int P, int MINB>
__global__ void __launch_bounds__(512, MINB) k_oneshot(KParams kp) {
  const int r = kp.rank0 + (int)blockIdx.y;
  if (r == kp.absent_rank) return;
  call_begin(kp, r);
  const int lo = 0, hi = kp.M;
  stamp(kp, 0);
  // groups of at most one slot per thread (the runtime sizes the grid for it up to two CTAs per
  // SM): every thread takes one slot -- its tensor lookup and its p remote loads in parallel
  // with every other thread's -- instead of a warp walking a 128-slot piece
  const bool flat = (int64_t)hi <= (int64_t)gridDim.x * blockDim.x;
  {
    CopyOutBody body{kp, r, 0, kp.stage[r] + stage_off()};
    if (flat) slot_loop_flat(kp, lo, hi, body);
    else slot_loop<unroll_for(1, MINB)>(kp, lo, hi, body);
  }
  if (!barrier_all(kp, r, BAR_ENTRY, true)) return;
  stamp(kp, 1);
  ReduceBody<OP, P, SRC_ONESHOT, false> body{kp, r, 0, nullptr};
  if (flat) slot_loop_flat(kp, lo, hi, body);
  else slot_loop<unroll_for(P, MINB)>(kp, lo, hi, body);
  stamp(kp, 2);
  stamp(kp, 3);
  stamp(kp, 4);
  call_end(kp, r);
  stamp(kp, 5);
}

// Low-latency: no barrier; each slot is pushed to every peer and its peers' words awaited.
template <int OP, int P, int MINB>
__global__ void __launch_bounds__(512, MINB) k_ll(KParams kp) {
  const int r = kp.rank0 + (int)blockIdx.y;
  if (r == kp.absent_rank) return;
  call_begin(kp, r);
  stamp(kp, 0);
  LLBody<OP, P> body{kp, r, (int)(ep() & 1u)};
  slot_loop_flat(kp, 0, kp.M, body);
  call_end(kp, r);
  stamp(kp, 5);
}

// ------------------------------------------------------------------ p = 1: TMA stream
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra W_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

// First element of a p = 1 tile: 64-bit, split over the .y (low) and .w (high) words, so tensors
// of 2^31 elements or more (8 GiB of fp32) are addressed correctly.
__device__ __forceinline__ int64_t tile_elem(const int4& tl) {
  return (int64_t)(uint32_t)tl.y | ((int64_t)tl.w << 32);
}

// p = 1 (no communication): the epilogue as one HBM stream, moved by the copy engine of each
// SM.  Tiles (<= kTileE elements inside one tensor, group-creation table) are dealt round-robin
// over the grid (DRAM locality, as the pieces of the other kernels); lane 0 of warp 0 issues
// cp.async.bulk loads of the tile's operands into local_stages() shared-memory stages (mbarrier
// complete_tx), the consumer warps apply elem<> from shared memory and store 16-B vectors.
// Tiles that are not 16-B aligned in every operand (or a tensor's last numel % 4 elements) are
// processed element by element straight from global memory, with the same arithmetic.
// Measured (tools/p2p_probe.cu, fused-SGD stream): TMA 6.26 TB/s vs 6.2 LDG; round 1's
// register-staged kernel (one piece per warp in flight) reached 87.5 us on ResNet-50, this 81.5.
template <int OP>
__global__ void __launch_bounds__(kTmaThreads, 1) k_local_tma(KParams kp) {
  using N = Needs<OP, PH_RS, 1>;
  constexpr int NA = local_na<OP>();            // operands per stage, packed: a, [b], [c], [d]
  static_assert(NA == local_ops(OP), "local_ops() disagrees with the operand needs");
  constexpr int NST = local_stages(NA);
  constexpr int IB = 1, IC = IB + (N::loadB ? 1 : 0), ID = IC + (N::loadC ? 1 : 0);
  extern __shared__ __align__(128) float4 sm4[];  // [NST][NA][kTileE / 4]
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const int r = kp.rank0 + (int)blockIdx.y;
  const int warp = threadIdx.x >> 5, lane_id = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])),
                   "r"(kTmaConsumerWarps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t row = (size_t)r * kp.T;
  auto aligned = [&](int t, int64_t e0, int n) {
    bool ok = (n & 3) == 0 && (((uintptr_t)(kp.a[row + t] + e0)) & 15) == 0;
    if constexpr (N::loadB) ok = ok && (((uintptr_t)(kp.b[row + t] + e0)) & 15) == 0;
    if constexpr (N::loadC) ok = ok && (((uintptr_t)(kp.c[row + t] + e0)) & 15) == 0;
    if constexpr (N::loadD) ok = ok && (((uintptr_t)(kp.d[row + t] + e0)) & 15) == 0;
    return ok;
  };
  if (warp == 0) {  // producer
    if (lane_id != 0) return;
    int k = 0;
    for (int i = blockIdx.x; i < kp.ntiles; i += gridDim.x, ++k) {
      const int s = k % NST;
      if (k >= NST) mbar_wait(&empty[s], (uint32_t)((k / NST - 1) & 1));
      const int4 tl = kp.tiles[i];
      const int64_t e0 = tile_elem(tl);
      if (!aligned(tl.x, e0, tl.z)) {  // consumers read global memory directly
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s]))
                     : "memory");
        continue;
      }
      const uint32_t bytes = (uint32_t)tl.z * 4;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       smem_u32(&full[s])),
                   "r"(NA * bytes)
                   : "memory");
      const float* src[4] = {kp.a[row + tl.x] + e0,
                             N::loadB ? kp.b[row + tl.x] + e0 : nullptr,
                             N::loadC ? kp.c[row + tl.x] + e0 : nullptr,
                             N::loadD ? kp.d[row + tl.x] + e0 : nullptr};
      int slot = 0;
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        if (src[o] == nullptr) continue;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(sm4 + ((size_t)s * NA + slot) * (kTileE / 4))),
            "l"(src[o]), "r"(bytes), "r"(smem_u32(&full[s]))
            : "memory");
        ++slot;
      }
    }
    return;
  }
  const int ct = threadIdx.x - 32, nct = kTmaThreads - 32;
  int k = 0;
  for (int i = blockIdx.x; i < kp.ntiles; i += gridDim.x, ++k) {
    const int s = k % NST;
    const int4 tl = kp.tiles[i];
    const int64_t e0 = tile_elem(tl);
    float* pa = kp.a[row + tl.x] + e0;
    float* pb = (N::loadB || N::storeB) ? kp.b[row + tl.x] + e0 : nullptr;
    float* pc = (N::loadC || N::storeC) ? kp.c[row + tl.x] + e0 : nullptr;
    const float* pd = N::loadD ? kp.d[row + tl.x] + e0 : nullptr;
    mbar_wait(&full[s], (uint32_t)((k / NST) & 1));
    if (aligned(tl.x, e0, tl.z)) {
      const float4* sa = sm4 + ((size_t)s * NA + 0) * (kTileE / 4);
      const float4* sb = sm4 + ((size_t)s * NA + IB) * (kTileE / 4);
      const float4* sc = sm4 + ((size_t)s * NA + IC) * (kTileE / 4);
      const float4* sd = sm4 + ((size_t)s * NA + ID) * (kTileE / 4);
      for (int v = ct; v < tl.z / 4; v += nct) {
        const float4 va = sa[v];
        float4 vb = N::loadB ? sb[v] : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 vc = N::loadC ? sc[v] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 vd = N::loadD ? sd[v] : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 oa;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          const float in[1] = {lane_of(va, l)};
          float la = 0.f, lb = lane_of(vb, l), lc = lane_of(vc, l);
          elem4<OP, PH_RS, 1>(kp, r, in, la, lb, lc, lane_of(vd, l));
          lane(oa, l) = la;
          lane(vb, l) = lb;
          lane(vc, l) = lc;
        }
        if constexpr (N::storeA) st16(pa + 4 * v, oa);
        if constexpr (N::storeB) st16(pb + 4 * v, vb);
        if constexpr (N::storeC) st16(pc + 4 * v, vc);
      }
    } else {
      for (int j = ct; j < tl.z; j += nct) {
        const float in[1] = {ld4(pa + j)};
        float la = 0.f, lb = N::loadB ? ld4(pb + j) : 0.f, lc = N::loadC ? ld4(pc + j) : 0.f;
        elem4<OP, PH_RS, 1>(kp, r, in, la, lb, lc, N::loadD ? ld4(pd + j) : 0.f);
        if constexpr (N::storeA) st4(pa + j, la);
        if constexpr (N::storeB) st4(pb + j, lb);
        if constexpr (N::storeC) st4(pc + j, lc);
      }
    }
    __syncwarp();
    if (lane_id == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s]))
                   : "memory");
  }
}

// ------------------------------------------------------------------ two-shot, TMA-staged
// The pulled two-shot with its data movement on the TMA engines.  Warp 0 is the producer:
// its 32 lanes fetch the descriptors of 32 tiles at once (one latency for 32 table walks),
// then issue cp.async.bulk copies of each tile's operands -- the p ranks' tensors in the
// reduce-scatter, the owner's staged chunk in the allgather, plus the local epilogue operands --
// into a ring of shared-memory stages, a stage holding G tiles when a phase has fewer operands
// than the stage has room for.  8 consumer warps reduce (float64, rank order), apply the
// epilogue and store.  Bytes in flight per CTA = the ring (up to 192 KiB), not one register
// load per thread, so a few CTAs drive the links and the other SMs stay free for computation
// running beside the collective (NEXT row f1).  Same tiles-to-CTA pairing (tile i of a chunk ->
// CTA i mod grid on every rank), staging, barriers and arithmetic as k_twoshot_pull.
struct T2Desc {
  float* a;     // this rank's tensors at the tile's first element
  float* b;
  float* c;
  float* st;    // staging at the tile's first slot: my chunk (RS) or the owner's (AG)
  const float* g;  // this rank's own gradient (ESGD), else nullptr
  int64_t e;    // element of the tile's first slot in tensor t (negative: shifted head)
  int t, n;     // tensor, slots
  int vec, pad; // 16-B aligned full slots in every operand: bulk path
};

__host__ __device__ constexpr int t2_pack(int x) {
  return x >= 8 ? 8 : x >= 4 ? 4 : x >= 2 ? 2 : 1;
}

// One tile of a TMA two-shot phase, processed by the consumer warps: a full tile and a partial
// slot from shared memory (operand o of this tile at so + o * V), the element path from global
// memory.
// Reduce-scatter tile of the asynchronous elastic update: operands are the P clients' x (slots
// 0..P-1) and this owner's center replica (slot P); every client's new x is stored straight into
// that client's tensor (a peer store over NVLink: only this owner touches this chunk of any
// client's x during the call), the final center into this rank's center and its staging.
template <int P, int V>
__device__ __forceinline__ void t2_tile_easync(const KParams& kp, const T2Desc& d,
                                               const float4* so, int ct, int nct) {
  const size_t T = (size_t)kp.T;
  float* px[P];
#pragma unroll
  for (int q = 0; q < P; ++q) px[q] = kp.a[q * T + d.t] + d.e;
  if (d.vec == 2) {  // one partial slot: only lanes inside the tensor are stored
    if (ct == 0) {
      const int lo_l = d.e < 0 ? (int)-d.e : 0;
      const int hi_l = (int)min((int64_t)4, kp.numel[d.t] - d.e);
      float4 c4 = so[P * V];
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        if (l < lo_l || l >= hi_l) continue;
        float in[P], out[P];
#pragma unroll
        for (int q = 0; q < P; ++q) in[q] = lane_of(so[q * V], l);
        float xc = lane_of(c4, l);
        easync1<P>(kp, in, out, xc);
#pragma unroll
        for (int q = 0; q < P; ++q) st4(px[q] + l, out[q]);
        st4(d.b + l, xc);
        lane(c4, l) = xc;
      }
      st16(d.st, c4);
    }
  } else if (d.vec) {
    for (int v = ct; v < d.n; v += nct) {
      float4 x[P], o[P];
#pragma unroll
      for (int q = 0; q < P; ++q) x[q] = so[q * V + v];
      float4 c4 = so[P * V + v];
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        float in[P], out[P];
#pragma unroll
        for (int q = 0; q < P; ++q) in[q] = lane_of(x[q], l);
        float xc = lane_of(c4, l);
        easync1<P>(kp, in, out, xc);
#pragma unroll
        for (int q = 0; q < P; ++q) lane(o[q], l) = out[q];
        lane(c4, l) = xc;
      }
#pragma unroll
      for (int q = 0; q < P; ++q) st16(px[q] + 4 * v, o[q]);
      st16(d.b + 4 * v, c4);
      st16(d.st + 4 * v, c4);
    }
  } else {  // element path
    const int64_t j0 = d.e < 0 ? -d.e : 0;
    const int64_t j1 = min(4 * (int64_t)d.n, kp.numel[d.t] - d.e);
    for (int64_t j = j0 + ct; j < j1; j += nct) {
      float in[P], out[P];
#pragma unroll
      for (int q = 0; q < P; ++q) in[q] = ld4(px[q] + j);
      float xc = ld4(d.b + j);
      easync1<P>(kp, in, out, xc);
#pragma unroll
      for (int q = 0; q < P; ++q) st4(px[q] + j, out[q]);
      st4(d.b + j, xc);
      st4(d.st + j, xc);
    }
  }
}

template <int OP, int P, int PH, int OPSP, int V>
__device__ __forceinline__ void t2_tile(const KParams& kp, int r, const T2Desc& d,
                                        const float4* so, int ct, int nct) {
  using N = Needs<OP, PH, PH == PH_RS ? P : 2>;
  const size_t T = (size_t)kp.T;
  if constexpr (OP == OP_EASYNC && PH == PH_RS) {
    t2_tile_easync<P, V>(kp, d, so, ct, nct);
    return;
  }
  // reduce-scatter sources: every rank's copy, or the root's alone (broadcast)
  constexpr int NSRC = OP == OP_BCAST ? 1 : P;
  if (d.vec == 2) {
    // one partial slot from shared memory: valid lanes [lo_l, hi_l) are stored
    if (ct == 0) {
      const int lo_l = d.e < 0 ? (int)-d.e : 0;
      const int hi_l = (int)min((int64_t)4, kp.numel[d.t] - d.e);
      if constexpr (PH == PH_RS) {
        constexpr int NB = N::loadB ? 1 : 0, NC = N::loadC ? 1 : 0;
        float4 b = N::loadB ? so[NSRC * V] : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 c = N::loadC ? so[(NSRC + NB) * V] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 g = N::loadD ? so[(NSRC + NB + NC) * V] : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 oa = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          if (l < lo_l || l >= hi_l) continue;
          float in[NSRC];
#pragma unroll
          for (int q = 0; q < NSRC; ++q) in[q] = lane_of(so[q * V], l);
          float la = 0.f, lb = lane_of(b, l), lc = lane_of(c, l);
          elem4<OP, PH_RS, NSRC>(kp, r, in, la, lb, lc, lane_of(g, l));
          lane(oa, l) = la;
          lane(b, l) = lb;
          if constexpr (N::storeA) st4(d.a + l, la);
          if constexpr (N::storeB) st4(d.b + l, lb);
          if constexpr (N::storeC) st4(d.c + l, lc);
        }
        st16(d.st, Needs<OP, PH_RS, P>::stageB ? b : oa);
      } else {
        constexpr int OA = 1, OB = 1 + N::loadA, OC = 1 + N::loadA + N::loadB;
        constexpr int OD = OC + N::loadC;
        const float4 x = so[0];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          if (l < lo_l || l >= hi_l) continue;
          const float in[1] = {lane_of(x, l)};
          float la = N::loadA ? lane_of(so[OA * V], l) : 0.f;
          float lb = N::loadB ? lane_of(so[OB * V], l) : 0.f;
          float lc = N::loadC ? lane_of(so[OC * V], l) : 0.f;
          elem4<OP, PH_AG, 2>(kp, r, in, la, lb, lc,
                              N::loadD ? lane_of(so[OD * V], l) : 0.f);
          if constexpr (N::storeA) st4(d.a + l, la);
          if constexpr (N::storeB) st4(d.b + l, lb);
          if constexpr (N::storeC) st4(d.c + l, lc);
        }
      }
    }
  } else if (d.vec) {
        constexpr int TU = kT2Unroll;
    for (int v0 = ct; v0 < d.n; v0 += nct * TU) {
      if constexpr (PH == PH_RS) {
        constexpr int NB = N::loadB ? 1 : 0, NC = N::loadC ? 1 : 0;
        float4 x[TU][NSRC], b[TU], c[TU], g[TU];
#pragma unroll
        for (int u = 0; u < TU; ++u) {
          const int v = v0 + u * nct;
          if (v < d.n) {
#pragma unroll
            for (int q = 0; q < NSRC; ++q) x[u][q] = so[q * V + v];
            b[u] = N::loadB ? so[NSRC * V + v] : make_float4(0.f, 0.f, 0.f, 0.f);
            c[u] = N::loadC ? so[(NSRC + NB) * V + v] : make_float4(0.f, 0.f, 0.f, 0.f);
            g[u] = N::loadD ? so[(NSRC + NB + NC) * V + v] : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < TU; ++u) {
          const int v = v0 + u * nct;
          if (v >= d.n) continue;
          float4 oa;
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            float in[NSRC];
#pragma unroll
            for (int q = 0; q < NSRC; ++q) in[q] = lane_of(x[u][q], l);
            float la = 0.f, lb = lane_of(b[u], l), lc = lane_of(c[u], l);
            elem4<OP, PH_RS, NSRC>(kp, r, in, la, lb, lc, lane_of(g[u], l));
            lane(oa, l) = la;
            lane(b[u], l) = lb;
            lane(c[u], l) = lc;
          }
          if constexpr (N::storeA) st16(d.a + 4 * v, oa);
          if constexpr (N::storeB) st16(d.b + 4 * v, b[u]);
          if constexpr (N::storeC) st16(d.c + 4 * v, c[u]);
          st16(d.st + 4 * v, Needs<OP, PH_RS, P>::stageB ? b[u] : oa);
        }
      } else {
        constexpr int OA = 1, OB = 1 + N::loadA, OC = 1 + N::loadA + N::loadB;
        constexpr int OD = OC + N::loadC;
        float4 x[TU], a[TU], b[TU], c[TU], g[TU];
#pragma unroll
        for (int u = 0; u < TU; ++u) {
          const int v = v0 + u * nct;
          if (v < d.n) {
            x[u] = so[v];
            a[u] = N::loadA ? so[OA * V + v] : make_float4(0.f, 0.f, 0.f, 0.f);
            b[u] = N::loadB ? so[OB * V + v] : make_float4(0.f, 0.f, 0.f, 0.f);
            c[u] = N::loadC ? so[OC * V + v] : make_float4(0.f, 0.f, 0.f, 0.f);
            g[u] = N::loadD ? so[OD * V + v] : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < TU; ++u) {
          const int v = v0 + u * nct;
          if (v >= d.n) continue;
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            const float in[1] = {lane_of(x[u], l)};
            float la = lane_of(a[u], l), lb = lane_of(b[u], l), lc = lane_of(c[u], l);
            elem4<OP, PH_AG, 2>(kp, r, in, la, lb, lc, lane_of(g[u], l));
            lane(a[u], l) = la;
            lane(b[u], l) = lb;
            lane(c[u], l) = lc;
          }
          if constexpr (N::storeA) st16(d.a + 4 * v, a[u]);
          if constexpr (N::storeB) st16(d.b + 4 * v, b[u]);
          if constexpr (N::storeC) st16(d.c + 4 * v, c[u]);
        }
      }
    }
  } else {
    // element path (shifted heads, partial tails, operands misaligned on some rank)
    const int64_t j0 = d.e < 0 ? -d.e : 0;
    const int64_t j1 = min(4 * (int64_t)d.n, kp.numel[d.t] - d.e);
    for (int64_t j = j0 + ct; j < j1; j += nct) {
      if constexpr (PH == PH_RS) {
        float in[NSRC];
#pragma unroll
        for (int q = 0; q < NSRC; ++q)
          in[q] = ld4(kp.a[(OP == OP_BCAST ? kp.root : q) * T + d.t] + d.e + j);
        float la = 0.f, lb = N::loadB ? ld4(d.b + j) : 0.f, lc = N::loadC ? ld4(d.c + j) : 0.f;
        elem4<OP, PH_RS, NSRC>(kp, r, in, la, lb, lc, N::loadD ? ld4(d.g + j) : 0.f);
        if constexpr (N::storeA) st4(d.a + j, la);
        if constexpr (N::storeB) st4(d.b + j, lb);
        if constexpr (N::storeC) st4(d.c + j, lc);
        st4(d.st + j, Needs<OP, PH_RS, P>::stageB ? lb : la);
      } else {
        const float in[1] = {ld4(d.st + j)};
        float la = N::loadA ? ld4(d.a + j) : 0.f;
        float lb = N::loadB ? ld4(d.b + j) : 0.f, lc = N::loadC ? ld4(d.c + j) : 0.f;
        elem4<OP, PH_AG, 2>(kp, r, in, la, lb, lc, N::loadD ? ld4(d.g + j) : 0.f);
        if constexpr (N::storeA) st4(d.a + j, la);
        if constexpr (N::storeB) st4(d.b + j, lb);
        if constexpr (N::storeC) st4(d.c + j, lc);
      }
    }
  }
}

template <int OP, int P, int PH, int G, int OPSP, int OPS, int NS>
__device__ __forceinline__ void t2_phase(const KParams& kp, int r, int qo, float* stagebuf,
                                         int& k, uint64_t* full, uint64_t* empty,
                                         T2Desc (*desc)[8], float4* sm4,
                                         unsigned long long& waited) {
  using N = Needs<OP, PH, PH == PH_RS ? P : 2>;
  constexpr int V = t2_slots(P);
  const int warp = threadIdx.x >> 5, lane_id = threadIdx.x & 31;
  const size_t T = (size_t)kp.T;
  const int lo = (int)((int64_t)kp.M * qo / P);
  const int first = kp.tile2_off[qo] + (int)blockIdx.x, end = kp.tile2_off[qo + 1];
  const int cnt = first < end ? (end - first + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  auto stage = [&](int s, int o) { return sm4 + ((size_t)s * OPS + o) * V; };
  if (warp == 0) {
    if (lane_id == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncwarp();
    for (int base = 0; base < cnt; base += 32) {
      const int j = base + lane_id;
      const bool valid = j < cnt;
      T2Desc d{};
      const float* src[OPSP];
      uint32_t bytes = 0;
      if (valid) {
        const int4 tl = kp.tiles2[first + j * (int)gridDim.x];
        d.t = tl.x;
        d.n = tl.z;
        d.e = (int64_t)(tl.y - kp.prefix[d.t]) * 4 - kp.shift[d.t];
        const size_t mine = (size_t)r * T + d.t;
        d.a = kp.a[mine] + d.e;
        d.b = (N::loadB || N::storeB) ? kp.b[mine] + d.e : nullptr;
        d.c = (N::loadC || N::storeC) ? kp.c[mine] + d.e : nullptr;
        d.g = N::loadD ? kp.d[mine] + d.e : nullptr;
        d.st = stagebuf + (size_t)(tl.y - lo) * 4;
        // full slots, or one partial slot (a shifted tensor's head, a tail) whose containing
        // 16-B block is bulk-copied whole (it lies inside the tensor's allocation: the
        // allocation base is 256-B aligned and sizes are rounded to 512 B), lanes outside the
        // tensor computed but never stored
        const bool part = d.e < 0 || d.e + 4 * (int64_t)d.n > kp.numel[d.t];
        bool vec = !part || d.n == 1;
        int o = 0;
        if constexpr (PH == PH_RS) {
          if constexpr (OP == OP_BCAST) {
            src[o++] = kp.a[(size_t)kp.root * T + d.t] + d.e;
          } else {
#pragma unroll
            for (int q = 0; q < P; ++q) src[o++] = kp.a[q * T + d.t] + d.e;
          }
        } else {
          src[o++] = d.st;
          if constexpr (N::loadA) src[o++] = d.a;
        }
        if constexpr (N::loadB) src[o++] = d.b;
        if constexpr (N::loadC) src[o++] = d.c;
        if constexpr (N::loadD) src[o++] = d.g;
#pragma unroll
        for (int x = 0; x < OPSP; ++x) vec = vec && (((uintptr_t)src[x] & 15) == 0);
        vec = vec && (((uintptr_t)d.a & 15) == 0);
        d.vec = vec ? (part ? 2 : 1) : 0;
        bytes = vec ? (uint32_t)d.n * 16 * OPSP : 0;
      }
      const int bc = min(32, cnt - base);
      for (int u0 = 0; u0 < bc; u0 += G) {
        const int s = k % NS;
        const bool in_unit = valid && lane_id >= u0 && lane_id < u0 + G;
        const uint32_t ub = __reduce_add_sync(0xffffffffu, in_unit ? bytes : 0u);
        if (lane_id == u0 && k >= NS) {
          const unsigned long long t0 = kp.prof ? globaltimer() : 0;
          mbar_wait(&empty[s], (uint32_t)((k / NS - 1) & 1));
          if (kp.prof) waited += globaltimer() - t0;
        }
        __syncwarp();
        if (in_unit) desc[s][lane_id - u0] = d;
        __syncwarp();
        if (lane_id == u0) {
          if (ub)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                             smem_u32(&full[s])),
                         "r"(ub)
                         : "memory");
          else
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s]))
                         : "memory");
        }
        __syncwarp();
        if (in_unit && d.vec) {
#pragma unroll
          for (int x = 0; x < OPSP; ++x)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                "%2, [%3];" ::"r"(smem_u32(stage(s, (lane_id - u0) * OPSP + x))),
                "l"(src[x]), "r"((uint32_t)d.n * 16), "r"(smem_u32(&full[s]))
                : "memory");
        }
        ++k;
      }
    }
    return;
  }
  // consumers
  const int ct = threadIdx.x - 32, nct = kT2Threads - 32;
  for (int base = 0; base < cnt; base += 32) {
    const int bc = min(32, cnt - base);
    for (int u0 = 0; u0 < bc; u0 += G) {
      const int s = k % NS;
      const int ut = min(G, bc - u0);
      {
        const unsigned long long t0 = kp.prof ? globaltimer() : 0;
        mbar_wait(&full[s], (uint32_t)((k / NS) & 1));
        if (kp.prof) waited += globaltimer() - t0;
      }
      for (int jt = 0; jt < ut; ++jt)
        t2_tile<OP, P, PH, OPSP, V>(kp, r, desc[s][jt], stage(s, jt * OPSP), ct, nct);
      __syncwarp();
      if (lane_id == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s]))
                     : "memory");
      ++k;
    }
  }
}

template <int OP, int P>
__global__ void __launch_bounds__(kT2Threads, 1) k_twoshot_tma(KParams kp) {
  using NR = Needs<OP, PH_RS, P>;
  using NG = Needs<OP, PH_AG, 2>;
  constexpr int OPS = t2_ops(OP, P), NS = t2_stages(OP, P);
  constexpr int OPS_RS = (OP == OP_BCAST ? 1 : P) + NR::loadB + NR::loadC + NR::loadD;
  constexpr int OPS_AG = 1 + NG::loadA + NG::loadB + NG::loadC + NG::loadD;
  constexpr int G_RS = t2_pack(OPS / OPS_RS), G_AG = t2_pack(OPS / OPS_AG);
  static_assert(OPS_RS <= OPS && OPS_AG <= OPS, "stage too small");
  extern __shared__ __align__(128) float4 sm4[];  // [NS][OPS][t2_slots(P)]
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  __shared__ T2Desc desc[NS][8];
  const int r = kp.rank0 + (int)blockIdx.y;
  if (r == kp.absent_rank) return;
  call_begin(kp, r);
  const int par = (int)(ep() & 1u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])),
                   "r"(kT2ConsumerWarps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  stamp(kp, 0);
  if (!barrier_all(kp, r, BAR_ENTRY, true)) return;
  stamp(kp, 1);
  int k = 0;  // position in the stage ring (continues across phases)
  unsigned long long waited = 0;  // profiling: producer waits for empty / consumers for full
  t2_phase<OP, P, PH_RS, G_RS, OPS_RS, OPS, NS>(kp, r, r, arena_stage(kp, r, par), k, full,
                                                 empty, desc, sm4, waited);
  stamp(kp, 2);
  if (!barrier_all(kp, r, BAR_MID, true)) return;
  stamp(kp, 3);
#pragma unroll 1
  for (int jq = 0; jq < P - 1; ++jq) {
    const int qo = (r + 1 + jq) % P;
    t2_phase<OP, P, PH_AG, G_AG, OPS_AG, OPS, NS>(kp, r, qo, arena_stage(kp, qo, par), k, full,
                                                   empty, desc, sm4, waited);
  }
  stamp(kp, 4);
  if (kp.prof != nullptr && threadIdx.x < 32)  // producer lanes each timed their own waits
    for (int o = 16; o > 0; o >>= 1) waited += __shfl_xor_sync(0xffffffffu, waited, o);
  if (kp.prof != nullptr && (threadIdx.x == 0 || threadIdx.x == 32)) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    // slot 6: producer waits for free stages; slot 7: consumer waits for data (low 40 bits) and
    // the SM the CTA ran on (high bits)
    kp.prof[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + (threadIdx.x ? 7 : 6)] =
        threadIdx.x ? (waited & ((1ull << 40) - 1)) | ((unsigned long long)smid << 40) : waited;
  }
  call_end(kp, r);
  stamp(kp, 5);
}


// ------------------------------------------------------------------ NVLS (switch reduction)
// The owner of a chunk reads every rank's copy of it reduced in the NVSwitch
// (multimem.ld_reduce on the multicast address: fp32 sums in the switch's order) and writes the
// result into every rank's copy with one multimem.st.  Per GPU: egress S (serving every owner's
// reductions) + S/p, ingress S/p + S -- (1 + 1/p) S each way against the two-shot's 2(p-1)/p S.
//
// Work: the owner chunk's tiles (the TMA two-shot's table: runs of <= 512 slots inside one
// tensor), tile i of a chunk on CTA i mod grid on every rank.  Inside a CTA the NVLS warps take
// the CTA's tiles round-robin, a round = one tile per NVLS warp (more when a CTA holds > 255
// rounds).  When every NVLS warp has reached the end of a round (named barrier 1), the signal
// warp fences at system scope and stores the round count into every rank's progress flag
// [BAR_PROG][this rank][this CTA].  Consumers on every rank (CTA b waits for CTA b of owner q):
//   SGD       -- the epilogue warps apply the update to round j's tiles of chunk q as soon as
//                owner q published round j: G (the stored sum) is written back already, w and
//                dw are updated from local memory -- the HBM epilogue overlaps the switch work;
//   allreduce -- the signal warp waits for every owner's last round (the call must not complete
//                before every owner's stores have landed here).
__device__ __forceinline__ float4 mm_ld_reduce16(const float* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ float mm_ld_reduce4(const float* p) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mm_st16(float* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_st4(float* p, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

constexpr int kNvlsWarps = kNvlsThreads / 32;
#ifndef TC_NV_RW_AR
#define TC_NV_RW_AR 12  // switch-reduction warps per CTA, plain allreduce
#endif
#ifndef TC_NV_RW_SGD
#define TC_NV_RW_SGD 4  // switch-reduction warps per CTA, fused SGD (the rest: signal + epilogue)
#endif
#ifndef TC_NV_RED_U_SGD
#define TC_NV_RED_U_SGD 4  // fused SGD: switch reductions in flight per lane
#endif
#ifndef TC_NV_RED_U_AR
#define TC_NV_RED_U_AR 4   // allreduce: switch reductions in flight per lane
#endif
#ifndef TC_NV_EPI_U
#define TC_NV_EPI_U 4   // fused SGD epilogue: 16-B slots per thread in flight
#endif
#ifndef TC_NV_ROUND
#define TC_NV_ROUND 1   // fused SGD: tiles per reduction warp per published round
#endif
__host__ __device__ constexpr int nvls_reduce_warps(int op) {
  return op == OP_ALLREDUCE ? TC_NV_RW_AR : TC_NV_RW_SGD;
}

// A tile of owner q's chunk as seen by this rank: element offset e of its first slot inside
// tensor t (negative for a shifted head), slot count n, vector path when the tile is whole
// 16-B slots.
struct NvTile {
  int t, n;
  int64_t e;
  bool full;
};
__device__ __forceinline__ NvTile nv_tile(const KParams& kp, int gi) {
  const int4 tl = kp.tiles2[gi];
  NvTile d;
  d.t = tl.x;
  d.n = tl.z;
  d.e = (int64_t)(tl.y - kp.prefix[d.t]) * 4 - kp.shift[d.t];
  d.full = d.e >= 0 && d.e + 4 * (int64_t)d.n <= kp.numel[d.t];
  return d;
}

// Tiles of owner q's chunk held by this CTA, and the tiles per published round: one tile per
// reduction warp for the SGD step (its epilogue follows the rounds), all of them at once for the
// plain allreduce (nothing to overlap: only the end is awaited).
template <int OP>
__device__ __forceinline__ void nv_counts(const KParams& kp, int q, int nw, int& cnt, int& tpr) {
  const int n = kp.tile2_off[q + 1] - kp.tile2_off[q];
  const int b = (int)blockIdx.x, G = (int)gridDim.x;
  cnt = n > b ? (n - b + G - 1) / G : 0;
  if constexpr (OP != OP_SGD) {
    tpr = cnt > 0 ? cnt : 1;
  } else {
    const int m = (cnt + 255 * nw - 1) / (255 * nw);
    tpr = nw * (m > TC_NV_ROUND ? m : TC_NV_ROUND);
  }
}
__device__ __forceinline__ uint32_t nv_flag_value(int rounds) {
  return (ep() << 8) | (uint32_t)rounds;
}

// Whole warp: switch-reduce one tile of this rank's chunk and multicast the result.
template <int OP>
__device__ __forceinline__ void nv_reduce_tile(const KParams& kp, const NvTile& d, int lane_id) {
  float* mc = kp.mc[d.t] + d.e;
  const bool vec = d.full && (((uintptr_t)mc & 15) == 0);
  auto fin = [&](float v) {
    return OP == OP_ALLREDUCE ? __double2float_rn(__dmul_rn((double)v, (double)kp.scale)) : v;
  };
  if (vec) {
    constexpr int U = OP == OP_SGD ? TC_NV_RED_U_SGD : TC_NV_RED_U_AR;  // in flight per lane
    for (int s0 = lane_id; s0 < d.n; s0 += 32 * U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (s0 + 32 * u < d.n) v[u] = mm_ld_reduce16(mc + 4 * (s0 + 32 * u));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (s0 + 32 * u >= d.n) continue;
        v[u] = make_float4(fin(v[u].x), fin(v[u].y), fin(v[u].z), fin(v[u].w));
        mm_st16(mc + 4 * (s0 + 32 * u), v[u]);
      }
    }
  } else {
    const int64_t j0 = d.e < 0 ? -d.e : 0;
    const int64_t j1 = min(4 * (int64_t)d.n, kp.numel[d.t] - d.e);
    for (int64_t j = j0 + lane_id; j < j1; j += 32) mm_st4(mc + j, fin(mm_ld_reduce4(mc + j)));
  }
}

// Threads ct of nct (the epilogue warps together): the SGD epilogue of one tile of any chunk,
// from local memory (G already stored by its owner).
__device__ __forceinline__ void nv_sgd_tile(const KParams& kp, int r, const NvTile& d, int ct,
                                            int nct) {
  const size_t mine = (size_t)r * kp.T + d.t;
  const float* pg = kp.a[mine] + d.e;
  float* pw = kp.b[mine] + d.e;
  float* pd = kp.c[mine] + d.e;
  const bool vec = d.full && ((((uintptr_t)pg | (uintptr_t)pw | (uintptr_t)pd) & 15) == 0);
  if (vec) {
    constexpr int U = TC_NV_EPI_U;  // slots per thread in flight (3 loads each)
    for (int s0 = ct; s0 < d.n; s0 += nct * U) {
      float4 g[U], w[U], dw[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = s0 + nct * u;
        if (s < d.n) {
          g[u] = ld16(pg + 4 * s);
          w[u] = ld16(pw + 4 * s);
          dw[u] = ld16(pd + 4 * s);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = s0 + nct * u;
        if (s >= d.n) continue;
#pragma unroll
        for (int l = 0; l < 4; ++l) sgd1(kp, lane_of(g[u], l), lane(w[u], l), lane(dw[u], l));
        st16(pw + 4 * s, w[u]);
        st16(pd + 4 * s, dw[u]);
      }
    }
  } else {
    const int64_t j0 = d.e < 0 ? -d.e : 0;
    const int64_t j1 = min(4 * (int64_t)d.n, kp.numel[d.t] - d.e);
    for (int64_t j = j0 + ct; j < j1; j += nct) {
      float w = ld4(pw + j), dw = ld4(pd + j);
      sgd1(kp, ld4(pg + j), w, dw);
      st4(pw + j, w);
      st4(pd + j, dw);
    }
  }
}

// One lane: wait until owner q's CTA (this CTA's index) has published `rounds` rounds.  Polls
// with relaxed loads and a short sleep (acquire loads in a tight loop from several warps slow the
// SM's other memory traffic), then one acquire load orders the data reads after the flag.
__device__ __forceinline__ bool nv_wait(const KParams& kp, int r, int q, int rounds) {
  const uint32_t* f = kp.flags[r] + flag_index(BAR_PROG, q, blockIdx.x);
  const uint32_t want = nv_flag_value(rounds);
  if ((int32_t)(ld_acquire_sys(f) - want) >= 0) return true;
  const unsigned long long t0 = globaltimer();
  while (true) {
    uint32_t v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if ((int32_t)(v - want) >= 0) break;
    __nanosleep(128);
    if (globaltimer() - t0 > kp.timeout_ns) {
      atomicCAS_system(kp.err, 0, (int)TC_ERR_TIMEOUT);
      return false;
    }
  }
  return (int32_t)(ld_acquire_sys(f) - want) >= 0;
}

template <int OP, int P>
__global__ void __launch_bounds__(32 * kNvlsWarps, 1) k_nvls(KParams kp) {
  // switch-reduction warps; warp NW signals.  The allreduce runs any block size of >= 2 warps
  // (up to 12 reduction warps; a 4-warp CTA can fit beside a compute kernel's CTA -- NEXT row
  // f1); the fused step has the fixed 16-warp split.
  const int NW = OP == OP_ALLREDUCE ? min(nvls_reduce_warps(OP), (int)(blockDim.x >> 5) - 1)
                                    : nvls_reduce_warps(OP);
  constexpr int NE = kNvlsWarps - nvls_reduce_warps(OP) - 1;  // SGD epilogue warps
  const int r = kp.rank0 + (int)blockIdx.y;
  if (r == kp.absent_rank) return;
  call_begin(kp, r);
  const int warp = threadIdx.x >> 5, lane_id = threadIdx.x & 31;
  const int b = (int)blockIdx.x, G = (int)gridDim.x;
  stamp(kp, 0);
  if (!barrier_all(kp, r, BAR_ENTRY, true)) return;  // every rank's data is in place
  stamp(kp, 1);
  int cnt, tpr;
  nv_counts<OP>(kp, r, NW, cnt, tpr);
  const int nr = (cnt + tpr - 1) / tpr;
  bool ok = true;
  if (warp < NW) {
    for (int j = 0; j < nr; ++j) {
      for (int k = j * tpr + warp; k < min(cnt, (j + 1) * tpr); k += NW)
        nv_reduce_tile<OP>(kp, nv_tile(kp, kp.tile2_off[r] + b + G * k), lane_id);
      __syncwarp();
      // every reduction warp syncs too: a warp must not arrive twice at one barrier phase
      asm volatile("bar.sync 1, %0;" ::"r"(32 * (NW + 1)) : "memory");
    }
    stamp(kp, 2);  // (diagnostics) reduction warps done
  } else if (warp == NW) {
    for (int j = 0; j < nr; ++j) {
      asm volatile("bar.sync 1, %0;" ::"r"(32 * (NW + 1)) : "memory");
      if (lane_id == 0) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        for (int q = 0; q < P; ++q)
          asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(
                           kp.flags[q] + flag_index(BAR_PROG, r, b)),
                       "r"(nv_flag_value(j + 1))
                       : "memory");
      }
      __syncwarp();
    }
    stamp(kp, 3, 32 * NW);  // (diagnostics) every round published
    if constexpr (OP != OP_SGD) {
      // every owner's stores have landed here before the call completes
      if (lane_id < P) {
        int cq, tq;
        nv_counts<OP>(kp, lane_id, NW, cq, tq);
        if (cq > 0) ok = nv_wait(kp, r, lane_id, (cq + tq - 1) / tq);
      }
      ok = __all_sync(0xffffffffu, ok);
      stamp(kp, 4, 32 * NW);  // (diagnostics) every owner's last round seen
    }
  } else if constexpr (OP == OP_SGD) {
    const int ew = warp - NW - 1;
    // round by round over every owner (round j of every chunk before round j + 1 of any): the
    // owners publish their rounds at about the same pace, so only the last round's epilogue
    // is left when the switch work ends
    int nmax = 0;
    for (int q = 0; q < P; ++q) {
      int cq, tq;
      nv_counts<OP>(kp, q, NW, cq, tq);
      nmax = max(nmax, (cq + tq - 1) / tq);
    }
    int item = 0;  // running index over (round, owner, tile): epilogue warp ew takes ew mod NE
#pragma unroll 1
    for (int j = 0; j < nmax && ok; ++j) {
#pragma unroll 1
      for (int jq = 0; jq < P && ok; ++jq) {
        const int q = (r + jq) % P;  // own chunk first: its round is published first
        int cq, tq;
        nv_counts<OP>(kp, q, NW, cq, tq);
        const int k0 = j * tq, k1 = min(cq, (j + 1) * tq);
        if (k0 >= k1) continue;
        int k = k0 + ((ew - item) % NE + NE) % NE;  // this warp's first item of the round
        item += k1 - k0;
        if (k >= k1) continue;
        if (lane_id == 0) ok = nv_wait(kp, r, q, j + 1);
        ok = __shfl_sync(0xffffffffu, ok, 0);
        __syncwarp();
        for (; k < k1 && ok; k += NE)
          nv_sgd_tile(kp, r, nv_tile(kp, kp.tile2_off[q] + b + G * k), lane_id, 32);
      }
      if (j == 0) stamp(kp, 6, 32 * (kNvlsWarps - 1));  // (diagnostics) first round done
      if (j == 1) stamp(kp, 7, 32 * (kNvlsWarps - 1));  // (diagnostics) second round done
    }
    stamp(kp, 4, 32 * (kNvlsWarps - 1));  // (diagnostics) last epilogue warp done
  }
  if (!__syncthreads_and(ok)) return;
  call_end(kp, r);
  stamp(kp, 5);
}

// Tensor broadcast through the switch (ALGO_NVLS, multicast-bound groups): the root reads its
// tensors and writes every rank's copy with one multimem.st per 16 B -- each byte leaves the root
// once (egress S, every rank's ingress S) instead of the scatter + allgather's 2(p-1)/p S out of
// the root.  A copy, so bit-exact.  ENTRY barrier (no rank still uses its old values); tile i of
// the whole group on CTA i mod grid, warps round-robin; the root's CTA b fences and publishes,
// every other rank's CTA b waits for it (the call completes once every tile has landed).
template <int P>
__global__ void __launch_bounds__(kNvlsThreads, 1) k_nvls_bcast(KParams kp) {
  const int r = kp.rank0 + (int)blockIdx.y;
  if (r == kp.absent_rank) return;
  call_begin(kp, r);
  const int warp = threadIdx.x >> 5, lane_id = threadIdx.x & 31;
  const int b = (int)blockIdx.x, G = (int)gridDim.x;
  if (!barrier_all(kp, r, BAR_ENTRY, true)) return;
  bool ok = true;
  if (r == kp.root) {
    const int n = kp.tile2_off[P] - kp.tile2_off[0];
    const size_t row = (size_t)r * kp.T;
    for (int k = warp; b + G * k < n; k += kNvlsWarps) {
      const NvTile d = nv_tile(kp, kp.tile2_off[0] + b + G * k);
      const float* src = kp.a[row + d.t] + d.e;
      float* mc = kp.mc[d.t] + d.e;
      if (d.full && ((((uintptr_t)src | (uintptr_t)mc) & 15) == 0)) {
        constexpr int U = 4;  // (8 and 16 in flight: same 220 us at p = 4 -- the switch's rate)
        for (int s0 = lane_id; s0 < d.n; s0 += 32 * U) {
          float4 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (s0 + 32 * u < d.n) v[u] = ld16(src + 4 * (s0 + 32 * u));
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (s0 + 32 * u < d.n) mm_st16(mc + 4 * (s0 + 32 * u), v[u]);
        }
      } else {
        const int64_t j0 = d.e < 0 ? -d.e : 0;
        const int64_t j1 = min(4 * (int64_t)d.n, kp.numel[d.t] - d.e);
        for (int64_t j = j0 + lane_id; j < j1; j += 32) mm_st4(mc + j, ld4(src + j));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int q = 0; q < P; ++q)
        if (q != r)
          asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(
                           kp.flags[q] + flag_index(BAR_PROG, r, b)),
                       "r"(nv_flag_value(1))
                       : "memory");
    }
  } else if (threadIdx.x == 0) {
    ok = nv_wait(kp, r, kp.root, 1);
  }
  if (!__syncthreads_and(ok)) return;
  call_end(kp, r);
}

template <int OP>
const void* kernel_ptr(int algo, int p) {
  if (algo == ALGO_LOCAL) return (const void*)k_local_tma<OP>;
#define TC_CASE(PP)                                                                          \
  case PP:                                                                                   \
    if constexpr (OP != OP_EASGD)                                                            \
      if (algo == ALGO_NVLS) return (const void*)k_nvls<OP, PP>;                             \
    if (algo == ALGO_NVLS) return nullptr;                                                   \
    if (algo == ALGO_TWOSHOT_TMA) return (const void*)k_twoshot_tma<OP, PP>;                 \
    if (algo == ALGO_LL) return (const void*)k_ll<OP, PP, 2>;                                \
    return algo == ALGO_TWOSHOT ? (const void*)k_twoshot_pull<OP, PP, 2>                     \
                                : (const void*)k_oneshot<OP, PP, 2>;
  switch (p) {
    TC_CASE(2) TC_CASE(3) TC_CASE(4) TC_CASE(5) TC_CASE(6) TC_CASE(7) TC_CASE(8)
    default: return nullptr;
  }
#undef TC_CASE
}

}  // namespace
}  // namespace tc
