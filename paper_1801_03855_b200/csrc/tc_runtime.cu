// libtc host runtime: communicators, CUDA-IPC peer mapping of caller tensors (no copies), the
// hot-path entry points of include/tc.h and their argument checking.
//
// The only cross-process traffic happens at create/destroy time through the caller's bootstrap
// allgather ("all the workers call MPI_Init()" -- here torch.distributed/gloo).  A
// hot-path call is host validation + ONE kernel launch on the caller's stream.
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <vector>

#include "tc_internal.h"

using namespace tc;

namespace {

// cuMemGetAddressRange through the runtime's driver entry point (libcuda is not linked, so the
// library also loads on machines without a driver -- the CPU test box).
typedef int (*PFN_addr_range)(unsigned long long*, size_t*, unsigned long long);

cudaError_t alloc_base(const void* p, void** base) {
  static PFN_addr_range fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !f) return cudaErrorNotSupported;
    fn = (PFN_addr_range)f;
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (unsigned long long)(uintptr_t)p) != 0) return cudaErrorInvalidValue;
  *base = (void*)(uintptr_t)b;
  return cudaSuccess;
}

#define TC_CUDA(expr)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      if (std::getenv("TC_DEBUG"))                                                          \
        std::fprintf(stderr, "libtc: %s failed: %s (%s:%d)\n", #expr, cudaGetErrorString(e_), \
                     __FILE__, __LINE__);                                                   \
      return TC_ERR_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

struct BusyGuard {
  std::atomic<bool>& f;
  bool ok;
  explicit BusyGuard(std::atomic<bool>& b) : f(b) { ok = !f.exchange(true); }
  ~BusyGuard() {
    if (ok) f.store(false);
  }
};

unsigned long long env_timeout_ns() {
  const char* s = std::getenv("TC_TIMEOUT_MS");
  long long ms = s ? std::atoll(s) : 30000;
  if (ms <= 0) ms = 30000;
  return (unsigned long long)ms * 1000000ull;
}

tc_status alloc_comm_buffers(Comm& c, int r) {
  TC_CUDA(cudaMalloc((void**)&c.flags[r], kFlagWords * sizeof(uint32_t)));
  TC_CUDA(cudaMemset(c.flags[r], 0, kFlagWords * sizeof(uint32_t)));
  TC_CUDA(cudaMalloc((void**)&c.stage[r], 2 * kStageCapacity + kLLBytes));
  TC_CUDA(cudaMemset((char*)c.stage[r] + 2 * kStageCapacity, 0, kLLBytes));
  return TC_OK;
}

tc_status finish_comm(Comm& c) {
  TC_CUDA(cudaHostAlloc((void**)&c.h_err, sizeof(int), cudaHostAllocMapped));
  *c.h_err = 0;
  TC_CUDA(cudaHostGetDevicePointer((void**)&c.d_err, c.h_err, 0));
  TC_CUDA(cudaMalloc((void**)&c.d_state, sizeof(DevState) * kMaxRanks));
  TC_CUDA(cudaMemset(c.d_state, 0, sizeof(DevState) * kMaxRanks));
  TC_CUDA(cudaMalloc((void**)&c.d_flags, sizeof(uint32_t*) * kMaxRanks));
  TC_CUDA(cudaMalloc((void**)&c.d_stage, sizeof(float*) * kMaxRanks));
  TC_CUDA(cudaMemcpy(c.d_flags, c.flags.data(), sizeof(uint32_t*) * kMaxRanks,
                     cudaMemcpyHostToDevice));
  TC_CUDA(cudaMemcpy(c.d_stage, c.stage.data(), sizeof(float*) * kMaxRanks,
                     cudaMemcpyHostToDevice));
  int sms = 0;
  TC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
  c.num_sms = sms;
  c.timeout_ns = env_timeout_ns();
  return TC_OK;
}

// Map (or reuse) peer `peer`'s allocation exported as `h`.
tc_status map_peer(Comm& c, int peer, const cudaIpcMemHandle_t& h, void** out,
                   std::pair<int, std::string>* key_out) {
  std::pair<int, std::string> key(peer, std::string(h.reserved, sizeof(h.reserved)));
  auto it = c.ipc_cache.find(key);
  if (it == c.ipc_cache.end()) {
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      if (std::getenv("TC_DEBUG"))
        std::fprintf(stderr, "libtc: cudaIpcOpenMemHandle(peer %d): %s\n", peer,
                     cudaGetErrorString(e));
      return TC_ERR_CUDA;
    }
    it = c.ipc_cache.emplace(key, MappedBase{p, 0}).first;
  }
  it->second.refs++;
  *out = it->second.ptr;
  if (key_out) *key_out = key;
  return TC_OK;
}

void unmap_peer(Comm& c, const std::pair<int, std::string>& key) {
  auto it = c.ipc_cache.find(key);
  if (it == c.ipc_cache.end()) return;
  if (--it->second.refs == 0) {
    cudaIpcCloseMemHandle(it->second.ptr);
    c.ipc_cache.erase(it);
  }
}

tc_status comm_barrier(Comm& c) {
  if (c.emulated || c.nranks == 1) return TC_OK;
  int32_t one = 1, all[kMaxRanks];
  return bootstrap_allgather(c.ag, c.ag_ctx, c.nranks, &one, all, sizeof(one));
}

// Collective status agreement: every rank learns the worst status of all ranks.
tc_status agree(Comm& c, tc_status mine) {
  if (c.emulated || c.nranks == 1) return mine;
  int32_t s = (int32_t)mine, all[kMaxRanks];
  tc_status bs = bootstrap_allgather(c.ag, c.ag_ctx, c.nranks, &s, all, sizeof(s));
  if (bs != TC_OK) return bs;
  for (int r = 0; r < c.nranks; ++r)
    if (all[r] != TC_OK) return (tc_status)all[r];
  return TC_OK;
}

void free_group_device(Group& g) {
  cudaFree(g.d_ptrs);
  cudaFree(g.d_prefix);
  cudaFree(g.d_block_t);
  cudaFree(g.d_numel);
  cudaFree(g.d_vec_ok);
  cudaFree(g.d_shift);
  g.d_shift = nullptr;
  cudaFree(g.d_mc);
  g.d_mc = nullptr;
  cudaFree(g.d_tiles);
  g.d_tiles = nullptr;
  g.ntiles = 0;
  cudaFree(g.d_tiles2);
  g.d_tiles2 = nullptr;
  cudaFree(g.d_tiles_nv);
  g.d_tiles_nv = nullptr;
  g.tile2_off.clear();
  g.d_ptrs = nullptr;
  g.d_prefix = nullptr;
  g.d_block_t = nullptr;
  g.d_numel = nullptr;
  g.d_vec_ok = nullptr;
}

// The device slot grid: tensor t (common misalignment m_t elements on every rank) occupies
// ceil((n_t + m_t)/4) slots, its first slot holding elements [0, 4 - m_t).
tc_status build_device_grid(Group& g, const std::vector<uint8_t>& vec_ok) {
  const Plan& pl = g.plan;
  g.dev_prefix.assign((size_t)pl.T + 1, 0);
  for (int t = 0; t < pl.T; ++t) {
    const int64_t n = pl.numel[(size_t)t];
    const int64_t m = vec_ok[(size_t)t] ? g.shift[(size_t)t] : 0;
    if (!vec_ok[(size_t)t]) g.shift[(size_t)t] = 0;
    g.dev_prefix[(size_t)t + 1] = g.dev_prefix[(size_t)t] + (n > 0 ? (n + m + 3) / 4 : 0);
  }
  g.M = g.dev_prefix[(size_t)pl.T];
  return g.M >= (int64_t(1) << 31) ? TC_ERR_INVALID_ARG : TC_OK;
}

tc_status upload_group(Group& g, const std::vector<uint8_t>& vec_ok) {
  const Plan& pl = g.plan;
  tc_status gs = build_device_grid(g, vec_ok);
  if (gs != TC_OK) return gs;
  std::vector<int> prefix(g.dev_prefix.begin(), g.dev_prefix.end());
  // tensor of the first slot of every 128-slot block (largest t with prefix[t] <= slot)
  std::vector<int> block_t((size_t)((g.M + kPiece - 1) >> kPieceShift) + 1, 0);
  for (size_t j = 0, t = 0; j < block_t.size(); ++j) {
    const int64_t slot = (int64_t)j << kPieceShift;
    while (t + 1 < (size_t)pl.T && g.dev_prefix[t + 1] <= slot) ++t;
    block_t[j] = (int)t;
  }
  TC_CUDA(cudaMalloc((void**)&g.d_block_t, sizeof(int) * block_t.size()));
  TC_CUDA(cudaMemcpy(g.d_block_t, block_t.data(), sizeof(int) * block_t.size(),
                     cudaMemcpyHostToDevice));
  TC_CUDA(cudaMalloc((void**)&g.d_ptrs, sizeof(float*) * g.h_ptrs.size()));
  TC_CUDA(cudaMalloc((void**)&g.d_prefix, sizeof(int) * prefix.size()));
  TC_CUDA(cudaMalloc((void**)&g.d_numel, sizeof(int64_t) * pl.numel.size()));
  TC_CUDA(cudaMalloc((void**)&g.d_vec_ok, vec_ok.size()));
  TC_CUDA(cudaMemcpy(g.d_ptrs, g.h_ptrs.data(), sizeof(float*) * g.h_ptrs.size(),
                     cudaMemcpyHostToDevice));
  TC_CUDA(cudaMemcpy(g.d_prefix, prefix.data(), sizeof(int) * prefix.size(),
                     cudaMemcpyHostToDevice));
  TC_CUDA(cudaMemcpy(g.d_numel, pl.numel.data(), sizeof(int64_t) * pl.numel.size(),
                     cudaMemcpyHostToDevice));
  TC_CUDA(cudaMemcpy(g.d_vec_ok, vec_ok.data(), vec_ok.size(), cudaMemcpyHostToDevice));
  TC_CUDA(cudaMalloc((void**)&g.d_shift, g.shift.size()));
  TC_CUDA(cudaMemcpy(g.d_shift, g.shift.data(), g.shift.size(), cudaMemcpyHostToDevice));
  if (g.comm->nranks == 1) {
    // p = 1 TMA stream: tiles of <= kTileE elements inside one tensor, starting on the
    // tensor's first 16-B boundary (the head before it, and the last (n - head) % 4 elements,
    // are tiles of their own on the element path).  The other operands take the vector path
    // when they share the misalignment (checked per tile in the kernel).
    std::vector<int4> tiles;
    for (int t = 0; t < pl.T; ++t) {
      const int64_t n = pl.numel[(size_t)t];
      const int64_t head = std::min<int64_t>(n, (4 - g.shift[(size_t)t]) & 3);
      const int64_t full = head + ((n - head) & ~(int64_t)3);
      // {tensor, first element (low 32 bits), elements, first element (high 32 bits)}
      auto tile = [&](int64_t e, int64_t cnt) {
        tiles.push_back(make_int4(t, (int)(uint32_t)(e & 0xffffffff), (int)cnt, (int)(e >> 32)));
      };
      if (head > 0) tile(0, head);
      for (int64_t e = head; e < full; e += kTileE) tile(e, std::min<int64_t>(kTileE, full - e));
      if (full < n) tile(full, n - full);
    }
    if (tiles.size() >= (size_t)INT32_MAX) return TC_ERR_INVALID_ARG;
    g.ntiles = (int)tiles.size();
    if (g.ntiles) {
      TC_CUDA(cudaMalloc((void**)&g.d_tiles, sizeof(int4) * tiles.size()));
      TC_CUDA(cudaMemcpy(g.d_tiles, tiles.data(), sizeof(int4) * tiles.size(),
                         cudaMemcpyHostToDevice));
    }
  }
  if (g.comm->nranks > 1) {
    // TMA two-shot: each owner chunk [M q / p, M (q+1) / p) of the device grid cut into tiles
    // of <= kT2Slots slots inside one tensor.  A shifted tensor's partial first slot and a
    // partial last slot are one-slot tiles of their own (element path in the kernel).  NVLS-
    // eligible groups get a second table with smaller tiles (kNvSlots: finer published rounds).
    const int p = g.comm->nranks;
    auto build = [&](int64_t cap, std::vector<int>& off) {
      std::vector<int4> tiles;
      off.assign((size_t)p + 1, 0);
      int t = 0;
      for (int q = 0; q < p; ++q) {
        off[(size_t)q] = (int)tiles.size();
        const int64_t lo = g.M * q / p, hi = g.M * (q + 1) / p;
        while (t < pl.T && g.dev_prefix[(size_t)t + 1] <= lo) ++t;
        for (int u = t; u < pl.T && g.dev_prefix[(size_t)u] < hi; ++u) {
          const int64_t pre = g.dev_prefix[(size_t)u], end = g.dev_prefix[(size_t)u + 1];
          int64_t a = std::max(lo, pre);
          const int64_t b = std::min(hi, end);
          if (a >= b) continue;
          const int64_t m = g.shift[(size_t)u], n = pl.numel[(size_t)u];
          const int64_t first_full = pre + (m ? 1 : 0);
          const int64_t full_end = end - (((n + m) & 3) ? 1 : 0);
          if (a < first_full) tiles.push_back(make_int4(u, (int)a++, 1, 0));
          const int64_t vend = std::min(b, full_end);
          for (int64_t x = a; x < vend; x += cap)
            tiles.push_back(make_int4(u, (int)x, (int)std::min<int64_t>(cap, vend - x), 0));
          const int64_t rest = std::max(a, vend);
          if (b > rest) tiles.push_back(make_int4(u, (int)rest, (int)(b - rest), 0));
        }
      }
      off[(size_t)p] = (int)tiles.size();
      return tiles;
    };
    std::vector<int4> tiles = build(t2_slots(p), g.tile2_off);
    if (!tiles.empty()) {
      TC_CUDA(cudaMalloc((void**)&g.d_tiles2, sizeof(int4) * tiles.size()));
      TC_CUDA(cudaMemcpy(g.d_tiles2, tiles.data(), sizeof(int4) * tiles.size(),
                         cudaMemcpyHostToDevice));
    }
    if (!g.h_mc.empty()) {
      std::vector<int4> nt = build(kNvSlots, g.tile_nv_off);
      if (!nt.empty()) {
        TC_CUDA(cudaMalloc((void**)&g.d_tiles_nv, sizeof(int4) * nt.size()));
        TC_CUDA(cudaMemcpy(g.d_tiles_nv, nt.data(), sizeof(int4) * nt.size(),
                           cudaMemcpyHostToDevice));
      }
    }
  }
  if (!g.h_mc.empty()) {
    TC_CUDA(cudaMalloc((void**)&g.d_mc, sizeof(float*) * g.h_mc.size()));
    TC_CUDA(cudaMemcpy(g.d_mc, g.h_mc.data(), sizeof(float*) * g.h_mc.size(),
                       cudaMemcpyHostToDevice));
  }
  return TC_OK;
}

bool finite(float v) { return std::isfinite(v); }

// Grow the per-rank arena (two parity-selected staging chunks of `cap` slots each) to
// hold owner chunks of `need` slots.  Collective (called from tc_group_create on every rank).
tc_status grow_arena(Comm& c, int64_t need) {
  const int p = c.nranks;
  if (p == 1 || need <= c.arena_cap) return TC_OK;
  int64_t cap = std::max<int64_t>(need, (int64_t)1 << 16);
  cap = (cap + 4095) & ~(int64_t)4095;
  const size_t bytes = (size_t)2 * (size_t)cap * 16;
  TC_CUDA(cudaDeviceSynchronize());
  tc_status st = comm_barrier(c);  // no kernel on any rank still uses the old arenas
  if (st != TC_OK) return st;
  for (auto& k : c.arena_keys) unmap_peer(c, k);
  c.arena_keys.clear();
  for (int r = 0; r < p; ++r) {
    if (c.emulated || r == c.rank) cudaFree(c.arena[r]);
    c.arena[r] = nullptr;
  }
  st = TC_OK;
  const int lo = c.emulated ? 0 : c.rank, hi = c.emulated ? p : c.rank + 1;
  for (int r = lo; r < hi && st == TC_OK; ++r)
    if (cudaMalloc((void**)&c.arena[r], bytes) != cudaSuccess) st = TC_ERR_CUDA;
  if (!c.emulated) {
    struct H { int32_t status; cudaIpcMemHandle_t h; } mine{}, all[kMaxRanks];
    mine.status = st;
    if (st == TC_OK && cudaIpcGetMemHandle(&mine.h, c.arena[c.rank]) != cudaSuccess)
      mine.status = TC_ERR_CUDA;
    st = bootstrap_allgather(c.ag, c.ag_ctx, p, &mine, all, sizeof(H));
    for (int r = 0; r < p && st == TC_OK; ++r)
      if (all[r].status != TC_OK) st = (tc_status)all[r].status;
    for (int r = 0; r < p && st == TC_OK; ++r) {
      if (r == c.rank) continue;
      void* ptr = nullptr;
      std::pair<int, std::string> key;
      st = map_peer(c, r, all[r].h, &ptr, &key);
      if (st == TC_OK) {
        c.arena[r] = (float*)ptr;
        c.arena_keys.push_back(key);
      }
    }
    st = agree(c, st);
  }
  if (st == TC_OK) {
    if (!c.d_arena) TC_CUDA(cudaMalloc((void**)&c.d_arena, sizeof(float*) * kMaxRanks));
    TC_CUDA(cudaMemcpy(c.d_arena, c.arena.data(), sizeof(float*) * kMaxRanks,
                       cudaMemcpyHostToDevice));
    c.arena_cap = cap;
  } else {
    c.arena_cap = 0;
  }
  return st;
}

// ------------------------------------------------------------------ hot-path dispatcher
tc_status run_hot(int op, Group* ga, Group* gb, Group* gc, float scale, float lr, float mu,
                  float wd, float rescale, float alpha, cudaStream_t stream,
                  Group* gd = nullptr, int root = 0, const int* order = nullptr) {
  Comm& c = *ga->comm;
  BusyGuard busy(c.busy);
  if (!busy.ok) return TC_ERR_BUSY;
  if (*(volatile int*)c.h_err) return (tc_status)*(volatile int*)c.h_err;
  const Plan& pl = ga->plan;
  const int p = c.nranks;
  const int64_t Mdev = ga->M;   // slots of the (shifted) device grid
  if (Mdev == 0) return TC_OK;  // empty group: nothing to reduce (still collective-safe)
  KParams kp;
  std::memset(&kp, 0, sizeof(kp));
  kp.p = p;
  kp.rank0 = c.emulated ? 0 : c.rank;
  kp.T = pl.T;
  kp.M = (int)Mdev;
  kp.prefix = ga->d_prefix;
  kp.block_t = ga->d_block_t;
  kp.numel = ga->d_numel;
  kp.vec_ok = ga->d_vec_ok;
  kp.a = ga->d_ptrs;
  kp.b = gb ? gb->d_ptrs : nullptr;
  kp.c = gc ? gc->d_ptrs : nullptr;
  kp.d = gd ? gd->d_ptrs : nullptr;
  kp.root = root;
  for (int j = 0; j < kMaxRanks; ++j) kp.order[j] = order ? (j < p ? order[j] : 0) : j;
  kp.mc = ga->d_mc;
  kp.flags = c.d_flags;
  kp.stage = c.d_stage;
  kp.ll_cap = (int)(kLLBytes / 2 / 8 / p) & ~(size_t)3;
  kp.arena = c.d_arena;
  kp.chunk_cap = (int)c.arena_cap;
  kp.scale = scale;
  kp.lr = lr;
  kp.mu = mu;
  kp.wd = wd;
  kp.rescale = rescale;
  kp.alpha = alpha;
  kp.timeout_ns = c.timeout_ns;
  kp.err = c.d_err;
  kp.absent_rank = c.emulated ? c.absent_rank : -1;
  // The vector path is taken for a tensor only if it is 16-B aligned in every group involved.
  kp.vec_ok_b = gb ? gb->d_vec_ok : nullptr;
  kp.vec_ok_c = gc ? gc->d_vec_ok : nullptr;
  kp.shift = ga->d_shift;
  kp.shift_b = gb ? gb->d_shift : nullptr;
  kp.shift_c = gc ? gc->d_shift : nullptr;

  const int threads = c.tune_threads;
  // per-group CTA budget (tc_group_set_num_ctas), else the comm's tuning
  const int tune_ctas = ga->num_ctas > 0 ? ga->num_ctas : c.tune_ctas;
  const int64_t bytes = Mdev * 16;
  int algo;
  if (p == 1) {
    algo = ALGO_LOCAL;
  } else if (op == OP_BCAST) {
    // a copy, so the switch path is bit-exact.  Multicast-bound groups take it from p = 4: the
    // root's bytes leave it once (S at ~480 GB/s: ResNet-50 group 214.5 us at p = 4 vs 246 for
    // the scatter + allgather, whose root sends 2(p-1)/p S; at p = 2 it loses, 212 vs 165 us)
    const bool mc = ga->d_mc != nullptr &&
                    (c.algo_override == ALGO_NVLS || (c.algo_override == 0 && p >= 4));
    algo = mc ? ALGO_NVLS : ALGO_TWOSHOT_TMA;
    if (!mc && (Mdev + p - 1) / p + 1 > c.arena_cap) return TC_ERR_CUDA;
  } else if (op == OP_EASYNC) {  // implemented by the TMA two-shot only
    algo = ALGO_TWOSHOT_TMA;
    if ((Mdev + p - 1) / p + 1 > c.arena_cap) return TC_ERR_CUDA;
  } else if (op == OP_ESGD) {
    algo = ALGO_TWOSHOT_TMA;
    if ((Mdev + p - 1) / p + 1 > c.arena_cap) return TC_ERR_CUDA;
  } else {
    // One-shot moves (p-1)S per GPU against 2(p-1)/p S for two-shot but needs one barrier
    // less.  Measured crossover against the TMA two-shot (config-5 sweep): p = 2 one-shot
    // 22-23 us at 4 MiB (TMA 24-35), two-shot from 16 MiB; p = 3 ties at 4 MiB (27.1-28.4 vs
    // 27.5-32.1 us); p = 4 ties at 2 MiB (24.4-25.4 vs 24.7-25.5) and loses at 4 MiB (33.6-35.2
    // vs TMA 28.3-33.3 for 1..1024 tensors, profiles/r01_oneshot_limit_p4.jsonl).
    const int64_t auto_lim = p == 2 ? (int64_t)kStageCapacity
                           : p == 3 ? (int64_t)kStageCapacity / 2
                           : p == 4 ? (int64_t)kStageCapacity / 4 : kDefaultOneshotMax;
    int64_t lim = c.tune_oneshot < 0 ? auto_lim : c.tune_oneshot;
    if (lim > (int64_t)kStageCapacity) lim = (int64_t)kStageCapacity;
    // Automatic choice (measured on B200, config-5 sweep and ResNet-50 group):
    // TMA-staged two-shot (p = 4: 16/64/256 MiB in 58-67/176-184/635-650 us; LDG pull
    // 72/189/679, pushed 95/210/737, NCCL 70/186/685).  NVLS, when the caller allowed switch
    // reduction (tolerance contract) and the group is multicast-bound: it moves (1 + 1/p) S per
    // GPU each way instead of 2(p-1)/p S.  At p = 4 (ResNet-50 group) it ties the two-shot:
    // allreduce 257 vs 257 us, fused SGD 289 vs 274 us -- per-direction rates 497 / 442 GB/s
    // against 596 / 559 for the two-shot, so by bytes NVLS wins from p = 5 (allreduce: p > 4.0,
    // SGD: p > 4.4); not measurable beyond 4 GPUs here.
    const bool nvls_ok = ga->d_mc != nullptr && op != OP_EASGD;
    // Low-latency (LL): every element travels once to every peer as an 8-byte {value, epoch}
    // word and is awaited in local memory -- no barrier round trip (small groups only).
    // Measured crossover vs one-shot (config-5 sweep): LL wins up to 1 MiB at p = 2 (12.6 vs
    // 20.6 us), up to 256 KiB at p = 4 (1 MiB: 29 vs 23 us).  Limits compare the group's data
    // bytes; the buffers' capacities the padded slot grid.
    const int64_t data_bytes = pl.N * 4;
    const int64_t ll_cap = (int64_t)(kLLBytes / 2 / 8 / p) & ~(size_t)3;
    // Against the flat one-shot (one slot per thread, profiles/r02_latency_probe_flat.jsonl,
    // 1 / 161 tensors): p = 2 LL up to 1 MiB (1 MiB 12.6 / 12.2 us vs 13.7 / 15.4; 2 MiB 17.3 /
    // 21.4 vs 14.6 / 21.3); p = 3 up to 512 KiB (13.9 / 13.8 vs 13.8 / 15.8; 1 MiB 22.1 vs
    // 15.1); p = 4 up to 256 KiB (512 KiB 17.2 / 18.3 vs 14.5 / 16.4).
    const int64_t ll_auto = p == 2 ? kDefaultLLMax : p == 3 ? kDefaultLLMax / 2
                          : p == 4 ? kDefaultLLMax / 4 : kDefaultLLMax / 8;
    const int64_t ll_lim = c.tune_ll < 0 ? ll_auto : c.tune_ll;
    if (data_bytes <= ll_lim && 4 * Mdev <= ll_cap) algo = ALGO_LL;
    else if (data_bytes <= lim && bytes <= (int64_t)kStageCapacity) algo = ALGO_ONESHOT;
    else if (c.algo_override == ALGO_TWOSHOT_TMA) algo = ALGO_TWOSHOT_TMA;
    else if (c.algo_override == ALGO_TWOSHOT) algo = ALGO_TWOSHOT;
    else if (nvls_ok && (c.algo_override == ALGO_NVLS ||
                         (c.algo_override == 0 && c.allow_switch && p >= 5)))
      algo = ALGO_NVLS;
    // TMA-staged two-shot: ResNet-50 group p = 2 allreduce 188 / SGD step 197 us (LDG pull
    // 208 / 226, NCCL allreduce 219); p = 4 262 / 278 us (pull 289 / 301, NCCL 274-276).
    else algo = ALGO_TWOSHOT_TMA;
    if ((algo == ALGO_TWOSHOT || algo == ALGO_TWOSHOT_TMA) &&
        (Mdev + p - 1) / p + 1 > c.arena_cap)
      return TC_ERR_CUDA;
  }
  const int nlocal = c.emulated ? p : 1;
  int occ = max_ctas_per_sm(op, algo, p, threads);
  if (occ < 1) return TC_ERR_CUDA;
  int cap = c.num_sms * occ / nlocal;  // co-resident CTAs per rank
  if (cap < 1) cap = 1;
  const bool twoshot = algo == ALGO_TWOSHOT;
  int64_t work_slots = twoshot ? (Mdev + p - 1) / p : Mdev;
  int64_t want = (work_slots + threads - 1) / threads;
  int ctas;
  if (algo == ALGO_TWOSHOT_TMA || algo == ALGO_NVLS) {
    // bytes in flight come from the stage ring, not from threads: one CTA per SM at most
    // (NVLS walks its own table of smaller tiles)
    const std::vector<int>& off = algo == ALGO_NVLS ? ga->tile_nv_off : ga->tile2_off;
    const int tiles_r = off[1] - off[0];
    ctas = tune_ctas > 0 ? tune_ctas : c.num_sms;
    ctas = std::max(1, std::min(ctas, std::max(tiles_r, 1)));
    kp.tiles2 = algo == ALGO_NVLS ? ga->d_tiles_nv : ga->d_tiles2;
    for (int q = 0; q <= p; ++q) kp.tile2_off[q] = off[(size_t)q];
  } else if (algo == ALGO_LOCAL) {  // TMA stream
    ctas = std::min(ga->ntiles, tune_ctas > 0 ? std::min(tune_ctas, c.num_sms * occ)
                                                : c.num_sms * occ);
    kp.tiles = ga->d_tiles;
    kp.ntiles = ga->ntiles;
  } else if (twoshot && tune_ctas > 0) {
    ctas = tune_ctas;
  } else if (algo == ALGO_ONESHOT && want <= (int64_t)c.num_sms * occ / nlocal) {
    // one slot per thread (the kernel's flat path): every slot's p remote loads in flight at
    // once -- p = 4, 1 MiB: 16.9-18.6 us against 21.3-23.8 for pieces walked by warps
    ctas = (int)want;
  } else {
    ctas = (int)std::min<int64_t>(
        want, (int64_t)c.num_sms * ((algo == ALGO_ONESHOT || algo == ALGO_LL) ? 1 : occ));
  }
  if (algo != ALGO_LOCAL) {
    if (ctas > kMaxCtas) ctas = kMaxCtas;
    if (ctas > cap) ctas = cap;
  }
  if (ctas < 1) ctas = 1;
  if (c.prof && (int64_t)ctas * nlocal <= c.prof_slots) kp.prof = c.prof;
  kp.state = c.d_state;
  cudaError_t e = launch_hot(op, algo, kp, ctas, threads, nlocal, c.emulated && p > 1, stream);
  if (e != cudaSuccess) {
    if (std::getenv("TC_DEBUG"))
      std::fprintf(stderr, "libtc: launch failed: %s\n", cudaGetErrorString(e));
    return TC_ERR_CUDA;
  }
  c.last_algo = algo;
  c.last_ctas = ctas;
  c.last_threads = launch_threads(op, algo, p, threads);
  return TC_OK;
}

bool congruent(const Group* a, const Group* b) {
  return a->comm == b->comm && a->plan.T == b->plan.T && a->plan.hash == b->plan.hash &&
         a->plan.numel == b->plan.numel;
}

}  // namespace

extern "C" {

int tc_version(void) { return 100; }

const char* tc_status_string(tc_status s) {
  switch (s) {
    case TC_OK: return "TC_OK";
    case TC_ERR_INVALID_ARG: return "TC_ERR_INVALID_ARG";
    case TC_ERR_SHAPE_MISMATCH: return "TC_ERR_SHAPE_MISMATCH";
    case TC_ERR_NOT_SHAREABLE: return "TC_ERR_NOT_SHAREABLE";
    case TC_ERR_BUSY: return "TC_ERR_BUSY";
    case TC_ERR_TIMEOUT: return "TC_ERR_TIMEOUT";
    case TC_ERR_CUDA: return "TC_ERR_CUDA";
    case TC_ERR_BOOTSTRAP: return "TC_ERR_BOOTSTRAP";
    case TC_ERR_UNSUPPORTED: return "TC_ERR_UNSUPPORTED";
  }
  return "TC_ERR_UNKNOWN";
}

tc_status tc_comm_create(int rank, int nranks, int cuda_device, tc_allgather_fn ag, void* ag_ctx,
                         tc_comm** out) {
  if (!out) return TC_ERR_INVALID_ARG;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || cuda_device < 0) return TC_ERR_INVALID_ARG;
  if (nranks > kMaxRanks) return TC_ERR_UNSUPPORTED;
  if (nranks > 1 && !ag) return TC_ERR_INVALID_ARG;
  TC_CUDA(cudaSetDevice(cuda_device));
  tc_comm* h = new tc_comm;
  Comm& c = h->c;
  c.rank = rank;
  c.nranks = nranks;
  c.device = cuda_device;
  c.ag = ag;
  c.ag_ctx = ag_ctx;
  tc_status st = alloc_comm_buffers(c, rank);
  struct Hello {
    int32_t status;
    int32_t sms;
    cudaIpcMemHandle_t hflags, hstage;
  } mine{}, all[kMaxRanks];
  mine.status = st;
  if (st == TC_OK && nranks > 1) {
    if (cudaIpcGetMemHandle(&mine.hflags, c.flags[rank]) != cudaSuccess ||
        cudaIpcGetMemHandle(&mine.hstage, c.stage[rank]) != cudaSuccess)
      mine.status = TC_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&mine.sms, cudaDevAttrMultiProcessorCount, cuda_device);
  st = bootstrap_allgather(ag, ag_ctx, nranks, &mine, all, sizeof(Hello));
  if (st == TC_OK)
    for (int r = 0; r < nranks; ++r)
      if (all[r].status != TC_OK) st = (tc_status)all[r].status;
  if (st == TC_OK) {
    for (int r = 0; r < nranks && st == TC_OK; ++r) {
      if (r == rank) continue;
      void* pf = nullptr;
      void* ps = nullptr;
      st = map_peer(c, r, all[r].hflags, &pf, nullptr);
      if (st == TC_OK) st = map_peer(c, r, all[r].hstage, &ps, nullptr);
      c.flags[r] = (uint32_t*)pf;
      c.stage[r] = (float*)ps;
    }
    st = agree(c, st);
  }
  if (st == TC_OK) st = finish_comm(c);
  if (st == TC_OK) {
    int min_sms = all[0].sms;
    for (int r = 1; r < nranks; ++r) min_sms = std::min(min_sms, (int)all[r].sms);
    c.num_sms = min_sms;  // identical grid on every rank (per-CTA barrier pairing)
    *out = h;
    return TC_OK;
  }
  for (auto& kv : c.ipc_cache) cudaIpcCloseMemHandle(kv.second.ptr);
  cudaFree(c.flags[rank]);
  cudaFree(c.stage[rank]);
  delete h;
  return st;
}

tc_status tc_comm_create_emulated(int nranks, int cuda_device, tc_comm** out) {
  if (!out) return TC_ERR_INVALID_ARG;
  *out = nullptr;
  if (nranks < 1 || cuda_device < 0) return TC_ERR_INVALID_ARG;
  if (nranks > kMaxRanks) return TC_ERR_UNSUPPORTED;
  TC_CUDA(cudaSetDevice(cuda_device));
  tc_comm* h = new tc_comm;
  Comm& c = h->c;
  c.rank = -1;
  c.nranks = nranks;
  c.emulated = true;
  c.device = cuda_device;
  tc_status st = TC_OK;
  for (int r = 0; r < nranks && st == TC_OK; ++r) st = alloc_comm_buffers(c, r);
  if (st == TC_OK) st = finish_comm(c);
  if (st != TC_OK) {
    for (int r = 0; r < nranks; ++r) {
      cudaFree(c.flags[r]);
      cudaFree(c.stage[r]);
    }
    delete h;
    return st;
  }
  *out = h;
  return TC_OK;
}

tc_status tc_comm_set_tuning(tc_comm* comm, int num_ctas, int threads, int64_t oneshot_max) {
  if (!comm) return TC_ERR_INVALID_ARG;
  if (num_ctas < 0 || num_ctas > kMaxCtas) return TC_ERR_INVALID_ARG;
  if (threads != 0 && (threads < 64 || threads > 512 || threads % 32)) return TC_ERR_INVALID_ARG;
  if (oneshot_max < -1) return TC_ERR_INVALID_ARG;
  comm->c.tune_ctas = num_ctas;
  comm->c.tune_threads = threads ? threads : 512;
  comm->c.tune_oneshot = oneshot_max;
  return TC_OK;
}

tc_status tc_comm_set_ll_max(tc_comm* comm, int64_t bytes) {
  if (!comm || bytes < -1) return TC_ERR_INVALID_ARG;
  comm->c.tune_ll = bytes;
  return TC_OK;
}

tc_status tc_comm_set_algorithm(tc_comm* comm, int algo) {
  if (!comm || (algo != 0 && algo != ALGO_TWOSHOT && algo != ALGO_NVLS &&
                algo != ALGO_TWOSHOT_TMA))
    return TC_ERR_INVALID_ARG;
  comm->c.algo_override = algo;
  return TC_OK;
}

tc_status tc_comm_set_switch_reduction(tc_comm* comm, int allow) {
  if (!comm || (allow != 0 && allow != 1)) return TC_ERR_INVALID_ARG;
  comm->c.allow_switch = allow != 0;
  return TC_OK;
}

tc_status tc_group_set_num_ctas(tc_group* group, int num_ctas) {
  if (!group || num_ctas < 0 || num_ctas > kMaxCtas) return TC_ERR_INVALID_ARG;
  group->g.num_ctas = num_ctas;
  return TC_OK;
}

tc_status tc_comm_set_debug_busy(tc_comm* comm, int hold) {
  if (!comm) return TC_ERR_INVALID_ARG;
  comm->c.busy.store(hold != 0);
  return TC_OK;
}

tc_status tc_comm_set_timeout(tc_comm* comm, int64_t timeout_ms) {
  if (!comm || timeout_ms <= 0) return TC_ERR_INVALID_ARG;
  comm->c.timeout_ns = (unsigned long long)timeout_ms * 1000000ull;
  return TC_OK;
}

tc_status tc_comm_set_debug_absent_rank(tc_comm* comm, int absent_rank) {
  if (!comm || !comm->c.emulated || absent_rank < -1 || absent_rank >= comm->c.nranks)
    return TC_ERR_INVALID_ARG;
  comm->c.absent_rank = absent_rank;
  return TC_OK;
}

tc_status tc_comm_set_profile_buffer(tc_comm* comm, void* device_buffer, int64_t bytes) {
  if (!comm || bytes < 0 || (bytes > 0 && !device_buffer)) return TC_ERR_INVALID_ARG;
  comm->c.prof = (unsigned long long*)device_buffer;
  comm->c.prof_slots = bytes / (8 * sizeof(unsigned long long));
  return TC_OK;
}

tc_status tc_comm_async_error(tc_comm* comm) {
  if (!comm) return TC_ERR_INVALID_ARG;
  return (tc_status) * (volatile int*)comm->c.h_err;
}

int tc_comm_rank(const tc_comm* comm) { return comm ? comm->c.rank : -1; }
int tc_comm_nranks(const tc_comm* comm) { return comm ? comm->c.nranks : -1; }

tc_status tc_comm_last_launch(const tc_comm* comm, int* algo, int* ctas, int* threads) {
  if (!comm || !algo || !ctas || !threads) return TC_ERR_INVALID_ARG;
  *algo = comm->c.last_algo;
  *ctas = comm->c.last_ctas;
  *threads = comm->c.last_threads;
  return TC_OK;
}

tc_status tc_comm_destroy(tc_comm* comm) {
  if (!comm) return TC_ERR_INVALID_ARG;
  Comm& c = comm->c;
  if (c.live_groups != 0) return TC_ERR_INVALID_ARG;
  cudaSetDevice(c.device);
  cudaDeviceSynchronize();
  tc_status st = comm_barrier(c);
  for (auto& kv : c.ipc_cache) cudaIpcCloseMemHandle(kv.second.ptr);
  c.ipc_cache.clear();
  for (int r = 0; r < c.nranks; ++r) {
    if (c.emulated || r == c.rank) {
      cudaFree(c.flags[r]);
      cudaFree(c.stage[r]);
      cudaFree(c.arena[r]);
    }
  }
  free_all_sym(c);
  cudaFree(c.d_state);
  cudaFree(c.d_arena);
  cudaFree(c.d_flags);
  cudaFree(c.d_stage);
  cudaFreeHost(c.h_err);
  delete comm;
  return st;
}

tc_status tc_group_create(tc_comm* comm, int ntensors, void* const* ptrs, const int64_t* numels,
                          tc_group** out) {
  if (!out) return TC_ERR_INVALID_ARG;
  *out = nullptr;
  if (!comm) return TC_ERR_INVALID_ARG;
  Comm& c = comm->c;
  BusyGuard busy(c.busy);  // one collective call per comm at a time
  if (!busy.ok) return TC_ERR_BUSY;
  const int p = c.nranks;
  const int myrank = c.emulated ? 0 : c.rank;
  Plan plan;
  tc_status st = build_plan(myrank, p, ntensors, numels, plan);
  const int nlocal = c.emulated ? p : 1;
  if (st == TC_OK && !ptrs) st = TC_ERR_INVALID_ARG;
  if (st == TC_OK) {
    for (int l = 0; l < nlocal && st == TC_OK; ++l)
      for (int t = 0; t < ntensors; ++t) {
        const void* q = ptrs[(size_t)l * ntensors + t];
        if (numels[t] > 0 && (q == nullptr || ((uintptr_t)q & 3u))) {
          st = TC_ERR_INVALID_ARG;
          break;
        }
      }
  }
  cudaSetDevice(c.device);

  // Header exchange: status, T, hash, number of distinct allocations (real comms).
  std::vector<void*> bases;
  std::vector<int32_t> base_idx(st == TC_OK ? ntensors : 0, -1);
  std::vector<int64_t> offs(st == TC_OK ? ntensors : 0, 0);
  std::vector<cudaIpcMemHandle_t> handles;
  if (st == TC_OK && !c.emulated && p > 1) {
    for (int t = 0; t < ntensors && st == TC_OK; ++t) {
      if (numels[t] == 0) continue;
      int64_t soff = 0;
      const int si = find_sym(c, ptrs[t], (size_t)numels[t] * 4, &soff);
      if (si >= 0) {  // symmetric allocation: peers already map it; index encoded as -(2 + i)
        base_idx[t] = -(2 + si);
        offs[t] = soff;
        continue;
      }
      void* base = nullptr;
      if (alloc_base(ptrs[t], &base) != cudaSuccess) {
        st = TC_ERR_NOT_SHAREABLE;
        break;
      }
      int idx = -1;
      for (size_t i = 0; i < bases.size(); ++i)
        if (bases[i] == base) idx = (int)i;
      if (idx < 0) {
        cudaIpcMemHandle_t h;
        if (cudaIpcGetMemHandle(&h, base) != cudaSuccess) {
          cudaGetLastError();
          st = TC_ERR_NOT_SHAREABLE;
          break;
        }
        idx = (int)bases.size();
        bases.push_back(base);
        handles.push_back(h);
      }
      base_idx[t] = idx;
      offs[t] = (int64_t)((const char*)ptrs[t] - (const char*)base);
    }
  }
  struct Hdr { int32_t status, T; uint64_t hash; int32_t nbases, pad; } mine{}, all[kMaxRanks];
  mine.status = st;
  mine.T = ntensors;
  mine.hash = st == TC_OK ? plan.hash : 0;
  mine.nbases = (int32_t)bases.size();
  if (!c.emulated && p > 1) {
    tc_status bs = bootstrap_allgather(c.ag, c.ag_ctx, p, &mine, all, sizeof(Hdr));
    if (bs != TC_OK) return bs;
    for (int r = 0; r < p; ++r)
      if (all[r].status != TC_OK) return (tc_status)all[r].status;
    for (int r = 0; r < p; ++r)
      if (all[r].T != all[0].T || all[r].hash != all[0].hash) return TC_ERR_SHAPE_MISMATCH;
  } else if (st != TC_OK) {
    return st;
  }

  tc_group* h = new tc_group;
  Group& g = h->g;
  g.comm = &c;
  g.plan = std::move(plan);
  const int T = ntensors;
  g.h_ptrs.assign((size_t)p * T, nullptr);
  std::vector<uint8_t> vec_ok((size_t)T, 1);
  g.shift.assign((size_t)T, 0);
  // misalignment (elements past a 16-B boundary) of tensor t on rank r; a tensor keeps the vector
  // path iff every rank has the same misalignment (0xFF: empty tensor, no constraint)
  auto note_mis = [&](int t, int r, uint8_t mis) {
    if (mis == 0xFF) return;
    if (r == 0 || g.shift[(size_t)t] == 0xFE) g.shift[(size_t)t] = mis;
    else if (g.shift[(size_t)t] != mis) vec_ok[(size_t)t] = 0;
  };
  for (int t = 0; t < T; ++t) g.shift[(size_t)t] = 0xFE;  // unset

  if (c.emulated || p == 1) {
    for (int l = 0; l < nlocal; ++l)
      for (int t = 0; t < T; ++t) {
        float* q = (float*)ptrs[(size_t)l * T + t];
        g.h_ptrs[(size_t)l * T + t] = q;
        note_mis(t, l == 0 ? 0 : 1, numels[t] ? (uint8_t)(((uintptr_t)q & 15u) >> 2) : 0xFF);
      }
  } else {
    // Payload exchange: handles, per-tensor (base index, offset), alignment bits.
    int maxb = 0;
    for (int r = 0; r < p; ++r) maxb = std::max(maxb, (int)all[r].nbases);
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    const size_t bytes = (size_t)maxb * hb + (size_t)T * (sizeof(int32_t) + sizeof(int64_t) + 1);
    std::vector<char> send(bytes, 0), recv(bytes * p);
    char* w = send.data();
    for (size_t i = 0; i < handles.size(); ++i) std::memcpy(w + i * hb, &handles[i], hb);
    w += (size_t)maxb * hb;
    std::memcpy(w, base_idx.data(), sizeof(int32_t) * T);
    w += sizeof(int32_t) * T;
    std::memcpy(w, offs.data(), sizeof(int64_t) * T);
    w += sizeof(int64_t) * T;
    for (int t = 0; t < T; ++t)
      w[t] = numels[t] ? (char)(((uintptr_t)ptrs[t] & 15u) >> 2) : (char)0xFF;
    st = bootstrap_allgather(c.ag, c.ag_ctx, p, send.data(), recv.data(), bytes);
    if (st != TC_OK) {
      delete h;
      return st;
    }
    // NVLS eligibility: every tensor in the same symmetric multicast allocation at the same
    // offset on every rank (then its multicast address is mc + offset everywhere).
    bool nvls = true;
    std::vector<float*> mc_ptrs((size_t)T, nullptr);
    for (int t = 0; t < T; ++t) {
      if (numels[t] == 0) continue;
      int32_t bi0 = 0;
      int64_t off0 = 0;
      for (int r = 0; r < p; ++r) {
        const char* rd = recv.data() + (size_t)r * bytes;
        int32_t bi;
        int64_t off;
        std::memcpy(&bi, rd + (size_t)maxb * hb + sizeof(int32_t) * t, sizeof(bi));
        std::memcpy(&off, rd + (size_t)maxb * hb + sizeof(int32_t) * T + sizeof(int64_t) * t,
                    sizeof(off));
        if (r == 0) {
          bi0 = bi;
          off0 = off;
        }
        if (bi > -2 || bi != bi0 || off != off0) nvls = false;
      }
      if (nvls) {
        const SymAlloc& sa = c.sym[(size_t)(-(bi0 + 2))];
        if (!sa.multicast) nvls = false;
        else mc_ptrs[t] = (float*)((char*)sa.mc + off0);
      }
    }
    if (nvls) g.h_mc = mc_ptrs;
    for (int r = 0; r < p && st == TC_OK; ++r) {
      const char* rd = recv.data() + (size_t)r * bytes;
      const int32_t* bi = (const int32_t*)(rd + (size_t)maxb * hb);
      int64_t off_r[1];
      const char* offp = rd + (size_t)maxb * hb + sizeof(int32_t) * T;
      const char* al = offp + sizeof(int64_t) * T;
      std::vector<void*> rbases(all[r].nbases, nullptr);
      if (r != c.rank) {
        for (int i = 0; i < all[r].nbases && st == TC_OK; ++i) {
          cudaIpcMemHandle_t hh;
          std::memcpy(&hh, rd + (size_t)i * hb, hb);
          std::pair<int, std::string> key;
          st = map_peer(c, r, hh, &rbases[i], &key);
          if (st == TC_OK) g.mapped_keys.push_back(key);
        }
      }
      for (int t = 0; t < T && st == TC_OK; ++t) {
        note_mis(t, r == 0 ? 0 : 1, (uint8_t)al[t]);
        if (numels[t] == 0) continue;
        if (r == c.rank) {
          g.h_ptrs[(size_t)r * T + t] = (float*)ptrs[t];
        } else {
          std::memcpy(off_r, offp + sizeof(int64_t) * t, sizeof(int64_t));
          int32_t bit;
          std::memcpy(&bit, &bi[t], sizeof(bit));
          if (bit <= -2)
            g.h_ptrs[(size_t)r * T + t] =
                (float*)((char*)c.sym[(size_t)(-(bit + 2))].uc[r] + off_r[0]);
          else
            g.h_ptrs[(size_t)r * T + t] = (float*)((char*)rbases[bit] + off_r[0]);
        }
      }
    }
    st = agree(c, st);
    if (st != TC_OK) {
      for (auto& k : g.mapped_keys) unmap_peer(c, k);
      delete h;
      return st;
    }
  }
  for (int t = 0; t < T; ++t)
    if (g.shift[(size_t)t] > 3) g.shift[(size_t)t] = 0;  // empty on every rank
  st = upload_group(g, vec_ok);
  if (!c.emulated && p > 1) st = agree(c, st);
  if (st == TC_OK) st = grow_arena(c, (g.M + p - 1) / p + 1);
  if (st != TC_OK) {
    free_group_device(g);
    for (auto& k : g.mapped_keys) unmap_peer(c, k);
    delete h;
    return st;
  }
  if (!c.emulated && p > 1) {
    // pin the symmetric allocations the tensors live in until the group is destroyed
    for (int t = 0; t < T; ++t) {
      if (base_idx[t] > -2) continue;
      void* b = c.sym[(size_t)(-(base_idx[t] + 2))].uc[c.rank];
      if (std::find(g.sym_bases.begin(), g.sym_bases.end(), b) == g.sym_bases.end())
        g.sym_bases.push_back(b);
    }
    for (void* b : g.sym_bases) sym_ref(c, b, +1);
  }
  c.live_groups++;
  *out = h;
  return TC_OK;
}

tc_status tc_group_destroy(tc_group* group) {
  if (!group) return TC_ERR_INVALID_ARG;
  Group& g = group->g;
  Comm& c = *g.comm;
  BusyGuard busy(c.busy);
  if (!busy.ok) return TC_ERR_BUSY;
  cudaSetDevice(c.device);
  cudaDeviceSynchronize();
  tc_status st = comm_barrier(c);  // no peer kernel can still read our tensors
  for (auto& k : g.mapped_keys) unmap_peer(c, k);
  for (void* b : g.sym_bases) sym_ref(c, b, -1);
  free_group_device(g);
  c.live_groups--;
  delete group;
  return st;
}

tc_status tc_allreduce(tc_group* x, float scale, void* stream) {
  if (!x || !finite(scale)) return TC_ERR_INVALID_ARG;
  return run_hot(OP_ALLREDUCE, &x->g, nullptr, nullptr, scale, 0, 0, 0, 0, 0,
                 (cudaStream_t)stream);
}

tc_status tc_sgd_step(tc_group* w, tc_group* g, tc_group* dw, float lr, float momentum, float wd,
                      float rescale, void* stream) {
  if (!w || !g || !dw) return TC_ERR_INVALID_ARG;
  if (!finite(lr) || !finite(momentum) || !finite(wd) || !finite(rescale))
    return TC_ERR_INVALID_ARG;
  if (!congruent(&g->g, &w->g) || !congruent(&g->g, &dw->g)) return TC_ERR_SHAPE_MISMATCH;
  return run_hot(OP_SGD, &g->g, &w->g, &dw->g, 1.0f, lr, momentum, wd, rescale, 0,
                 (cudaStream_t)stream);
}

tc_status tc_esgd_step(tc_group* x, tc_group* center, tc_group* g, tc_group* dw, float alpha,
                       float lr, float momentum, float wd, float rescale, void* stream) {
  if (!x || !center || !g || !dw) return TC_ERR_INVALID_ARG;
  if (!finite(alpha) || alpha < 0.f || alpha > 1.f || !finite(lr) || !finite(momentum) ||
      !finite(wd) || !finite(rescale))
    return TC_ERR_INVALID_ARG;
  if (!congruent(&x->g, &center->g) || !congruent(&x->g, &g->g) || !congruent(&x->g, &dw->g))
    return TC_ERR_SHAPE_MISMATCH;
  return run_hot(OP_ESGD, &x->g, &center->g, &dw->g, 1.0f, lr, momentum, wd, rescale, alpha,
                 (cudaStream_t)stream, &g->g);
}

tc_status tc_broadcast(tc_group* x, int root, void* stream) {
  if (!x || root < 0 || root >= x->g.comm->nranks) return TC_ERR_INVALID_ARG;
  if (x->g.comm->nranks == 1) return TC_OK;  // the root's tensors are the result
  return run_hot(OP_BCAST, &x->g, nullptr, nullptr, 1.0f, 0, 0, 0, 0, 0, (cudaStream_t)stream,
                 nullptr, root);
}

tc_status tc_easgd_async_update(tc_group* x, tc_group* center, float alpha, const int* order,
                                void* stream) {
  if (!x || !center || !finite(alpha) || alpha < 0.f || alpha > 1.f) return TC_ERR_INVALID_ARG;
  if (!congruent(&x->g, &center->g)) return TC_ERR_SHAPE_MISMATCH;
  const int p = x->g.comm->nranks;
  int ord[kMaxRanks];
  bool seen[kMaxRanks] = {};
  for (int j = 0; j < p; ++j) {
    ord[j] = order ? order[j] : j;
    if (ord[j] < 0 || ord[j] >= p || seen[ord[j]]) return TC_ERR_INVALID_ARG;
    seen[ord[j]] = true;
  }
  if (p == 1)  // one arrival: Eqs. elastic1/elastic2 exactly (the local elastic stream)
    return run_hot(OP_EASGD, &x->g, &center->g, nullptr, 1.0f, 0, 0, 0, 0, alpha,
                   (cudaStream_t)stream);
  return run_hot(OP_EASYNC, &x->g, &center->g, nullptr, 1.0f, 0, 0, 0, 0, alpha,
                 (cudaStream_t)stream, nullptr, 0, ord);
}

tc_status tc_easgd_update(tc_group* x, tc_group* center, float alpha, void* stream) {
  if (!x || !center || !finite(alpha) || alpha < 0.f || alpha > 1.f) return TC_ERR_INVALID_ARG;
  if (!congruent(&x->g, &center->g)) return TC_ERR_SHAPE_MISMATCH;
  return run_hot(OP_EASGD, &x->g, &center->g, nullptr, 1.0f, 0, 0, 0, 0, alpha,
                 (cudaStream_t)stream);
}

}  // extern "C"
