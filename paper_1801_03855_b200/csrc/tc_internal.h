// Internal structures of libtc shared by the host runtime (tc_runtime.cu) and the kernels
// (tc_kernels.cu).  Not part of the ABI.
#pragma once

#include <cstdint>
#include <cstddef>
#include <vector>
#include <map>
#include <atomic>
#include <string>
#include <array>

#include <cuda_runtime.h>

#include "../../include/tc.h"

namespace tc {

constexpr int kMaxRanks = TC_MAX_RANKS;
constexpr int kMaxCtas = 1024;                 // per barrier and source rank
constexpr int kNumBarriers = 3;                // entry, mid, NVLS progress
constexpr size_t kFlagWords = (size_t)kNumBarriers * kMaxRanks * kMaxCtas;
constexpr size_t kStageCapacity = 8u << 20;    // one-shot staging bytes per parity
constexpr size_t kLLBytes = 16u << 20;         // low-latency receive buffers (after staging)
constexpr int64_t kDefaultLLMax = 1 << 20;
constexpr int64_t kDefaultOneshotMax = 256 << 10;
constexpr int kPieceShift = 7;                 // work piece = 128 slots = 2 KiB per operand
constexpr int kPiece = 1 << kPieceShift;
// p = 1 TMA stream (k_local_tma): tiles of up to kTileE elements inside one tensor, kTmaStages
// x 3 tiles of shared-memory stages (tc_kernels.cuh local_stages), one producer warp +
// kTmaConsumerWarps.
#ifndef TC_TILE_E
#define TC_TILE_E 2048
#endif
#ifndef TC_TMA_STAGES
#define TC_TMA_STAGES 4
#endif
#ifndef TC_TMA_CW
#define TC_TMA_CW 8
#endif
constexpr int kTileE = TC_TILE_E;
constexpr int kTmaStages = TC_TMA_STAGES;
constexpr int kTmaConsumerWarps = TC_TMA_CW;
constexpr int kTmaThreads = 32 * (1 + kTmaConsumerWarps);
// Two-shot, TMA-staged (k_twoshot_tma): owner-chunk tiles of <= kT2Slots slots inside one
// tensor; each stage holds every operand of one tile; as many stages as fit kT2SmemCap.
#ifndef TC_T2_SLOTS
#define TC_T2_SLOTS 512
#endif
#ifndef TC_T2_SMEM
#define TC_T2_SMEM (192 * 1024)
#endif
constexpr int kT2Slots = TC_T2_SLOTS;
// p = 2 moves half the group per phase through one peer: 1024-slot tiles (16 KiB per operand)
// measured faster there (allreduce 172 vs 175 us, fused step 173 vs 185 us); 512 elsewhere
constexpr int t2_slots(int p) { return p == 2 ? 2 * kT2Slots : kT2Slots; }
constexpr int kT2SmemCap = TC_T2_SMEM;
// The fused SGD step runs faster with fewer bytes in flight per SM (tools/algo_bench.py, ring
// caps 128 / 160 / 192 KiB: p = 4 step 268.5-269.3 / 268.4-269.4 / 274.5-276.4 us, p = 2
// 188.3-188.4 / 188.3-188.4 / 191.4-192.5; allreduce and EASGD flat within 1 us;
// profiles/r02_ring_p24.txt): 160 KiB keeps two stages at p = 8
#ifndef TC_T2_SMEM_SGD
#define TC_T2_SMEM_SGD (160 * 1024)
#endif
#ifndef TC_T2_SMEM_EL
#define TC_T2_SMEM_EL (192 * 1024)   // elastic ops (EASGD, fused elastic + SGD, async EASGD)
#endif
constexpr int t2_cap(int op) {
  return op == 1 ? TC_T2_SMEM_SGD : (op == 2 || op == 3 || op == 5) ? TC_T2_SMEM_EL : kT2SmemCap;
}
constexpr int kT2MaxStages = 16;
#ifndef TC_T2_CW
#define TC_T2_CW 8
#endif
#ifndef TC_T2_U
#define TC_T2_U 1
#endif
constexpr int kT2ConsumerWarps = TC_T2_CW;
constexpr int kT2Unroll = TC_T2_U;
constexpr int kT2Threads = 32 * (1 + kT2ConsumerWarps);
// operands per stage: reduce-scatter p sources (+ w, dw for SGD; + center for EASGD);
// allgather the staged value (+ w, dw for SGD; + x, center for EASGD)
// (ESGD, NEXT row f2: + w (= x), center, dw and the local gradient g)
constexpr int t2_ops(int op, int p) {
  if (op == 4) return 1;  // broadcast: the root's copy, then the owner's staged chunk
  if (op == 5) return p + 1;  // async EASGD: every client's x + the center; then the center
  const int rs = p + (op == 1 ? 2 : op == 2 ? 1 : op == 3 ? 3 : 0);
  const int ag = 1 + (op == 0 ? 0 : op == 3 ? 4 : 2);
  return rs > ag ? rs : ag;
}
constexpr int t2_stages(int op, int p) {
  const int n = t2_cap(op) / (t2_ops(op, p) * t2_slots(p) * 16);
  return n > kT2MaxStages ? kT2MaxStages : n;
}
constexpr int t2_smem(int op, int p) {
  return t2_stages(op, p) * t2_ops(op, p) * t2_slots(p) * 16;
}

constexpr int kNvlsThreads = 512;              // NVLS: 16 warps (reduction / signal / epilogue)
#ifndef TC_NV_SLOTS
#define TC_NV_SLOTS 512
#endif
constexpr int kNvSlots = TC_NV_SLOTS;           // NVLS tile: <= 512 slots = 8 KiB per operand
enum Barrier { BAR_ENTRY = 0, BAR_MID = 1, BAR_PROG = 2 };  // PROG: NVLS round progress
enum Op { OP_ALLREDUCE = 0, OP_SGD = 1, OP_EASGD = 2, OP_ESGD = 3, OP_BCAST = 4, OP_EASYNC = 5 };
// p = 1 TMA stream: operands per stage -- g (SGD: + w, dw), x + center (EASGD, async EASGD),
// x, center, dw, g (fused elastic + SGD) -- and stages: the ring holds kTmaStages x 3 tiles
// (96 KiB, two CTAs per SM) whatever the count, so every op keeps the SGD step's bytes in flight
// (allreduce 12 stages, EASGD 6, SGD 4, fused elastic + SGD 3).  tc_kernels.cuh checks the
// counts against the kernels' operand needs.
constexpr int local_ops(int op) {
  return op == OP_SGD ? 3 : (op == OP_EASGD || op == OP_EASYNC) ? 2 : op == OP_ESGD ? 4 : 1;
}
constexpr int kTmaMaxStages = 12;
constexpr int local_stages(int na) {
  return kTmaStages * 3 / na < kTmaMaxStages ? kTmaStages * 3 / na : kTmaMaxStages;
}
constexpr int local_smem(int op) { return local_stages(local_ops(op)) * local_ops(op) * kTileE * 4; }
enum Algo {
  ALGO_LOCAL = 0,
  ALGO_TWOSHOT = 1,
  ALGO_ONESHOT = 2,
  // 3 (register push two-shot) and 7 (TMA two-shot with claimed tiles): removed in round 2,
  // measured never faster than 6
  ALGO_NVLS = 4,
  ALGO_LL = 5,
  ALGO_TWOSHOT_TMA = 6,
};

// ---------------------------------------------------------------- A1 descriptor (host)
struct Plan {
  int rank = 0, nranks = 1, T = 0;
  std::vector<int64_t> numel;        // [T]
  std::vector<int64_t> slot_prefix;  // [T+1]
  int64_t N = 0, M = 0;
  uint64_t hash = 0;
  struct Segment { int tensor, owner; int64_t lo, hi; };
  std::vector<Segment> segments;
  int64_t owner_lo(int r) const { return M * r / nranks; }
  int64_t owner_hi(int r) const { return M * (r + 1) / nranks; }
};

struct Comm;
int find_sym(const Comm& c, const void* p, size_t bytes, int64_t* offset);
void sym_ref(Comm& c, const void* base, int delta);
bool multicast_supported(int device);
void free_all_sym(Comm& c);

tc_status build_plan(int rank, int nranks, int ntensors, const int64_t* numels, Plan& out);
uint64_t plan_hash(int ntensors, const int64_t* numels);
// Collective allgather through the caller's callback; returns TC_ERR_BOOTSTRAP on failure.
tc_status bootstrap_allgather(tc_allgather_fn ag, void* ctx, int nranks, const void* send,
                              void* recv, size_t bytes);

// ---------------------------------------------------------------- kernel parameters
// Per-rank device state of a comm: the epoch of the last completed call and the count of CTAs
// that finished the current one (the last one advances the epoch).
struct DevState {
  uint32_t epoch;
  uint32_t done;
  uint32_t pad;
};

// Passed by value to every hot-path kernel.  Tables are device arrays.
struct KParams {
  int p;                 // ranks in the comm
  int rank0;             // comm rank of blockIdx.y == 0
  int T;
  int M;                 // total 16-B slots
  const int* prefix;     // [T+1] slot prefix
  const int* block_t;    // [ceil(M/128)] tensor holding the first slot of each 128-slot block
  const int64_t* numel;  // [T]
  const uint8_t* vec_ok; // [T] primary group 16-B aligned on every rank
  const uint8_t* vec_ok_b; // [T] same for group b (nullptr if unused)
  const uint8_t* vec_ok_c; // [T] same for group c (nullptr if unused)
  const uint8_t* shift;    // [T] slot-grid shift (elements past a 16-B boundary) of group a
  const uint8_t* shift_b;  // [T] same for group b / c (a vector path needs equal shifts)
  const uint8_t* shift_c;
  float* const* a;       // [p*T] primary group: x (allreduce, easgd) or g (sgd)
  float* const* b;       // [p*T] w (sgd) or center (easgd)
  float* const* c;       // [p*T] dw (sgd, esgd)
  float* const* d;       // [p*T] this rank's gradient (esgd), else nullptr
  float* const* mc;      // [T] multicast addresses of the primary group (NVLS), or nullptr
  uint32_t* const* flags;// [p] flag buffers (peer-mapped)
  float* const* stage;   // [p] one-shot staging (+ low-latency buffers), peer-mapped
  int ll_cap;            // low-latency elements per source per parity
  float* const* arena;   // [p] per-rank arena: staging chunk x2 (parity)
  int chunk_cap;         // slots per arena region (>= the largest owner chunk)
  DevState* state;       // [p] device-side call epochs (this process's ranks are valid)
  float scale, lr, mu, wd, rescale, alpha;
  int root;              // broadcast root
  int order[kMaxRanks];  // async EASGD: client arrival order (a permutation of 0..p-1)
  unsigned long long timeout_ns;
  int* err;              // host-mapped sticky error word
  int absent_rank;       // fault injection (emulated only), -1 off
  unsigned long long* prof; // optional per-CTA phase timestamps [nlocal*ctas][8] (ns)
  const int4* tiles;     // p = 1 TMA stream: {tensor, first element lo32, elements, first element hi32}
  int ntiles;
  const int4* tiles2;    // p >= 2 TMA two-shot: {tensor, first slot, slots, 0} per tile,
  int tile2_off[kMaxRanks + 1];  // owner q's tiles: [tile2_off[q], tile2_off[q + 1])
};

// Kernel launchers (tc_kernels.cu).
cudaError_t launch_hot(int op, int algo, const KParams& kp, int ctas, int threads, int nlocal,
                       bool cooperative, cudaStream_t stream);
int max_ctas_per_sm(int op, int algo, int p, int threads);
int launch_threads(int op, int algo, int p, int threads);

// ---------------------------------------------------------------- runtime objects
// One symmetric allocation (tc_mem_alloc): every rank's physical memory mapped locally (uc[r]),
// plus the multicast mapping when NVSwitch multicast is available.
struct SymAlloc {
  size_t size = 0;
  int device = 0;
  bool multicast = false;
  uint64_t phys[kMaxRanks] = {};
  void* uc[kMaxRanks] = {};
  uint64_t mc_handle = 0;
  void* mc = nullptr;
  int refs = 0;          // live groups with tensors in this allocation (tc_mem_free refuses)
};

struct MappedBase {
  void* ptr = nullptr;
  int refs = 0;
};

struct Comm {
  int rank = 0;            // -1 when emulated
  int nranks = 1;
  bool emulated = false;
  int device = 0;
  int num_sms = 148;
  tc_allgather_fn ag = nullptr;
  void* ag_ctx = nullptr;
  // per-rank buffers: own (index = rank) allocated here, peers IPC-mapped.
  std::array<uint32_t*, kMaxRanks> flags{};
  std::array<float*, kMaxRanks> stage{};
  uint32_t** d_flags = nullptr;   // device table [p]
  float** d_stage = nullptr;      // device table [p]
  int* h_err = nullptr;           // host-mapped
  int* d_err = nullptr;
  DevState* d_state = nullptr;    // [kMaxRanks] device-side epochs
  std::array<float*, kMaxRanks> arena{};
  float** d_arena = nullptr;      // device table [p]
  int64_t arena_cap = 0;          // slots per region
  std::vector<std::pair<int, std::string>> arena_keys;  // peer arena mappings held
  int algo_override = 0;          // 0 auto, else an Algo
  bool allow_switch = false;      // automatic choice may use NVLS (fp32 sums in the switch)
  int tune_ctas = 0, tune_threads = 512;
  int64_t tune_oneshot = -1;
  int64_t tune_ll = -1;
  unsigned long long timeout_ns = 30ull * 1000 * 1000 * 1000;
  int absent_rank = -1;
  unsigned long long* prof = nullptr;
  int64_t prof_slots = 0;
  int last_algo = -1, last_ctas = 0, last_threads = 0;
  std::atomic<bool> busy{false};
  int live_groups = 0;
  std::vector<SymAlloc> sym;      // symmetric allocations, in creation order (same on all ranks)
  // IPC mapping cache: (peer, handle bytes) -> mapping
  std::map<std::pair<int, std::string>, MappedBase> ipc_cache;
};

struct Group {
  Comm* comm = nullptr;
  Plan plan;
  std::vector<float*> h_ptrs;    // [p*T] (peer-mapped pointers for real comms)
  float** d_ptrs = nullptr;      // device copy
  int* d_prefix = nullptr;
  int* d_block_t = nullptr;
  int64_t* d_numel = nullptr;
  uint8_t* d_vec_ok = nullptr;
  uint8_t* d_shift = nullptr;
  std::vector<uint8_t> shift;    // [T] common misalignment in elements (0 if ranks differ)
  std::vector<int64_t> dev_prefix;  // [T+1] slot prefix of the shifted grid
  int64_t M = 0;                 // slots of the shifted grid
  std::vector<std::pair<int, std::string>> mapped_keys;  // ipc_cache keys held
  std::vector<float*> h_mc;      // [T] multicast addresses (NVLS-eligible groups only)
  float** d_mc = nullptr;
  int4* d_tiles = nullptr;       // p = 1: tile table of the TMA stream (k_local_tma)
  int ntiles = 0;
  int4* d_tiles2 = nullptr;      // p >= 2: owner-chunk tiles of the TMA two-shot
  std::vector<int> tile2_off;    // [p + 1]
  int4* d_tiles_nv = nullptr;    // NVLS-eligible groups: owner-chunk tiles of <= kNvSlots slots
  std::vector<int> tile_nv_off;  // [p + 1]
  std::vector<void*> sym_bases;  // symmetric allocations (this rank's base) the group uses
  int num_ctas = 0;              // per-group CTA budget (0 = the comm's tuning)
};

}  // namespace tc

struct tc_plan { tc::Plan p; };
struct tc_comm { tc::Comm c; };
struct tc_group { tc::Group g; };
