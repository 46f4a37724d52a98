// A1: the tensor-group descriptor (host only; no CUDA calls).
//
// PAPER.md:325-326 (§6.1) defines a "tensor" as a group of vectors operated on as one object,
// and P:331 (§6.2) partitions "the buffer from each process ... into nearly equal parts".
// Reading R2: the partition is over 16-byte slots of 4 fp32 elements, so every
// owner chunk starts on a 16-B boundary inside its tensor and the kernels can move 16-B
// vectors.  Nothing is copied: the flat index space is a table of (tensor, slot) ranges over
// the caller's own allocations.
#include <cstring>
#include <vector>

#include "tc_internal.h"

namespace tc {

uint64_t plan_hash(int ntensors, const int64_t* numels) {
  // FNV-1a over (T, n_0 .. n_{T-1}); congruence check across ranks and between groups.
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= (v >> (8 * i)) & 0xff;
      h *= 1099511628211ull;
    }
  };
  mix((uint64_t)ntensors);
  for (int t = 0; t < ntensors; ++t) mix((uint64_t)numels[t]);
  return h;
}

tc_status build_plan(int rank, int nranks, int ntensors, const int64_t* numels, Plan& out) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return TC_ERR_INVALID_ARG;
  if (nranks > kMaxRanks) return TC_ERR_UNSUPPORTED;
  if (ntensors < 1 || numels == nullptr) return TC_ERR_INVALID_ARG;
  Plan p;
  p.rank = rank;
  p.nranks = nranks;
  p.T = ntensors;
  p.numel.assign(numels, numels + ntensors);
  p.slot_prefix.resize((size_t)ntensors + 1);
  p.slot_prefix[0] = 0;
  for (int t = 0; t < ntensors; ++t) {
    if (numels[t] < 0) return TC_ERR_INVALID_ARG;
    p.N += numels[t];
    p.slot_prefix[t + 1] = p.slot_prefix[t] + (numels[t] + 3) / 4;
  }
  p.M = p.slot_prefix[ntensors];
  if (p.M >= (int64_t(1) << 31)) return TC_ERR_INVALID_ARG;  // kernels index slots in int32
  p.hash = plan_hash(ntensors, numels);
  // Segments: maximal runs inside one tensor and one owner chunk.
  for (int t = 0; t < ntensors; ++t) {
    int64_t lo = p.slot_prefix[t], hi = p.slot_prefix[t + 1];
    while (lo < hi) {
      // owner of slot lo: largest r with floor(M*r/p) <= lo
      int r = (int)((lo * nranks) / (p.M ? p.M : 1));
      while (r + 1 < nranks && p.owner_lo(r + 1) <= lo) ++r;
      while (r > 0 && p.owner_lo(r) > lo) --r;
      int64_t end = hi < p.owner_hi(r) ? hi : p.owner_hi(r);
      p.segments.push_back({t, r, lo, end});
      lo = end;
    }
  }
  out = std::move(p);
  return TC_OK;
}

tc_status bootstrap_allgather(tc_allgather_fn ag, void* ctx, int nranks, const void* send,
                              void* recv, size_t bytes) {
  if (nranks == 1) {
    std::memcpy(recv, send, bytes);
    return TC_OK;
  }
  if (ag == nullptr) return TC_ERR_BOOTSTRAP;
  return ag(ctx, send, recv, bytes) == 0 ? TC_OK : TC_ERR_BOOTSTRAP;
}

}  // namespace tc

using namespace tc;

extern "C" {

tc_status tc_plan_create(int rank, int nranks, int ntensors, const int64_t* numels,
                         tc_allgather_fn ag, void* ag_ctx, tc_plan** out) {
  if (out == nullptr) return TC_ERR_INVALID_ARG;
  *out = nullptr;
  Plan p;
  tc_status st = build_plan(rank, nranks, ntensors, numels, p);
  if (ag != nullptr && nranks > 1) {
    // Collective congruence check: every rank learns every rank's (status, T, hash), so all
    // ranks return the same status (no rank is left waiting in a later collective).
    struct Hdr { int32_t status, T; uint64_t hash; } mine{(int32_t)st, ntensors,
                                                          st == TC_OK ? p.hash : 0}, all[kMaxRanks];
    if (nranks > kMaxRanks) return TC_ERR_UNSUPPORTED;
    tc_status bs = bootstrap_allgather(ag, ag_ctx, nranks, &mine, all, sizeof(Hdr));
    if (bs != TC_OK) return bs;
    for (int r = 0; r < nranks; ++r)
      if (all[r].status != TC_OK) return all[r].status == TC_ERR_UNSUPPORTED ? TC_ERR_UNSUPPORTED
                                                                          : TC_ERR_INVALID_ARG;
    for (int r = 0; r < nranks; ++r)
      if (all[r].T != all[0].T || all[r].hash != all[0].hash) return TC_ERR_SHAPE_MISMATCH;
  }
  if (st != TC_OK) return st;
  tc_plan* h = new tc_plan;
  h->p = std::move(p);
  *out = h;
  return TC_OK;
}

void tc_plan_destroy(tc_plan* plan) { delete plan; }

int64_t tc_plan_num_elements(const tc_plan* plan) { return plan ? plan->p.N : -1; }
int64_t tc_plan_num_slots(const tc_plan* plan) { return plan ? plan->p.M : -1; }
uint64_t tc_plan_hash(const tc_plan* plan) { return plan ? plan->p.hash : 0; }

tc_status tc_plan_tensor_slots(const tc_plan* plan, int t, int64_t* first, int64_t* n) {
  if (!plan || t < 0 || t >= plan->p.T || !first || !n) return TC_ERR_INVALID_ARG;
  *first = plan->p.slot_prefix[t];
  *n = plan->p.slot_prefix[t + 1] - plan->p.slot_prefix[t];
  return TC_OK;
}

tc_status tc_plan_owner_range(const tc_plan* plan, int r, int64_t* lo, int64_t* hi) {
  if (!plan || r < 0 || r >= plan->p.nranks || !lo || !hi) return TC_ERR_INVALID_ARG;
  *lo = plan->p.owner_lo(r);
  *hi = plan->p.owner_hi(r);
  return TC_OK;
}

int tc_plan_num_segments(const tc_plan* plan) { return plan ? (int)plan->p.segments.size() : -1; }

tc_status tc_plan_segment(const tc_plan* plan, int i, int* tensor, int* owner, int64_t* lo,
                          int64_t* hi) {
  if (!plan || i < 0 || i >= (int)plan->p.segments.size() || !tensor || !owner || !lo || !hi)
    return TC_ERR_INVALID_ARG;
  const auto& s = plan->p.segments[(size_t)i];
  *tensor = s.tensor;
  *owner = s.owner;
  *lo = s.lo;
  *hi = s.hi;
  return TC_OK;
}

int tc_plan_buckets(const tc_plan* plan, int64_t bucket_bytes, int* bucket_of_tensor) {
  // NEXT row f1 (gradients "can be aggregated in parallel with the backward phase"):
  // consecutive tensors, taken from the last to the first -- the order a backward pass produces
  // them -- are grouped while the bucket stays within bucket_bytes; a larger tensor is a bucket
  // of its own.  Bucket 0 is the first ready (it holds the last tensors).
  if (!plan || !bucket_of_tensor || bucket_bytes <= 0) return -1;
  const Plan& p = plan->p;
  int b = 0;
  int64_t fill = 0;
  bool open = false;
  for (int t = p.T - 1; t >= 0; --t) {
    const int64_t bytes = p.numel[(size_t)t] * 4;
    if (open && fill + bytes > bucket_bytes) {
      ++b;
      fill = 0;
      open = false;
    }
    bucket_of_tensor[t] = b;
    fill += bytes;
    open = true;
  }
  return open ? b + 1 : b;
}

}  // extern "C"
