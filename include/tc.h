/*
 * tc.h -- C ABI of libtc, the B200-native tensor-collective hot path of MXNET-MPI
 *         (arXiv 1801.03855).  PAPER.md line n is cited as P:n, SPEC.md line n as S:n.
 *
 * What it computes:
 *   tc_allreduce    -- the *tensor allreduce* of §6: the T tensors a rank holds are
 *                      one flat logical vector ("a group of vectors on a node as a single
 *                      object"), reduced by reduce-scatter + allgather.
 *   tc_sgd_step     -- that allreduce fused with the SGD update of Eq. 1 with the
 *                      1/mini_batch "rescale" of Fig. code-snippet-2 and momentum.
 *   tc_easgd_update -- the elastic-averaging update, Eqs. elastic1/elastic2, in the
 *                      synchronous sum form  x_i -= a(x_i - xc);  xc += a * sum_i (x_i - xc).
 *
 * Data types: fp32 tensors only (the paper never states a precision; fp32 is implied, R19).
 *
 * Ownership: the caller owns every tensor.  A tensor passed to tc_group_create must stay
 * allocated and unmoved until tc_group_destroy returns on all ranks.  libtc owns its flag,
 * staging and descriptor buffers and its CUDA-IPC mappings.  Streams belong to the caller:
 * hot-path calls enqueue one kernel on `stream` (a cudaStream_t, NULL = legacy default
 * stream) and return; completion is stream-ordered.
 *
 * Collectives: every call on a comm (create, group create/destroy, the three hot-path calls)
 * is COLLECTIVE -- every rank of the comm makes the same calls, in the same order, with the
 * same scalar arguments ("the operations are enqueued in order to avoid deadlocks").
 * Consecutive hot-path calls on one comm must be stream-ordered on each rank.
 *
 * Errors: every function returns a tc_status synchronously; nothing throws across the ABI.
 * Non-finite *data* is not checked on the hot path (NaN/Inf propagate).
 */
#ifndef TC_H_
#define TC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TC_OK = 0,
  TC_ERR_INVALID_ARG = 1,     /* null pointer, bad count/size/alignment, bad hyper-parameter   */
  TC_ERR_SHAPE_MISMATCH = 2,  /* ranks disagree on (T, n_t), or groups not congruent   */
  TC_ERR_NOT_SHAREABLE = 3,   /* a tensor's allocation cannot be exported with CUDA IPC        */
  TC_ERR_BUSY = 4,            /* another host thread is inside a call on this comm     */
  TC_ERR_TIMEOUT = 5,         /* a peer did not arrive at a device barrier (sticky)     */
  TC_ERR_CUDA = 6,            /* a CUDA runtime call failed                                     */
  TC_ERR_BOOTSTRAP = 7,       /* the caller's allgather callback failed                         */
  TC_ERR_UNSUPPORTED = 8      /* e.g. nranks > TC_MAX_RANKS                                      */
} tc_status;

#define TC_MAX_RANKS 8        /* one NVSwitch box */

#if defined(__GNUC__)
#define TC_API __attribute__((visibility("default")))
#else
#define TC_API
#endif

typedef struct tc_plan tc_plan;    /* A1 descriptor: flat slot space + owner partition (host) */
typedef struct tc_comm tc_comm;    /* ranks (GPUs) with peer-mapped flag/staging buffers      */
typedef struct tc_group tc_group;  /* caller tensors flattened over a comm, peer-mapped        */

/* Bootstrap allgather supplied by the caller (torch.distributed over gloo in the Python
 * binding).  Gathers `bytes_per_rank` bytes from every rank of the comm into `recv`
 * (rank-major, nranks * bytes_per_rank bytes).  Returns 0 on success. */
typedef int (*tc_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes_per_rank);

/* Library version (major*10000 + minor*100 + patch). */
TC_API int tc_version(void);

/* Human-readable name of a status code (static storage; never NULL). */
TC_API const char* tc_status_string(tc_status s);

/* ---------------------------------------------------------------------------------------
 * A1: group descriptor (host only, no CUDA).  P:331 "the buffer from each process is
 * partitioned into nearly equal parts"; reading R2: 16-byte slots.  Tensor t of n_t fp32
 * elements occupies ceil(n_t/4) consecutive slots of one flat slot space of M slots (the last
 * slot of a tensor may be partial).  Rank r owns slots [floor(M*r/p), floor(M*(r+1)/p)).
 * A segment is a maximal run of slots inside one tensor and one owner (<= T+p-1 of them).
 * --------------------------------------------------------------------------------------- */

/* Builds the plan for `ntensors` tensors of `numels[t]` elements (numels[t] >= 0) over
 * `nranks` ranks.  If `ag` is non-NULL the call is collective: every rank's (T, numels) is
 * checked through `ag` and TC_ERR_SHAPE_MISMATCH is returned on EVERY rank if any differ.
 * With ag == NULL the plan is local.  Errors: TC_ERR_INVALID_ARG (nranks < 1, rank out of
 * range, ntensors < 1, numels NULL or negative, M >= 2^31 slots), TC_ERR_UNSUPPORTED
 * (nranks > TC_MAX_RANKS), TC_ERR_BOOTSTRAP.  *out is owned by the caller (tc_plan_destroy). */
TC_API tc_status tc_plan_create(int rank, int nranks, int ntensors, const int64_t* numels,
                         tc_allgather_fn ag, void* ag_ctx, tc_plan** out);
TC_API void tc_plan_destroy(tc_plan* plan);
TC_API int64_t tc_plan_num_elements(const tc_plan* plan);              /* N = sum_t n_t            */
TC_API int64_t tc_plan_num_slots(const tc_plan* plan);                 /* M                        */
TC_API uint64_t tc_plan_hash(const tc_plan* plan);                     /* congruence hash of (T,n) */
/* First slot and slot count of tensor t. */
TC_API tc_status tc_plan_tensor_slots(const tc_plan* plan, int t, int64_t* first_slot, int64_t* nslots);
/* Owner slot range [lo, hi) of rank r. */
TC_API tc_status tc_plan_owner_range(const tc_plan* plan, int r, int64_t* lo, int64_t* hi);
TC_API int tc_plan_num_segments(const tc_plan* plan);
/* Segment i: tensor index, owner rank, and its global slot range [slot_lo, slot_hi). */
TC_API tc_status tc_plan_segment(const tc_plan* plan, int i, int* tensor, int* owner,
                          int64_t* slot_lo, int64_t* slot_hi);

/* NEXT row f1 -- bucketed reduction overlapped with the backward pass (gradients "can be
 * aggregated in parallel with the backward phase").  Assigns every tensor a bucket: tensors are
 * taken from the last to the first (backward order) and grouped while a bucket holds at most
 * `bucket_bytes` (a larger tensor is a bucket of its own).  Writes bucket_of_tensor[T] (bucket 0
 * = first ready) and returns the number of buckets, or -1 on a bad argument.  Each bucket is
 * then an ordinary tc_group whose reduction (tc_allreduce / tc_sgd_step) is launched on a side
 * stream as soon as its last gradient is produced. */
TC_API int tc_plan_buckets(const tc_plan* plan, int64_t bucket_bytes, int* bucket_of_tensor);

/* ---------------------------------------------------------------------------------------
 * Communicators.
 * --------------------------------------------------------------------------------------- */

/* One rank per process (the production layout).  Collective over `nranks` processes; `ag`
 * is the bootstrap allgather over exactly those processes (rank order = comm rank order).
 * Allocates the flag and one-shot staging buffers on `cuda_device`, exports them with
 * cudaIpcGetMemHandle and maps every peer's.  Errors: TC_ERR_INVALID_ARG,
 * TC_ERR_UNSUPPORTED (nranks > TC_MAX_RANKS), TC_ERR_CUDA, TC_ERR_BOOTSTRAP. */
TC_API tc_status tc_comm_create(int rank, int nranks, int cuda_device, tc_allgather_fn ag,
                         void* ag_ctx, tc_comm** out);

/* All `nranks` ranks live in this process on ONE device (test/debug layout): every hot-path
 * call launches ONE cooperative kernel whose blockIdx.y is the rank, running exactly the
 * per-rank code and flag protocol of the multi-process layout (peer "mappings" are plain
 * local pointers).  Not collective. */
TC_API tc_status tc_comm_create_emulated(int nranks, int cuda_device, tc_comm** out);

/* Launch tuning, must be identical on all ranks.  num_ctas: CTAs per rank for two-shot and NVLS
 * calls (0 = automatic: a full wave of the GPU); threads: threads per CTA of the register kernels
 * and of the NVLS allreduce (0 = 512; a multiple of 32 in [64, 512]; the TMA kernels and the
 * NVLS fused step keep their fixed block sizes); oneshot_max_bytes: groups of at most this many bytes use the one-shot
 * algorithm (-1 = automatic: 8 MiB at p = 2, 4 MiB at p = 3, 2 MiB at p = 4, 256 KiB beyond;
 * 0 = never; capped by the staging capacity).  Applies to later
 * calls.  Errors: TC_ERR_INVALID_ARG. */
TC_API tc_status tc_comm_set_tuning(tc_comm* comm, int num_ctas, int threads, int64_t oneshot_max_bytes);

/* Groups of at most `bytes` of data (-1 = automatic: 1 MiB at p = 2, 512 KiB at p = 3,
 * 256 KiB at p = 4, 128 KiB beyond; 0 = never) use the low-latency algorithm:
 * every rank stores each element to every peer as one 8-byte {value, call epoch} word and waits
 * for its peers' words in local memory, so a call costs one NVLink crossing and no barrier.
 * Same arithmetic (float64, rank order) as the other P2P algorithms.  Capped by the LL buffer
 * (16 MiB / (16 p) elements).  Must be identical on all ranks.  Errors: TC_ERR_INVALID_ARG. */
TC_API tc_status tc_comm_set_ll_max(tc_comm* comm, int64_t bytes);

/* Large-group algorithm (must be identical on all ranks): 0 = automatic; 1 = two-shot with the
 * reduce-scatter and allgather pulled by the SMs' 16-B loads (register kernels); 6 = two-shot
 * with the data moved by TMA bulk copies through a shared-memory stage ring (one CTA per SM at
 * most; tc_comm_set_tuning's num_ctas or tc_group_set_num_ctas sets how many SMs it occupies);
 * 1 and 6 give bit-identical results (float64, rank order).  4 = NVLS (switch reduction,
 * multimem.ld_reduce + multimem.st; only for groups in tc_mem_alloc memory, else two-shot): the
 * switch sums in fp32 in its own order -- exact for integer-valued data, else within the
 * BASELINE tolerance 1e-5 * sum_k |x_k| of the float64 sum; identical on every rank.
 * Automatic (0): low-latency / one-shot for small groups, 6 above (measured fastest); NVLS only
 * when tc_comm_set_switch_reduction(comm, 1) allowed it.  Errors: TC_ERR_INVALID_ARG. */
TC_API tc_status tc_comm_set_algorithm(tc_comm* comm, int algo);

/* Whether the AUTOMATIC choice may use the NVSwitch reduction (algorithm 4) for groups in
 * tc_mem_alloc memory (must be identical on all ranks).  0 (default): never -- every automatic
 * result is bit-identical to the float64 rank-order oracle.  1: allowed where it moves fewer
 * bytes per GPU than the two-shot ((1 + 1/p) S against 2(p-1)/p S, with the p = 4
 * measured rates: from p = 5 for tc_allreduce and tc_sgd_step) -- results then
 * follow algorithm 4's tolerance contract.
 * Errors: TC_ERR_INVALID_ARG (allow not 0 or 1). */
TC_API tc_status tc_comm_set_switch_reduction(tc_comm* comm, int allow);

/* Device-barrier timeout in milliseconds (default 30000, or env TC_TIMEOUT_MS). */
TC_API tc_status tc_comm_set_timeout(tc_comm* comm, int64_t timeout_ms);

/* Fault injection for tests: while hold != 0 the comm is marked busy exactly as if another
 * host thread were inside a call on it, so every call that takes the comm (hot path, group
 * create/destroy) returns TC_ERR_BUSY ("one collective call per communicator at a
 * time").  Not collective. */
TC_API tc_status tc_comm_set_debug_busy(tc_comm* comm, int hold);

/* Fault injection for tests (emulated comms only): the CTAs of rank `absent_rank` return
 * immediately without arriving at any barrier (-1 = off), so the other ranks time out. */
TC_API tc_status tc_comm_set_debug_absent_rank(tc_comm* comm, int absent_rank);

/* Diagnostics: when `device_buffer` is non-NULL, hot-path kernels with at most bytes/64 CTAs
 * (all local ranks) record %globaltimer (ns) at their phase boundaries: slot [cta][0..5] =
 * start, after entry barrier, after reduce-scatter, after mid barrier, after allgather, end
 * (CTA index = rank_local * ctas + blockIdx.x).  NULL turns it off.  Not collective. */
TC_API tc_status tc_comm_set_profile_buffer(tc_comm* comm, void* device_buffer, int64_t bytes);

/* Sticky device-side error: TC_ERR_TIMEOUT once any barrier timed out, else TC_OK.  Reads
 * host-mapped memory; does not synchronize.  After a timeout the comm must be destroyed. */
TC_API tc_status tc_comm_async_error(tc_comm* comm);

TC_API int tc_comm_rank(const tc_comm* comm);      /* -1 for an emulated comm */
TC_API int tc_comm_nranks(const tc_comm* comm);

/* Collective: synchronizes the device, waits for every rank (bootstrap barrier), unmaps and
 * frees.  All groups of the comm must have been destroyed first (TC_ERR_INVALID_ARG). */
TC_API tc_status tc_comm_destroy(tc_comm* comm);

/* ---------------------------------------------------------------------------------------
 * Symmetric memory (for the NVSwitch multicast algorithm).
 * --------------------------------------------------------------------------------------- */

/* Collective over a one-rank-per-process comm: allocates `bytes` (rounded up to the
 * allocation granularity) of device memory on every rank, maps every peer's copy into this
 * process, and -- when NVSwitch multicast is supported -- binds all copies to one multicast
 * object.  Returns this rank's pointer.  Tensors placed at the SAME offset of the same
 * symmetric allocation on every rank can be reduced in the switch (algorithm 4, NVLS:
 * multimem.ld_reduce / multimem.st).  Freed only by tc_mem_free (collective) or
 * tc_comm_destroy.  Errors: TC_ERR_INVALID_ARG, TC_ERR_UNSUPPORTED (emulated comm or no VMM
 * driver entry points), TC_ERR_CUDA, TC_ERR_BOOTSTRAP. */
TC_API tc_status tc_mem_alloc(tc_comm* comm, size_t bytes, void** ptr);
/* Collective.  `ptr` must be a pointer tc_mem_alloc returned.  TC_ERR_INVALID_ARG if it is not,
 * or while a live group still has tensors in the allocation (destroy those groups first). */
TC_API tc_status tc_mem_free(tc_comm* comm, void* ptr);
/* 1 if this comm's device supports NVSwitch multicast + reduction, else 0. */
TC_API int tc_comm_multicast_supported(const tc_comm* comm);

/* ---------------------------------------------------------------------------------------
 * Tensor groups (the paper's "tensor", generalized to T tensors per rank).
 * --------------------------------------------------------------------------------------- */

/* Collective.  `ptrs[t]` is this rank's device pointer to tensor t (fp32, 4-byte aligned,
 * contiguous), `numels[t]` its element count (0 allowed, then ptrs[t] may be NULL).  For an
 * emulated comm `ptrs` holds nranks*ntensors pointers, rank-major (ptrs[r*ntensors + t]).
 * Nothing is copied: each pointer's cudaMalloc allocation is exported with CUDA IPC and
 * mapped by every peer (allocations shared by several tensors are mapped once).  Tensors whose
 * pointers sit the same number of elements past a 16-byte boundary on every rank use 16-byte
 * vector (and TMA bulk) copies; others a scalar path.  The bulk copies may READ (never write)
 * the rest of the 16-byte block holding a tensor's first or last element, which lies inside
 * the same allocation for every CUDA allocator (bases 256-B aligned, sizes rounded up).
 * Errors: TC_ERR_INVALID_ARG, TC_ERR_SHAPE_MISMATCH (ranks disagree on T or any n_t; returned
 * on every rank), TC_ERR_NOT_SHAREABLE (e.g. PyTorch expandable_segments allocations),
 * TC_ERR_BUSY (another call on the comm is in progress), TC_ERR_CUDA, TC_ERR_BOOTSTRAP. */
TC_API tc_status tc_group_create(tc_comm* comm, int ntensors, void* const* ptrs, const int64_t* numels,
                          tc_group** out);

/* Collective: synchronizes the device, waits for every rank, then unmaps. */
TC_API tc_status tc_group_destroy(tc_group* group);

/* CTA budget of this group's hot-path launches (0 = the comm's tc_comm_set_tuning value), so
 * e.g. the buckets of an overlapped step can run on a few SMs without changing the comm's
 * state for other groups.  Must be identical on all ranks (the per-CTA barriers pair CTA b of
 * every rank).  Not collective.  Errors: TC_ERR_INVALID_ARG (num_ctas outside [0, 1024]). */
TC_API tc_status tc_group_set_num_ctas(tc_group* group, int num_ctas);

/* ---------------------------------------------------------------------------------------
 * Hot path.  One kernel launch per call on `stream`.
 * --------------------------------------------------------------------------------------- */

/* A3+A4 (or A5 one-shot for small groups): in place, on every rank,
 *     x[t][j] := round_fp32( (sum_{k=0..p-1} x_k[t][j]) * scale )
 * summed in float64 in canonical rank order k = 0..p-1 and rounded once (readings R3, R4), so
 * the result is bit-identical on every rank and for every P2P algorithm (NVLS, algorithm 4:
 * see tc_comm_set_algorithm).  Errors:
 * TC_ERR_INVALID_ARG (NULL group, non-finite scale), TC_ERR_TIMEOUT (sticky), TC_ERR_BUSY,
 * TC_ERR_CUDA (launch failure). */
TC_API tc_status tc_allreduce(tc_group* x, float scale, void* stream);

/* A6: gradient allreduce fused with the SGD(-momentum) update, on every rank, per element:
 *     G   = sum_k g_k                (float64, rank order, rounded once; written back to g)
 *     t   = (rescale*G) + (wd*w)                        each op rounded to fp32, no FMA
 *     dw := (momentum*dw) - (lr*t)                      (reading R12; Eq. 1 at momentum=wd=0)
 *     w  := w + dw                                      (Eq. 1: w_{t+1} = w_t + dw)
 * w, g, dw must be congruent groups on the same comm (same T and n_t) -- normally w and dw
 * are replicated, so every rank ends with identical w, dw.  Errors: TC_ERR_INVALID_ARG
 * (NULL, non-finite hyper-parameter), TC_ERR_SHAPE_MISMATCH, TC_ERR_TIMEOUT, TC_ERR_BUSY,
 * TC_ERR_CUDA. */
TC_API tc_status tc_sgd_step(tc_group* w, tc_group* g, tc_group* dw, float lr, float momentum,
                      float wd, float rescale, void* stream);

/* A7: elastic averaging over a comm with one rank per client (c = nranks), per element:
 *     d_i  = x_i - xc                     (each client's params vs the replicated center)
 *     x_i := x_i - alpha*d_i              (Eq. elastic2)
 *     xc  := xc + alpha*(d_0 + d_1 + ... + d_{c-1})   (Eq. elastic1 summed over clients, R10)
 * all in fp32 with every op rounded (fp32 mirror), sums in client order.  `center` is
 * replicated and stays bit-identical on every rank.  alpha in [0, 1].  Errors:
 * TC_ERR_INVALID_ARG, TC_ERR_SHAPE_MISMATCH, TC_ERR_TIMEOUT, TC_ERR_BUSY, TC_ERR_CUDA. */
TC_API tc_status tc_easgd_update(tc_group* x, tc_group* center, float alpha, void* stream);

/* NEXT row f2: the elastic update of tc_easgd_update followed, in the same
 * pass over memory, by the SGD-momentum update of tc_sgd_step applied to the elastically moved
 * parameters with THIS rank's own gradient (not reduced: one GPU per client, as in config 1's
 * "4 workers" or Fig. code-snippet-4 at one GPU per worker; the paper's order is Elastic2 then
 * SGD.Update in the same iteration).  Per element, fp32 with every op rounded:
 *     d   = x - xc;                xe  = x - alpha*d
 *     xc := xc + alpha*(d_0 + ... + d_{c-1})          (client order)
 *     t   = rescale*g + wd*xe;     dw := momentum*dw - lr*t;     x := xe + dw
 * x, center, g, dw: congruent groups on one comm (one rank per client); g is read only.
 * One kernel: the TMA two-shot (p >= 2) or the TMA stream (p = 1).  Reads x, xc, g, dw once and
 * writes x, xc, dw once (8S of HBM per GPU instead of 10S for tc_easgd_update + a local
 * tc_sgd_step), NVLink traffic as tc_easgd_update.  Errors: as tc_sgd_step; alpha in [0, 1]. */
TC_API tc_status tc_esgd_step(tc_group* x, tc_group* center, tc_group* g, tc_group* dw,
                              float alpha, float lr, float momentum, float wd, float rescale,
                              void* stream);

/* NEXT row f2, asynchronous server: elastic averaging as the paper's parameter server applies
 * it -- Elastic1 on the server as each client's push arrives, Elastic2 on the client (P:66
 * "elastic1 is done on the server and elastic2 is done on the client"; Fig. code-snippet-4,
 * P:302-312) -- with the arrivals in the recorded order `order` (host array of nranks
 * client indices, a permutation; NULL = client order 0..c-1; identical on all ranks).  The
 * center is sharded by owner (the owner of a chunk is its server shard) and replicated after
 * the call.  Per element, for i = order[0], order[1], ... with the center as the earlier
 * arrivals left it, fp32 with every op rounded (oracle.easgd_async, reading R20):
 *     d = x_i - xc;     xc := xc + alpha*d   (Eq. elastic1);     x_i := x_i - alpha*d   (Eq. elastic2)
 * c = 1 is exactly tc_easgd_update.  One kernel (TMA two-shot): the owner pulls every client's
 * chunk, applies the arrivals, stores each client's new chunk straight into that client's
 * tensor over NVLink, stages the center; the allgather brings the center.  Per GPU: NVLink
 * ingress 2(c-1)/c S, egress 2(c-1)/c S.  Errors: TC_ERR_INVALID_ARG (alpha outside [0, 1],
 * order not a permutation), TC_ERR_SHAPE_MISMATCH, TC_ERR_TIMEOUT, TC_ERR_BUSY, TC_ERR_CUDA. */
TC_API tc_status tc_easgd_async_update(tc_group* x, tc_group* center, float alpha,
                                       const int* order, void* stream);

/* Tensor broadcast (MPI_Bcast of the weights at initialisation; the KVStore.pull
 * broadcast): every rank's group := the root's group, bit for bit.  Groups in
 * multicast-bound tc_mem_alloc memory at p >= 4 (or with tc_comm_set_algorithm(4)): the root
 * writes every rank's copy with NVSwitch multicast stores (each byte leaves the root once; a
 * copy, so exact).  Otherwise: scatter from the root (each rank copies its owner
 * chunk of the root's tensors) then the allgather of the two-shot (the root sends
 * 2(p-1)/p S).  Collective; root identical on all ranks.  p = 1: no-op.  Errors:
 * TC_ERR_INVALID_ARG (root outside [0, nranks)), TC_ERR_TIMEOUT, TC_ERR_BUSY, TC_ERR_CUDA. */
TC_API tc_status tc_broadcast(tc_group* x, int root, void* stream);

/* Introspection of the most recent hot-path launch on this comm (for benchmarks):
 * algorithm (0 = local p=1, 1 = two-shot (register), 2 = one-shot, 4 = NVLS, 5 = low-latency,
 * 6 = two-shot TMA), grid CTAs per rank, threads per CTA. */
TC_API tc_status tc_comm_last_launch(const tc_comm* comm, int* algo, int* ctas, int* threads);

#ifdef __cplusplus
}
#endif
#endif /* TC_H_ */
