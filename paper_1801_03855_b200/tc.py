"""Thin Python binding of libtc (include/tc.h) -- argument marshalling only.

Every step of the hot path runs in libtc's CUDA kernels; PyTorch supplies device memory, the
current stream and the torch.distributed (gloo) allgather used to bootstrap a communicator.
There is no CPU fallback: if libtc.so is missing this module raises on import.

    comm  = Comm.from_process_group()              # one rank per process (torchrun)
    comm  = Comm.emulated(4, device=0)             # 4 ranks in this process on one GPU (tests)
    g     = Group(comm, grads)                     # list of fp32 CUDA tensors (no copy)
    allreduce(g)                                   # x := sum over ranks, in place
    sgd_step(w, g, dw, lr=0.1, momentum=0.9, wd=1e-4, rescale=1/256)
    easgd_update(x, center, alpha=0.1)
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TC_LIB", os.path.join(_HERE, "libtc.so"))

STATUS = {
    0: "TC_OK", 1: "TC_ERR_INVALID_ARG", 2: "TC_ERR_SHAPE_MISMATCH", 3: "TC_ERR_NOT_SHAREABLE",
    4: "TC_ERR_BUSY", 5: "TC_ERR_TIMEOUT", 6: "TC_ERR_CUDA", 7: "TC_ERR_BOOTSTRAP",
    8: "TC_ERR_UNSUPPORTED",
}
TC_OK, TC_ERR_INVALID_ARG, TC_ERR_SHAPE_MISMATCH, TC_ERR_NOT_SHAREABLE = 0, 1, 2, 3
TC_ERR_BUSY, TC_ERR_TIMEOUT, TC_ERR_CUDA, TC_ERR_BOOTSTRAP, TC_ERR_UNSUPPORTED = 4, 5, 6, 7, 8
ALGO_NAMES = {0: "local", 1: "two-shot", 2: "one-shot", 4: "nvls", 5: "ll", 6: "two-shot-tma"}
ALGO_AUTO, ALGO_TWOSHOT_PULL, ALGO_NVLS, ALGO_TWOSHOT_TMA = 0, 1, 4, 6

ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_size_t)

_c_int, _c_int64, _c_float, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p
_pp = ctypes.POINTER(ctypes.c_void_p)
_SIGS = {
    "tc_version": (_c_int, []),
    "tc_status_string": (ctypes.c_char_p, [_c_int]),
    "tc_plan_create": (_c_int, [_c_int, _c_int, _c_int, ctypes.POINTER(_c_int64), ALLGATHER_FN,
                                _vp, _pp]),
    "tc_plan_destroy": (None, [_vp]),
    "tc_plan_buckets": (_c_int, [_vp, _c_int64, ctypes.POINTER(_c_int)]),
    "tc_plan_num_elements": (_c_int64, [_vp]),
    "tc_plan_num_slots": (_c_int64, [_vp]),
    "tc_plan_hash": (ctypes.c_uint64, [_vp]),
    "tc_plan_tensor_slots": (_c_int, [_vp, _c_int, ctypes.POINTER(_c_int64),
                                      ctypes.POINTER(_c_int64)]),
    "tc_plan_owner_range": (_c_int, [_vp, _c_int, ctypes.POINTER(_c_int64),
                                     ctypes.POINTER(_c_int64)]),
    "tc_plan_num_segments": (_c_int, [_vp]),
    "tc_plan_segment": (_c_int, [_vp, _c_int, ctypes.POINTER(_c_int), ctypes.POINTER(_c_int),
                                 ctypes.POINTER(_c_int64), ctypes.POINTER(_c_int64)]),
    "tc_comm_create": (_c_int, [_c_int, _c_int, _c_int, ALLGATHER_FN, _vp, _pp]),
    "tc_comm_create_emulated": (_c_int, [_c_int, _c_int, _pp]),
    "tc_comm_set_tuning": (_c_int, [_vp, _c_int, _c_int, _c_int64]),
    "tc_comm_set_timeout": (_c_int, [_vp, _c_int64]),
    "tc_comm_set_algorithm": (_c_int, [_vp, _c_int]),
    "tc_comm_set_switch_reduction": (_c_int, [_vp, _c_int]),
    "tc_comm_set_debug_busy": (_c_int, [_vp, _c_int]),
    "tc_group_set_num_ctas": (_c_int, [_vp, _c_int]),
    "tc_comm_set_ll_max": (_c_int, [_vp, _c_int64]),
    "tc_mem_alloc": (_c_int, [_vp, ctypes.c_size_t, _pp]),
    "tc_mem_free": (_c_int, [_vp, _vp]),
    "tc_comm_multicast_supported": (_c_int, [_vp]),
    "tc_comm_set_debug_absent_rank": (_c_int, [_vp, _c_int]),
    "tc_comm_async_error": (_c_int, [_vp]),
    "tc_comm_set_profile_buffer": (_c_int, [_vp, _vp, _c_int64]),
    "tc_comm_rank": (_c_int, [_vp]),
    "tc_comm_nranks": (_c_int, [_vp]),
    "tc_comm_destroy": (_c_int, [_vp]),
    "tc_comm_last_launch": (_c_int, [_vp, ctypes.POINTER(_c_int), ctypes.POINTER(_c_int),
                                     ctypes.POINTER(_c_int)]),
    "tc_group_create": (_c_int, [_vp, _c_int, _pp, ctypes.POINTER(_c_int64), _pp]),
    "tc_group_destroy": (_c_int, [_vp]),
    "tc_allreduce": (_c_int, [_vp, _c_float, _vp]),
    "tc_sgd_step": (_c_int, [_vp, _vp, _vp, _c_float, _c_float, _c_float, _c_float, _vp]),
    "tc_easgd_update": (_c_int, [_vp, _vp, _c_float, _vp]),
    "tc_easgd_async_update": (_c_int, [_vp, _vp, _c_float, ctypes.POINTER(_c_int), _vp]),
    "tc_broadcast": (_c_int, [_vp, _c_int, _vp]),
    "tc_esgd_step": (_c_int, [_vp, _vp, _vp, _vp, _c_float, _c_float, _c_float, _c_float,
                              _c_float, _vp]),
}


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libtc.so not built at {path}: run `python build_libtc.py`"
                          " (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = load()


class TcError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        super().__init__(f"{what}: {STATUS.get(status, status)}")


def _check(st: int, what: str):
    if st != TC_OK:
        raise TcError(st, what)


def _stream_ptr(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def make_allgather(pg=None):
    """A tc_allgather_fn over a torch.distributed (gloo/CPU) group."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(pg)

    def cb(ctx, send, recv, nbytes):
        try:
            buf = torch.empty(nbytes, dtype=torch.uint8)
            ctypes.memmove(buf.data_ptr(), send, nbytes)
            outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(outs, buf, group=pg)
            for r, o in enumerate(outs):
                ctypes.memmove(recv + r * nbytes, o.data_ptr(), nbytes)
            return 0
        except Exception:  # noqa: BLE001 -- reported to C as TC_ERR_BOOTSTRAP
            return 1

    return ALLGATHER_FN(cb)


class Plan:
    """A1 descriptor (host only).  Collective over `pg` when given."""

    def __init__(self, numels: Sequence[int], nranks: int = 1, rank: int = 0, pg=None):
        arr = (ctypes.c_int64 * len(numels))(*[int(n) for n in numels])
        self._ag = make_allgather(pg) if pg is not None else ALLGATHER_FN()
        h = ctypes.c_void_p()
        _check(LIB.tc_plan_create(rank, nranks, len(numels), arr, self._ag, None, ctypes.byref(h)),
               "tc_plan_create")
        self.h = h
        self.num_tensors = len(numels)

    def __del__(self):
        if getattr(self, "h", None):
            LIB.tc_plan_destroy(self.h)
            self.h = None

    @property
    def num_elements(self) -> int:
        return LIB.tc_plan_num_elements(self.h)

    @property
    def num_slots(self) -> int:
        return LIB.tc_plan_num_slots(self.h)

    @property
    def hash(self) -> int:
        return LIB.tc_plan_hash(self.h)

    def tensor_slots(self, t: int):
        a, n = ctypes.c_int64(), ctypes.c_int64()
        _check(LIB.tc_plan_tensor_slots(self.h, t, ctypes.byref(a), ctypes.byref(n)), "tensor_slots")
        return a.value, n.value

    def owner_range(self, r: int):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(LIB.tc_plan_owner_range(self.h, r, ctypes.byref(a), ctypes.byref(b)), "owner_range")
        return a.value, b.value

    def buckets(self, bucket_bytes: int):
        """Bucket index of every tensor (backward order, bucket 0 first ready)."""
        out = (ctypes.c_int * self.num_tensors)()
        n = LIB.tc_plan_buckets(self.h, int(bucket_bytes), out)
        if n < 0:
            raise TcError(TC_ERR_INVALID_ARG, "tc_plan_buckets")
        return list(out), n

    def segments(self):
        out = []
        for i in range(LIB.tc_plan_num_segments(self.h)):
            t, o, lo, hi = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
            _check(LIB.tc_plan_segment(self.h, i, ctypes.byref(t), ctypes.byref(o),
                                       ctypes.byref(lo), ctypes.byref(hi)), "segment")
            out.append((t.value, o.value, lo.value, hi.value))
        return out


class Comm:
    """A tc_comm.  Use :meth:`from_process_group` (one rank per process) or :meth:`emulated`."""

    def __init__(self, handle, ag=None, pg=None):
        self.h = handle
        self._ag = ag      # keeps the ctypes callback alive
        self._pg = pg
        self.groups = 0

    @classmethod
    def from_process_group(cls, pg=None, device: int | None = None):
        """Collective over the ranks of `pg`.  The bootstrap allgather runs on CPU tensors, so
        `pg` must be a gloo group (create sub-communicators with
        ``dist.new_group(ranks, backend="gloo")`` on every rank).  With pg=None a gloo group over
        the whole world is created (a collective over all ranks).  The data path never touches
        the process group."""
        import torch
        import torch.distributed as dist

        if device is None:
            device = torch.cuda.current_device()
        boot = dist.new_group(backend="gloo") if pg is None else pg
        ag = make_allgather(boot)
        h = ctypes.c_void_p()
        _check(LIB.tc_comm_create(dist.get_rank(boot), dist.get_world_size(boot), device, ag, None,
                                  ctypes.byref(h)), "tc_comm_create")
        return cls(h, ag, boot)

    @classmethod
    def single(cls, device: int = 0):
        h = ctypes.c_void_p()
        _check(LIB.tc_comm_create(0, 1, device, ALLGATHER_FN(), None, ctypes.byref(h)),
               "tc_comm_create")
        return cls(h)

    @classmethod
    def emulated(cls, nranks: int, device: int = 0):
        h = ctypes.c_void_p()
        _check(LIB.tc_comm_create_emulated(nranks, device, ctypes.byref(h)),
               "tc_comm_create_emulated")
        return cls(h)

    @property
    def rank(self) -> int:
        return LIB.tc_comm_rank(self.h)

    @property
    def nranks(self) -> int:
        return LIB.tc_comm_nranks(self.h)

    @property
    def is_emulated(self) -> bool:
        return self.rank < 0

    def set_tuning(self, num_ctas: int = 0, threads: int = 0, oneshot_max_bytes: int = -1):
        _check(LIB.tc_comm_set_tuning(self.h, num_ctas, threads, oneshot_max_bytes), "set_tuning")

    @property
    def multicast_supported(self) -> bool:
        return bool(LIB.tc_comm_multicast_supported(self.h))

    def alloc_symmetric(self, numel: int):
        """Collective: a float32 CUDA tensor of `numel` elements in symmetric, multicast-bound
        memory (tc_mem_alloc).  Groups of views at the same offsets on every rank can use the
        NVLS algorithm.  The memory lives until free_symmetric() or destroy()."""
        import torch
        p = ctypes.c_void_p()
        _check(LIB.tc_mem_alloc(self.h, int(numel) * 4, ctypes.byref(p)), "tc_mem_alloc")
        dev = torch.cuda.current_device()

        class _Cai:
            __cuda_array_interface__ = {"shape": (int(numel),), "typestr": "<f4",
                                        "data": (p.value, False), "version": 3, "strides": None}
        t = torch.as_tensor(_Cai(), device=f"cuda:{dev}")
        assert t.data_ptr() == p.value
        self._sym = getattr(self, "_sym", []) + [t]
        return t

    def free_symmetric(self, tensor):
        _check(LIB.tc_mem_free(self.h, tensor.data_ptr()), "tc_mem_free")
        self._sym = [t for t in getattr(self, "_sym", []) if t is not tensor]

    def set_algorithm(self, algo: int):
        """0 = automatic, 1 = register two-shot, 6 = TMA two-shot (identical results),
        4 = NVLS for groups in symmetric memory."""
        _check(LIB.tc_comm_set_algorithm(self.h, int(algo)), "set_algorithm")

    def set_switch_reduction(self, allow: bool):
        """Let the automatic choice use NVLS (fp32 sums in the switch; tolerance contract)."""
        _check(LIB.tc_comm_set_switch_reduction(self.h, int(bool(allow))),
               "set_switch_reduction")

    def set_debug_busy(self, hold: bool):
        """Tests: mark the comm busy as if another thread were inside a call on it."""
        _check(LIB.tc_comm_set_debug_busy(self.h, int(bool(hold))), "set_debug_busy")

    def set_ll_max(self, nbytes: int):
        """Groups up to nbytes use the low-latency algorithm (-1 automatic, 0 never)."""
        _check(LIB.tc_comm_set_ll_max(self.h, int(nbytes)), "set_ll_max")

    def set_timeout(self, ms: int):
        _check(LIB.tc_comm_set_timeout(self.h, int(ms)), "set_timeout")

    def set_debug_absent_rank(self, r: int):
        _check(LIB.tc_comm_set_debug_absent_rank(self.h, r), "set_debug_absent_rank")

    def set_profile_buffer(self, tensor=None):
        """Diagnostics: phase timestamps into a CUDA int64 tensor of shape [ctas, 8] (or None)."""
        if tensor is None:
            _check(LIB.tc_comm_set_profile_buffer(self.h, None, 0), "set_profile_buffer")
        else:
            _check(LIB.tc_comm_set_profile_buffer(self.h, tensor.data_ptr(),
                                                  tensor.numel() * tensor.element_size()),
                   "set_profile_buffer")

    def async_error(self) -> int:
        return LIB.tc_comm_async_error(self.h)

    def last_launch(self):
        a, c, t = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(LIB.tc_comm_last_launch(self.h, ctypes.byref(a), ctypes.byref(c), ctypes.byref(t)),
               "last_launch")
        return ALGO_NAMES.get(a.value, "none"), c.value, t.value

    def destroy(self):
        if self.h:
            st = LIB.tc_comm_destroy(self.h)
            self.h = None
            _check(st, "tc_comm_destroy")

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()


def _check_tensor(t):
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_cuda \
            or not t.is_contiguous():
        raise TypeError("tc tensors must be contiguous float32 CUDA tensors")


class Group:
    """A tc_group over `tensors` (this rank's list; for an emulated comm a list per rank)."""

    def __init__(self, comm: Comm, tensors):
        self.comm = comm
        if comm.is_emulated:
            per_rank = [list(ts) for ts in tensors]
            if len(per_rank) != comm.nranks:
                raise ValueError("emulated comm: need one tensor list per rank")
            T = len(per_rank[0])
            if any(len(ts) != T for ts in per_rank):
                raise ValueError("emulated comm: ranks disagree on the number of tensors")
            flat = [t for ts in per_rank for t in ts]
            numels = [t.numel() for t in per_rank[0]]
            if any([t.numel() for t in ts] != numels for ts in per_rank):
                raise TcError(TC_ERR_SHAPE_MISMATCH, "tc_group_create")
        else:
            flat = list(tensors)
            T = len(flat)
            numels = [t.numel() for t in flat]
        for t in flat:
            _check_tensor(t)
        self.tensors = flat  # keeps the memory alive while the group exists
        self.numels = numels
        ptrs = (ctypes.c_void_p * len(flat))(*[t.data_ptr() if t.numel() else None for t in flat])
        arr = (ctypes.c_int64 * T)(*numels)
        h = ctypes.c_void_p()
        _check(LIB.tc_group_create(comm.h, T, ptrs, arr, ctypes.byref(h)), "tc_group_create")
        self.h = h
        comm.groups += 1

    def set_num_ctas(self, num_ctas: int):
        """CTA budget of this group's launches (0 = the comm's tuning); identical on all ranks."""
        _check(LIB.tc_group_set_num_ctas(self.h, int(num_ctas)), "tc_group_set_num_ctas")

    def destroy(self):
        if self.h:
            st = LIB.tc_group_destroy(self.h)
            self.h = None
            self.comm.groups -= 1
            _check(st, "tc_group_destroy")

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()


def allreduce(x: Group, scale: float = 1.0, stream=None):
    _check(LIB.tc_allreduce(x.h, float(scale), _stream_ptr(stream)), "tc_allreduce")


def sgd_step(w: Group, g: Group, dw: Group, lr: float, momentum: float = 0.0, wd: float = 0.0,
             rescale: float = 1.0, stream=None):
    _check(LIB.tc_sgd_step(w.h, g.h, dw.h, float(lr), float(momentum), float(wd), float(rescale),
                           _stream_ptr(stream)), "tc_sgd_step")


def easgd_update(x: Group, center: Group, alpha: float, stream=None):
    _check(LIB.tc_easgd_update(x.h, center.h, float(alpha), _stream_ptr(stream)),
           "tc_easgd_update")


def easgd_async_update(x: Group, center: Group, alpha: float, order=None, stream=None):
    """NEXT row f2: server-side Elastic1 per client arrival in `order` (a permutation of the
    clients; None = client order), Elastic2 at each client."""
    arr = None
    if order is not None:
        arr = (_c_int * len(order))(*[int(i) for i in order])
    _check(LIB.tc_easgd_async_update(x.h, center.h, float(alpha), arr, _stream_ptr(stream)),
           "tc_easgd_async_update")


def broadcast(x: Group, root: int = 0, stream=None):
    """Every rank's group := the root's (weight initialisation)."""
    _check(LIB.tc_broadcast(x.h, int(root), _stream_ptr(stream)), "tc_broadcast")


def esgd_step(x: Group, center: Group, g: Group, dw: Group, alpha: float, lr: float,
              momentum: float = 0.0, wd: float = 0.0, rescale: float = 1.0, stream=None):
    """NEXT row f2: elastic update then SGD-momentum with this rank's own gradient, one pass."""
    _check(LIB.tc_esgd_step(x.h, center.h, g.h, dw.h, float(alpha), float(lr), float(momentum),
                            float(wd), float(rescale), _stream_ptr(stream)), "tc_esgd_step")


class BucketedStep:
    """Bucketed, overlapped step (NEXT row f1).

    The gradient group is split into buckets (tc_plan_buckets, backward order).  After the
    backward pass has produced every gradient of a bucket (``grad_ready(t)`` for each of its
    tensors, called on the compute stream in production order), the bucket's collective is
    enqueued on a side stream behind an event, so it overlaps the backward computation of later
    layers.  ``finish()`` makes the compute stream wait for all buckets.  All ranks must produce
    the gradients in the same order (the bucket calls are collective).

    fused (split=False): each bucket runs tc_sgd_step (allreduce + update in one kernel), or
    tc_allreduce when w/dw are None.
    split (split=True): each bucket runs only tc_allreduce (link-bound, few SMs suffice:
    ``ctas``), and finish() runs the SGD update once over the whole group as a local HBM
    stream (tc_sgd_step on a single-rank comm).  Bit-identical to the fused step on the P2P
    algorithms: the allreduce rounds the float64 sum once and the local step's "sum" of one rank
    is that value.  (With switch reduction -- NVLS, tc_comm_set_switch_reduction / algorithm 4 --
    both are within the NVLS tolerance instead, and identical on every rank.)
    """

    # defaults from a graph-captured ResNet-50 backward on B200 (bench_train.py):
    # 25 MiB buckets, a 48-CTA budget and a highest-priority side stream hid 0.44 / 0.49 of the
    # step at p = 4 with 8 / 4 images per GPU (the full grid hid none: the buckets then take SMs
    # the backward's next kernels need)
    def __init__(self, comm, g, w=None, dw=None, bucket_bytes=25 << 20, stream=None, ctas=48,
                 split=False):
        import torch
        numels = [t.numel() for t in (g[0] if comm.is_emulated else g)]
        plan = Plan(numels)
        self.bucket_of, self.nbuckets = plan.buckets(bucket_bytes)
        self.comm = comm
        self.stream = stream or torch.cuda.Stream(priority=torch.cuda.Stream.priority_range()[1])
        members = [[] for _ in range(self.nbuckets)]
        for t in range(len(numels)):
            members[self.bucket_of[t]].append(t)
        self.members = members

        def pick(ts, idx):
            return [[x[i] for i in idx] for x in ts] if comm.is_emulated else [ts[i] for i in idx]

        self.split = bool(split) and w is not None
        self.G = [Group(comm, pick(g, m)) for m in members]
        self.W = self.D = None
        self.local = []
        if self.split:
            # the update after the last bucket: one local HBM stream per rank of this process
            self.lcomm = Comm.single(g[0][0].device.index if comm.is_emulated
                                     else g[0].device.index)
            ranks = range(comm.nranks) if comm.is_emulated else [None]
            for k in ranks:
                sel = (lambda x: x[k]) if k is not None else (lambda x: x)
                self.local.append((Group(self.lcomm, sel(w)), Group(self.lcomm, sel(g)),
                                   Group(self.lcomm, sel(dw))))
        elif w is not None:
            self.W = [Group(comm, pick(w, m)) for m in members]
            self.D = [Group(comm, pick(dw, m)) for m in members]
        self.ctas = ctas
        if ctas:  # the CTA budget applies to the bucket launches only (per group, not the comm)
            for grp in self.G:
                grp.set_num_ctas(ctas)
        self.hp = {}
        self.reset()

    def reset(self):
        self.missing = [len(m) for m in self.members]

    def grad_ready(self, t, compute_stream=None, **hp):
        """Tensor t's gradient has been written (on compute_stream).  Launches its bucket's
        collective when it was the bucket's last tensor."""
        b = self.bucket_of[t]
        self.missing[b] -= 1
        if self.missing[b]:
            self.hp = hp
            return
        self.bucket_ready(b, compute_stream, **hp)

    def bucket_ready(self, b, compute_stream=None, **hp):
        """Every gradient of bucket b has been written (on compute_stream): launch its collective
        on the side stream behind an event.  The caller must know that all of them are written
        (grad_ready counts them); calling it early races the collective with the backward pass."""
        import torch
        self.hp = hp
        self.missing[b] = 0
        ev = torch.cuda.Event()
        ev.record(compute_stream or torch.cuda.current_stream())
        self.stream.wait_event(ev)
        if self.W is not None:
            sgd_step(self.W[b], self.G[b], self.D[b], stream=self.stream, **hp)
        else:
            allreduce(self.G[b], 1.0 if self.split else hp.get("scale", 1.0), stream=self.stream)

    def finish(self, compute_stream=None):
        import torch
        for W, G, D in self.local:
            sgd_step(W, G, D, stream=self.stream, **self.hp)
        ev = torch.cuda.Event()
        ev.record(self.stream)
        (compute_stream or torch.cuda.current_stream()).wait_event(ev)
        self.reset()

    def destroy(self):
        for gs in (self.G, self.W or [], self.D or [], [x for t in self.local for x in t]):
            for grp in gs:
                grp.destroy()
        if self.local:
            self.lcomm.destroy()
