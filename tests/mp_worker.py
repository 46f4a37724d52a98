"""Multi-process parity worker: one rank per GPU, launched by torchrun (test_gpu_multiproc.py).

Every rank regenerates every rank's seeded inputs, so each rank checks its own outputs against
the CPU oracle independently; a failure raises (non-zero exit code).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402
from oracle import tc_oracle as O  # noqa: E402
from gpu_util import to_dev, to_host, assert_bitwise  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, p = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    comm = tc.Comm.from_process_group(device=local)
    assert comm.rank == rank and comm.nranks == p

    # allreduce: tiny config (integer), both algorithms; ragged grad-valued groups
    cases = [(W.TINY, "int", 0), (W.TINY, "int", 1 << 20),
             ([7, 13, 1000, 0, 50001, 3, 262144], "grad", 0),
             ([7, 13, 1000, 0, 5001, 3], "grad", 1 << 20)]
    for (numels, kind, oneshot), algo in [(c, a) for c in cases for a in (1, 5, 6)]:
        comm.set_tuning(0, 0, oneshot)
        comm.set_ll_max(1 << 30 if algo == 5 else 0)
        comm.set_algorithm(algo if algo != 5 else 0)
        xs = [W.group(numels, kind, 60, 0, k, W.GRAD) for k in range(p)]
        dev = to_dev(xs[rank])
        with tc.Group(comm, dev) as g:
            tc.allreduce(g)
            assert_bitwise(to_host(dev), O.allreduce(xs), f"allreduce {numels[:4]} rank {rank}")
        assert comm.async_error() == 0

    # SGD (fused) and EASGD, two-shot and one-shot
    for oneshot, algo in ((0, 1), (1 << 20, 0), (0, 5), (0, 6)):
        comm.set_tuning(0, 0, oneshot)
        comm.set_ll_max(1 << 30 if algo == 5 else 0)
        comm.set_algorithm(algo if algo != 5 else 0)
        numels = [7, 13, 1000, 4096, 65]
        gs = [W.group(numels, "grad", 61, 0, k, W.GRAD) for k in range(p)]
        w = W.group(numels, "param", 61, 0, 0, W.PARAM)
        dw = W.group(numels, "dw", 61, 0, 0, W.DW)
        dg, dwt, ddw = to_dev(gs[rank]), to_dev(w), to_dev(dw)
        hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (p * 128))
        with tc.Group(comm, dg) as G, tc.Group(comm, dwt) as Wg, tc.Group(comm, ddw) as D:
            tc.sgd_step(Wg, G, D, **hp)
            Gw, Ws, Dws = O.sgd_step([w] * p, gs, [dw] * p, **hp)
            assert_bitwise(to_host(dg), Gw, "sgd g")
            assert_bitwise(to_host(dwt), Ws[rank], "sgd w")
            assert_bitwise(to_host(ddw), Dws[rank], "sgd dw")
        center = W.group(numels, "center", 62, 0, 0, W.CENTER)
        xs = [W.client_params(numels, center, 62, 0, i) for i in range(p)]
        dx, dc = to_dev(xs[rank]), to_dev(center)
        with tc.Group(comm, dx) as X, tc.Group(comm, dc) as C:
            tc.easgd_update(X, C, 0.1)
            wx, wc = O.easgd_update(xs, center, 0.1)
            assert_bitwise(to_host(dx), wx[rank], "easgd x")
            assert_bitwise(to_host(dc), wc, "easgd center")
        assert comm.async_error() == 0

    # a pointer CUDA IPC cannot export (pinned host memory on rank 0): every rank gets
    # TC_ERR_NOT_SHAREABLE from the collective tc_group_create
    import ctypes
    host = torch.zeros(1024, dtype=torch.float32).pin_memory()
    devt = torch.zeros(1024, dtype=torch.float32, device="cuda")
    ptr = host.data_ptr() if rank == 0 else devt.data_ptr()
    out = ctypes.c_void_p()
    st = tc.LIB.tc_group_create(comm.h, 1, (ctypes.c_void_p * 1)(ptr),
                                (ctypes.c_int64 * 1)(1024), ctypes.byref(out))
    assert st == tc.tc.TC_ERR_NOT_SHAREABLE, st
    assert not out.value

    # tensor broadcast from the last rank
    numels = [7, 13, 1000, 0, 50001]
    xs = [W.group(numels, "grad", 64, 0, k, W.GRAD) for k in range(p)]
    dev = to_dev(xs[rank])
    with tc.Group(comm, dev) as g:
        tc.broadcast(g, p - 1)
        assert_bitwise(to_host(dev), O.broadcast(xs, p - 1)[rank], "broadcast")
    assert comm.async_error() == 0

    # NEXT row f2: fused elastic + SGD with each rank's own gradient (one GPU per client)
    comm.set_tuning(0, 0, -1)
    comm.set_ll_max(-1)
    comm.set_algorithm(0)
    numels = [7, 13, 1000, 4096, 65, 30001]
    center = W.group(numels, "center", 63, 0, 0, W.CENTER)
    xs = [W.client_params(numels, center, 63, 0, i) for i in range(p)]
    gs = [W.group(numels, "grad", 63, 1, i, W.GRAD) for i in range(p)]
    dws = [W.group(numels, "dw", 63, 2, i, W.DW) for i in range(p)]
    hp = dict(alpha=0.1, lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / 128)
    dx, dc, dg, dd = to_dev(xs[rank]), to_dev(center), to_dev(gs[rank]), to_dev(dws[rank])
    with tc.Group(comm, dx) as X, tc.Group(comm, dc) as C, tc.Group(comm, dg) as G, \
            tc.Group(comm, dd) as D:
        tc.esgd_step(X, C, G, D, **hp)
        wx, wc, wd = O.esgd_step(xs, center, gs, dws, **hp)
        assert_bitwise(to_host(dx), wx[rank], "esgd x")
        assert_bitwise(to_host(dc), wc, "esgd center")
        assert_bitwise(to_host(dd), wd[rank], "esgd dw")
    assert comm.async_error() == 0

    # NEXT row f2, asynchronous server: arrivals in a recorded order, owners store every
    # client's new chunk into the client's tensor over NVLink
    order = list(reversed(range(p)))
    dx, dc = to_dev(xs[rank]), to_dev(center)
    with tc.Group(comm, dx) as X, tc.Group(comm, dc) as C:
        tc.easgd_async_update(X, C, 0.1, order)
        wx, wc = O.easgd_async(xs, center, 0.1, order)
        assert_bitwise(to_host(dx), wx[rank], "easgd_async x")
        assert_bitwise(to_host(dc), wc, "easgd_async center")
    assert comm.async_error() == 0

    # symmetric (tc_mem_alloc) memory: P2P algorithms bit-exact; NVLS (switch reduction) exact on
    # integers, within the BASELINE tolerance on gradients, identical on every rank
    numels = [7, 13, 1000, 0, 50001, 3, 262144]
    sym = comm.alloc_symmetric(sum(numels) + 64)
    views = list(torch.split(sym[:sum(numels)], numels))
    algos = [1, 6] + ([4] if comm.multicast_supported else [])
    comm.set_tuning(0, 0, 0)
    comm.set_ll_max(0)
    with tc.Group(comm, views) as g:
        # NVLS allreduce also on small CTAs (the comm's thread count: 2 and 4 warps, 1 and 3
        # reducing) and a partial grid -- the launch shapes a co-running bucket uses (f1)
        runs = [(a, c, t) for a in algos for c, t in ([(0, 0)] + ([(0, 128), (32, 64)]
                                                                  if a == 4 else []))]
        for algo, ctas, thr in runs:
            comm.set_algorithm(algo)
            comm.set_tuning(ctas, thr, 0)
            for kind in ("int", "grad"):
                xs = [W.group(numels, kind, 63, 0, k, W.GRAD) for k in range(p)]
                for v, a in zip(views, xs[rank]):
                    v.copy_(torch.from_numpy(a))
                tc.allreduce(g)
                assert comm.last_launch()[0] == tc.tc.ALGO_NAMES[algo]
                if algo == 4:
                    assert comm.last_launch()[2] == (thr or 512), comm.last_launch()
                got = to_host(views)
                if algo != 4 or kind == "int":
                    assert_bitwise(got, O.allreduce(xs), f"sym allreduce algo {algo} {kind}")
                else:
                    ref = O.allreduce_f64(xs)
                    for t, n in enumerate(numels):
                        bound = 1e-5 * sum(np.abs(xs[k][t].astype(np.float64)) for k in range(p))
                        assert (np.abs(got[t] - ref[t]) <= bound).all(), f"nvls tolerance t={t}"
                    # every rank holds the same bits
                    import hashlib
                    dig = hashlib.sha256(b"".join(a.tobytes() for a in got)).digest()
                    h = torch.tensor([int.from_bytes(dig[:7], "little")])
                    hs = [torch.zeros_like(h) for _ in range(p)]
                    dist.all_gather(hs, h)
                    assert all(int(x) == int(hs[0]) for x in hs), "nvls ranks differ"
        comm.set_tuning(0, 0, 0)
        if comm.multicast_supported:
            # fused SGD over NVLS: G within tolerance, epilogue bit-exact given G
            comm.set_algorithm(4)
            gs = [W.group(numels, "grad", 64, 0, k, W.GRAD) for k in range(p)]
            w = W.group(numels, "param", 64, 0, 0, W.PARAM)
            dw = W.group(numels, "dw", 64, 0, 0, W.DW)
            for v, a in zip(views, gs[rank]):
                v.copy_(torch.from_numpy(a))
            dwt, ddw = to_dev(w), to_dev(dw)
            hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (p * 128))
            with tc.Group(comm, dwt) as Wg, tc.Group(comm, ddw) as D:
                tc.sgd_step(Wg, g, D, **hp)
                assert comm.last_launch()[0] == "nvls"
                G = to_host(views)
                ref = O.allreduce_f64(gs)
                for t in range(len(numels)):
                    bound = 1e-5 * sum(np.abs(gs[k][t].astype(np.float64)) for k in range(p))
                    assert (np.abs(G[t] - ref[t]) <= bound).all()
                _, Ws, Dws = O.sgd_step([w], [G], [dw], **hp)
                assert_bitwise(to_host(dwt), Ws[0], "nvls sgd w")
                assert_bitwise(to_host(ddw), Dws[0], "nvls sgd dw")
        # tensor broadcast through the switch (a copy: bit-exact), chosen automatically for a
        # multicast-bound group; the TMA scatter + allgather when forced
        mc = comm.multicast_supported
        for algo, want in ((0, "nvls" if mc and p >= 4 else "two-shot-tma"),
                           (4, "nvls" if mc else "two-shot-tma"), (6, "two-shot-tma")):
            comm.set_algorithm(algo)
            xs = [W.group(numels, "grad", 65, algo, k, W.GRAD) for k in range(p)]
            for v, a in zip(views, xs[rank]):
                v.copy_(torch.from_numpy(a))
            tc.broadcast(g, p - 1)
            assert comm.last_launch()[0] == want, comm.last_launch()
            assert_bitwise(to_host(views), O.broadcast(xs, p - 1)[rank], f"broadcast {want}")
        comm.set_algorithm(0)
        # tc_mem_free refuses while a live group still points into the allocation
        st = tc.LIB.tc_mem_free(comm.h, sym.data_ptr())
        assert st == tc.tc.TC_ERR_INVALID_ARG, st
    comm.free_symmetric(sym)
    assert comm.async_error() == 0
    if rank == 0:
        print(f"symmetric memory: algorithms {algos} ok (multicast={comm.multicast_supported})",
              flush=True)

    # full-size ResNet-50 gradient group, fused SGD, on the kernel bench.py times at N = p (the
    # automatic choice: TMA two-shot on the full 148-CTA grid), whole arrays vs the oracle
    comm.set_tuning(0, 0, -1)
    comm.set_ll_max(-1)
    comm.set_algorithm(0)
    numels = W.RESNET50
    gs = [W.group(numels, "grad", W.CFG_RESNET50, 0, k, W.GRAD) for k in range(p)]
    w = W.group(numels, "param", W.CFG_RESNET50, 0, 0, W.PARAM)
    dw = W.group(numels, "dw", W.CFG_RESNET50, 0, 0, W.DW)
    dg, dwt, ddw = to_dev(gs[rank]), to_dev(w), to_dev(dw)
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (p * 128))
    with tc.Group(comm, dg) as G, tc.Group(comm, dwt) as Wg, tc.Group(comm, ddw) as D:
        tc.sgd_step(Wg, G, D, **hp)
        algo, ctas, _ = comm.last_launch()
        assert algo == "two-shot-tma", algo
        hg, hw, hd = to_host(dg), to_host(dwt), to_host(ddw)
    Gw, Ws, Dws = O.sgd_step([w], gs, [dw], **hp)
    assert_bitwise(hg, Gw, "resnet50 g")
    assert_bitwise(hw, Ws[0], "resnet50 w")
    assert_bitwise(hd, Dws[0], "resnet50 dw")
    if rank == 0:
        print(f"full-size resnet50 sgd_step: {algo} on {ctas} CTAs per rank, whole arrays "
              "bit-exact", flush=True)
    assert comm.async_error() == 0
    comm.destroy()
    dist.barrier()
    if rank == 0:
        print(f"MP_WORKER_OK p={p}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
