#!/usr/bin/env python
"""Config 5 (BASELINE.json): tensor-group shape sweep, libtc vs NCCL on the flattened buffer.

    torchrun --nproc-per-node N bench_sweep.py [--out FILE]

T in {1, 2, 8, 32, 161, 512, 1024} tensors, total size 1 KiB * 4^k (k = 0..10: 1 KiB .. 1 GiB,
including the paper's 4/16/64 MiB), per-tensor sizes a seeded log-uniform split with
unaligned tails (tc_workloads.sweep_numels).  Per cell: tc_allreduce on the T tensors (scale
1/p keeps the values fixed) and torch.distributed NCCL all_reduce on one flat buffer of the same
N fp32, each timed with CUDA events (max over ranks).  Rank 0 prints one JSON line per cell.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402


def timed(fn, iters, warm=3, graph=False):
    """Device time per call (us, max over ranks).  graph=True captures `iters` calls in one CUDA
    graph and times a replay, removing host launch overhead (both libtc and NCCL capture)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
            fn()
    torch.cuda.synchronize()
    g = None
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(iters):
                fn()
        g.replay()
        torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        if g is not None:
            g.replay()
        else:
            for _ in range(iters):
                fn()
        e1.record(s)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t) * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--max-k", type=int, default=10)
    ap.add_argument("--algo", type=int, default=0, help="0 auto, 1 pull, 3 push, 4 NVLS")
    ap.add_argument("--oneshot", type=int, default=-1, help="one-shot limit in bytes (-1 auto)")
    ap.add_argument("--sizes", default="", help="comma list of k (total = 1 KiB * 4^k)")
    ap.add_argument("--ll", type=int, default=-1, help="low-latency limit in bytes (-1 auto)")
    ap.add_argument("--tensors", default="1,2,8,32,161,512,1024")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, p = dist.get_rank(), dist.get_world_size()
    comm = tc.Comm.from_process_group(device=local)
    comm.set_algorithm(a.algo)
    comm.set_tuning(0, 0, a.oneshot)
    comm.set_ll_max(a.ll)
    out = open(a.out, "w") if (a.out and rank == 0) else None
    ks = [int(x) for x in a.sizes.split(",")] if a.sizes else range(a.max_k + 1)
    for k in ks:
        total = 1024 * 4 ** k
        N = total // 4
        flat = torch.randn(N, device="cuda")
        nccl_buf = torch.randn(N, device="cuda")
        iters = 200 if total <= (1 << 20) else (50 if total <= (64 << 20) else 5)
        graph = total <= (64 << 20)
        t_nccl = timed(lambda: dist.all_reduce(nccl_buf), iters, graph=graph)
        for T in [int(x) for x in a.tensors.split(",")]:
            numels = W.sweep_numels(total, T)
            if not numels:
                continue
            views = list(torch.split(flat, numels))
            with tc.Group(comm, views) as g:
                t_tc = timed(lambda: tc.allreduce(g, 1.0 / p,
                                                  stream=torch.cuda.current_stream()),
                             iters, graph=graph)
                algo = comm.last_launch()[0]
            rec = {"p": p, "T": T, "bytes": total, "tc_us": t_tc, "nccl_us": t_nccl,
                   "cuda_graph": graph,
                   "tc_busbw_gbs": total * 2 * (p - 1) / p / t_tc / 1e3,
                   "nccl_busbw_gbs": total * 2 * (p - 1) / p / t_nccl / 1e3,
                   "speedup_vs_nccl": t_nccl / t_tc, "algo": algo}
            if rank == 0:
                line = json.dumps(rec)
                print(line, flush=True)
                if out:
                    out.write(line + "\n")
        del flat, nccl_buf
        torch.cuda.empty_cache()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
