#!/usr/bin/env python
"""Latency probe for the 0.25-4 MiB range (DESIGN.md §12 "Latency at 1 MiB, p = 4").

    torchrun --nproc-per-node N tools/latency_probe.py

For each total size and tensor count: the automatic choice, the one-shot at several CTA counts
and block sizes, the low-latency (LL) path forced, the TMA two-shot forced, and NCCL on the flat
buffer -- each as a CUDA-graph replay timed with CUDA events (max over ranks, us).  Rank 0 prints
one JSON line per cell.
"""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402
from bench_sweep import timed  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, p = dist.get_rank(), dist.get_world_size()
    comm = tc.Comm.from_process_group(device=local)
    big = 64 << 20
    variants = [("auto", 0, 0, 0, -1, -1), ("ll", 0, 0, 0, -1, big),
                ("tma", 6, 0, 0, 0, 0), ("oneshot", 0, 0, 0, big, 0)]
    if os.environ.get("LAT_SHAPES"):
        for ctas in (16, 32, 64, 96, 148):
            for thr in (256, 512):
                variants.append((f"oneshot_c{ctas}_t{thr}", 0, ctas, thr, big, 0))
    sizes = [int(x) << 10 for x in os.environ.get(
        "LAT_KIB", "16,64,256,512,1024,2048,4096,8192,16384").split(",")]
    for total in sizes:
        N = total // 4
        flat = torch.randn(N, device="cuda")
        nccl_buf = torch.randn(N, device="cuda")
        t_nccl = timed(lambda: dist.all_reduce(nccl_buf), 200, graph=True)
        for T in (1, 161):
            numels = W.sweep_numels(total, T)
            views = list(torch.split(flat, numels))
            rec = {"p": p, "T": T, "bytes": total, "nccl_us": round(t_nccl, 2)}
            with tc.Group(comm, views) as g:
                for name, algo, ctas, thr, os_lim, ll in variants:
                    comm.set_algorithm(algo)
                    comm.set_tuning(ctas, thr, os_lim)
                    comm.set_ll_max(ll)
                    try:
                        t = timed(lambda: tc.allreduce(g, 1.0 / p,
                                                       stream=torch.cuda.current_stream()),
                                  200, graph=True)
                        rec[name] = [round(t, 2), comm.last_launch()[0]]
                    except tc.TcError as e:  # e.g. a launch shape the path rejects
                        rec[name] = str(e)
            comm.set_algorithm(0)
            comm.set_tuning(0, 0, -1)
            comm.set_ll_max(-1)
            if rank == 0:
                print(json.dumps(rec), flush=True)
        del flat, nccl_buf
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
