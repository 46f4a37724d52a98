"""Quick per-algorithm timing on the ResNet-50 group (diagnostics, not the bench contract).

    torchrun --nproc-per-node N tools/algo_bench.py [--algos 6,4] [--steps 50] [--ops ar,sgd,bc,ea]

Gradients in tc_mem_alloc memory (NVLS-eligible), refreshed before every fused step; CUDA events
around each kernel, max over ranks.  One JSON line per (op, algo) on rank 0.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algos", default="6,4")
    ap.add_argument("--ops", default="ar,sgd")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--config", default="resnet50")
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0, help="register kernels / NVLS allreduce")
    a = ap.parse_args()
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    numels = W.GROUPS[a.config]
    S = 4 * sum(numels)
    comm = tc.Comm.from_process_group(device=local)
    comm.set_tuning(a.ctas, a.threads, -1)
    pristine = torch.from_numpy(np.concatenate(W.group(numels, "grad", 2, 0, rank, W.GRAD))).cuda()
    g_flat = comm.alloc_symmetric(sum(numels))
    g_flat.copy_(pristine)
    w = torch.from_numpy(np.concatenate(W.group(numels, "param", 2, 0, 0, W.PARAM))).cuda()
    dw = torch.from_numpy(np.concatenate(W.group(numels, "dw", 2, 0, 0, W.DW))).cuda()
    split = lambda f: list(torch.split(f, numels))  # noqa: E731
    G, Wg, D = tc.Group(comm, split(g_flat)), tc.Group(comm, split(w)), tc.Group(comm, split(dw))
    center = torch.from_numpy(np.concatenate(W.group(numels, "param", 3, 0, 0, W.PARAM))).cuda()
    C = tc.Group(comm, split(center))
    s = torch.cuda.Stream()
    for op in a.ops.split(","):
        for algo in [int(x) for x in a.algos.split(",")]:
            comm.set_algorithm(algo)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(a.steps)]
            with torch.cuda.stream(s):
                for i in range(5 + a.steps):
                    g_flat.copy_(pristine)
                    if i >= 5:
                        ev[i - 5][0].record(s)
                    if op == "ar":
                        tc.allreduce(G, 1.0 / p, stream=s)
                    elif op == "bc":
                        tc.broadcast(G, 0, stream=s)
                    elif op == "ea":  # elastic averaging, one client per rank (c = p)
                        tc.easgd_update(Wg, C, 0.1, stream=s)
                    else:
                        tc.sgd_step(Wg, G, D, lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (128 * p),
                                    stream=s)
                    if i >= 5:
                        ev[i - 5][1].record(s)
                s.synchronize()
            ts = sorted(x.elapsed_time(y) * 1e3 for x, y in ev)
            t = torch.tensor([ts[len(ts) // 2], sum(ts) / len(ts)], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            name, ctas, thr = comm.last_launch()
            if rank == 0:
                print(json.dumps({"p": p, "op": op, "algo": name, "ctas": ctas, "threads": thr,
                                  "median_us": t[0].item(),
                                  "mean_us": t[1].item(),
                                  "busbw_gbs": 2 * (p - 1) / p * S / t[1].item() / 1e3}), flush=True)
    for grp in (G, Wg, D, C):
        grp.destroy()
    comm.free_symmetric(g_flat)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
