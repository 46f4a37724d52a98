"""Per-phase timing of the two-shot kernel from in-kernel %globaltimer stamps (diagnostics).

    torchrun --nproc-per-node N tools/phase_probe.py [--config resnet50] [--ctas C] [--threads T]

Prints, per rank and op, the median / max over CTAs of: entry barrier, reduce-scatter, mid
barrier, allgather, exit barrier, and the kernel span (first start -> last end).
"""
import argparse
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
    ap.add_argument("--config", default="resnet50")
    ap.add_argument("--numel", type=int, default=0, help="one flat tensor of this many elements")
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--algo", type=int, default=1)
    ap.add_argument("--oneshot", type=int, default=0, help="one-shot limit in bytes (-1 auto)")
    ap.add_argument("--sym", action="store_true", help="gradients in tc_mem_alloc memory")
    ap.add_argument("--smid", action="store_true", help="TMA two-shot: RS time by SM")
    a = ap.parse_args()
    dist.init_process_group("gloo")
    rank, p = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    numels = W.GROUPS[a.config] if a.numel <= 0 else [a.numel]
    S = 4 * sum(numels)

    def flat(kind, role):
        f = torch.from_numpy(np.concatenate(W.group(numels, kind, 2, 0, rank, role))).cuda()
        return list(torch.split(f, numels))

    g, w, dw = flat("grad", W.GRAD), flat("param", W.PARAM), flat("dw", W.DW)
    comm = tc.Comm.from_process_group(device=local)
    if a.sym:
        sym = comm.alloc_symmetric(sum(numels))
        sym.copy_(torch.cat(g))
        g = list(torch.split(sym, numels))
    comm.set_tuning(a.ctas, a.threads, a.oneshot)
    comm.set_algorithm(a.algo)
    prof = torch.zeros(1024 * 8, dtype=torch.int64, device="cuda")
    G, Wg, D = tc.Group(comm, g), tc.Group(comm, w), tc.Group(comm, dw)
    names = (["entry", "reduce", "signal", "epilogue/wait", "end"] if a.algo == 4 else
             ["entry", "RS", "mid", "AG", "exit"])
    for op in ("allreduce", "sgd"):
        comm.set_profile_buffer(None)
        for i in range(a.iters):
            if i == a.iters - 1:
                comm.set_profile_buffer(prof)
            if op == "allreduce":
                tc.allreduce(G, 1.0 / p)
            else:
                tc.sgd_step(Wg, G, D, lr=1e-3, momentum=0.9, wd=0.0, rescale=1.0 / p)
        torch.cuda.synchronize()
        _, ctas, thr = comm.last_launch()
        t = prof[: ctas * 8].view(ctas, 8).cpu().numpy().astype(np.int64)
        d = np.diff(t[:, :6], axis=1) / 1e3
        span = (t[:, 5].max() - t[:, 0].min()) / 1e3
        line = " ".join(f"{n}={np.median(d[:, i]):7.1f}/{d[:, i].max():7.1f}" for i, n in enumerate(names))
        if a.algo == 4 and op == "sgd":  # NVLS: epilogue of the own chunk / the next one done
            line += (f" | epilogue of round 0 done at {np.median(t[:, 6] - t[:, 1]) / 1e3:7.1f}"
                     f", round 1 at {np.median(t[:, 7] - t[:, 1]) / 1e3:7.1f} (from entry)")
        if a.algo == 6:  # TMA two-shot: producer waiting for free stages / consumers for data
            wf = t[:, 7] & ((1 << 40) - 1)
            smid = t[:, 7] >> 40
            line += (f" | wait_empty={np.median(t[:, 6]) / 1e3:7.1f}"
                     f" wait_full={np.median(wf) / 1e3:7.1f}")
            if a.smid:
                rs = d[:, 1]
                order = np.argsort(rs)
                line += ("\n   RS by SM (fast..slow): " +
                         " ".join(f"{smid[i]}:{rs[i]:.0f}" for i in order[::max(1, len(order) // 24)]) +
                         f"\n   mean RS on SMs < 74: {rs[smid < 74].mean():.1f}, >= 74: {rs[smid >= 74].mean():.1f}"
                         f"; even SM: {rs[smid % 2 == 0].mean():.1f}, odd: {rs[smid % 2 == 1].mean():.1f}")
        msg = (f"rank {rank} algo{a.algo} {op:9s} ctas={ctas} thr={thr} span={span:7.1f}us "
               f"(busbw@span {S * 2 * (p - 1) / p / span / 1e3:6.1f} GB/s) | med/max us: {line}")
        for r in range(p):
            dist.barrier()
            if r == rank:
                print(msg, flush=True)
    comm.set_profile_buffer(None)
    for grp in (G, Wg, D):
        grp.destroy()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
