#!/usr/bin/env python
"""Benchmark of the tensor-collective hot path (BASELINE.json metric) on 1..8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config resnet50|alexnet|vgg16]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...        # the CPU oracle as the reference arm

A step is one pass of the hot path over one batch of synthetic gradients: tc_sgd_step =
reduce-scatter + allgather of the whole ResNet-50 gradient group (161 tensors, 25.6 M fp32,
102.2 MB per rank) fused with the SGD-momentum update, one kernel.
Each step's gradients are fresh (copied in from a pristine buffer before the step, as a backward
pass would write them); the copy is outside the timed kernel.  Inputs (3 groups, 307 MB per
GPU) exceed the 126 MB L2, so no L2 flush is needed.

value = all ranks' gradient bytes reduced per second = N * S / t_step  (GB/s).  The BASELINE
"bus GB/s" (nccl-tests convention, 2(p-1)/p * S / t per rank) is reported as busbw_gbs and is the
roofline's achieved figure for N >= 2 (bound: NVLink).  At N = 1 there is no communication and
the roofline is HBM (5 S bytes per step).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import tc_workloads as W  # noqa: E402

METRIC = ("tensor-allreduce + fused SGD-momentum step, gradient GB/s reduced (N*S/t; "
          "busbw_gbs = BASELINE bus GB/s), ResNet-50 grad group")
UNIT = "GB/s"
NVLINK_PEER_GBS = 770.0     # B200_PROFILING.md: measured peer copy per direction (900 nominal)
NVLINK_NOMINAL_GBS = 900.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks during timing
class ClockSampler:
    REASONS = {
        "nvmlClocksEventReasonGpuIdle": "gpu_idle",
        "nvmlClocksEventReasonApplicationsClocksSetting": "applications_clocks_setting",
        "nvmlClocksEventReasonSwPowerCap": "sw_power_cap",
        "nvmlClocksEventReasonHwSlowdown": "hw_slowdown",
        "nvmlClocksEventReasonSyncBoost": "sync_boost",
        "nvmlClocksEventReasonSwThermalSlowdown": "sw_thermal_slowdown",
        "nvmlClocksEventReasonHwThermalSlowdown": "hw_thermal_slowdown",
        "nvmlClocksEventReasonHwPowerBrakeSlowdown": "hw_power_brake_slowdown",
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[device_index]) if vis else device_index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for attr, name in self.REASONS.items():
            bit = getattr(nv, attr, 0)
            if bit and mask & bit and name != "gpu_idle":
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                return
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self.nv:
            self._stop.set()
            self._t.join()
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                pass

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ distributed helpers
def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


# ------------------------------------------------------------------ CPU oracle baseline
def cpu_baseline_sgd(numels, p, budget_s=12.0, max_steps=20):
    """The oracle as it stands (numpy, one thread) on the same workload: sgd_step over p
    simulated ranks.  Bounded: the full group when it fits the time budget, else a contiguous
    prefix of the group's tensors."""
    from oracle import tc_oracle as O
    gs = [W.group(numels, "grad", W.CFG_RESNET50, 0, k, W.GRAD) for k in range(p)]
    w = W.group(numels, "param", W.CFG_RESNET50, 0, 0, W.PARAM)
    dw = W.group(numels, "dw", W.CFG_RESNET50, 0, 0, W.DW)
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (p * 128))
    t0 = time.perf_counter()
    steps = 0
    while steps < max_steps and (time.perf_counter() - t0) < budget_s:
        O.sgd_step([w] * p, gs, [dw] * p, **hp)
        steps += 1
    dt = (time.perf_counter() - t0) / steps
    S = 4 * sum(numels)
    return {"value": p * S / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"full group ({len(numels)} tensors, {S/1e6:.1f} MB/rank) x {p} ranks, "
                      f"{steps} oracle steps, {dt:.3f} s/step"}


# ------------------------------------------------------------------ the reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import tc_oracle as O
    p = max(args.gpus, 1)
    numels = W.GROUPS[args.config]
    # bounded sample per step: a prefix of the group of at most 4 M elements
    sample, tot = [], 0
    for n in numels:
        if tot + n > 4_000_000 and sample:
            break
        sample.append(n)
        tot += n
    gs = [W.group(sample, "grad", W.CFG_RESNET50, 0, k, W.GRAD) for k in range(p)]
    w = W.group(sample, "param", W.CFG_RESNET50, 0, 0, W.PARAM)
    dw = W.group(sample, "dw", W.CFG_RESNET50, 0, 0, W.DW)
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (p * 128))
    for _ in range(args.warmup):
        O.sgd_step([w] * p, gs, [dw] * p, **hp)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.sgd_step([w] * p, gs, [dw] * p, **hp)
    dt = (time.perf_counter() - t0) / args.steps
    S = 4 * tot
    v = p * S / dt / 1e9
    desc = (f"prefix of {len(sample)} of {len(numels)} {args.config} tensors ({S/1e6:.1f} MB/rank) "
            f"x {p} simulated ranks per step")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": f"{args.config} grad group, oracle sgd_step",
                                        "p": p, "sample": desc},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------ the product arm
def config4_sequence(args, p, rank, local, numels, dev, ecomm, cen, stream, timed_calls):
    """BASELINE config 4 (MPI Elastic SGD, Fig. code-snippet-4): 2 clients of p/2 GPUs each;
    every step each client runs the fused allreduce + SGD over its GPUs, and every tau = 4 steps
    the counterpart pairs (k, k + p/2) first run the elastic update of the client parameters
    (P:309-313).  Reports the mean step over 16 steps (4 elastic updates)."""
    import torch.distributed as dist
    import paper_1801_03855_b200 as tc
    half = p // 2
    mine = None
    for c in range(2):
        grp = dist.new_group(list(range(c * half, (c + 1) * half)), backend="gloo")
        if rank // half == c:
            mine = grp
    ccomm = tc.Comm.single(local) if half == 1 else tc.Comm.from_process_group(mine, device=local)
    _, w4 = dev(W.group(numels, "param", W.CFG_EASGD, 3, rank // half, W.PARAM))
    _, g4 = dev(W.group(numels, "grad", W.CFG_EASGD, 4, rank, W.GRAD))
    _, d4 = dev(W.group(numels, "dw", W.CFG_EASGD, 5, rank // half, W.DW))
    W4, G4, D4 = tc.Group(ccomm, w4), tc.Group(ccomm, g4), tc.Group(ccomm, d4)
    X4 = tc.Group(ecomm, w4)
    C4 = tc.Group(ecomm, cen)
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (half * 128))
    steps, tau = 16, 4

    def sequence():
        for t in range(steps):
            if t % tau == 0:
                tc.easgd_update(X4, C4, 0.1, stream=stream)
            tc.sgd_step(W4, G4, D4, stream=stream, **hp)

    t_seq = timed_calls(sequence)
    t_sgd = timed_calls(lambda: tc.sgd_step(W4, G4, D4, stream=stream, **hp))
    out = {"clients": 2, "gpus_per_client": half, "tau": tau, "steps": steps,
           "mean_step_us": t_seq / steps, "sgd_step_us": t_sgd,
           "easgd_amortised_us": t_seq / steps - t_sgd,
           "note": "BASELINE config 4: fused allreduce+SGD inside each client every step, "
                   "elastic update across counterpart pairs every tau steps"}
    extra_groups = []
    if half == 1:
        # one GPU per client: the elastic steps can use the fused tc_esgd_step (NEXT row f2)
        G4e, D4e = tc.Group(ecomm, g4), tc.Group(ecomm, d4)
        extra_groups = [G4e, D4e]

        def fused():
            for t in range(steps):
                if t % tau == 0:
                    tc.esgd_step(X4, C4, G4e, D4e, 0.1, stream=stream, **hp)
                else:
                    tc.sgd_step(W4, G4, D4, stream=stream, **hp)

        out["mean_step_fused_us"] = timed_calls(fused) / steps
    for grp in [W4, G4, D4, X4, C4] + extra_groups:
        grp.destroy()
    if ccomm is not None:
        ccomm.destroy()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="tc", choices=["tc", "reference"])
    ap.add_argument("--config", default="resnet50", choices=["resnet50", "alexnet", "vgg16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--algo", type=int, default=0,
                    help="0 auto, 1 two-shot pull, 3 two-shot push, 4 NVLS")
    ap.add_argument("--no-sym", action="store_true",
                    help="keep gradients in torch memory (no NVLS) instead of tc_mem_alloc")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1801_03855_b200 as tc

    p = world
    numels = W.GROUPS[args.config]
    S = 4 * sum(numels)
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (p * 128))
    stream = torch.cuda.Stream()
    def dev(grp):
        """The group's tensors as views of one flat allocation (a gradient bucket, as frameworks
        lay them out); libtc still receives T separate pointers and assumes nothing."""
        flat = torch.from_numpy(np.concatenate(grp)).cuda()
        return flat, list(torch.split(flat, [int(n) for n in numels]))

    gp_flat, g_pristine = dev(W.group(numels, "grad", W.CFG_RESNET50, 0, rank, W.GRAD))
    g_flat, g = dev(W.group(numels, "zeros", 0, 0, 0, 0))
    g_flat.copy_(gp_flat)
    w_flat, w = dev(W.group(numels, "param", W.CFG_RESNET50, 0, 0, W.PARAM))
    dw_flat, dw = dev(W.group(numels, "dw", W.CFG_RESNET50, 0, 0, W.DW))
    torch.cuda.synchronize()

    comm = tc.Comm.single(local) if p == 1 else tc.Comm.from_process_group(device=local)
    comm.set_algorithm(args.algo)
    sym = p > 1 and not args.no_sym
    if sym:
        # the gradient bucket in symmetric multicast memory (tc_mem_alloc): NVLS-eligible
        g_flat = comm.alloc_symmetric(sum(numels))
        g_flat.copy_(gp_flat)
        g = list(torch.split(g_flat, [int(n) for n in numels]))
    G, Wg, D = tc.Group(comm, g), tc.Group(comm, w), tc.Group(comm, dw)
    refresh = p > 1  # at p = 1 the gradient is not modified by the step

    def refresh_g():  # the next batch's gradients (one D2D copy, outside the timed kernel)
        g_flat.copy_(gp_flat, non_blocking=True)

    def step():
        tc.sgd_step(Wg, G, D, stream=stream, **hp)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            if refresh:
                refresh_g()
            step()
    barrier(world)

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(K)]
    with ClockSampler(local) as clocks, torch.cuda.stream(stream):
        barrier(world)
        t_wall0 = time.perf_counter()
        if refresh:
            # per-step events around the kernel: the refresh copy between steps is not timed
            for i in range(K):
                refresh_g()
                ev[i][0].record(stream)
                step()
                ev[i][1].record(stream)
        else:
            # the step is the kernel alone: one event pair around the K back-to-back steps
            ev[0][0].record(stream)
            for i in range(K):
                step()
            ev[0][1].record(stream)
        stream.synchronize()
        barrier(world)
        t_wall = time.perf_counter() - t_wall0
    kernel_ms = (sum(a.elapsed_time(b) for a, b in ev) if refresh
                 else ev[0][0].elapsed_time(ev[0][1])) / K
    t_ms = max_over_ranks(kernel_ms, world)
    algo, ctas, threads = comm.last_launch()
    t_s = t_ms / 1e3
    value = p * S / t_s / 1e9
    algbw = S / t_s / 1e9
    busbw = algbw * 2 * (p - 1) / p if p > 1 else 0.0
    hbm_peak, hbm_src = peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"{args.config}_p{p}_sgd")
    except Exception:  # noqa: BLE001
        pass
    if p == 1:
        hbm_bytes = 5 * S  # read g, w, dw; write w, dw
        roofline = {"bound": "hbm", "achieved": hbm_bytes / t_s / 1e9, "peak": hbm_peak,
                    "unit": "GB/s", "frac": hbm_bytes / t_s / 1e9 / hbm_peak, "traffic": traffic,
                    "peak_source": hbm_src, "algorithmic_bytes_per_launch": hbm_bytes}
    else:
        nvl_bytes = 2 * (p - 1) / p * S
        roofline = {"bound": "nvlink", "achieved": busbw, "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                    "frac": busbw / NVLINK_PEER_GBS, "frac_of_nominal_900": busbw / NVLINK_NOMINAL_GBS,
                    "traffic": traffic,
                    "peak_source": "measured peer copy per direction (B200_PROFILING.md)",
                    "algorithmic_bytes_per_launch": nvl_bytes}

    extra = {}
    # allreduce alone (scale 1/p keeps the values fixed from call to call)
    if p > 1:
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                tc.allreduce(G, 1.0 / p, stream=stream)
            barrier(world)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(K):
                tc.allreduce(G, 1.0 / p, stream=stream)
            e1.record(stream)
            stream.synchronize()
        ta = max_over_ranks(e0.elapsed_time(e1) / K, world) / 1e3
        extra["allreduce_only"] = {"t_us": ta * 1e6, "busbw_gbs": S / ta / 1e9 * 2 * (p - 1) / p,
                                   "algo": comm.last_launch()[0]}
        # tensor broadcast from rank 0 (weight initialisation): scatter + allgather
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                tc.broadcast(G, 0, stream=stream)
            barrier(world)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(K):
                tc.broadcast(G, 0, stream=stream)
            e1.record(stream)
            stream.synchronize()
        tb = max_over_ranks(e0.elapsed_time(e1) / K, world) / 1e3
        extra["broadcast"] = {"t_us": tb * 1e6, "algbw_gbs": S / tb / 1e9,
                              "busbw_gbs": S / tb / 1e9 * (p - 1) / p,
                              "algo": comm.last_launch()[0]}
        if not args.no_nccl:
            import torch.distributed as dist
            flat = torch.empty(sum(numels), dtype=torch.float32, device="cuda")
            flat.normal_()
            with torch.cuda.stream(stream):
                for _ in range(args.warmup):
                    dist.all_reduce(flat)
                barrier(world)
                e0.record(stream)
                for _ in range(K):
                    dist.all_reduce(flat)
                e1.record(stream)
                stream.synchronize()
            tn = max_over_ranks(e0.elapsed_time(e1) / K, world) / 1e3
            extra["nccl_allreduce_flat"] = {"t_us": tn * 1e6,
                                            "busbw_gbs": S / tn / 1e9 * 2 * (p - 1) / p,
                                            "note": "torch.distributed NCCL all_reduce on one flat "
                                                    "buffer of N fp32 (comparison only)"}
            del flat

    # EASGD update (A7) on the ResNet-50 params: pairs (k, k + N/2) as in config 4
    _, x_c = dev(W.group(numels, "param", W.CFG_EASGD, 0, 0, W.PARAM))
    _, cen = dev(W.group(numels, "center", W.CFG_EASGD, 0, 0, W.CENTER))
    if p == 1:
        ecomm = comm
    else:
        import torch.distributed as dist
        mine = None
        if p % 2 == 0:
            half = p // 2
            for k in range(half):
                grp = dist.new_group([k, k + half], backend="gloo")
                if rank in (k, k + half):
                    mine = grp
        else:
            mine = dist.new_group(backend="gloo")
        ecomm = tc.Comm.from_process_group(mine, device=local) if mine is not None else None
    if ecomm is not None:
        X, C = tc.Group(ecomm, x_c), tc.Group(ecomm, cen)
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                tc.easgd_update(X, C, 0.1, stream=stream)
            barrier(world)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(K):
                tc.easgd_update(X, C, 0.1, stream=stream)
            e1.record(stream)
            stream.synchronize()
        te = max_over_ranks(e0.elapsed_time(e1) / K, world) / 1e3
        c = ecomm.nranks
        extra["easgd"] = {"t_us": te * 1e6, "clients": c,
                          "nvlink_ingress_gbs": (c - 1) * S / te / 1e9 if c > 1 else 0.0,
                          "hbm_gbs_local": 4 * S / te / 1e9 if c == 1 else None,
                          "algo": ecomm.last_launch()[0]}
        # NEXT row f2: the same update fused with each client's own SGD step (tc_esgd_step),
        # against the separate calls (tc_easgd_update + a local tc_sgd_step)
        _, g_c = dev(W.group(numels, "grad", W.CFG_EASGD, 1, rank, W.GRAD))
        _, d_c = dev(W.group(numels, "dw", W.CFG_EASGD, 2, rank, W.DW))
        Gc, Dc = tc.Group(ecomm, g_c), tc.Group(ecomm, d_c)
        lcomm = comm if p == 1 else tc.Comm.single(local)
        Wl, Gl, Dl = tc.Group(lcomm, x_c), tc.Group(lcomm, g_c), tc.Group(lcomm, d_c)
        ehp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / 128)

        def timed_calls(fn):
            with torch.cuda.stream(stream):
                for _ in range(args.warmup):
                    fn()
                barrier(world)
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                for _ in range(K):
                    fn()
                a1.record(stream)
                stream.synchronize()
            return max_over_ranks(a0.elapsed_time(a1) / K, world) * 1e3

        t_fused = timed_calls(lambda: tc.esgd_step(X, C, Gc, Dc, 0.1, stream=stream, **ehp))
        t_sep = timed_calls(lambda: (tc.easgd_update(X, C, 0.1, stream=stream),
                                     tc.sgd_step(Wl, Gl, Dl, stream=stream, **ehp)))
        extra["esgd_fused"] = {"t_us": t_fused, "t_separate_us": t_sep, "clients": c,
                               "algo": ecomm.last_launch()[0],
                               "note": "NEXT row f2: tc_esgd_step vs tc_easgd_update + local "
                                       "tc_sgd_step, one GPU per client"}
        for grp in (Gc, Dc, Wl, Gl, Dl):
            grp.destroy()
        if lcomm is not comm:
            lcomm.destroy()
        if p >= 2 and p % 2 == 0:
            extra["config4"] = config4_sequence(args, p, rank, local, numels, dev, ecomm, cen,
                                                stream, timed_calls)
        X.destroy()
        C.destroy()
        if ecomm is not comm:
            ecomm.destroy()

    # e2e through the public API with host buffers: pinned H2D of the step's gradients,
    # tc_sgd_step, D2H of the updated parameters.
    e2e = None
    if not args.no_e2e:
        # Every step copies its gradients in from pinned host memory and the updated
        # parameters out.  The copies are pipelined the way a training loop would: the next
        # step's gradients travel H2D (into the other of two gradient buffers) while this step's
        # kernel runs and its parameters travel D2H; a step's kernel waits for its gradients and
        # for the previous parameter read-out (it overwrites w).
        h_g = gp_flat.cpu().pin_memory()
        h_w = torch.empty_like(w_flat, device="cpu").pin_memory()
        if sym:
            g2_flat = comm.alloc_symmetric(sum(numels))
        else:
            g2_flat = torch.empty_like(g_flat)
        g2 = list(torch.split(g2_flat, [int(n) for n in numels]))
        bufs, groups = [g_flat, g2_flat], [G, tc.Group(comm, g2)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        Ke = min(K, 20)
        ev = lambda: torch.cuda.Event()  # noqa: E731
        for rep in range(2):  # rep 0 = warm-up
            barrier(world)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s_in.wait_stream(stream)
            s_out.wait_stream(stream)
            h2d_done, k_done, d2h_done = [None] * Ke, [None] * Ke, [None] * Ke
            with torch.cuda.stream(s_in):
                bufs[0].copy_(h_g, non_blocking=True)
                h2d_done[0] = ev()
                h2d_done[0].record(s_in)
            for i in range(Ke):
                if i + 1 < Ke:  # next step's gradients, into the buffer step i-1 used
                    with torch.cuda.stream(s_in):
                        if i >= 1:
                            s_in.wait_event(k_done[i - 1])
                        bufs[(i + 1) % 2].copy_(h_g, non_blocking=True)
                        h2d_done[i + 1] = ev()
                        h2d_done[i + 1].record(s_in)
                stream.wait_event(h2d_done[i])
                if i >= 1:
                    stream.wait_event(d2h_done[i - 1])
                tc.sgd_step(Wg, groups[i % 2], D, stream=stream, **hp)
                k_done[i] = ev()
                k_done[i].record(stream)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(k_done[i])
                    h_w.copy_(w_flat, non_blocking=True)
                    d2h_done[i] = ev()
                    d2h_done[i].record(s_out)
            stream.wait_event(d2h_done[Ke - 1])
            e1.record(stream)
            stream.synchronize()
        tt = max_over_ranks(e0.elapsed_time(e1) / Ke, world) / 1e3
        e2e = {"value": p * S / tt / 1e9, "unit": UNIT, "h2d_bytes_per_step": S,
               "d2h_bytes_per_step": S, "ms_per_step": tt * 1e3,
               "pipelining": "H2D of step i+1 overlaps step i's kernel and D2H"}
        groups[1].destroy()
        if sym:
            comm.free_symmetric(g2_flat)

    cpu = None
    if rank == 0 and p == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sgd(numels, 1)

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": p, "steps": K,
        "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded; torchvision ResNet-50 parameter shapes, SURVEY.md App. A)",
        "config": {"workload": f"{args.config} gradient group: tc_sgd_step (allreduce + fused "
                               f"SGD-momentum), {len(numels)} tensors, {S/1e6:.2f} MB per rank",
                   "global_batch": None, "p": p, "algo": algo, "ctas": ctas, "threads": threads,
                   "grad_memory": "tc_mem_alloc (symmetric, multicast)" if sym else "torch",
                   "l2": "inputs larger than L2 (3 groups, %.0f MB per GPU); no flush" % (3 * S / 1e6),
                   "parallelism": f"dp{p}"},
        "busbw_gbs": busbw, "algbw_gbs": algbw, "t_us": t_ms * 1e3,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": K, "clocks": clocks.summary(), "wall_s_timed_region": t_wall,
    }
    out.update(extra)
    for grp in (G, Wg, D):
        grp.destroy()
    comm.destroy()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
