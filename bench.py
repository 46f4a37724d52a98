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

value (BASELINE.json metric):
  N >= 2: the step's bus bandwidth, busbw = 2(N-1)/N * S / t (nccl-tests convention; the
          paper's bandwidth term), the roofline's achieved figure (bound: NVLink);
  N = 1:  no communication -- the fused step's HBM bandwidth 5S / t (bound: HBM).
whole_job_gbs = N * S / t is reported beside it.  Rank 0 prints ONE JSON line.
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

METRIC = ("tensor-allreduce bus GB/s of the fused allreduce + SGD-momentum step, ResNet-50 grad "
          "group (N>=2: busbw = 2(N-1)/N*S/t; N=1: HBM GB/s of the step, 5S/t)")
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




# ------------------------------------------------------------------ CPU oracle (baselines)
# The oracle as it stands: oracle.sgd_step over p simulated ranks.  Its arithmetic is
# elementwise within each tensor, so the all-cores baseline runs the same function on contiguous
# slices of the flattened group in a multiprocessing pool ("a multiprocessing
# pool over contiguous flat-space slices, len(os.sched_getaffinity(0)) workers"); the inputs
# live in shared memory.
_POOL = {}


def _pool_sgd(ab):
    from oracle import tc_oracle as O
    a, b = ab
    st = _POOL
    G, Ws, Ds = O.sgd_step([[st["w"][a:b]]], [[g[a:b]] for g in st["g"]], [[st["dw"][a:b]]],
                           **st["hp"])
    st["G_out"][a:b] = G[0]
    st["w_out"][a:b] = Ws[0][0]
    st["dw_out"][a:b] = Ds[0][0]
    return b - a


class OracleSGD:
    """The p-rank fused step of config 2 on the host: inputs generated from the same seeds as
    the GPU run (rank k's gradient group, the replicated w and dw), flattened."""

    def __init__(self, numels, p, cfg=W.CFG_RESNET50):
        from multiprocessing import shared_memory
        self.numels, self.p = numels, p
        self.N = int(sum(numels))
        self.hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (p * 128))
        self._shm = []

        def shared(fill=None):
            m = shared_memory.SharedMemory(create=True, size=4 * self.N)
            self._shm.append(m)
            a = np.ndarray((self.N,), np.float32, buffer=m.buf)
            if fill is not None:
                a[:] = np.concatenate(fill)
            return a

        self.g = [shared(W.group(numels, "grad", cfg, 0, k, W.GRAD)) for k in range(p)]
        self.w = shared(W.group(numels, "param", cfg, 0, 0, W.PARAM))
        self.dw = shared(W.group(numels, "dw", cfg, 0, 0, W.DW))
        self.outs = [shared() for _ in range(3)]
        self.pool = None
        self.cores = 1

    def step_single(self):
        """One thread: the oracle over the whole group, as the tests call it."""
        from oracle import tc_oracle as O
        O.sgd_step([[self.w]], [[g] for g in self.g], [[self.dw]], **self.hp)

    def start_pool(self):
        import multiprocessing as mp
        self.cores = len(os.sched_getaffinity(0))
        _POOL.update(g=self.g, w=self.w, dw=self.dw, hp=self.hp, G_out=self.outs[0],
                     w_out=self.outs[1], dw_out=self.outs[2])
        self.pool = mp.get_context("fork").Pool(self.cores)
        n = 4 * self.cores
        cuts = [self.N * i // n for i in range(n + 1)]
        self.slices = [(cuts[i], cuts[i + 1]) for i in range(n) if cuts[i + 1] > cuts[i]]

    def step_pool(self):
        assert sum(self.pool.map(_pool_sgd, self.slices)) == self.N

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
        for m in self._shm:
            m.close()
            m.unlink()


def step_value(p, S, t_s):
    """The BASELINE metric of one step of t_s seconds: busbw (p >= 2) or 5S/t (p = 1)."""
    return (2 * (p - 1) / p * S if p > 1 else 5 * S) / t_s / 1e9


def workload_config(config, numels, p):
    """The `config` object, identical in both arms (the reference arm runs the same workload)."""
    S = 4 * sum(numels)
    return {"workload": f"{config} gradient group: allreduce + fused SGD-momentum step "
                        f"(tc_sgd_step), {len(numels)} tensors, {S/1e6:.2f} MB per rank",
            "global_batch": None, "p": p, "parallelism": f"dp{p}",
            "hyper": "lr 0.1, momentum 0.9, wd 1e-4, rescale 1/(128 p)",
            "l2": "inputs larger than L2 (3 groups, %.0f MB per GPU); no flush" % (3 * S / 1e6)}


def cpu_baseline_sgd(numels, p, budget_s=20.0):
    """Our arm's cpu_baseline (rank 0, N = 1): the oracle on the same workload, bounded to about
    `budget_s` of CPU work -- one thread, then all cores."""
    o = OracleSGD(numels, p)
    S = 4 * sum(numels)
    try:
        t0 = time.perf_counter()
        n1 = 0
        while n1 < 3 and time.perf_counter() - t0 < budget_s / 2:
            o.step_single()
            n1 += 1
        t1 = (time.perf_counter() - t0) / n1
        o.start_pool()
        o.step_pool()  # warm the workers
        t0 = time.perf_counter()
        nall = 0
        while nall < 20 and time.perf_counter() - t0 < budget_s / 2:
            o.step_pool()
            nall += 1
        tall = (time.perf_counter() - t0) / nall
    finally:
        o.close()
    desc = f"full group ({len(numels)} tensors, {S/1e6:.1f} MB/rank) x {p} ranks per step"
    return {"value": step_value(p, S, tall), "unit": UNIT, "cores": o.cores, "kind": "oracle",
            "sample": f"{desc}; all cores: {nall} steps, {tall:.3f} s/step",
            "single_thread": {"value": step_value(p, S, t1), "cores": 1,
                              "sample": f"{desc}; {n1} steps, {t1:.3f} s/step"}}


# ------------------------------------------------------------------ the reference arm
def run_reference(args, jsonout):
    """The tier's reference arm: the CPU oracle as it stands, on our arm's workload (the whole
    p-rank fused step on the full group every step), on all host cores of rank 0."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    p = max(args.gpus, 1)
    numels = W.GROUPS[args.config]
    S = 4 * sum(numels)
    o = OracleSGD(numels, p)
    try:
        o.start_pool()
        for _ in range(args.warmup):
            o.step_pool()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            o.step_pool()
        dt = (time.perf_counter() - t0) / args.steps
    finally:
        o.close()
    v = step_value(p, S, dt)
    desc = (f"full {args.config} group ({len(numels)} tensors, {S/1e6:.1f} MB/rank) x {p} "
            f"simulated ranks every step, {o.cores} worker processes over flat slices")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded; torchvision ResNet-50 parameter shapes, SURVEY.md App. A)",
        "config": workload_config(args.config, numels, p),
        "whole_job_gbs": p * S / dt / 1e9,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": o.cores, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), file=jsonout, flush=True)


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


def nccl_allreduce_us(flat, stream, warmup, K, world, group=None):
    import torch
    import torch.distributed as dist
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            dist.all_reduce(flat, group=group)
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(K):
            dist.all_reduce(flat, group=group)
        e1.record(stream)
        stream.synchronize()
    return max_over_ranks(e0.elapsed_time(e1) / K, world) * 1e3


def claim_stdout():
    """Only the JSON line may reach stdout: the process's fd 1 is pointed at stderr (NCCL prints
    its version banner there) and the returned file writes to the original stdout."""
    sys.stdout.flush()
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    return out


def p2p_pull_peak(S, p, rank, local, stream, timed_us):
    """The roofline against a P2P peak measured in the same run: every GPU
    pulls S/p from every peer at once with TMA bulk copies (tools/nvl_probe.cu, our kernel, no
    arithmetic) -- GB/s per GPU per direction, best of two launch shapes from the probe sweep
    (profiles/r02_nvl_probe_p*.jsonl)."""
    import ctypes
    import torch
    import torch.distributed as dist
    so = os.path.join(ROOT, "tools", "bin", "libnvl_probe.so")
    if not os.path.exists(so):
        return {"unavailable": "tools/bin/libnvl_probe.so not built (__graft_entry__.build)"}
    try:
        import torch.distributed._symmetric_memory as symm
        lib = ctypes.CDLL(so)
        try:
            symm.enable_symm_mem_for_group(dist.group.WORLD.group_name)
        except Exception:  # noqa: BLE001 -- not needed on newer torch
            pass
        buf = symm.empty(S // 4, dtype=torch.float32, device=f"cuda:{local}")
        hdl = symm.rendezvous(buf, dist.group.WORLD.group_name)
        arr = (ctypes.c_void_p * 8)(*[hdl.buffer_ptrs[q] for q in range(p) if q != rank])
        part = (S // p) - (S // p) % (1 << 16)
        rows = []
        for ctas, tile, depth in ((148, 16384, 12), (32, 32768, 6)):
            c = max(1, ctas // (p - 1)) * (p - 1)
            st = ctypes.c_void_p(stream.cuda_stream)

            def f(c=c, tile=tile, depth=depth, st=st):
                if lib.probe_tma(0, arr, p - 1, ctypes.c_long(part), tile, depth, c, rank, st):
                    raise RuntimeError("probe_tma launch failed")
            t = timed_us(f)
            rows.append({"gbs_per_dir": (p - 1) * part / t / 1e3, "t_us": t, "ctas": c,
                         "tile_bytes": tile, "stages": depth})
        torch.cuda.synchronize()
        del hdl, buf
        best = max(rows, key=lambda r: r["gbs_per_dir"])
        return dict(best, kernel="tma_pull_kernel (tools/nvl_probe.cu): all peers at once, "
                    f"(p-1) x {part} B ingress per GPU", shapes=rows)
    except Exception as e:  # noqa: BLE001 -- a diagnostic field, never the bench's value
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}


def main():
    jsonout = claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="tc", choices=["tc", "reference"])
    ap.add_argument("--config", default="resnet50", choices=["resnet50", "alexnet", "vgg16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="only the step (and e2e): skip allreduce/broadcast/NCCL/EASGD/config-4")
    ap.add_argument("--algo", type=int, default=0,
                    help="0 auto, 1 register two-shot, 4 NVLS, 6 TMA two-shot")
    ap.add_argument("--switch", default="auto", choices=["auto", "on", "off"],
                    help="let the automatic choice use NVLS (tc_comm_set_switch_reduction): "
                         "auto = from N = 5, where it moves fewer bytes than the two-shot")
    ap.add_argument("--no-sym", action="store_true",
                    help="keep gradients in torch memory (no NVLS) instead of tc_mem_alloc")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args, jsonout)

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

    cfg_id = W.CFG_RESNET50
    gp_flat, _ = dev(W.group(numels, "grad", cfg_id, 0, rank, W.GRAD))
    g_flat, g = dev(W.group(numels, "zeros", 0, 0, 0, 0))
    g_flat.copy_(gp_flat)
    w_flat, w = dev(W.group(numels, "param", cfg_id, 0, 0, W.PARAM))
    dw_flat, dw = dev(W.group(numels, "dw", cfg_id, 0, 0, W.DW))
    torch.cuda.synchronize()

    comm = tc.Comm.single(local) if p == 1 else tc.Comm.from_process_group(device=local)
    comm.set_algorithm(args.algo)
    switch = args.switch == "on" or (args.switch == "auto" and p >= 5)
    if switch:
        comm.set_switch_reduction(True)
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
    value = step_value(p, S, t_s)
    algbw = S / t_s / 1e9
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
                    "achieved_is": "algorithmic bytes (5S) / CUDA-event time of the step kernel",
                    "peak_source": hbm_src, "algorithmic_bytes_per_launch": hbm_bytes,
                    "kernel": "k_local_tma<OP_SGD>"}
    else:
        # the step's own link bytes per GPU per direction: 2(p-1)/p S for the two-shot, (1 + 1/p) S
        # when the switch reduces (NVLS) -- value stays BASELINE's busbw either way
        nvls = algo == "nvls"
        nvl_bytes = (1 + 1 / p) * S if nvls else 2 * (p - 1) / p * S
        achieved = nvl_bytes / t_s / 1e9
        roofline = {"bound": "nvlink", "achieved": achieved, "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                    "frac": achieved / NVLINK_PEER_GBS,
                    "frac_of_nominal_900": achieved / NVLINK_NOMINAL_GBS, "traffic": traffic,
                    "achieved_is": ("algorithmic NVLink bytes per GPU per direction, (1 + 1/p) S "
                                    "(switch reduction)" if nvls else
                                    "algorithmic NVLink bytes per GPU 2(p-1)/p S") +
                                   " / CUDA-event time",
                    "peak_source": "measured peer copy per direction (B200_PROFILING.md)",
                    "algorithmic_bytes_per_launch": nvl_bytes, "kernel": f"{algo} (OP_SGD)"}

    extra = {}
    if p > 1 and not args.no_extras:
        def timed_us(fn):
            with torch.cuda.stream(stream):
                for _ in range(args.warmup):
                    fn()
                barrier(world)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(K):
                    fn()
                e1.record(stream)
                stream.synchronize()
            return max_over_ranks(e0.elapsed_time(e1) / K, world) * 1e3

        # the same-run P2P ceiling: an all-peer TMA pull copy, no arithmetic
        roofline["p2p_pull_peak"] = p2p_pull_peak(S, p, rank, local, stream, timed_us)
        pk = roofline["p2p_pull_peak"].get("gbs_per_dir")
        if pk:
            roofline["frac_of_p2p_pull_peak"] = achieved / pk
        # allreduce alone (scale 1/p keeps the values fixed from call to call)
        ta = timed_us(lambda: tc.allreduce(G, 1.0 / p, stream=stream))
        extra["allreduce_only"] = {"t_us": ta, "busbw_gbs": 2 * (p - 1) / p * S / ta / 1e3,
                                   "algo": comm.last_launch()[0]}
        if sym and comm.multicast_supported:
            comm.set_algorithm(4)
            tn = timed_us(lambda: tc.allreduce(G, 1.0 / p, stream=stream))
            extra["allreduce_nvls"] = {"t_us": tn, "busbw_gbs": 2 * (p - 1) / p * S / tn / 1e3,
                                       "link_gbs_per_dir": (1 + 1 / p) * S / tn / 1e3,
                                       "note": "algorithm 4 (switch reduction, fp32 in the "
                                               "switch: tolerance contract)"}
            # the fused step on the switch (fresh gradients before every kernel, as the step)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(K)]
            with torch.cuda.stream(stream):
                for i in range(args.warmup + K):
                    refresh_g()
                    if i >= args.warmup:
                        evs[i - args.warmup][0].record(stream)
                    step()
                    if i >= args.warmup:
                        evs[i - args.warmup][1].record(stream)
                stream.synchronize()
            ts = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs) / K, world) * 1e3
            extra["sgd_step_nvls"] = {"t_us": ts, "busbw_gbs": 2 * (p - 1) / p * S / ts / 1e3,
                                      "algo": comm.last_launch()[0],
                                      "note": "tc_sgd_step on algorithm 4: switch reduction, "
                                              "HBM epilogue overlapped per published round"}
            comm.set_algorithm(args.algo)
            refresh_g()
        # tensor broadcast from rank 0 (weight initialisation): through the switch for
        # the multicast-bound gradient bucket, else scatter + allgather (both timed)
        tb = timed_us(lambda: tc.broadcast(G, 0, stream=stream))
        extra["broadcast"] = {"t_us": tb, "algbw_gbs": S / tb / 1e3,
                              "busbw_gbs": S / tb / 1e3 * (p - 1) / p,
                              "algo": comm.last_launch()[0]}
        if comm.last_launch()[0] == "nvls":
            comm.set_algorithm(6)
            tb2 = timed_us(lambda: tc.broadcast(G, 0, stream=stream))
            extra["broadcast"]["two_shot_t_us"] = tb2
            comm.set_algorithm(args.algo)
        if not args.no_nccl:
            import torch.distributed as dist
            flat = torch.empty(sum(numels), dtype=torch.float32, device="cuda")
            flat.normal_()
            tn = nccl_allreduce_us(flat, stream, args.warmup, K, world)
            extra["nccl_allreduce_flat"] = {"t_us": tn, "busbw_gbs": 2 * (p - 1) / p * S / tn / 1e3,
                                            "note": "torch.distributed NCCL all_reduce on one flat "
                                                    "buffer of N fp32, default algorithm "
                                                    "(comparison only)"}
            # NCCL_ALGO is read when a communicator is created: a new group created with it set
            old = os.environ.get("NCCL_ALGO")
            os.environ["NCCL_ALGO"] = "Ring"
            ring = dist.new_group(backend="nccl")
            dist.all_reduce(flat, group=ring)  # creates the ring communicator now
            torch.cuda.synchronize()
            if old is None:
                del os.environ["NCCL_ALGO"]
            else:
                os.environ["NCCL_ALGO"] = old
            tr = nccl_allreduce_us(flat, stream, args.warmup, K, world, group=ring)
            extra["nccl_ring_allreduce_flat"] = {
                "t_us": tr, "busbw_gbs": 2 * (p - 1) / p * S / tr / 1e3,
                "note": "NCCL with NCCL_ALGO=Ring at communicator creation (the paper's ring "
                        "design (b), P:504), same flat buffer"}
            dist.destroy_process_group(ring)
            del flat

    # EASGD update (A7) on the ResNet-50 params: pairs (k, k + N/2) as in config 4
    _, x_c = dev(W.group(numels, "param", W.CFG_EASGD, 0, 0, W.PARAM))
    _, cen = dev(W.group(numels, "center", W.CFG_EASGD, 0, 0, W.CENTER))
    ecomm = None
    if p == 1:
        ecomm = comm
    elif not args.no_extras:
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
    if ecomm is not None and not args.no_extras:
        X, C = tc.Group(ecomm, x_c), tc.Group(ecomm, cen)

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

        te = timed_calls(lambda: tc.easgd_update(X, C, 0.1, stream=stream))
        c = ecomm.nranks
        extra["easgd"] = {"t_us": te, "clients": c,
                          "nvlink_ingress_gbs": (c - 1) * S / te / 1e3 if c > 1 else 0.0,
                          "hbm_gbs_local": 4 * S / te / 1e3 if c == 1 else None,
                          "algo": ecomm.last_launch()[0]}
        if c > 1:
            order = list(reversed(range(c)))
            tas = timed_calls(lambda: tc.easgd_async_update(X, C, 0.1, order, stream=stream))
            extra["easgd_async"] = {"t_us": tas, "clients": c, "order": order,
                                    "algo": ecomm.last_launch()[0],
                                    "note": "NEXT row f2: server-side Elastic1 per arrival"}
        # NEXT row f2: the same update fused with each client's own SGD step (tc_esgd_step),
        # against the separate calls (tc_easgd_update + a local tc_sgd_step)
        _, g_c = dev(W.group(numels, "grad", W.CFG_EASGD, 1, rank, W.GRAD))
        _, d_c = dev(W.group(numels, "dw", W.CFG_EASGD, 2, rank, W.DW))
        Gc, Dc = tc.Group(ecomm, g_c), tc.Group(ecomm, d_c)
        lcomm = comm if p == 1 else tc.Comm.single(local)
        Wl, Gl, Dl = tc.Group(lcomm, x_c), tc.Group(lcomm, g_c), tc.Group(lcomm, d_c)
        ehp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / 128)
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
    if ecomm is not None and ecomm is not comm:
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
        e2e = {"value": step_value(p, S, tt), "unit": UNIT, "h2d_bytes_per_step": S,
               "d2h_bytes_per_step": S, "ms_per_step": tt * 1e3, "whole_job_gbs": p * S / tt / 1e9,
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
        "config": workload_config(args.config, numels, p),
        "launch": {"algo": algo, "ctas": ctas, "threads": threads,
                   "grad_memory": "tc_mem_alloc (symmetric, multicast)" if sym else "torch",
                   "switch_reduction_allowed": switch},
        "whole_job_gbs": p * S / t_s / 1e9, "busbw_gbs": value if p > 1 else 0.0,
        "algbw_gbs": algbw, "t_us": t_ms * 1e3,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": K, "clocks": clocks.summary(), "wall_s_timed_region": t_wall,
    }
    out.update(extra)
    for grp in (G, Wg, D):
        grp.destroy()
    comm.destroy()
    if rank == 0:
        print(json.dumps(out), file=jsonout, flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
