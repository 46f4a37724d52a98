"""Seeded synthetic inputs shared by the CPU oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no sums, no SGD, no elastic update): only
tensor-group shapes, seeds and value distributions.  It is the one module both sides of the
parity check may use.

Shapes: the gradient groups of the paper's ImageNet-1K CNNs ("resnet-50",
SURVEY.md Appendix A; torchvision ``named_parameters()`` order, BN running stats excluded).
Seeds: ``SeedSequence([180103855, cfg_id, step, rank, role, tensor_idx])``.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 180103855

# roles (SURVEY.md §8(d) "Seeds")
GRAD, PARAM, DW, CENTER = 0, 1, 2, 3

# config ids (BASELINE.json "configs", 1-based as in SURVEY.md §8(d))
CFG_TINY, CFG_RESNET50, CFG_ALEX_VGG, CFG_EASGD, CFG_SWEEP = 1, 2, 3, 4, 5


def _rle(spec: str) -> list[int]:
    out: list[int] = []
    for tok in spec.split():
        if "x" in tok:
            a, k = tok.split("x")
            out += [int(a)] * int(k)
        else:
            out.append(int(tok))
    return out


RESNET50 = _rle(
    "9408 64x2 4096 64x2 36864 64x2 16384 256x2 16384 256x2 16384 64x2 36864 64x2 16384 256x2 "
    "16384 64x2 36864 64x2 16384 256x2 32768 128x2 147456 128x2 65536 512x2 131072 512x2 65536 "
    "128x2 147456 128x2 65536 512x2 65536 128x2 147456 128x2 65536 512x2 65536 128x2 147456 128x2 "
    "65536 512x2 131072 256x2 589824 256x2 262144 1024x2 524288 1024x2 262144 256x2 589824 256x2 "
    "262144 1024x2 262144 256x2 589824 256x2 262144 1024x2 262144 256x2 589824 256x2 262144 "
    "1024x2 262144 256x2 589824 256x2 262144 1024x2 262144 256x2 589824 256x2 262144 1024x2 "
    "524288 512x2 2359296 512x2 1048576 2048x2 2097152 2048x2 1048576 512x2 2359296 512x2 "
    "1048576 2048x2 1048576 512x2 2359296 512x2 1048576 2048x2 2048000 1000")
ALEXNET = _rle("23232 64 307200 192 663552 384 884736 256 589824 256 37748736 4096 16777216 4096 "
               "4096000 1000")
VGG16 = _rle("1728 64 36864 64 73728 128 147456 128 294912 256 589824 256 589824 256 1179648 512 "
             "2359296 512 2359296 512 2359296 512 2359296 512 2359296 512 102760448 4096 16777216 "
             "4096 4096000 1000")
TINY = [7, 13, 1000]  # BASELINE.json configs[0]

GROUPS = {"tiny": TINY, "resnet50": RESNET50, "alexnet": ALEXNET, "vgg16": VGG16}

assert len(RESNET50) == 161 and sum(RESNET50) == 25_557_032
assert len(ALEXNET) == 16 and sum(ALEXNET) == 61_100_840
assert len(VGG16) == 32 and sum(VGG16) == 138_357_544


def rng(cfg_id: int, step: int, rank: int, role: int, tensor_idx: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(
        [SEED_BASE, cfg_id, step, rank, role, tensor_idx]))


def draw(kind: str, n: int, g: np.random.Generator) -> np.ndarray:
    """One tensor of ``n`` fp32 values with distribution ``kind``."""
    if kind == "int":      # integers uniform in [-1000, 1000]; no -0
        return g.integers(-1000, 1001, size=n).astype(np.float32)
    if kind == "grad":     # per-tensor sigma_t = 10^U(-4,-1)
        sigma = 10.0 ** g.uniform(-4.0, -1.0)
        return (sigma * g.standard_normal(n)).astype(np.float32)
    if kind == "param":    # N(0, 0.05^2)
        return (0.05 * g.standard_normal(n)).astype(np.float32)
    if kind == "dw":       # N(0, 1e-6)
        return (1e-3 * g.standard_normal(n)).astype(np.float32)
    if kind == "center":   # N(0, 0.05^2)
        return (0.05 * g.standard_normal(n)).astype(np.float32)
    if kind == "client":   # perturbation of a client's params around the center: N(0, 0.01^2)
        return (0.01 * g.standard_normal(n)).astype(np.float32)
    if kind == "zeros":
        return np.zeros(n, np.float32)
    raise ValueError(kind)


def group(numels, kind: str, cfg_id: int, step: int, rank: int, role: int) -> list[np.ndarray]:
    """A tensor group: one seeded fp32 array per tensor."""
    return [draw(kind, int(n), rng(cfg_id, step, rank, role, t)) for t, n in enumerate(numels)]


def client_params(numels, center: list[np.ndarray], cfg_id: int, step: int, client: int):
    """x_i = center + N(0, 0.01^2), generated as data (the addition here is input synthesis,
    not the method's arithmetic)."""
    out = []
    for t, n in enumerate(numels):
        e = draw("client", int(n), rng(cfg_id, step, 1000 + client, CENTER, t))
        out.append((center[t] + e).astype(np.float32))
    return out


def sweep_numels(total_bytes: int, T: int, seed_idx: int = 0) -> list[int]:
    """Config 5: a seeded log-uniform split of N = total_bytes/4 into T tensors, every n_t >= 1
    (tails unaligned on purpose).  Returns [] when T > N (cell skipped)."""
    N = total_bytes // 4
    if T > N:
        return []
    g = rng(CFG_SWEEP, seed_idx, T, 0, total_bytes & 0x7FFFFFFF)
    w = np.exp(g.uniform(0.0, np.log(1000.0), size=T))
    extra = N - T
    parts = np.floor(w / w.sum() * extra).astype(np.int64)
    rem = extra - int(parts.sum())
    parts[: rem] += 1
    return [int(1 + x) for x in parts]


def random_numels(g: np.random.Generator, T: int, max_n: int, allow_zero: bool = True) -> list[int]:
    """Random ragged group shapes for property tests (zero-length tensors allowed)."""
    lo = 0 if allow_zero else 1
    return [int(x) for x in g.integers(lo, max_n + 1, size=T)]
