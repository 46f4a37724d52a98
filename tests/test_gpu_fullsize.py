"""T2 at the benchmarked sizes: the kernels bench.py times, on the gradient groups it times,
compared with the CPU oracle ELEMENT BY ELEMENT over the whole arrays (no sampling).

On one B200 the p >= 2 paths run as emulated comms (one cooperative kernel whose blockIdx.y is
the rank: the same per-rank code, tile table, stage ring and flag protocol as the one-process-
per-GPU layout; the grid is 148/p CTAs per rank instead of 148, so the tile -> CTA deal differs
from the real run -- tests/mp_worker.py covers the 148-CTA grid over real processes).

Covered (BASELINE.json configs):
  * config 2 -- ResNet-50 group (161 tensors, 25,557,032 fp32 per rank):
      p = 1: the TMA stream (k_local_tma) with allreduce scale != 1, the fused SGD step, the
             elastic update and the fused elastic + SGD step; 12.5k tiles, so the 4-stage ring
             wraps thousands of times;
      p = 2, 4, 8: TMA two-shot (algorithm 6, the bench default) for allreduce, fused SGD, EASGD
             and fused elastic + SGD, and the register two-shot (algorithm 1) for the first three.
  * config 3 -- AlexNet (61.1 M) and VGG-16 (138.4 M) at p = 1, 2, 4 (default algorithm).
  * config 4 -- 2 clients x 4 ranks on the ResNet-50 parameters, 16 steps, tau = 4.
  * config 5 -- 4 / 16 / 64 / 256 MiB (the paper's 4/16/64 MB sizes, plus 256 MiB)
      x T in {1, 161, 1024} x p in {2, 4, 8}, as views of one flat buffer (bench_sweep.py).
Values: the SURVEY.md §8(d) distributions (gradients sigma_t N(0,1), params, momentum).
Hyper-parameters: the perf set (lr 0.1, mu 0.9, wd 1e-4, rescale 1/(128 p)), alpha 0.1.
"""
import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402
from oracle import tc_oracle as O  # noqa: E402
from gpu_util import to_dev, to_host, assert_bitwise  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SGD_HP = dict(lr=0.1, momentum=0.9, wd=1e-4)
ALPHA = 0.1
ALGO = {"tma": 6, "pull": 1, "auto": 0}


@functools.lru_cache(maxsize=24)
def _grp(name, kind, cfg, step, rank, role):
    return tuple(W.group(W.GROUPS[name], kind, cfg, step, rank, role))


def grp(name, kind, cfg, step, rank, role):
    return list(_grp(name, kind, cfg, step, rank, role))


@functools.lru_cache(maxsize=16)
def _client(name, cfg, step, i):
    center = grp(name, "center", cfg, step, 0, W.CENTER)
    return tuple(W.client_params(W.GROUPS[name], center, cfg, step, i))


@pytest.fixture(scope="module", autouse=True)
def _drop_cache():
    yield
    _grp.cache_clear()
    _client.cache_clear()


def _comm(p, algo):
    if p == 1:
        return tc.Comm.single(0)
    c = tc.Comm.emulated(p, 0)
    c.set_algorithm(ALGO[algo])
    return c


def _pick(p):
    return (lambda v: v) if p > 1 else (lambda v: v[0])


def _want_algo(p, algo):
    return "local" if p == 1 else ("two-shot" if algo == "pull" else "two-shot-tma")


def _check_allreduce(name, p, algo, cfg, scale=0.37):
    xs = [grp(name, "grad", cfg, 0, k, W.GRAD) for k in range(p)]
    comm = _comm(p, algo)
    dev = [to_dev(x) for x in xs]
    g = tc.Group(comm, _pick(p)(dev))
    tc.allreduce(g, scale)
    got = [to_host(d) for d in dev]
    launched = comm.last_launch()[0]
    assert comm.async_error() == 0
    g.destroy()
    comm.destroy()
    del dev
    want = O.allreduce(xs, scale)
    for r in range(p):
        assert_bitwise(got[r], want, f"{name} allreduce p={p} rank {r}")
    return launched


def _check_sgd(name, p, algo, cfg):
    rescale = 1.0 / (128 * p)
    gs = [grp(name, "grad", cfg, 0, k, W.GRAD) for k in range(p)]
    w = grp(name, "param", cfg, 0, 0, W.PARAM)
    dw = grp(name, "dw", cfg, 0, 0, W.DW)
    comm = _comm(p, algo)
    dg, dwt, ddw = [to_dev(g) for g in gs], [to_dev(w) for _ in range(p)], [to_dev(dw) for _ in range(p)]
    G, Wg, D = (tc.Group(comm, _pick(p)(v)) for v in (dg, dwt, ddw))
    tc.sgd_step(Wg, G, D, rescale=rescale, **SGD_HP)
    got = [(to_host(dg[r]), to_host(dwt[r]), to_host(ddw[r])) for r in range(p)]
    launched = comm.last_launch()[0]
    assert comm.async_error() == 0
    for x in (G, Wg, D):
        x.destroy()
    comm.destroy()
    del dg, dwt, ddw
    Gw, Ws, Dws = O.sgd_step([w], gs, [dw], rescale=rescale, **SGD_HP)  # w, dw replicated
    for r in range(p):
        assert_bitwise(got[r][0], Gw, f"{name} sgd g p={p} rank {r}")
        assert_bitwise(got[r][1], Ws[0], f"{name} sgd w p={p} rank {r}")
        assert_bitwise(got[r][2], Dws[0], f"{name} sgd dw p={p} rank {r}")
    return launched


def _check_easgd(name, p, algo):
    center = grp(name, "center", W.CFG_EASGD, 0, 0, W.CENTER)
    xs = [list(_client(name, W.CFG_EASGD, 0, i)) for i in range(p)]
    comm = _comm(p, algo)
    dx, dc = [to_dev(x) for x in xs], [to_dev(center) for _ in range(p)]
    X, C = tc.Group(comm, _pick(p)(dx)), tc.Group(comm, _pick(p)(dc))
    tc.easgd_update(X, C, ALPHA)
    got = [(to_host(dx[i]), to_host(dc[i])) for i in range(p)]
    launched = comm.last_launch()[0]
    assert comm.async_error() == 0
    X.destroy()
    C.destroy()
    comm.destroy()
    del dx, dc
    wx, wc = O.easgd_update(xs, center, ALPHA)
    for i in range(p):
        assert_bitwise(got[i][0], wx[i], f"{name} easgd x p={p} client {i}")
        assert_bitwise(got[i][1], wc, f"{name} easgd center p={p} replica {i}")
    return launched


def _check_esgd(name, p, algo):
    center = grp(name, "center", W.CFG_EASGD, 0, 0, W.CENTER)
    xs = [list(_client(name, W.CFG_EASGD, 0, i)) for i in range(p)]
    gs = [grp(name, "grad", W.CFG_EASGD, 1, i, W.GRAD) for i in range(p)]
    dws = [grp(name, "dw", W.CFG_EASGD, 2, i, W.DW) for i in range(p)]
    hp = dict(alpha=ALPHA, rescale=1.0 / 128, **SGD_HP)
    comm = _comm(p, algo)
    dx, dc = [to_dev(x) for x in xs], [to_dev(center) for _ in range(p)]
    dg, dd = [to_dev(g) for g in gs], [to_dev(d) for d in dws]
    X, C, G, D = (tc.Group(comm, _pick(p)(v)) for v in (dx, dc, dg, dd))
    tc.esgd_step(X, C, G, D, **hp)
    got = [(to_host(dx[i]), to_host(dc[i]), to_host(dd[i]), to_host(dg[i])) for i in range(p)]
    launched = comm.last_launch()[0]
    assert comm.async_error() == 0
    for x in (X, C, G, D):
        x.destroy()
    comm.destroy()
    del dx, dc, dg, dd
    wx, wc, wd = O.esgd_step(xs, center, gs, dws, **hp)
    for i in range(p):
        assert_bitwise(got[i][0], wx[i], f"{name} esgd x p={p} client {i}")
        assert_bitwise(got[i][1], wc, f"{name} esgd center p={p} replica {i}")
        assert_bitwise(got[i][2], wd[i], f"{name} esgd dw p={p} client {i}")
        assert_bitwise(got[i][3], gs[i], f"{name} esgd g (read only) p={p} client {i}")
    return launched


OPS = {"allreduce": lambda name, p, algo: _check_allreduce(name, p, algo, W.CFG_RESNET50),
       "sgd": lambda name, p, algo: _check_sgd(name, p, algo, W.CFG_RESNET50),
       "easgd": _check_easgd, "esgd": _check_esgd}


# ------------------------------------------------------------------ config 2: ResNet-50
@pytest.mark.parametrize("op", sorted(OPS))
def test_resnet50_p1_tma_stream(op):
    """bench.py N = 1: k_local_tma over the whole group (296 CTAs, 4-stage ring)."""
    assert OPS[op]("resnet50", 1, "auto") == "local"


@pytest.mark.parametrize("algo", ["tma", "pull"])
@pytest.mark.parametrize("op", sorted(OPS))
@pytest.mark.parametrize("p", [2, 4, 8])
def test_resnet50_twoshot(p, op, algo):
    """bench.py N >= 2 default (algorithm 6, TMA two-shot) and the register two-shot (1), an
    independent implementation of the same arithmetic (ESGD exists in the TMA kernels only)."""
    if op == "esgd" and algo == "pull":
        pytest.skip("the fused elastic + SGD step is implemented by the TMA kernels only")
    assert OPS[op]("resnet50", p, algo) == _want_algo(p, algo)


def test_resnet50_default_choice_is_benched_kernel():
    """At N >= 2 the automatic choice for the ResNet-50 group is the kernel bench.py times."""
    for p in (2, 4, 8):
        assert _check_sgd("resnet50", p, "auto", W.CFG_RESNET50) == "two-shot-tma"


# ------------------------------------------------------------------ config 3: AlexNet, VGG-16
@pytest.mark.parametrize("p", [1, 2, 4])
@pytest.mark.parametrize("name", ["alexnet", "vgg16"])
def test_config3_allreduce(name, p):
    algo = _check_allreduce(name, p, "auto", W.CFG_ALEX_VGG, scale=1.0 / 3)
    assert algo == ("local" if p == 1 else "two-shot-tma")


@pytest.mark.parametrize("p", [1, 2, 4])
def test_config3_alexnet_sgd(p):
    assert _check_sgd("alexnet", p, "auto", W.CFG_ALEX_VGG) == ("local" if p == 1 else "two-shot-tma")


def test_config3_vgg16_sgd_p2():
    assert _check_sgd("vgg16", 2, "auto", W.CFG_ALEX_VGG) == "two-shot-tma"


# ------------------------------------------------------------------ config 4 at ResNet-50 shapes
def test_config4_resnet50_sequence():
    """2 clients x 4 ranks, synchronous fused allreduce + SGD inside each client, elastic update
    across the counterpart pairs (k, k+4) every tau = 4 steps, 16 steps (Fig. code-snippet-4,
    P:301-315), on the full ResNet-50 parameters -- vs oracle.esgd_sequence."""
    name, C, Q, steps, tau = "resnet50", 2, 4, 16, 4
    numels = W.GROUPS[name]
    hp = dict(alpha=ALPHA, rescale=1.0 / (Q * 128), **SGD_HP)
    center = grp(name, "center", W.CFG_EASGD, 0, 0, W.CENTER)
    x0 = [list(_client(name, W.CFG_EASGD, 0, i)) for i in range(C)]
    dw0 = [grp(name, "dw", W.CFG_EASGD, 0, i, W.DW) for i in range(C)]

    x = [to_dev(x0[g // Q]) for g in range(C * Q)]
    dw = [to_dev(dw0[g // Q]) for g in range(C * Q)]
    xc = [to_dev(center) for _ in range(C * Q)]
    g = [to_dev(W.group(numels, "zeros", 0, 0, 0, 0)) for _ in range(C * Q)]
    clients = [tc.Comm.emulated(Q, 0) for _ in range(C)]
    pairs = [tc.Comm.emulated(C, 0) for _ in range(Q)]
    G = [tc.Group(clients[i], [g[Q * i + k] for k in range(Q)]) for i in range(C)]
    Wt = [tc.Group(clients[i], [x[Q * i + k] for k in range(Q)]) for i in range(C)]
    D = [tc.Group(clients[i], [dw[Q * i + k] for k in range(Q)]) for i in range(C)]
    X = [tc.Group(pairs[k], [x[Q * i + k] for i in range(C)]) for k in range(Q)]
    XC = [tc.Group(pairs[k], [xc[Q * i + k] for i in range(C)]) for k in range(Q)]

    def grads(t, i):
        """Every GPU of every step draws a fresh gradient.  The oracle asks for client i's
        gradients of step t exactly when the GPU run needs them (t outer, i inner, after the
        elastic update of step t), so the GPU side runs here, in lockstep, and only one step's
        gradients are ever held on the host."""
        gr = [W.group(numels, "grad", W.CFG_EASGD, 100 + t, Q * i + k, W.GRAD) for k in range(Q)]
        if i == 0 and t % tau == 0:
            for k in range(Q):
                tc.easgd_update(X[k], XC[k], hp["alpha"])
        for k in range(Q):
            for dst, src in zip(g[Q * i + k], gr[k]):
                dst.copy_(torch.from_numpy(src))
        tc.sgd_step(Wt[i], G[i], D[i], lr=hp["lr"], momentum=hp["momentum"], wd=hp["wd"],
                    rescale=hp["rescale"])
        assert clients[i].last_launch()[0] == "two-shot-tma"
        torch.cuda.synchronize()  # the host arrays are handed to the oracle next
        return gr

    wx, wc, wdw = O.esgd_sequence(x0, center, dw0, grads, steps, tau, **hp)
    got = [(to_host(x[q]), to_host(dw[q]), to_host(xc[q])) for q in range(C * Q)]
    for cm in clients + pairs:
        assert cm.async_error() == 0
    for grp_ in G + Wt + D + X + XC:
        grp_.destroy()
    for cm in clients + pairs:
        cm.destroy()
    del x, dw, xc, g
    for q in range(C * Q):
        i = q // Q
        assert_bitwise(got[q][0], wx[i], f"x gpu {q}")
        assert_bitwise(got[q][1], wdw[i], f"dw gpu {q}")
        assert_bitwise(got[q][2], wc, f"center gpu {q}")


# ------------------------------------------------------------------ config 5 at real sizes
@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("T", [1, 161, 1024])
@pytest.mark.parametrize("mib", [4, 16, 64, 256])
def test_config5_sweep(mib, T, p):
    """The paper's message sizes (4/16/64 MB) and 256 MiB, T tensors as views of one
    flat buffer with unaligned tails, automatic algorithm choice -- whole arrays vs the oracle."""
    total = mib << 20
    numels = W.sweep_numels(total, T)
    xs = [W.group(numels, "grad", W.CFG_SWEEP, 0, k, W.GRAD) for k in range(p)]
    comm = tc.Comm.emulated(p, 0)
    flats = [torch.from_numpy(np.concatenate(x)).cuda() for x in xs]
    views = [list(torch.split(f, numels)) for f in flats]
    g = tc.Group(comm, views)
    tc.allreduce(g, 0.5)
    got = [to_host(v) for v in views]
    launched = comm.last_launch()[0]
    assert comm.async_error() == 0
    g.destroy()
    comm.destroy()
    del flats, views
    want = O.allreduce(xs, 0.5)
    for r in range(p):
        assert_bitwise(got[r], want, f"{mib} MiB T={T} p={p} rank {r} ({launched})")


# ------------------------------------------------------------------ NEXT row f2: async-server EASGD
@pytest.mark.parametrize("p", [2, 4, 8])
def test_resnet50_easgd_async(p):
    """The asynchronous-server elastic update on the full ResNet-50 parameters, arrivals in a
    shuffled recorded order, whole arrays vs oracle.easgd_async."""
    name = "resnet50"
    center = grp(name, "center", W.CFG_EASGD, 0, 0, W.CENTER)
    xs = [list(_client(name, W.CFG_EASGD, 0, i)) for i in range(p)]
    order = [int(i) for i in np.random.default_rng(p).permutation(p)]
    comm = tc.Comm.emulated(p, 0)
    dx, dc = [to_dev(x) for x in xs], [to_dev(center) for _ in range(p)]
    X, C = tc.Group(comm, dx), tc.Group(comm, dc)
    tc.easgd_async_update(X, C, ALPHA, order)
    got = [(to_host(dx[i]), to_host(dc[i])) for i in range(p)]
    assert comm.last_launch()[0] == "two-shot-tma"
    assert comm.async_error() == 0
    X.destroy()
    C.destroy()
    comm.destroy()
    del dx, dc
    wx, wc = O.easgd_async(xs, center, ALPHA, order)
    for i in range(p):
        assert_bitwise(got[i][0], wx[i], f"async x p={p} client {i}")
        assert_bitwise(got[i][1], wc, f"async center p={p} replica {i}")


# ------------------------------------------------------------------ tensors of >= 2^31 elements
def test_p1_tensor_over_2g_elements():
    """A single tensor of 2^31 + 13 fp32 elements (8 GiB) between two small ones on the p = 1
    TMA stream: tiles past element 2^31 need the 64-bit tile offsets.  With scale 1/2 the result
    is exactly x / 2 for every finite x (a power-of-two scale rounds nothing) -- a property that
    holds at any size, checked element by element on the device against a kept copy."""
    n_big = (1 << 31) + 13
    free, _ = torch.cuda.mem_get_info()
    if free < 2.6 * 4 * n_big:
        pytest.skip("needs ~23 GB of free device memory")
    gen = torch.Generator(device="cuda").manual_seed(7)
    xs = [torch.randn(5, device="cuda", generator=gen),
          torch.randn(n_big, device="cuda", generator=gen),
          torch.randn(7, device="cuda", generator=gen)]
    keep = [x.clone() for x in xs]
    comm = tc.Comm.single(0)
    g = tc.Group(comm, xs)
    tc.allreduce(g, 0.5)
    torch.cuda.synchronize()
    assert comm.last_launch()[0] == "local"
    assert comm.async_error() == 0
    g.destroy()
    comm.destroy()
    assert torch.equal(xs[0], keep[0] * 0.5) and torch.equal(xs[2], keep[2] * 0.5)
    chunk = 1 << 28
    for lo in range(0, n_big, chunk):
        assert torch.equal(xs[1][lo:lo + chunk], keep[1][lo:lo + chunk] * 0.5), lo
