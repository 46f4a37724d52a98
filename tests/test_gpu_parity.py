"""T2: GPU parity of libtc against the CPU oracle, on one B200.

Multi-rank paths run on one GPU through an *emulated* comm: one cooperative kernel whose
blockIdx.y is the rank, executing the same per-rank code and flag protocol as the
one-process-per-GPU layout (test_gpu_multiproc.py covers real multi-GPU runs).

Bar: allreduce bit-exact vs the float64-accumulating oracle for every finite
input (same canonical order, one rounding); SGD and EASGD bit-exact vs the oracle's fp32
mirror; every rank bit-identical; and, as the BASELINE bound, within 1e-5 * sum|x| of the
float64 reference.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_03855_b200 as tc  # noqa: E402
import tc_workloads as W  # noqa: E402
from oracle import tc_oracle as O  # noqa: E402
from gpu_util import to_dev, to_host, assert_bitwise  # noqa: E402

pytestmark = pytest.mark.gpu

ONESHOT = 1 << 20   # force one-shot
TWOSHOT = 0         # force two-shot (pull reduce-scatter)
LL = -3             # force the low-latency algorithm
TMA = -4            # force the TMA-staged two-shot
ALGOS = [("two-shot", TWOSHOT), ("one-shot", ONESHOT), ("ll", LL), ("two-shot-tma", TMA)]


def _comm(p, oneshot=-1, ctas=0):
    c = tc.Comm.single(0) if p == 1 else tc.Comm.emulated(p, 0)
    if oneshot == LL:
        c.set_ll_max(1 << 30)
        return c
    if oneshot != -1:
        c.set_ll_max(0)
    if oneshot == TMA:
        c.set_algorithm(6)
        oneshot = 0
    elif oneshot == TWOSHOT and p > 1:
        c.set_algorithm(1)
    c.set_tuning(ctas, 0, oneshot)
    return c


def run_allreduce(xs, scale=1.0, oneshot=-1, offset=0, ctas=0):
    """offset: elements each tensor starts past its allocation (int, or a callable of the rank)."""
    p = len(xs)
    comm = _comm(p, oneshot, ctas)
    off = offset if callable(offset) else (lambda k: offset)
    dev = [to_dev(x, offset=off(k)) for k, x in enumerate(xs)]
    grp = tc.Group(comm, dev if p > 1 else dev[0])
    tc.allreduce(grp, scale)
    out = [to_host(d) for d in dev]
    algo = comm.last_launch()[0]
    assert comm.async_error() == 0
    grp.destroy()
    comm.destroy()
    return out, algo


# ------------------------------------------------------------------ allreduce
@pytest.mark.parametrize("name,oneshot", ALGOS)
@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_tiny_config_allreduce_int(p, name, oneshot):
    """Config 1 (tiny: 3 tensors of 7, 13, 1000 elems, integer-valued) at p ranks."""
    xs = [W.group(W.TINY, "int", W.CFG_TINY, 0, k, W.GRAD) for k in range(p)]
    out, algo = run_allreduce(xs, oneshot=oneshot)
    assert algo == name
    want = O.allreduce(xs)
    for r in range(p):
        assert_bitwise(out[r], want, f"rank {r}")


@pytest.mark.parametrize("name,oneshot", ALGOS)
@pytest.mark.parametrize("p", [2, 4, 5, 8])
def test_random_groups_grad_values(p, name, oneshot):
    """Ragged groups (zero-length, 1-element, tails of 1..3) with gradient-like values:
    bit-exact vs the float64 oracle and within the BASELINE tolerance of the f64 reference."""
    g = np.random.default_rng(1000 + p)
    numels = W.random_numels(g, 37, 3000) + [1, 2, 3, 0, 5]
    xs = [W.group(numels, "grad", 77, 0, k, W.GRAD) for k in range(p)]
    out, algo = run_allreduce(xs, oneshot=oneshot, scale=0.125)
    assert algo == name
    want = O.allreduce(xs, 0.125)
    ref = O.allreduce_f64(xs, 0.125)
    for r in range(p):
        assert_bitwise(out[r], want, f"rank {r}")
    for t in range(len(numels)):
        bound = 1e-5 * 0.125 * sum(np.abs(xs[k][t].astype(np.float64)) for k in range(p))
        assert (np.abs(out[0][t] - ref[t]) <= bound).all()


@pytest.mark.parametrize("extra", [-1, 0, 1, 515])
@pytest.mark.parametrize("p", [2, 3, 4])
def test_oneshot_flat_boundary(p, extra):
    """The one-shot deals one slot per thread when the group's M slots fit a grid of up to
    2 CTAs/SM per local rank (512 threads), else 128-slot pieces over that grid: groups of
    limit-1, limit, limit+1 and limit+515 slots (ragged tensors, 2 tails) stay bit-exact."""
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    limit = (2 * sms // p) * 512
    m = limit + extra
    numels = [4 * (m // 3) - 1, 4 * (m // 3) - 2]
    numels.append(4 * (m - 2 * (m // 3)))
    assert tc.Plan(numels).num_slots == m
    xs = [W.group(numels, "int", 900 + extra, 0, k, W.GRAD) for k in range(p)]
    comm = _comm(p, 8 << 20)
    dev = [to_dev(x) for x in xs]
    grp = tc.Group(comm, dev)
    tc.allreduce(grp, 0.5)
    algo, ctas, _ = comm.last_launch()
    assert algo == "one-shot"
    assert ctas == (-(-m // 512) if extra <= 0 else 2 * sms // p), ctas
    want = O.allreduce(xs, 0.5)
    for r in range(p):
        assert_bitwise(to_host(dev[r]), want, f"rank {r}")
    assert comm.async_error() == 0
    grp.destroy()
    comm.destroy()


@pytest.mark.parametrize("offset", [1, 2, 3, "per-rank"])
@pytest.mark.parametrize("p", [1, 2, 4])
def test_unaligned_tensors(p, offset):
    """Tensors starting 1-3 elements past a 16-B boundary.  Same misalignment on every rank:
    shifted slot grid, vector path.  Misalignment differing by rank: scalar path."""
    numels = [7, 13, 1000, 4096, 3, 1, 2]
    xs = [W.group(numels, "int", 76, 0, k, W.GRAD) for k in range(p)]
    off = (lambda k: k % 4) if offset == "per-rank" else offset
    for oneshot in (TWOSHOT, ONESHOT, LL, TMA):
        out, _ = run_allreduce(xs, oneshot=oneshot, offset=off)
        for r in range(p):
            assert_bitwise(out[r], O.allreduce(xs), f"rank {r}")


@pytest.mark.parametrize("p", [1, 3])
def test_sgd_mixed_alignment(p):
    """g as views of one flat buffer (odd sizes: misaligned), w and dw separate allocations:
    the primary grid is shifted, the other operands fall back to the scalar path (p = 1: the
    TMA stream's element path for tiles misaligned in any operand)."""
    numels = [7, 13, 1000, 4097, 3, 2048, 6001]
    gs = [W.group(numels, "grad", 70, 0, k, W.GRAD) for k in range(p)]
    w = W.group(numels, "param", 70, 0, 0, W.PARAM)
    dw = W.group(numels, "dw", 70, 0, 0, W.DW)
    comm = _comm(p, TWOSHOT)
    flats = [torch.from_numpy(np.concatenate(gs[k])).cuda() for k in range(p)]
    dg = [list(torch.split(f, numels)) for f in flats]
    dwt = [to_dev(w) for _ in range(p)]
    ddw = [to_dev(dw, offset=2) for _ in range(p)]
    pick = (lambda x: x) if p > 1 else (lambda x: x[0])
    G, Wg, D = tc.Group(comm, pick(dg)), tc.Group(comm, pick(dwt)), tc.Group(comm, pick(ddw))
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / 384)
    tc.sgd_step(Wg, G, D, **hp)
    Gw, Ws, Dws = O.sgd_step([w] * p, gs, [dw] * p, **hp)
    for r in range(p):
        assert_bitwise(to_host(dg[r]), Gw, f"g rank {r}")
        assert_bitwise(to_host(dwt[r]), Ws[r], f"w rank {r}")
        assert_bitwise(to_host(ddw[r]), Dws[r], f"dw rank {r}")
    for grp in (G, Wg, D):
        grp.destroy()
    comm.destroy()


@pytest.mark.parametrize("p", [4, 8])
def test_fewer_slots_than_ranks(p):
    """N < p: some owners have empty chunks."""
    numels = [1, 2] if p == 4 else [3, 0, 1]
    xs = [W.group(numels, "int", 75, 0, k, W.GRAD) for k in range(p)]
    for oneshot in (TWOSHOT, TMA):
        out, _ = run_allreduce(xs, oneshot=oneshot)
        for r in range(p):
            assert_bitwise(out[r], O.allreduce(xs), f"rank {r}")


def test_many_tensors_1024():
    p = 4
    g = np.random.default_rng(5)
    numels = W.random_numels(g, 1024, 700)
    xs = [W.group(numels, "grad", 74, 0, k, W.GRAD) for k in range(p)]
    for oneshot in (TWOSHOT, ONESHOT, LL, TMA):
        out, _ = run_allreduce(xs, oneshot=oneshot)
        for r in range(p):
            assert_bitwise(out[r], O.allreduce(xs), f"rank {r}")


@pytest.mark.parametrize("ctas", [1, 3, 17])
def test_cta_counts(ctas):
    """Sub-range partition across CTAs, including few CTAs (many slots per CTA)."""
    p = 3
    numels = [7, 13, 1000, 50000, 9]
    xs = [W.group(numels, "grad", 73, 0, k, W.GRAD) for k in range(p)]
    for oneshot in (TWOSHOT, TMA):
        out, _ = run_allreduce(xs, oneshot=oneshot, ctas=ctas)
        for r in range(p):
            assert_bitwise(out[r], O.allreduce(xs), f"rank {r}")


def test_single_rank_scale():
    xs = [W.group([7, 13, 1000, 4097], "grad", 72, 0, 0, W.GRAD)]
    out, algo = run_allreduce(xs, scale=0.37)
    assert algo == "local"
    assert_bitwise(out[0], O.allreduce(xs, 0.37))


@pytest.mark.parametrize("offset", [0, 1, 2])
def test_single_rank_tile_boundaries(offset):
    """p = 1 TMA stream: tensors around the 2048-element tile size, several tiles per tensor,
    ragged tails, 1-2 element tensors; aligned (offset 0) and shifted starts."""
    numels = [2048, 2047, 2049, 4096, 4099, 1, 2, 3, 10000, 6143, 12288]
    xs = [W.group(numels, "grad", 79, 0, 0, W.GRAD)]
    out, algo = run_allreduce(xs, scale=0.25, offset=offset)
    assert algo == "local"
    assert_bitwise(out[0], O.allreduce(xs, 0.25))


def test_repeated_calls_epochs():
    """Many consecutive calls rotating algorithms on one comm (epoch and staging-parity
    bookkeeping), each call changing the data: with scale 1/2 at p = 4 the first call gives
    y = sum_k x_k / 2 and every later call doubles it (every rank holds y), exactly for integer
    data -- so a skipped or stale call fails the check made after EVERY call."""
    p = 4
    comm = tc.Comm.emulated(p, 0)
    numels = [7, 13, 1000, 5000]
    xs = [W.group(numels, "int", 71, 0, k, W.GRAD) for k in range(p)]
    dev = [to_dev(x) for x in xs]
    grp = tc.Group(comm, dev)
    want = O.allreduce(xs, 0.5)
    for i in range(60):
        comm.set_algorithm((1, 6)[i % 2])
        comm.set_tuning(0, 0, ONESHOT if i % 3 == 0 else TWOSHOT)
        comm.set_ll_max(1 << 30 if i % 5 == 0 else 0)
        tc.allreduce(grp, 0.5)
        for r in range(p):
            assert_bitwise(to_host(dev[r]), want, f"call {i} rank {r}")
        want = O.allreduce([want] * p, 0.5)
    assert comm.async_error() == 0
    grp.destroy()
    comm.destroy()


def test_repeated_sgd_steps_fresh_gradients():
    """Eight consecutive fused SGD steps on one comm, a fresh gradient every step and the
    algorithm rotating (register pull, TMA two-shot, one-shot, LL): w and dw carry every step
    into the next, so a skipped or repeated call fails."""
    p = 4
    numels = [7, 13, 1000, 4096, 65, 20000]
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (p * 128))
    w = W.group(numels, "param", 78, 0, 0, W.PARAM)
    dw = W.group(numels, "dw", 78, 0, 0, W.DW)
    comm = tc.Comm.emulated(p, 0)
    dg = [to_dev(W.group(numels, "zeros", 0, 0, 0, 0)) for _ in range(p)]
    dwt, ddw = [to_dev(w) for _ in range(p)], [to_dev(dw) for _ in range(p)]
    G, Wg, D = tc.Group(comm, dg), tc.Group(comm, dwt), tc.Group(comm, ddw)
    shapes = [(1, 0, 0), (6, 0, 0), (0, ONESHOT, 0), (0, 0, 1 << 30)]
    for step in range(8):
        gs = [W.group(numels, "grad", 78, 10 + step, k, W.GRAD) for k in range(p)]
        for k in range(p):
            for dst, src in zip(dg[k], gs[k]):
                dst.copy_(torch.from_numpy(src))
        a, one, ll = shapes[step % len(shapes)]
        comm.set_algorithm(a)
        comm.set_tuning(0, 0, one)
        comm.set_ll_max(ll)
        tc.sgd_step(Wg, G, D, **hp)
        _, Ws, Dws = O.sgd_step([w], gs, [dw], **hp)
        w, dw = Ws[0], Dws[0]
        for r in range(p):
            assert_bitwise(to_host(dwt[r]), w, f"step {step} w rank {r}")
            assert_bitwise(to_host(ddw[r]), dw, f"step {step} dw rank {r}")
    assert comm.async_error() == 0
    for x in (G, Wg, D):
        x.destroy()
    comm.destroy()


# ------------------------------------------------------------------ SGD (A6)
SGD_PERF = dict(lr=0.1, momentum=0.9, wd=1e-4)
SGD_DYADIC = dict(lr=0.5, momentum=0.5, wd=0.0)


def run_sgd(p, numels, kind, hp, oneshot=-1, cfg=W.CFG_RESNET50):
    rescale = 1.0 / (p * 128)
    gs = [W.group(numels, kind, cfg, 0, k, W.GRAD) for k in range(p)]
    w = W.group(numels, "int" if kind == "int" else "param", cfg, 0, 0, W.PARAM)
    dw = W.group(numels, "int" if kind == "int" else "dw", cfg, 0, 0, W.DW)
    comm = _comm(p, oneshot)
    dg = [to_dev(g) for g in gs]
    dwt = [to_dev(w) for _ in range(p)]
    ddw = [to_dev(dw) for _ in range(p)]
    pick = (lambda x: x) if p > 1 else (lambda x: x[0])
    G, Wg, Dg = (tc.Group(comm, pick(x)) for x in (dg, dwt, ddw))
    tc.sgd_step(Wg, G, Dg, rescale=rescale, **hp)
    res = [(to_host(dg[r]), to_host(dwt[r]), to_host(ddw[r])) for r in range(p)]
    algo = comm.last_launch()[0]
    assert comm.async_error() == 0
    for grp in (G, Wg, Dg):
        grp.destroy()
    comm.destroy()
    want = O.sgd_step([w] * p, gs, [dw] * p, rescale=rescale, **hp)
    return res, want, algo, (gs, w, dw, rescale)


@pytest.mark.parametrize("name,oneshot", ALGOS + [("local", -1)])
@pytest.mark.parametrize("hp", [SGD_PERF, SGD_DYADIC], ids=["perf", "dyadic"])
def test_sgd_step(name, oneshot, hp):
    p = 1 if name == "local" else 4
    numels = [7, 13, 1000, 4096, 1, 0, 65]
    res, (G, Ws, Dws), algo, _ = run_sgd(p, numels, "grad" if hp is SGD_PERF else "int", hp,
                                         oneshot)
    assert algo == name
    for r in range(p):
        assert_bitwise(res[r][0], G, f"g rank {r}")
        assert_bitwise(res[r][1], Ws[r], f"w rank {r}")
        assert_bitwise(res[r][2], Dws[r], f"dw rank {r}")


def test_sgd_tolerance_vs_f64():
    p = 8
    numels = [5000, 3, 77]
    res, _, _, (gs, w, dw, rescale) = run_sgd(p, numels, "grad", SGD_PERF, TWOSHOT)
    _, wr, dwr = O.sgd_step_f64([w] * p, gs, [dw] * p, rescale=rescale, **SGD_PERF)
    for t in range(len(numels)):
        sabs = sum(np.abs(gs[k][t].astype(np.float64)) for k in range(p))
        bd = 1e-5 * (0.9 * np.abs(dw[t]) + 0.1 * (rescale * sabs + 1e-4 * np.abs(w[t])))
        assert (np.abs(res[0][2][t] - dwr[0][t]) <= bd + 1e-30).all()
        bw = 1e-5 * (np.abs(w[t]) + np.abs(res[0][2][t]))
        assert (np.abs(res[0][1][t] - wr[0][t]) <= bw + 1e-30).all()


# ------------------------------------------------------------------ EASGD (A7)
def run_easgd(c, numels, alpha, oneshot=-1, kind="float"):
    if kind == "int":
        center = W.group(numels, "int", W.CFG_EASGD, 0, 0, W.CENTER)
        xs = [W.group(numels, "int", W.CFG_EASGD, 0, i, W.PARAM) for i in range(c)]
    else:
        center = W.group(numels, "center", W.CFG_EASGD, 0, 0, W.CENTER)
        xs = [W.client_params(numels, center, W.CFG_EASGD, 0, i) for i in range(c)]
    comm = _comm(c, oneshot)
    dx = [to_dev(x) for x in xs]
    dc = [to_dev(center) for _ in range(c)]
    pick = (lambda x: x) if c > 1 else (lambda x: x[0])
    X, C = tc.Group(comm, pick(dx)), tc.Group(comm, pick(dc))
    tc.easgd_update(X, C, alpha)
    res = [(to_host(dx[i]), to_host(dc[i])) for i in range(c)]
    algo = comm.last_launch()[0]
    assert comm.async_error() == 0
    X.destroy()
    C.destroy()
    comm.destroy()
    return res, xs, center, algo


@pytest.mark.parametrize("name,oneshot,c", [a + (c,) for a in ALGOS for c in (2, 4, 8)] +
                         [("local", -1, 1)])
@pytest.mark.parametrize("alpha", [0.1, 0.5, 0.0])
def test_easgd(name, oneshot, c, alpha):
    numels = [7, 13, 1000, 4096, 0, 2]
    res, xs, center, algo = run_easgd(c, numels, alpha, oneshot)
    assert algo == name
    wx, wc = O.easgd_update(xs, center, alpha)
    for i in range(c):
        assert_bitwise(res[i][0], wx[i], f"x client {i}")
        assert_bitwise(res[i][1], wc, f"center replica {i}")


@pytest.mark.parametrize("xoff,coff", [(0, 0), (1, 1), (0, 3)])
def test_easgd_single_client_tiles(xoff, coff):
    """c = 1 on the p = 1 TMA stream: tile-boundary shapes, x and center shifted alike (vector
    path) or differently (element path)."""
    numels = [2048, 2049, 4099, 1, 10000, 6143]
    center = W.group(numels, "center", W.CFG_EASGD, 1, 0, W.CENTER)
    x = W.client_params(numels, center, W.CFG_EASGD, 1, 0)
    comm = tc.Comm.single(0)
    dx, dc = to_dev(x, offset=xoff), to_dev(center, offset=coff)
    X, C = tc.Group(comm, dx), tc.Group(comm, dc)
    tc.easgd_update(X, C, 0.1)
    assert comm.last_launch()[0] == "local"
    wx, wc = O.easgd_update([x], center, 0.1)
    assert_bitwise(to_host(dx), wx[0], "x")
    assert_bitwise(to_host(dc), wc, "center")
    X.destroy()
    C.destroy()
    comm.destroy()


def test_tiny_config_easgd_int_conservation():
    """Config 1's EASGD step (4 workers = 4 clients, alpha = 0.1) on integer inputs, plus the
    alpha = 0.5 conservation pin on the GPU result itself."""
    c = 4
    res, xs, center, _ = run_easgd(c, W.TINY, 0.1, kind="int")
    wx, wc = O.easgd_update(xs, center, 0.1)
    for i in range(c):
        assert_bitwise(res[i][0], wx[i])
        assert_bitwise(res[i][1], wc)
    res, xs, center, _ = run_easgd(c, W.TINY, 0.5, kind="int", oneshot=TMA)
    for t in range(3):
        before = sum(xs[i][t].astype(np.float64) for i in range(c)) + center[t]
        after = sum(res[i][0][t].astype(np.float64) for i in range(c)) + res[0][1][t]
        assert (before == after).all()


# ------------------------------------------------------------------ errors and faults (T3)
def test_errors():
    comm = tc.Comm.emulated(2, 0)
    a = [to_dev([np.zeros(5, np.float32)]) for _ in range(2)]
    b = [to_dev([np.zeros(6, np.float32)]) for _ in range(2)]
    with pytest.raises(tc.TcError) as e:
        tc.Group(comm, [a[0], b[0]])  # ranks disagree on n_t
    assert e.value.status == tc.tc.TC_ERR_SHAPE_MISMATCH
    ga, gb = tc.Group(comm, a), tc.Group(comm, b)
    with pytest.raises(tc.TcError) as e:
        tc.easgd_update(ga, gb, 0.1)  # not congruent
    assert e.value.status == tc.tc.TC_ERR_SHAPE_MISMATCH
    with pytest.raises(tc.TcError) as e:
        tc.easgd_update(ga, ga, 1.5)  # alpha outside [0, 1]
    assert e.value.status == tc.tc.TC_ERR_INVALID_ARG
    with pytest.raises(tc.TcError) as e:
        tc.allreduce(ga, float("nan"))
    assert e.value.status == tc.tc.TC_ERR_INVALID_ARG
    ga.destroy()
    gb.destroy()
    comm.destroy()


def test_timeout_when_a_rank_is_absent():
    """A rank that never arrives: the others time out, the error is sticky, later calls fail."""
    comm = tc.Comm.emulated(2, 0)
    comm.set_timeout(200)
    comm.set_debug_absent_rank(1)
    xs = [to_dev([np.ones(4096, np.float32)]) for _ in range(2)]
    grp = tc.Group(comm, xs)
    comm.set_tuning(0, 0, TWOSHOT)
    comm.set_algorithm(1)
    tc.allreduce(grp)
    torch.cuda.synchronize()
    assert comm.async_error() == tc.tc.TC_ERR_TIMEOUT
    with pytest.raises(tc.TcError) as e:
        tc.allreduce(grp)
    assert e.value.status == tc.tc.TC_ERR_TIMEOUT
    grp.destroy()
    comm.destroy()


# ------------------------------------------------------------------ config-5 shapes, small totals
# (full-size configs 2-5, whole arrays: tests/test_gpu_fullsize.py)
@pytest.mark.parametrize("p", [1, 2, 4])
@pytest.mark.parametrize("T", [1, 2, 8, 32, 161, 512, 1024])
def test_config5_sweep_shapes(p, T):
    """Config 5 shapes (seeded log-uniform splits, unaligned tails) at the small totals the
    oracle covers fully (16 KiB, 1 MiB), as views of one flat buffer like bench_sweep.py."""
    for total in (16 << 10, 1 << 20):
        numels = W.sweep_numels(total, T)
        if not numels:
            continue
        xs = [W.group(numels, "grad", W.CFG_SWEEP, 0, k, W.GRAD) for k in range(p)]
        for oneshot in ((TWOSHOT,) if p == 1 else (TWOSHOT, ONESHOT, LL, TMA)):
            if oneshot == LL and total > (64 << 10):
                continue
            comm = _comm(p, oneshot)
            flats = [torch.from_numpy(np.concatenate(x)).cuda() for x in xs]
            views = [list(torch.split(f, numels)) for f in flats]
            grp = tc.Group(comm, views if p > 1 else views[0])
            tc.allreduce(grp, 0.5)
            want = O.allreduce(xs, 0.5)
            for r in range(p):
                assert_bitwise(to_host(views[r]), want, f"T={T} total={total} rank {r}")
            grp.destroy()
            comm.destroy()


# ------------------------------------------------------------------ NEXT row f2: fused elastic + SGD
@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("offset", [0, 1])
def test_esgd_step(p, offset):
    """tc_esgd_step (one GPU per client) bit-exact vs oracle.esgd_step: ragged groups with
    multi-tile tensors; offset 1 shifts every tensor off its 16-B boundary (element path at
    p = 1 heads, shifted grid at p >= 2)."""
    numels = [7, 13, 1000, 4096, 0, 2, 3001, 9000]
    center = W.group(numels, "center", W.CFG_EASGD, 5, 0, W.CENTER)
    xs = [W.client_params(numels, center, W.CFG_EASGD, 5, i) for i in range(p)]
    gs = [W.group(numels, "grad", W.CFG_EASGD, 6, i, W.GRAD) for i in range(p)]
    dws = [W.group(numels, "dw", W.CFG_EASGD, 7, i, W.DW) for i in range(p)]
    hp = dict(alpha=0.1, lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / 128)
    comm = tc.Comm.single(0) if p == 1 else tc.Comm.emulated(p, 0)
    dx = [to_dev(x, offset=offset) for x in xs]
    dc = [to_dev(center, offset=offset) for _ in range(p)]
    dg = [to_dev(g, offset=offset) for g in gs]
    dd = [to_dev(d, offset=offset) for d in dws]
    pick = (lambda v: v) if p > 1 else (lambda v: v[0])
    X, C, G, D = (tc.Group(comm, pick(v)) for v in (dx, dc, dg, dd))
    tc.esgd_step(X, C, G, D, **hp)
    assert comm.last_launch()[0] == ("local" if p == 1 else "two-shot-tma")
    assert comm.async_error() == 0
    wx, wc, wd = O.esgd_step(xs, center, gs, dws, **hp)
    for i in range(p):
        assert_bitwise(to_host(dx[i]), wx[i], f"x client {i}")
        assert_bitwise(to_host(dc[i]), wc, f"center replica {i}")
        assert_bitwise(to_host(dd[i]), wd[i], f"dw client {i}")
        assert_bitwise(to_host(dg[i]), gs[i], f"g client {i} (read only)")
    for grp in (X, C, G, D):
        grp.destroy()
    comm.destroy()


def test_esgd_step_errors():
    comm = tc.Comm.emulated(2, 0)
    a = [to_dev(W.group([5, 9], "grad", 1, 0, k, W.GRAD)) for k in range(2)]
    b = [to_dev(W.group([5, 8], "grad", 1, 0, k, W.GRAD)) for k in range(2)]
    ga, gb = tc.Group(comm, a), tc.Group(comm, b)
    with pytest.raises(tc.TcError) as e:
        tc.esgd_step(ga, ga, gb, ga, 0.1, 0.1)  # not congruent
    assert e.value.status == tc.tc.TC_ERR_SHAPE_MISMATCH
    with pytest.raises(tc.TcError) as e:
        tc.esgd_step(ga, ga, ga, ga, 1.5, 0.1)  # alpha outside [0, 1]
    assert e.value.status == tc.tc.TC_ERR_INVALID_ARG
    ga.destroy()
    gb.destroy()
    comm.destroy()


# ------------------------------------------------------------------ tensor broadcast
@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("offset", [0, 1])
def test_broadcast(p, offset):
    numels = [7, 13, 1000, 4096, 0, 2, 3001, 9000]
    xs = [W.group(numels, "grad", 84, 0, k, W.GRAD) for k in range(p)]
    for root in sorted({0, p // 2, p - 1}):  # p >= 3: the root owns no chunk (first/middle/last)
        comm = tc.Comm.single(0) if p == 1 else tc.Comm.emulated(p, 0)
        dev = [to_dev(x, offset=offset) for x in xs]
        g = tc.Group(comm, dev if p > 1 else dev[0])
        tc.broadcast(g, root)
        if p > 1:
            assert comm.last_launch()[0] == "two-shot-tma"
        want = O.broadcast(xs, root)
        for r in range(p):
            assert_bitwise(to_host(dev[r]), want[r], f"rank {r} root {root}")
        assert comm.async_error() == 0
        with pytest.raises(tc.TcError):
            tc.broadcast(g, p)  # root outside the comm
        g.destroy()
        comm.destroy()


def test_busy_one_call_per_comm():
    """S:246 "one collective call per communicator at a time": while another call holds the
    comm (fault injection marks it busy) every call that takes it returns TC_ERR_BUSY and does
    nothing; once released the same calls succeed.  Then two host threads hammer one comm:
    every call either succeeds or reports TC_ERR_BUSY, never anything else."""
    import threading
    comm = tc.Comm.emulated(2, 0)
    xs = [W.group([7, 13, 1000], "int", 80, 0, k, W.GRAD) for k in range(2)]
    dev = [to_dev(x) for x in xs]
    g = tc.Group(comm, dev)
    comm.set_debug_busy(True)
    with pytest.raises(tc.TcError) as e:
        tc.allreduce(g)
    assert e.value.status == tc.tc.TC_ERR_BUSY
    with pytest.raises(tc.TcError) as e:
        tc.Group(comm, [to_dev(x) for x in xs])
    assert e.value.status == tc.tc.TC_ERR_BUSY
    for r in range(2):  # nothing ran
        assert_bitwise(to_host(dev[r]), xs[r], f"rank {r} untouched")
    comm.set_debug_busy(False)
    tc.allreduce(g, 0.5)
    want = O.allreduce(xs, 0.5)
    for r in range(2):
        assert_bitwise(to_host(dev[r]), want, f"rank {r}")

    seen = {"ok": 0, "busy": 0, "other": []}
    lock = threading.Lock()

    def hammer():
        for _ in range(300):
            st = tc.LIB.tc_allreduce(g.h, 0.5, None)
            with lock:
                if st == tc.tc.TC_OK:
                    seen["ok"] += 1
                elif st == tc.tc.TC_ERR_BUSY:
                    seen["busy"] += 1
                else:
                    seen["other"].append(st)

    th = [threading.Thread(target=hammer) for _ in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not seen["other"], seen
    assert seen["ok"] + seen["busy"] == 600 and seen["ok"] >= 1, seen
    assert comm.async_error() == 0
    g.destroy()
    comm.destroy()


def test_group_cta_budget():
    """tc_group_set_num_ctas: a per-group CTA budget (the comm's tuning is untouched), same
    results."""
    p = 4
    numels = [7, 13, 1000, 40000, 3]
    xs = [W.group(numels, "grad", 81, 0, k, W.GRAD) for k in range(p)]
    comm = _comm(p, TMA)
    dev = [to_dev(x) for x in xs]
    g = tc.Group(comm, dev)
    g.set_num_ctas(3)
    tc.allreduce(g, 0.25)
    assert comm.last_launch()[:2] == ("two-shot-tma", 3)
    want = O.allreduce(xs, 0.25)
    for r in range(p):
        assert_bitwise(to_host(dev[r]), want, f"rank {r}")
    g.set_num_ctas(0)
    tc.allreduce(g, 1.0)
    assert comm.last_launch()[1] > 3
    with pytest.raises(tc.TcError):
        g.set_num_ctas(-1)
    g.destroy()
    comm.destroy()


# ------------------------------------------------------------------ NEXT row f2: async-server EASGD
@pytest.mark.parametrize("c", [2, 3, 4, 8])
@pytest.mark.parametrize("offset", [0, 1, "per-rank"])
def test_easgd_async(c, offset):
    """Server-side Elastic1 per arrival in a recorded order, Elastic2 at the client, bit-exact
    vs oracle.easgd_async: ragged multi-tile groups, aligned / shifted / per-rank misaligned
    tensors (vector, shifted and element paths), several orders."""
    numels = [7, 13, 1000, 4096, 0, 2, 3001, 9000, 70001]
    center = W.group(numels, "center", W.CFG_EASGD, 8, 0, W.CENTER)
    xs = [W.client_params(numels, center, W.CFG_EASGD, 8, i) for i in range(c)]
    g = np.random.default_rng(c)
    off = (lambda k: k % 4) if offset == "per-rank" else (lambda k: offset)
    for order in (None, list(reversed(range(c))), [int(i) for i in g.permutation(c)]):
        comm = tc.Comm.emulated(c, 0)
        dx = [to_dev(x, offset=off(i)) for i, x in enumerate(xs)]
        dc = [to_dev(center, offset=off(i)) for i in range(c)]
        X, C = tc.Group(comm, dx), tc.Group(comm, dc)
        tc.easgd_async_update(X, C, 0.1, order)
        assert comm.last_launch()[0] == "two-shot-tma"
        assert comm.async_error() == 0
        wx, wc = O.easgd_async(xs, center, 0.1, order)
        for i in range(c):
            assert_bitwise(to_host(dx[i]), wx[i], f"x client {i} order {order}")
            assert_bitwise(to_host(dc[i]), wc, f"center replica {i} order {order}")
        X.destroy()
        C.destroy()
        comm.destroy()


def test_easgd_async_single_client_and_errors():
    numels = [7, 13, 1000, 4099]
    center = W.group(numels, "center", W.CFG_EASGD, 9, 0, W.CENTER)
    x = W.client_params(numels, center, W.CFG_EASGD, 9, 0)
    comm = tc.Comm.single(0)
    dx, dc = to_dev(x), to_dev(center)
    X, C = tc.Group(comm, dx), tc.Group(comm, dc)
    tc.easgd_async_update(X, C, 0.25, [0])
    wx, wc = O.easgd_async([x], center, 0.25)
    assert_bitwise(to_host(dx), wx[0])
    assert_bitwise(to_host(dc), wc)
    X.destroy()
    C.destroy()
    comm.destroy()
    comm = tc.Comm.emulated(3, 0)
    dx = [to_dev(x) for _ in range(3)]
    dc = [to_dev(center) for _ in range(3)]
    X, C = tc.Group(comm, dx), tc.Group(comm, dc)
    for bad in ([0, 0, 1], [0, 1, 3]):
        with pytest.raises(tc.TcError) as e:
            tc.easgd_async_update(X, C, 0.1, bad)
        assert e.value.status == tc.tc.TC_ERR_INVALID_ARG
    X.destroy()
    C.destroy()
    comm.destroy()


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_degenerate_groups(p):
    """Degenerate groups: every tensor empty (the calls are no-ops and succeed), and a single
    element over p ranks (one owner holds it, the others own nothing)."""
    comm = tc.Comm.single(0) if p == 1 else tc.Comm.emulated(p, 0)
    pick = (lambda v: v) if p > 1 else (lambda v: v[0])
    empty = [[torch.empty(0, device="cuda"), torch.empty(0, device="cuda")] for _ in range(p)]
    g = tc.Group(comm, pick(empty))
    tc.allreduce(g, 0.5)
    tc.sgd_step(g, g, g, lr=0.1)
    tc.easgd_update(g, g, 0.1)
    g.destroy()
    xs = [[np.array([float(k + 1)], np.float32)] for k in range(p)]
    for algo in ((0, -1, -1), (1, 0, 0), (6, 0, 0), (0, 1 << 20, 0), (0, 0, 1 << 20)):
        if p > 1:
            comm.set_algorithm(algo[0])
            comm.set_tuning(0, 0, algo[1])
            comm.set_ll_max(algo[2])
        dev = [to_dev(x) for x in xs]
        g = tc.Group(comm, pick(dev))
        tc.allreduce(g, 1.0)
        want = O.allreduce(xs)
        for r in range(p):
            assert_bitwise(to_host(dev[r]), want, f"algo {algo} rank {r}")
        g.destroy()
    assert comm.async_error() == 0
    comm.destroy()
