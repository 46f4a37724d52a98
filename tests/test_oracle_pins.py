"""T0: the CPU oracle pinned against what the paper and mathematics fix (not against itself).

Each test names the passage it pins.  P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import tc_workloads as W
from oracle import tc_oracle as O

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _grp(vals):
    return [np.asarray(v, np.float32) for v in vals]


# ------------------------------------------------------------------ allreduce
def test_golden_lane_reduce():
    ex = GOLDEN["lane_reduce"]
    out = O.allreduce([_grp([x]) for x in ex["inputs"]])
    assert out[0].tolist() == ex["expected"]


def test_golden_reduce_scatter_p2():
    ex = GOLDEN["reduce_scatter_p2"]
    # two 1-element tensors per rank so each rank owns one (slot-granular partition, R2)
    xs = [_grp([[v] for v in x]) for x in ex["inputs"]]
    pieces = [O.reduce_scatter(xs, r) for r in range(2)]
    got = [[float(v) for (_, _, _, vals) in pc for v in vals] for pc in pieces]
    assert got == ex["expected_rank_pieces"]


def test_golden_allreduce_rank_lanes():
    ex = GOLDEN["allreduce_rank_lanes"]
    xs = [_grp([[w]]) for w in range(ex["workers"]) for _ in range(ex["lanes"])]
    assert O.allreduce(xs)[0].tolist() == [ex["expected"]]


def test_golden_partition_sizes():
    ex = GOLDEN["allgather_p3_n7"]
    _, owners = O.slot_partition([4 * ex["n"]], ex["p"])
    assert sorted([b - a for a, b in owners], reverse=True) == ex["expected_sizes"]


def test_golden_kvstore_ones():
    ex = GOLDEN["kvstore_ones"]
    xs = [[np.ones(ex["shape"], np.float32) for _ in ex["keys"]] for _ in range(ex["gpus"])]
    for t in O.allreduce(xs):
        assert (t == ex["expected"]).all()


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8])
def test_allreduce_bruteforce_integers(p):
    """Brute force: integer-valued fp32 in [-1000,1000], p<=8 -> every order exact; compare
    with Python int sums element by element (pins dropped terms, wrong index or sign)."""
    numels = [7, 13, 1000, 1, 0, 33]
    xs = [W.group(numels, "int", 99, 0, k, W.GRAD) for k in range(p)]
    out = O.allreduce(xs)
    for t, n in enumerate(numels):
        for j in range(n):
            assert float(out[t][j]) == sum(int(xs[k][t][j]) for k in range(p))


def test_allreduce_scale_exact():
    xs = [W.group([50], "int", 98, 0, k, W.GRAD) for k in range(4)]
    out = O.allreduce(xs, scale=0.25)
    for j in range(50):
        assert Fraction(float(out[0][j])) == Fraction(sum(int(xs[k][0][j]) for k in range(4)), 4)


def test_allreduce_special_cases():
    g = W.group([9, 4], "grad", 97, 0, 0, W.GRAD)
    # p = 1, scale = 1 is the identity
    out = O.allreduce([g])
    assert all((a == b).all() for a, b in zip(out, g))
    # all-ones -> p
    assert (O.allreduce([[np.ones(5, np.float32)]] * 6)[0] == 6).all()
    # rank-valued -> p(p-1)/2
    p = 7
    assert (O.allreduce([[np.full(3, k, np.float32)] for k in range(p)])[0] == p * (p - 1) / 2).all()


@pytest.mark.parametrize("p", [2, 4, 8])
def test_allreduce_correctly_rounded(p):
    """Within the paper's error bound, in fact exact: for gradient-like fp32 inputs the float64
    sequential sum of p<=8 addends is exact, so the oracle equals the correctly rounded exact
    sum (math.fsum) bit for bit."""
    xs = [W.group([3000], "grad", 96, 0, k, W.GRAD) for k in range(p)]
    out = O.allreduce(xs)[0]
    exact = np.array([math.fsum(float(xs[k][0][j]) for k in range(p)) for j in range(3000)])
    assert (out == exact.astype(np.float32)).all()


def test_allreduce_same_on_every_rank_and_split_invariant():
    """Invariant: one result for all ranks; re-splitting the same flat data into different
    tensors gives the same bits (the group is one object)."""
    p = 4
    flat = [np.concatenate(W.group([4000], "grad", 95, 0, k, W.GRAD)) for k in range(p)]
    a = np.concatenate(O.allreduce([[f] for f in flat]))
    splits = [7, 13, 980, 3000]
    xs = [np.split(f, np.cumsum(splits)[:-1]) for f in flat]
    b = np.concatenate(O.allreduce(xs))
    assert (a == b).all()


@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_allreduce_equals_ring_algorithm_and_bytes(p):
    """allgather(reduce_scatter) == allreduce via the paper's bucket algorithm
    on exact integer inputs, and the byte count 2(p-1)/p n per rank."""
    n = 4 * p * 25
    flat = [W.draw("int", n, W.rng(94, 0, k, 0, 0)) for k in range(p)]
    res, sent, steps = O.ring_allreduce_sim(flat)
    ref = O.allreduce([[f] for f in flat])[0]
    for r in range(p):
        assert (res[r].astype(np.float32) == ref).all()
        assert sent[r] == 2 * n * (p - 1) // p
    assert steps == 2 * (p - 1)
    assert O.bus_bytes_per_rank(p, 4 * n) == 4 * sent[0]


def test_reduce_scatter_then_allgather_is_allreduce():
    p = 3
    numels = [7, 13, 1000]
    xs = [W.group(numels, "grad", 93, 0, k, W.GRAD) for k in range(p)]
    pieces = [O.reduce_scatter(xs, r) for r in range(p)]
    full = O.allgather(pieces, numels)
    ref = O.allreduce(xs)
    assert all((a == b).all() for a, b in zip(full, ref))


def test_predict_cost_golden():
    ex = GOLDEN["predict_cost"]
    assert O.predict_cost(ex["p"], ex["n"], ex["alpha"], ex["beta"], ex["gamma"]) == ex["expected"]
    assert O.predict_cost(1, 1e6, 3, 1, 1) == 0


def test_allreduce_tolerance_vs_f64():
    p = 8
    xs = [W.group([5000], "grad", 92, 0, k, W.GRAD) for k in range(p)]
    out = O.allreduce(xs)[0].astype(np.float64)
    ref = O.allreduce_f64(xs)[0]
    bound = 1e-5 * sum(np.abs(xs[k][0].astype(np.float64)) for k in range(p))
    assert (np.abs(out - ref) <= bound).all()


# ------------------------------------------------------------------ partition (A1)
@pytest.mark.parametrize("p", [1, 2, 3, 4, 7, 8])
def test_slot_partition_invariants(p):
    numels = [7, 13, 1000, 0, 1, 64, 5]
    prefix, owners = O.slot_partition(numels, p)
    M = prefix[-1]
    assert prefix == [0, 2, 6, 256, 256, 257, 273, 275]
    assert owners[0][0] == 0 and owners[-1][1] == M
    for r in range(p - 1):
        assert owners[r][1] == owners[r + 1][0]
    sizes = [b - a for a, b in owners]
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == M


# ------------------------------------------------------------------ SGD (Eq. 1)
def test_golden_sgd():
    ex = GOLDEN["sgd_update"]
    G, w, dw = O.sgd_step([_grp([ex["w"]])], [_grp([ex["g"]])], [_grp([[0.0]])],
                          lr=ex["lr"], momentum=0.0, wd=0.0, rescale=ex["rescale"])
    assert w[0][0].tolist() == np.asarray(ex["expected_f32"], np.float32).tolist()


def test_sgd_mu0_is_eq1_exact():
    """mu = 0, wd = 0 reduces to Eq. 1: w' = w - lr * rescale * sum_k g_k (dyadic lr, rescale so
    every step is exact; compared with exact rational arithmetic)."""
    p = 4
    numels = [7, 13, 100]
    gs = [W.group(numels, "int", 91, 0, k, W.GRAD) for k in range(p)]
    w = W.group(numels, "int", 91, 0, 0, W.PARAM)
    dw = W.group(numels, "int", 91, 0, 0, W.DW)
    lr, rescale = 0.5, 1.0 / (p * 128)
    G, ws, dws = O.sgd_step([w] * p, gs, [dw] * p, lr, 0.0, 0.0, rescale)
    for t, n in enumerate(numels):
        for j in range(n):
            g = sum(Fraction(float(gs[k][t][j])) for k in range(p))
            assert Fraction(float(G[t][j])) == g
            assert Fraction(float(ws[1][t][j])) == Fraction(float(w[t][j])) - Fraction(lr) * Fraction(rescale) * g


def test_sgd_dyadic_exact_rational():
    """Reading R12 (momentum form), evaluated in exact rationals on dyadic inputs where no
    rounding occurs: pins operation order, signs and every term (rescale, wd, mu, lr)."""
    p = 2
    numels = [64]
    gs = [W.group(numels, "int", 90, 0, k, W.GRAD) for k in range(p)]
    w = W.group(numels, "int", 90, 0, 0, W.PARAM)
    dw = W.group(numels, "int", 90, 0, 0, W.DW)
    lr, mu, wd, rs = 0.5, 0.5, 0.25, 0.125
    _, ws, dws = O.sgd_step([w] * p, gs, [dw] * p, lr, mu, wd, rs)
    Fr = Fraction
    for j in range(64):
        g = sum(Fr(float(gs[k][0][j])) for k in range(p))
        t = Fr(rs) * g + Fr(wd) * Fr(float(w[0][j]))
        d = Fr(mu) * Fr(float(dw[0][j])) - Fr(lr) * t
        assert Fr(float(dws[0][0][j])) == d
        assert Fr(float(ws[0][0][j])) == Fr(float(w[0][j])) + d


def test_sgd_momentum_geometric_series():
    """Closed form: constant summed gradient G, wd=0, dw0=0: after K steps
    dw_K = -lr*rescale*G*(1-mu^K)/(1-mu) (dyadic values keep it exact)."""
    G = np.float32(8.0)
    w = [np.zeros(1, np.float32)]
    dw = [np.zeros(1, np.float32)]
    lr, mu, rs = 0.5, 0.5, 0.25
    for _ in range(6):
        _, ws, dws = O.sgd_step([w], [[np.array([G], np.float32)]], [dw], lr, mu, 0.0, rs)
        w, dw = ws[0], dws[0]
    K = 6
    assert Fraction(float(dw[0][0])) == -Fraction(lr) * Fraction(rs) * 8 * (1 - Fraction(mu) ** K) / (1 - Fraction(mu))


def test_sgd_momentum_matches_library_optimizer():
    """R12's momentum form (P:158 names "momentum SGD") against an independent library routine:
    torch.optim.SGD (buf <- mu*buf + g + wd*w; w <- w - lr*buf, dampening 0) is the same
    trajectory for constant lr with dw = -lr*buf.  Several steps, p = 3 ranks, float64; the
    gradient the optimiser sees is rescale * (the plain sum over ranks)."""
    import torch
    p, n, steps = 3, 257, 5
    lr, mu, wd, rs = 0.125, 0.875, 0.0078125, 0.25  # exact in fp32 (they cross a C float)
    w = W.group([n], "param", 61, 0, 0, W.PARAM)
    dw = [np.zeros(n, np.float32)]
    tw = torch.tensor(w[0].astype(np.float64), requires_grad=True)
    opt = torch.optim.SGD([tw], lr=lr, momentum=mu, weight_decay=wd, dampening=0.0)
    ws_o, dws_o = [w] * p, [dw] * p
    for s in range(steps):
        gs = [W.group([n], "grad", 61, s, k, W.GRAD) for k in range(p)]
        _, ws_o, dws_o = O.sgd_step_f64(ws_o, gs, dws_o, lr, mu, wd, rs)
        tw.grad = torch.tensor(rs * np.stack([g[0].astype(np.float64) for g in gs]).sum(0))
        opt.step()
    ref = tw.detach().numpy()
    for k in range(p):
        np.testing.assert_allclose(ws_o[k][0], ref, rtol=1e-12, atol=1e-15)
    buf = opt.state[tw]["momentum_buffer"].numpy()
    np.testing.assert_allclose(dws_o[0][0], -lr * buf, rtol=1e-12, atol=1e-15)


def test_sgd_zero_grad_identity():
    w = W.group([33], "param", 89, 0, 0, W.PARAM)
    z = [np.zeros(33, np.float32)]
    _, ws, dws = O.sgd_step([w], [z], [z], 0.1, 0.9, 0.0, 1.0)
    assert (ws[0][0] == w[0]).all() and (dws[0][0] == 0).all()


def test_sgd_tolerance_vs_f64():
    p = 4
    numels = [4000]
    gs = [W.group(numels, "grad", 88, 0, k, W.GRAD) for k in range(p)]
    w = W.group(numels, "param", 88, 0, 0, W.PARAM)
    dw = W.group(numels, "dw", 88, 0, 0, W.DW)
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / (p * 128))
    _, ws, dws = O.sgd_step([w] * p, gs, [dw] * p, **hp)
    _, wr, dwr = O.sgd_step_f64([w] * p, gs, [dw] * p, **hp)
    sabs = sum(np.abs(gs[k][0].astype(np.float64)) for k in range(p))
    bd = 1e-5 * (0.9 * np.abs(dw[0]) + 0.1 * (hp["rescale"] * sabs + 1e-4 * np.abs(w[0])))
    assert (np.abs(dws[0][0] - dwr[0][0]) <= bd + 1e-30).all()
    bw = 1e-5 * (np.abs(w[0]) + np.abs(dws[0][0]))
    assert (np.abs(ws[0][0] - wr[0][0]) <= bw + 1e-30).all()


# ------------------------------------------------------------------ EASGD
def test_golden_elastic_c1():
    ec, el = GOLDEN["elastic_center_update"], GOLDEN["elastic_local_update"]
    xs, c = O.easgd_update([_grp([ec["w"]])], _grp([ec["center"]]), ec["alpha"])
    assert c[0].tolist() == ec["expected"]
    xs, c = O.easgd_update([_grp([el["w"]])], _grp([el["center"]]), el["alpha"])
    assert xs[0][0].tolist() == el["expected"]


def test_elastic_c1_is_eq_elastic1_elastic2_exact():
    """c = 1 with dyadic alpha on integer inputs: exactly Eq. elastic1 and Eq. elastic2."""
    x = W.group([200], "int", 87, 0, 0, W.PARAM)
    xc = W.group([200], "int", 87, 0, 0, W.CENTER)
    a = Fraction(0.25)
    xs, c = O.easgd_update([x], xc, 0.25)
    for j in range(200):
        w, wt = Fraction(float(x[0][j])), Fraction(float(xc[0][j]))
        assert Fraction(float(c[0][j])) == wt + a * (w - wt)        # elastic1
        assert Fraction(float(xs[0][0][j])) == w - a * (w - wt)     # elastic2


@pytest.mark.parametrize("c", [2, 3, 4])
def test_elastic_sum_form_exact_rational(c):
    """Reading R10 (synchronous sum form): x_i' = x_i - a(x_i - xc), xc' = xc + a sum_i(x_i - xc)."""
    xs = [W.group([100], "int", 86, 0, i, W.PARAM) for i in range(c)]
    xc = W.group([100], "int", 86, 0, 0, W.CENTER)
    a = Fraction(0.125)
    xo, co = O.easgd_update(xs, xc, 0.125)
    for j in range(100):
        wt = Fraction(float(xc[0][j]))
        s = sum(Fraction(float(xs[i][0][j])) - wt for i in range(c))
        assert Fraction(float(co[0][j])) == wt + a * s
        for i in range(c):
            w = Fraction(float(xs[i][0][j]))
            assert Fraction(float(xo[i][0][j])) == w - a * (w - wt)


def test_elastic_alpha0_identity_and_fixed_point():
    xs = [W.group([300], "param", 85, 0, i, W.PARAM) for i in range(4)]
    xc = W.group([300], "center", 85, 0, 0, W.CENTER)
    xo, co = O.easgd_update(xs, xc, 0.0)
    assert all((xo[i][0] == xs[i][0]).all() for i in range(4)) and (co[0] == xc[0]).all()
    xo, co = O.easgd_update([xc] * 3, xc, 0.1)
    assert all((xo[i][0] == xc[0]).all() for i in range(3)) and (co[0] == xc[0]).all()


@pytest.mark.parametrize("alpha", [0.5, 0.25])
def test_elastic_conservation_exact(alpha):
    """sum_i x_i + xc is conserved (each client counted once), exactly for dyadic alpha."""
    c = 4
    xs = [W.group([500], "int", 84, 0, i, W.PARAM) for i in range(c)]
    xc = W.group([500], "int", 84, 0, 0, W.CENTER)
    xo, co = O.easgd_update(xs, xc, alpha)
    before = sum(xs[i][0].astype(np.float64) for i in range(c)) + xc[0]
    after = sum(xo[i][0].astype(np.float64) for i in range(c)) + co[0]
    assert (before == after).all()


def test_elastic_conservation_bounded_alpha01():
    c = 4
    center = W.group([20000], "center", 83, 0, 0, W.CENTER)
    xs = [W.client_params([20000], center, 83, 0, i) for i in range(c)]
    xo, co = O.easgd_update(xs, center, 0.1)
    before = sum(xs[i][0].astype(np.float64) for i in range(c)) + center[0]
    after = sum(xo[i][0].astype(np.float64) for i in range(c)) + co[0].astype(np.float64)
    mag = sum(np.abs(xs[i][0].astype(np.float64)) for i in range(c)) + np.abs(center[0])
    assert (np.abs(after - before) <= (c + 1) * 2.0 ** -24 * mag).all()


def test_elastic_contraction_c1():
    """c = 1: |x' - xc'| = |1 - 2a| |x - xc|, exact for dyadic a on integers; the
    alpha = 0.5 midpoint closes the gap."""
    x = W.group([300], "int", 82, 0, 0, W.PARAM)
    xc = W.group([300], "int", 82, 0, 0, W.CENTER)
    for a in (0.25, 0.5):
        xo, co = O.easgd_update([x], xc, a)
        gap0 = np.abs(x[0].astype(np.float64) - xc[0])
        gap1 = np.abs(xo[0][0].astype(np.float64) - co[0])
        assert (gap1 == abs(1 - 2 * a) * gap0).all()


def test_elastic_tolerance_vs_f64():
    c = 4
    center = W.group([5000], "center", 81, 0, 0, W.CENTER)
    xs = [W.client_params([5000], center, 81, 0, i) for i in range(c)]
    xo, co = O.easgd_update(xs, center, 0.1)
    xr, cr = O.easgd_update_f64(xs, center, 0.1)
    d = [np.abs(xs[i][0].astype(np.float64) - center[0]) for i in range(c)]
    for i in range(c):
        assert (np.abs(xo[i][0] - xr[i][0]) <= 1e-5 * (np.abs(xs[i][0]) + 0.1 * d[i])).all()
    assert (np.abs(co[0] - cr[0]) <= 1e-5 * (np.abs(center[0]) + 0.1 * sum(d))).all()


# ------------------------------------------------------------------ config 4 sequence
def test_esgd_sequence_composition():
    """8 steps (two elastic updates), tau = 4, 2 clients x 2 GPUs on integer data with dyadic
    hyper-parameters: every intermediate is exact, so the sequence equals an exact rational
    re-computation of Fig. code-snippet-4's order (Elastic2 before SGD.Update in the same
    iteration).  (At 16 steps the dyadic denominators outgrow fp32's 24-bit
    significand and the oracle rounds, as it must; config 4's 16-step sequence is pinned on the
    GPU side against this composition, tests/test_gpu_fullsize.py.)"""
    numels = [5, 11]
    c, q, steps, tau = 2, 2, 8, 4
    center = W.group(numels, "int", 80, 0, 0, W.CENTER)
    x0 = [W.group(numels, "int", 80, 0, i, W.PARAM) for i in range(c)]
    dw0 = [[np.zeros(n, np.float32) for n in numels] for _ in range(c)]
    grads = lambda t, i: [W.group(numels, "int", 80, t, 10 * i + k, W.GRAD) for k in range(q)]
    hp = dict(alpha=0.25, lr=0.5, momentum=0.5, wd=0.0, rescale=0.125)
    x, xc, dw = O.esgd_sequence(x0, center, dw0, grads, steps, tau, **hp)
    Fr = Fraction
    for t_idx, n in enumerate(numels):
        for j in range(n):
            X = [Fr(float(x0[i][t_idx][j])) for i in range(c)]
            D = [Fr(0)] * c
            C = Fr(float(center[t_idx][j]))
            for t in range(steps):
                if t % tau == 0:
                    d = [X[i] - C for i in range(c)]
                    X = [X[i] - Fr(hp["alpha"]) * d[i] for i in range(c)]
                    C = C + Fr(hp["alpha"]) * sum(d)
                for i in range(c):
                    g = sum(Fr(float(a[t_idx][j])) for a in grads(t, i))
                    D[i] = Fr(hp["momentum"]) * D[i] - Fr(hp["lr"]) * Fr(hp["rescale"]) * g
                    X[i] = X[i] + D[i]
            assert Fr(float(xc[t_idx][j])) == C
            for i in range(c):
                assert Fr(float(x[i][t_idx][j])) == X[i]


# ------------------------------------------------------------------ NEXT row f2: esgd_step
def test_esgd_step_exact_rational():
    """Elastic2 then SGD.Update in one iteration, one GPU per client, c = 3, on
    integer data with dyadic hyper-parameters: every fp32 intermediate is exact, so the oracle
    equals the formula evaluated in exact rationals."""
    numels = [6, 9]
    c = 3
    center = W.group(numels, "int", 81, 0, 0, W.CENTER)
    xs = [W.group(numels, "int", 81, 0, i, W.PARAM) for i in range(c)]
    gs = [W.group(numels, "int", 81, 1, i, W.GRAD) for i in range(c)]
    dws = [W.group(numels, "int", 81, 2, i, W.DW) for i in range(c)]
    hp = dict(alpha=0.25, lr=0.5, momentum=0.5, wd=0.25, rescale=0.125)
    x, xc, dw = O.esgd_step(xs, center, gs, dws, **hp)
    Fr = Fraction
    a, lr, mu, wd, rs = (Fr(hp[k]) for k in ("alpha", "lr", "momentum", "wd", "rescale"))
    for t, n in enumerate(numels):
        for j in range(n):
            C = Fr(float(center[t][j]))
            d = [Fr(float(xs[i][t][j])) - C for i in range(c)]
            assert Fr(float(xc[t][j])) == C + a * sum(d)
            for i in range(c):
                xe = Fr(float(xs[i][t][j])) - a * d[i]
                D = mu * Fr(float(dws[i][t][j])) - lr * (rs * Fr(float(gs[i][t][j])) + wd * xe)
                assert Fr(float(dw[i][t][j])) == D
                assert Fr(float(x[i][t][j])) == xe + D


def test_esgd_step_special_cases():
    """alpha = 0: exactly the local SGD step of every client (Eq. 1 with momentum); lr = 0 and
    momentum = 0: exactly the elastic update, with the momentum cleared."""
    numels = [7, 13, 100]
    c = 2
    center = W.group(numels, "center", 82, 0, 0, W.CENTER)
    xs = [W.client_params(numels, center, 82, 0, i) for i in range(c)]
    gs = [W.group(numels, "grad", 82, 1, i, W.GRAD) for i in range(c)]
    dws = [W.group(numels, "dw", 82, 2, i, W.DW) for i in range(c)]
    x, xc, dw = O.esgd_step(xs, center, gs, dws, 0.0, 0.1, 0.9, 1e-4, 0.5)
    for i in range(c):
        _, w1, d1 = O.sgd_step([xs[i]], [gs[i]], [dws[i]], 0.1, 0.9, 1e-4, 0.5)
        for t in range(len(numels)):
            assert np.array_equal(x[i][t], w1[0][t]) and np.array_equal(dw[i][t], d1[0][t])
    for t in range(len(numels)):
        assert np.array_equal(xc[t], center[t])
    x, xc, dw = O.esgd_step(xs, center, gs, dws, 0.1, 0.0, 0.0, 1e-4, 0.5)
    xe, ce = O.easgd_update(xs, center, 0.1)
    for t in range(len(numels)):
        assert np.array_equal(xc[t], ce[t])
        for i in range(c):
            assert np.array_equal(x[i][t], xe[i][t]) and not dw[i][t].any()


# ------------------------------------------------------------------ tensor broadcast
def test_broadcast_definition():
    numels = [7, 13, 0, 1000]
    xs = [W.group(numels, "grad", 83, 0, k, W.GRAD) for k in range(4)]
    for root in range(4):
        out = O.broadcast(xs, root)
        for r in range(4):
            for t in range(len(numels)):
                assert out[r][t].tobytes() == xs[root][t].tobytes()
                assert out[r][t] is not xs[root][t]


# ------------------------------------------------------------------ NEXT row f2: async server EASGD
def test_easgd_async_c1_is_eq_elastic1_elastic2_exact():
    """c = 1: one arrival is exactly Eq. elastic1 at the server and Eq. elastic2 at the client
    (P:69-78), evaluated in exact rationals on integer data with dyadic alpha."""
    x = W.group([300], "int", 90, 0, 0, W.PARAM)
    xc = W.group([300], "int", 90, 0, 0, W.CENTER)
    a = Fraction(0.25)
    xs, c = O.easgd_async([x], xc, 0.25)
    for j in range(300):
        w, wt = Fraction(float(x[0][j])), Fraction(float(xc[0][j]))
        assert Fraction(float(c[0][j])) == wt + a * (w - wt)        # elastic1
        assert Fraction(float(xs[0][0][j])) == w - a * (w - wt)     # elastic2


@pytest.mark.parametrize("order", [(0, 1, 2), (2, 0, 1), (1, 2, 0)])
def test_easgd_async_midpoint_closed_form(order):
    """alpha = 1/2: each arriving client and the center move to their midpoint, so after the
    arrivals i_1, i_2, i_3: x_{i_1}' = xc_1 = (xc + x_{i_1})/2, x_{i_k}' = xc_k =
    (xc_{k-1} + x_{i_k})/2 -- a closed form independent of the update formulas' code."""
    c = 3
    xs = [W.group([256], "int", 91, 0, i, W.PARAM) for i in range(c)]
    xc = W.group([256], "int", 91, 0, 0, W.CENTER)
    xo, co = O.easgd_async(xs, xc, 0.5, order)
    for j in range(256):
        cur = Fraction(float(xc[0][j]))
        for i in order:
            cur = (cur + Fraction(float(xs[i][0][j]))) / 2
            assert Fraction(float(xo[i][0][j])) == cur
        assert Fraction(float(co[0][j])) == cur


@pytest.mark.parametrize("alpha", [0.5, 0.25])
def test_easgd_async_conservation_exact(alpha):
    """Every arrival moves the center by +a d and the client by -a d, so sum_i x_i + xc is
    conserved -- exactly on integer data with dyadic alpha (no rounding occurs)."""
    c = 5
    xs = [W.group([400], "int", 92, 0, i, W.PARAM) for i in range(c)]
    xc = W.group([400], "int", 92, 0, 0, W.CENTER)
    xo, co = O.easgd_async(xs, xc, alpha, [3, 1, 4, 0, 2])
    before = sum(xs[i][0].astype(np.float64) for i in range(c)) + xc[0]
    after = sum(xo[i][0].astype(np.float64) for i in range(c)) + co[0]
    assert (before == after).all()


def test_easgd_async_alpha0_and_relabelling():
    """alpha = 0 is the identity; and the result depends on the clients only through the
    arrival sequence: permuting the clients together with the order permutes the outputs."""
    c = 4
    xs = [W.group([200], "param", 93, 0, i, W.PARAM) for i in range(c)]
    xc = W.group([200], "center", 93, 0, 0, W.CENTER)
    xo, co = O.easgd_async(xs, xc, 0.0, [2, 0, 3, 1])
    assert all((xo[i][0] == xs[i][0]).all() for i in range(c)) and (co[0] == xc[0]).all()
    order = [2, 0, 3, 1]
    perm = [3, 1, 0, 2]                      # new label of old client i is perm[i]
    ys = [None] * c
    for i in range(c):
        ys[perm[i]] = xs[i]
    xo, co = O.easgd_async(xs, xc, 0.1, order)
    yo, cy = O.easgd_async(ys, xc, 0.1, [perm[i] for i in order])
    assert all(np.array_equal(yo[perm[i]][0], xo[i][0]) for i in range(c))
    assert np.array_equal(cy[0], co[0])


def test_easgd_async_differs_from_sync_by_order():
    """c >= 2: the server's center moves between arrivals (the asynchronous form), unlike the
    synchronous sum form, which uses the pre-update center for every client (reading R10):
    the first arrival agrees with easgd_update's x_i', later ones do not in general."""
    c = 3
    xs = [W.group([500], "param", 94, 0, i, W.PARAM) for i in range(c)]
    xc = W.group([500], "center", 94, 0, 0, W.CENTER)
    xa, ca = O.easgd_async(xs, xc, 0.1, [1, 0, 2])
    xsync, _ = O.easgd_update(xs, xc, 0.1)
    assert np.array_equal(xa[1][0], xsync[1][0])
    assert not np.array_equal(xa[2][0], xsync[2][0])
    with pytest.raises(ValueError):
        O.easgd_async(xs, xc, 0.1, [0, 0, 1])
