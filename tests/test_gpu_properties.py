"""Property-based GPU parity (hypothesis): random ragged groups, rank counts, start offsets,
algorithms and ops, each bit-exact against the CPU oracle (T2 of SURVEY.md §4.2)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
from hypothesis import given, settings, strategies as st  # noqa: E402

import paper_1801_03855_b200 as tc  # noqa: E402
from oracle import tc_oracle as O  # noqa: E402
from gpu_util import to_dev, to_host, assert_bitwise  # noqa: E402

pytestmark = pytest.mark.gpu

# (algorithm id for set_algorithm, one-shot limit, LL limit)
ALGOS = {"auto": (0, -1, -1), "pull": (1, 0, 0), "tma": (6, 0, 0),
         "oneshot": (0, 1 << 30, 0), "ll": (0, 0, 1 << 30)}


@settings(max_examples=60, deadline=None)
@given(numels=st.lists(st.integers(0, 5000), min_size=1, max_size=24),
       p=st.sampled_from([1, 2, 3, 4, 8]), offset=st.integers(0, 3),
       algo=st.sampled_from(sorted(ALGOS)), op=st.sampled_from(["allreduce", "sgd", "easgd", "esgd"]),
       seed=st.integers(0, 2 ** 31 - 1))
def test_random_groups(numels, p, offset, algo, op, seed):
    if sum(numels) == 0:
        return
    rng = np.random.default_rng(seed)

    def group(scale):
        return [(rng.standard_normal(n) * scale).astype(np.float32) for n in numels]

    comm = tc.Comm.single(0) if p == 1 else tc.Comm.emulated(p, 0)
    a, oneshot, ll = ALGOS[algo]
    if p > 1:
        comm.set_algorithm(a)
        comm.set_tuning(0, 0, oneshot)
        comm.set_ll_max(ll)
    pick = (lambda v: v) if p > 1 else (lambda v: v[0])
    hp = dict(lr=0.1, momentum=0.9, wd=1e-4, rescale=1.0 / 64)
    if op == "allreduce":
        xs = [group(1e-2) for _ in range(p)]
        dev = [to_dev(x, offset=offset) for x in xs]
        g = tc.Group(comm, pick(dev))
        tc.allreduce(g, 0.5)
        want = O.allreduce(xs, 0.5)
        for r in range(p):
            assert_bitwise(to_host(dev[r]), want, f"rank {r}")
        groups = [g]
    elif op == "sgd":
        gs = [group(1e-2) for _ in range(p)]
        w, dw = group(5e-2), group(1e-3)
        dg = [to_dev(x, offset=offset) for x in gs]
        dwt = [to_dev(w) for _ in range(p)]
        ddw = [to_dev(dw, offset=offset) for _ in range(p)]
        groups = [tc.Group(comm, pick(v)) for v in (dg, dwt, ddw)]
        tc.sgd_step(groups[1], groups[0], groups[2], **hp)
        G, Ws, Ds = O.sgd_step([w] * p, gs, [dw] * p, **hp)
        for r in range(p):
            assert_bitwise(to_host(dg[r]), G, f"g rank {r}")
            assert_bitwise(to_host(dwt[r]), Ws[r], f"w rank {r}")
            assert_bitwise(to_host(ddw[r]), Ds[r], f"dw rank {r}")
    elif op == "easgd":
        center = group(5e-2)
        xs = [[c + (rng.standard_normal(c.size) * 1e-2).astype(np.float32) for c in center]
              for _ in range(p)]
        dx = [to_dev(x, offset=offset) for x in xs]
        dc = [to_dev(center, offset=offset) for _ in range(p)]
        groups = [tc.Group(comm, pick(v)) for v in (dx, dc)]
        tc.easgd_update(groups[0], groups[1], 0.1)
        wx, wc = O.easgd_update(xs, center, 0.1)
        for r in range(p):
            assert_bitwise(to_host(dx[r]), wx[r], f"x rank {r}")
            assert_bitwise(to_host(dc[r]), wc, f"center rank {r}")
    else:
        center = group(5e-2)
        xs = [[c + (rng.standard_normal(c.size) * 1e-2).astype(np.float32) for c in center]
              for _ in range(p)]
        gs, dws = [group(1e-2) for _ in range(p)], [group(1e-3) for _ in range(p)]
        dx = [to_dev(x, offset=offset) for x in xs]
        dc = [to_dev(center, offset=offset) for _ in range(p)]
        dg = [to_dev(x, offset=offset) for x in gs]
        dd = [to_dev(x, offset=offset) for x in dws]
        groups = [tc.Group(comm, pick(v)) for v in (dx, dc, dg, dd)]
        tc.esgd_step(*groups, 0.1, **hp)
        wx, wc, wd = O.esgd_step(xs, center, gs, dws, 0.1, **hp)
        for r in range(p):
            assert_bitwise(to_host(dx[r]), wx[r], f"x rank {r}")
            assert_bitwise(to_host(dc[r]), wc, f"center rank {r}")
            assert_bitwise(to_host(dd[r]), wd[r], f"dw rank {r}")
    assert comm.async_error() == 0
    for grp in groups:
        grp.destroy()
    comm.destroy()
