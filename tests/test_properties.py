"""Property-based checks (hypothesis) of the oracle (CPU) against what mathematics fixes, on
random ragged groups: integer-valued sums are exact, allgather(reduce_scatter) = allreduce
(S:237), and the result does not depend on how the flat vector is split into tensors (the
paper's "group of vectors as a single object")."""
import numpy as np
from hypothesis import given, settings, strategies as st

from oracle import tc_oracle as O

groups = st.lists(st.integers(min_value=0, max_value=40), min_size=1, max_size=12)


def _int_group(numels, seed, k):
    rng = np.random.default_rng([seed, k])
    return [rng.integers(-1000, 1001, size=n).astype(np.float32) for n in numels]


@settings(max_examples=60, deadline=None)
@given(numels=groups, p=st.integers(1, 8), seed=st.integers(0, 2 ** 31 - 1))
def test_integer_sums_exact(numels, p, seed):
    xs = [_int_group(numels, seed, k) for k in range(p)]
    out = O.allreduce(xs)
    for t, n in enumerate(numels):
        want = [sum(int(xs[k][t][j]) for k in range(p)) for j in range(n)]
        assert [int(v) for v in out[t]] == want


@settings(max_examples=60, deadline=None)
@given(numels=groups, p=st.integers(1, 8), seed=st.integers(0, 2 ** 31 - 1))
def test_allgather_of_reduce_scatter_is_allreduce(numels, p, seed):
    if sum(numels) == 0:
        return
    rng = np.random.default_rng(seed)
    xs = [[(rng.standard_normal(n) * 1e-2).astype(np.float32) for n in numels] for _ in range(p)]
    pieces = [O.reduce_scatter(xs, r) for r in range(p)]
    got = O.allgather(pieces, numels)
    want = O.allreduce(xs)
    for a, b in zip(got, want):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@settings(max_examples=60, deadline=None)
@given(numels=groups, cut=st.lists(st.integers(0, 200), min_size=1, max_size=6),
       p=st.integers(1, 6), seed=st.integers(0, 2 ** 31 - 1))
def test_split_invariance(numels, cut, p, seed):
    N = sum(numels)
    rng = np.random.default_rng(seed)
    flats = [(rng.standard_normal(N) * 1e-2).astype(np.float32) for _ in range(p)]
    # a second split of the same flat vectors
    cuts = sorted({min(c, N) for c in cut})
    edges = [0] + cuts + [N]
    other = [b - a for a, b in zip(edges[:-1], edges[1:])]

    def split(f, ns):
        return list(np.split(f, np.cumsum(ns)[:-1])) if ns else []

    a = np.concatenate(O.allreduce([split(f, numels) for f in flats]) or [np.zeros(0, np.float32)])
    b = np.concatenate(O.allreduce([split(f, other) for f in flats]) or [np.zeros(0, np.float32)])
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
