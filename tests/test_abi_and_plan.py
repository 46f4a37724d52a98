"""T1 (CPU): the C-ABI library loads, exports every symbol include/tc.h declares, and its host-only
descriptor (A1, tc_plan_*) matches the plain definition of the partition.  No CUDA calls."""
import os
import re

import numpy as np
import pytest

import paper_1801_03855_b200 as tc
from paper_1801_03855_b200.tc import LIB, TcError
from oracle import tc_oracle as O
import tc_workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tc.h")).read()
    return sorted(set(re.findall(r"^TC_API [^(]*?\b(tc_\w+)\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for need in ("tc_group_create", "tc_allreduce", "tc_sgd_step", "tc_easgd_update",
                 "tc_comm_create", "tc_comm_destroy", "tc_group_destroy", "tc_plan_create"):
        assert need in names


def test_library_exports_every_declared_symbol():
    import ctypes
    lib = ctypes.CDLL(tc.LIB_PATH)
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


def test_status_strings():
    for code, name in tc.STATUS.items():
        assert LIB.tc_status_string(code).decode() == name
    assert LIB.tc_version() >= 100


@pytest.mark.parametrize("p", [1, 2, 3, 4, 7, 8])
@pytest.mark.parametrize("group", ["tiny", "resnet50", "alexnet", "vgg16", "ragged"])
def test_plan_matches_definition(p, group):
    numels = W.random_numels(np.random.default_rng(3), 200, 50) + [0, 1, 2, 3, 5] \
        if group == "ragged" else W.GROUPS[group]
    plan = tc.Plan(numels, nranks=p)
    prefix, owners = O.slot_partition(numels, p)
    assert plan.num_elements == sum(numels)
    assert plan.num_slots == prefix[-1]
    for t in range(len(numels)):
        assert plan.tensor_slots(t) == (prefix[t], prefix[t + 1] - prefix[t])
    for r in range(p):
        assert plan.owner_range(r) == owners[r]
    segs = plan.segments()
    # segments tile the slot space in order, never cross a tensor or an owner boundary
    pos = 0
    for t, owner, lo, hi in segs:
        assert lo == pos and hi > lo
        assert prefix[t] <= lo and hi <= prefix[t + 1]
        assert owners[owner][0] <= lo and hi <= owners[owner][1]
        pos = hi
    assert pos == prefix[-1]
    assert len(segs) <= sum(1 for n in numels if n) + p - 1


def test_plan_hash_is_congruence():
    a = tc.Plan([7, 13, 1000])
    assert a.hash == tc.Plan([7, 13, 1000], nranks=4).hash
    assert a.hash != tc.Plan([7, 1000, 13]).hash
    assert a.hash != tc.Plan([7, 13]).hash


def test_plan_errors():
    with pytest.raises(TcError) as e:
        tc.Plan([5, -1])
    assert e.value.status == tc.tc.TC_ERR_INVALID_ARG
    with pytest.raises(TcError) as e:
        tc.Plan([5], nranks=9)
    assert e.value.status == tc.tc.TC_ERR_UNSUPPORTED
    with pytest.raises(TcError) as e:
        tc.Plan([], nranks=1)
    assert e.value.status == tc.tc.TC_ERR_INVALID_ARG
    with pytest.raises(TcError) as e:
        tc.Plan([1 << 33])  # 2^31 slots: beyond the int32 slot index
    assert e.value.status == tc.tc.TC_ERR_INVALID_ARG


def test_hot_path_rejects_null_handles_without_a_gpu():
    assert LIB.tc_allreduce(None, 1.0, None) == tc.tc.TC_ERR_INVALID_ARG
    assert LIB.tc_sgd_step(None, None, None, 0.1, 0.9, 0.0, 1.0, None) == tc.tc.TC_ERR_INVALID_ARG
    assert LIB.tc_easgd_update(None, None, 0.1, None) == tc.tc.TC_ERR_INVALID_ARG
    assert LIB.tc_comm_async_error(None) == tc.tc.TC_ERR_INVALID_ARG


@pytest.mark.parametrize("cap", [1 << 10, 1 << 20, 25 << 20, 1 << 40])
def test_buckets_backward_order(cap):
    """NEXT row f1: buckets are runs of consecutive tensors in backward order, within the byte cap
    unless a single tensor exceeds it, covering every tensor once."""
    numels = W.RESNET50
    b, n = tc.Plan(numels).buckets(cap)
    assert n >= 1 and sorted(set(b)) == list(range(n))
    assert b[-1] == 0 and b == sorted(b, reverse=True)      # backward order, bucket 0 first
    for k in range(n):
        members = [t for t in range(len(numels)) if b[t] == k]
        assert members == list(range(members[0], members[-1] + 1))
        size = 4 * sum(numels[t] for t in members)
        assert size <= cap or len(members) == 1
        if k + 1 < n:  # greedy: the next tensor would not have fitted
            nxt = members[0] - 1
            assert size + 4 * numels[nxt] > cap
