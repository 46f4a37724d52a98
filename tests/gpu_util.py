"""Helpers shared by the GPU parity tests: upload seeded host groups, download results."""
import numpy as np
import torch


def to_dev(group, device="cuda", offset=0):
    """Upload a list of fp32 numpy arrays as separate CUDA tensors.  offset > 0 makes every
    tensor a view starting `offset` elements into its own allocation (4-B but not 16-B aligned
    when offset % 4 != 0), exercising the scalar path."""
    out = []
    for a in group:
        if offset:
            base = torch.empty(a.size + offset, dtype=torch.float32, device=device)
            t = base[offset:]
            t.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        else:
            t = torch.from_numpy(np.ascontiguousarray(a)).to(device)
        out.append(t)
    return out


def to_host(tensors):
    torch.cuda.synchronize()
    return [t.detach().cpu().numpy() for t in tensors]


def assert_bitwise(got, want, what=""):
    assert len(got) == len(want)
    for t, (a, b) in enumerate(zip(got, want)):
        a = np.asarray(a, np.float32)
        b = np.asarray(b, np.float32)
        assert a.shape == b.shape, (what, t, a.shape, b.shape)
        bad = np.flatnonzero(a.view(np.uint32) != b.view(np.uint32))
        assert bad.size == 0, f"{what}: tensor {t}: {bad.size} mismatches, first at {bad[0]}: " \
                              f"got {a[bad[0]]!r} want {b[bad[0]]!r}"
