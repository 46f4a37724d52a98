"""Plain, slow, obviously-correct CPU oracle of the MXNET-MPI data-parallel hot path.

TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It shares no code with the CUDA library
(paper_1801_03855_b200/csrc) and never imports it.

Citations: ``P:n`` = /root/reference/PAPER.md line n (arXiv 1801.03855), ``S:n`` = SPEC.md line n.
Readings of silent/garbled passages are numbered R1.. and listed in DESIGN.md §3.

Data model: a *tensor group* is a Python list of T one-dimensional numpy fp32 arrays (the
"group of vectors ... as a single object").  A multi-rank input is a list over
ranks k = 0..p-1 of tensor groups.

Notation: F(v) = float64(v), R(v) = round-to-nearest-even to float32.

Pins (tests/test_oracle_pins.py, -m "not gpu"):
  allreduce        -- pinned: brute-force integer sums, SPEC worked examples, exact (fsum)
                      rounding, ring-algorithm simulation, split invariance, rank identity.
  sgd_step         -- pinned: Eq. 1 at mu=0, wd=0; SPEC example S:364; exact rational
                      arithmetic on dyadic inputs; closed-form geometric series for momentum.
                      The momentum *form* itself is reading R12 (the paper only names
                      "momentum SGD") -- pinned to its own closed form, not to the paper.
  easgd_update     -- pinned: Eqs. elastic1/elastic2 at c=1; SPEC S:373/S:382;
                      alpha=0 identity; conservation; contraction; exact rational arithmetic.
  slot_partition   -- pinned: exact integer invariants (cover, disjoint, balance).
  esgd_sequence    -- composed of the three pinned parts (no closed form).
  broadcast        -- the plain definition (copies of the root's group); pinned by rank
                      identity and the root's group unchanged, bit for bit.
  esgd_step        -- NEXT row f2 (elastic then SGD with each client's own gradient): pinned by
                      exact rational evaluation on dyadic data and its special cases (alpha = 0
                      -> local sgd_step; lr = momentum = 0 -> easgd_update).
  easgd_async      -- NEXT row f2 (the server applies Elastic1 per client, in arrival order):
                      pinned at c = 1 to Eqs. elastic1/elastic2 in exact rationals, by the
                      alpha = 1/2 closed form (each arriving client meets the center at their
                      midpoint), exact conservation of sum_i x_i + xc on integer data with
                      dyadic alpha, the alpha = 0 identity, and relabelling invariance.
  The momentum term (mu != 0) follows reading R12; the paper fixes no formula for it (P:158 names
  "momentum SGD" only), so it is pinned to its own closed form and to an independent library
  routine for the standard heavy-ball form (torch.optim.SGD, float64, several steps:
  tests/test_oracle_pins.py::test_sgd_momentum_matches_library_optimizer).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "allreduce", "allreduce_f64", "reduce_scatter", "allgather",
    "sgd_step", "sgd_step_f64", "easgd_update", "easgd_update_f64", "esgd_sequence", "esgd_step",
    "easgd_async",
    "broadcast",
    "slot_partition", "bus_bytes_per_rank", "predict_cost", "ring_allreduce_sim",
    "F", "R",
]


def F(v):
    return np.asarray(v, dtype=np.float64)


def R(v):
    return np.asarray(v, dtype=np.float64).astype(np.float32)


def _f32(x) -> np.float32:
    """A hyper-parameter as it crosses the C ABI (a C ``float``)."""
    return np.float32(x)


# ----------------------------------------------------------------------------------------
# A3+A4: tensor allreduce = reduce-scatter followed by allgather, whose result is the
# plain definition: every rank ends with the elementwise sum over ranks.
# ----------------------------------------------------------------------------------------
def allreduce(xs, scale: float = 1.0):
    """out[t][j] = R( (sum_{k=0..p-1} F(xs[k][t][j])) * F(float32(scale)) ).

    The sum is an explicit sequential loop in canonical rank order k = 0..p-1 in float64
    (reading R3/R4: the paper fixes neither order nor accumulator precision),
    rounded once.  The same array is the result on every rank.
    """
    p = len(xs)
    T = len(xs[0])
    s = F(_f32(scale))
    out = []
    for t in range(T):
        acc = F(xs[0][t])
        for k in range(1, p):
            acc = acc + F(xs[k][t])
        out.append(R(acc * s))
    return out


def allreduce_f64(xs, scale: float = 1.0):
    """Tolerance reference: same sum, kept in float64 (not rounded)."""
    p = len(xs)
    s = F(_f32(scale))
    out = []
    for t in range(len(xs[0])):
        acc = F(xs[0][t])
        for k in range(1, p):
            acc = acc + F(xs[k][t])
        out.append(acc * s)
    return out


# ----------------------------------------------------------------------------------------
# A1: the flat index space and owner partition ("the buffer from each process is
# partitioned into nearly equal parts"; reading R2: 16-byte slots of 4 fp32 elements).
# ----------------------------------------------------------------------------------------
def slot_partition(numels, p: int):
    """Returns (slot_prefix, owner_ranges).

    Tensor t has ceil(n_t/4) slots; slot_prefix[t] = sum_{u<t} slots_u, M = slot_prefix[T].
    Rank r owns slots [floor(M*r/p), floor(M*(r+1)/p)).
    """
    slots = [(int(n) + 3) // 4 for n in numels]
    prefix = [0]
    for s in slots:
        prefix.append(prefix[-1] + s)
    M = prefix[-1]
    owners = [(M * r // p, M * (r + 1) // p) for r in range(p)]
    return prefix, owners


def _flat_to_group(flat, numels):
    out, o = [], 0
    for n in numels:
        out.append(flat[o:o + n])
        o += n
    return out


def reduce_scatter(xs, r: int, scale: float = 1.0):
    """Rank r's piece of the reduced sum: the elements of the slots it owns, as a list
    of (tensor index, element lo, element hi, values)."""
    numels = [len(a) for a in xs[0]]
    prefix, owners = slot_partition(numels, len(xs))
    lo, hi = owners[r]
    full = allreduce(xs, scale)
    pieces = []
    for t, n in enumerate(numels):
        a, b = max(lo, prefix[t]), min(hi, prefix[t + 1])
        if a < b:
            e0, e1 = (a - prefix[t]) * 4, min(n, (b - prefix[t]) * 4)
            pieces.append((t, e0, e1, full[t][e0:e1].copy()))
    return pieces


def allgather(pieces_per_rank, numels):
    """Concatenate every rank's owned pieces into the full group."""
    out = [np.zeros(n, np.float32) for n in numels]
    for pieces in pieces_per_rank:
        for t, e0, e1, v in pieces:
            out[t][e0:e1] = v
    return out


# ----------------------------------------------------------------------------------------
# A6: SGD step fused with the gradient allreduce (Eq. 1; rescale).
# ----------------------------------------------------------------------------------------
def sgd_step(ws, gs, dws, lr, momentum, wd, rescale):
    """fp32 mirror.  Per rank k, per element (reading R12 for the momentum form, R13 rescale):

        G   = allreduce(g, 1)                       (written back to g on every rank, R15)
        t   = R( R(rescale*G) + R(wd*w) )
        dw' = R( R(momentum*dw) - R(lr*t) )
        w'  = R( w + dw' )                          (Eq. 1: w_{t+1} = w_t + dw)

    Hyper-parameters are fp32 (C ``float`` at the ABI).  Returns (G, [w'_k], [dw'_k]).
    """
    lr, mu, wd, rs = _f32(lr), _f32(momentum), _f32(wd), _f32(rescale)
    G = allreduce(gs, 1.0)
    w_out, dw_out = [], []
    for w, dw in zip(ws, dws):
        wk, dwk = [], []
        for t in range(len(G)):
            tt = (rs * G[t]).astype(np.float32) + (wd * w[t]).astype(np.float32)
            tt = tt.astype(np.float32)
            d = (mu * dw[t]).astype(np.float32) - (lr * tt).astype(np.float32)
            d = d.astype(np.float32)
            wk.append((w[t] + d).astype(np.float32))
            dwk.append(d)
        w_out.append(wk)
        dw_out.append(dwk)
    return G, w_out, dw_out


def sgd_step_f64(ws, gs, dws, lr, momentum, wd, rescale):
    """Tolerance reference: the same formulas in float64 from the stored fp32 inputs."""
    lr, mu, wd, rs = (F(_f32(v)) for v in (lr, momentum, wd, rescale))
    G = allreduce_f64(gs, 1.0)
    w_out, dw_out = [], []
    for w, dw in zip(ws, dws):
        wk, dwk = [], []
        for t in range(len(G)):
            tt = rs * G[t] + wd * F(w[t])
            d = mu * F(dw[t]) - lr * tt
            wk.append(F(w[t]) + d)
            dwk.append(d)
        w_out.append(wk)
        dw_out.append(dwk)
    return G, w_out, dw_out


# ----------------------------------------------------------------------------------------
# A7: Elastic averaging, synchronous sum form (Eqs. elastic1/elastic2; reading R10).
# ----------------------------------------------------------------------------------------
def easgd_update(xs, center, alpha):
    """fp32 mirror for c clients, per element (a = alpha as fp32):

        d_i  = R(x_i - xc)                      for every client i
        x_i' = R(x_i - R(a*d_i))                (Eq. elastic2)
        s    = d_0;  s = R(s + d_i), i = 1..c-1 (client order)
        xc'  = R(xc + R(a*s))                   (Eq. elastic1, summed over clients)

    Returns ([x_i'], xc').  At c = 1 these are exactly Eqs. elastic2 and elastic1.
    """
    a = _f32(alpha)
    c = len(xs)
    x_out = [[None] * len(center) for _ in range(c)]
    c_out = []
    for t in range(len(center)):
        xc = center[t]
        d = [(xs[i][t] - xc).astype(np.float32) for i in range(c)]
        for i in range(c):
            x_out[i][t] = (xs[i][t] - (a * d[i]).astype(np.float32)).astype(np.float32)
        s = d[0]
        for i in range(1, c):
            s = (s + d[i]).astype(np.float32)
        c_out.append((xc + (a * s).astype(np.float32)).astype(np.float32))
    return x_out, c_out


def easgd_update_f64(xs, center, alpha):
    """Tolerance reference: the same update in float64 from the stored fp32 inputs."""
    a = F(_f32(alpha))
    c = len(xs)
    x_out = [[None] * len(center) for _ in range(c)]
    c_out = []
    for t in range(len(center)):
        xc = F(center[t])
        d = [F(xs[i][t]) - xc for i in range(c)]
        for i in range(c):
            x_out[i][t] = F(xs[i][t]) - a * d[i]
        s = d[0]
        for i in range(1, c):
            s = s + d[i]
        c_out.append(xc + a * s)
    return x_out, c_out


def easgd_async(xs, center, alpha, order=None):
    """Asynchronous elastic averaging at a parameter server ("The update elastic1 is done
    on the server and elastic2 is done on the client"; Fig. code-snippet-4):
    clients arrive one at a time, in `order` (a permutation of 0..c-1, the recorded ticket
    order; default client order).  On client i's arrival, with the center as the earlier
    arrivals left it (fp32 mirror, a = alpha as fp32):

        d_i  = R(x_i - xc)
        xc   = R(xc + R(a*d_i))        (Eq. elastic1, at the server)
        x_i' = R(x_i - R(a*d_i))       (Eq. elastic2, at the client, same w~_t; reading R20)

    Returns ([x_i'], xc').  At c = 1 this is exactly easgd_update (Eqs. elastic1/elastic2).
    """
    a = _f32(alpha)
    c = len(xs)
    order = list(range(c)) if order is None else [int(i) for i in order]
    if sorted(order) != list(range(c)):
        raise ValueError("order must be a permutation of the clients")
    x_out = [[np.array(t, dtype=np.float32, copy=True) for t in x] for x in xs]
    c_out = [np.array(t, dtype=np.float32, copy=True) for t in center]
    for i in order:
        for t in range(len(center)):
            d = (x_out[i][t] - c_out[t]).astype(np.float32)
            ad = (a * d).astype(np.float32)
            c_out[t] = (c_out[t] + ad).astype(np.float32)
            x_out[i][t] = (x_out[i][t] - ad).astype(np.float32)
    return x_out, c_out


# ----------------------------------------------------------------------------------------
# Tensor broadcast (MPI_Bcast of the weights at initialisation; KVStore.pull).
# ----------------------------------------------------------------------------------------
def broadcast(xs, root: int):
    """Every rank's group becomes a copy of the root's (plain definition)."""
    return [[np.array(a, dtype=np.float32, copy=True) for a in xs[root]] for _ in xs]


# ----------------------------------------------------------------------------------------
# NEXT row f2: elastic averaging then SGD in the same iteration, one GPU per client
# (Fig. code-snippet-4: Elastic2 before SGD.Update; reading R10 for the center).
# ----------------------------------------------------------------------------------------
def esgd_step(xs, center, gs, dws, alpha, lr, momentum, wd, rescale):
    """Client i (one rank) holds params xs[i], momentum dws[i] and its own gradient gs[i]; the
    center is replicated.  easgd_update across the clients, then every client's sgd_step with
    its own (unreduced) gradient applied to its elastically moved params.  Returns
    ([x_i''], xc', [dw_i'])."""
    x_el, c_new = easgd_update(xs, center, alpha)
    x_out, dw_out = [], []
    for i in range(len(xs)):
        _, w_new, dw_new = sgd_step([x_el[i]], [gs[i]], [dws[i]], lr, momentum, wd, rescale)
        x_out.append(w_new[0])
        dw_out.append(dw_new[0])
    return x_out, c_new, dw_out


# ----------------------------------------------------------------------------------------
# Config 4: MPI Elastic SGD loop (Fig. code-snippet-4; reading R9/R10/R11).
# ----------------------------------------------------------------------------------------
def esgd_sequence(x0, center0, dw0, grads, steps, tau, alpha, lr, momentum, wd, rescale):
    """x0[i], dw0[i]: client i's params / momentum (replicated on its GPUs); center0: the
    center group; grads(step, i) -> list over client-i GPUs of gradient groups.

    For t = 0..steps-1: if t % tau == 0, easgd_update across clients (params before this
    step's SGD); then every client runs sgd_step over its own GPUs' gradients.
    Returns (x, center, dw) after the last step.
    """
    x = [list(g) for g in x0]
    dw = [list(g) for g in dw0]
    center = list(center0)
    for t in range(steps):
        if t % tau == 0:
            x, center = easgd_update(x, center, alpha)
        for i in range(len(x)):
            gs = grads(t, i)
            q = len(gs)
            _, w_new, dw_new = sgd_step([x[i]] * q, gs, [dw[i]] * q, lr, momentum, wd, rescale)
            x[i], dw[i] = w_new[0], dw_new[0]
    return x, center, dw


# ----------------------------------------------------------------------------------------
# Cost model: (p-1)alpha + 2(p-1)/p n beta + (p-1)/p n gamma
# ----------------------------------------------------------------------------------------
def bus_bytes_per_rank(p: int, S: float) -> float:
    """Bytes each rank must send (and receive) for an allreduce of S bytes."""
    return 2.0 * (p - 1) / p * S


def predict_cost(p: int, n: float, alpha: float, beta: float, gamma: float) -> float:
    """The bucket-algorithm cost of P:331, reading R6 for the garbled parentheses."""
    return (p - 1) * alpha + 2.0 * (p - 1) / p * n * beta + (p - 1) / p * n * gamma


def ring_allreduce_sim(flat_per_rank):
    """The bucket (ring) algorithm of: p-1 reduce-scatter steps then p-1 allgather
    steps around the ring 0->1->..->p-1->0 on element partitions (first n mod p parts one
    longer).  float64 accumulation.  Returns (results per rank as float64, elements
    sent per rank, communication steps).  Used only to pin the byte count and
    allgather(reduce_scatter) == allreduce."""
    p = len(flat_per_rank)
    n = len(flat_per_rank[0])
    sizes = [n // p + (1 if i < n % p else 0) for i in range(p)]
    starts = [sum(sizes[:i]) for i in range(p)]
    buf = [F(x).copy() for x in flat_per_rank]
    sent = [0] * p
    steps = 0
    if p == 1:
        return buf, sent, steps
    for s in range(p - 1):              # reduce-scatter
        msgs = []
        for r in range(p):
            c = (r - s) % p
            a, b = starts[c], starts[c] + sizes[c]
            msgs.append(((r + 1) % p, c, buf[r][a:b].copy()))
            sent[r] += b - a
        for dst, c, v in msgs:
            a = starts[c]
            buf[dst][a:a + len(v)] += v
        steps += 1
    for s in range(p - 1):              # allgather
        msgs = []
        for r in range(p):
            c = (r + 1 - s) % p
            a, b = starts[c], starts[c] + sizes[c]
            msgs.append(((r + 1) % p, c, buf[r][a:b].copy()))
            sent[r] += b - a
        for dst, c, v in msgs:
            a = starts[c]
            buf[dst][a:a + len(v)] = v
        steps += 1
    return buf, sent, steps
