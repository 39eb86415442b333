"""Row-sharded ascend (lcb_ascend_rows; north star 5, SURVEY 8e "row-sharding of A"):
ranks hold disjoint CSR row ranges and their slice of the state, exchange the new rows
every iteration and OR-reduce the early-exit bits.  Run as 1-3 loopback ranks (threads
of this process on one GPU, the same code path as NCCL ranks).  Contract: the result
equals ``ascend`` on the whole graph -- fp64 bit for bit against the oracle (itself pinned
to the reference), fp32 bit for bit against the unsharded K1 step (same CSR-order sums,
same op sequence) -- for any partition, including an empty range and a range holding
only hub rows, with and without early exit, unlifted and lifted.
"""
import threading

import numpy as np
import pytest

import oracle as O
from paper_2509_18612_b200 import LCB_FP32, LCB_FP64
from paper_2509_18612_b200 import liftcut as lc
from paper_2509_18612_b200.dist import Comm, LoopbackGroup

pytestmark = pytest.mark.gpu


def ba_like(n, m, seed):
    rng = np.random.default_rng(seed)
    us, vs, rep = [], [], list(range(m))
    for v in range(m, n):
        chosen = set()
        while len(chosen) < m:
            chosen.add(int(rep[rng.integers(0, len(rep))]))
        for u in chosen:
            us.append(u)
            vs.append(v)
        rep += list(chosen) + [v] * m
    return O.csr_from_edges(n, us, vs)


def sharded_ascend(cg, x, l, B, params, prec, cuts):
    """Run lcb_ascend_rows over len(cuts)-1 loopback ranks; rank q owns [cuts[q], cuts[q+1])."""
    nr = len(cuts) - 1
    full = x.reshape(B, l, cg.n)
    out = full.copy()
    grp = LoopbackGroup(nr) if nr > 1 else None
    comms = [Comm.loopback(grp, r, 0) for r in range(nr)] if nr > 1 else [None]
    err = []

    def work(q):
        r0, r1 = cuts[q], cuts[q + 1]
        sl = np.ascontiguousarray(full[:, :, r0:r1])
        off = cg.off[r0:r1 + 1] - cg.off[r0]
        adj = cg.adj[cg.off[r0]:cg.off[r1]]
        try:
            lc.ascend_rows(cg.n, r0, r1, off, adj, sl, l, B, params, comm=comms[q], precision=prec)
            out[:, :, r0:r1] = sl
        except Exception as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=work, args=(q,)) for q in range(nr)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in comms:
        if c is not None:
            c.close()
    if grp is not None:
        grp.close()
    if err:
        raise err[0]
    return out.reshape(-1)


@pytest.fixture(scope="module")
def graph():
    return ba_like(2600, 4, 3)  # hubs (degree > 100) in the first rows


def start(rng, n, l, B):
    return rng.choice([-1e-4, 1e-4], B * l * n) + rng.normal(0, 9e-5, B * l * n)


PARTS = [[0, 2600], [0, 1000, 2600], [0, 7, 1500, 2600], [0, 0, 1300, 2600]]


@pytest.mark.parametrize("cuts", PARTS)
@pytest.mark.parametrize("l,B,ee", [(1, 40, False), (1, 40, True), (2, 20, True)])
def test_rowshard_fp64_bitwise_vs_oracle(graph, cuts, l, B, ee):
    rng = np.random.default_rng(len(cuts) * 10 + l)
    x = start(rng, graph.n, l, B)
    for T in (1, 9, 60):
        want, _ = O.ascend(graph, x, l, B, 0.05, T, 0.9, ee)
        got = sharded_ascend(graph, x, l, B, lc.AscentParams(0.05, T, 0.9, ee), LCB_FP64, cuts)
        assert np.array_equal(got, want), (cuts, l, B, ee, T)


@pytest.mark.parametrize("cuts", PARTS[1:])
def test_rowshard_fp32_equals_unsharded_k1(graph, cuts):
    rng = np.random.default_rng(7)
    l, B, T = 1, 64, 40
    x = start(rng, graph.n, l, B)
    s = lc.DenseState(graph.n, l, B)
    s.values[:] = x
    with lc.options(resident=0, stream=0, signrec=0, chunk=0):
        lc.ascend(lc.Graph.from_csr(graph.n, graph.off, graph.adj), s, lc.AscentParams(0.05, T, 0.9, True),
                  precision=LCB_FP32)
    got = sharded_ascend(graph, x, l, B, lc.AscentParams(0.05, T, 0.9, True), LCB_FP32, cuts)
    assert np.array_equal(got, s.values)


def test_rowshard_rejects_a_bad_partition(graph):
    x = start(np.random.default_rng(1), graph.n, 1, 8)
    with pytest.raises(lc.ValidationError):
        sharded_ascend(graph, x, 1, 8, lc.AscentParams(0.05, 3, 0.9), LCB_FP64, [0, 1000, 2500])
    with pytest.raises(lc.ValidationError):  # rows 0..999 owned by no rank
        sharded_ascend(graph, x, 1, 8, lc.AscentParams(0.05, 3, 0.9), LCB_FP64, [1000, 2600, 2600])


def test_rowshard_numeric_error_names_iteration_and_member(graph):
    x = start(np.random.default_rng(2), graph.n, 1, 4)
    with pytest.raises(lc.NumericError) as e:
        sharded_ascend(graph, x, 1, 4, lc.AscentParams(1e308, 5, 0.0), LCB_FP64, [0, 1300, 2600])
    assert "iteration" in str(e.value) and "member" in str(e.value)
