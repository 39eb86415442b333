"""The product's multi-rank solve (member sharding + per-batch exchange) executed on one GPU.

Two ranks run as threads of this process over a loopback communicator
(lcb_comm_create_loopback): the same Solver code path as NCCL ranks (member_base =
rank * B, allreduce(max) of the packed key, of the winner bits and allreduce(min) of
the error slots), with the collectives through device staging buffers and a host
barrier.  Contract (parallel.hpp:22-50, test_solver.cpp:272-308): results do not depend
on the partition — a 2-rank solve with batch_size B equals the 1-rank solve with 2B
(fp64 bit for bit: cut, assignment, batch / phase / search traces).
"""
import threading

import numpy as np
import pytest

import oracle as O
from paper_2509_18612_b200 import LCB_FP64
from paper_2509_18612_b200 import liftcut as lc
from paper_2509_18612_b200.dist import Comm, LoopbackGroup

pytestmark = pytest.mark.gpu


def pg(c):
    return lc.Graph.from_csr(c.n, c.off, c.adj)


def sharded(fn, nranks, *args, **kw):
    """Run fn(rank, comm) on `nranks` threads sharing one loopback group."""
    grp = LoopbackGroup(nranks)
    comms = [Comm.loopback(grp, r, 0) for r in range(nranks)]
    out, err = [None] * nranks, []

    def work(r):
        try:
            out[r] = fn(r, comms[r])
        except Exception as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in comms:
        c.close()
    grp.close()
    assert not err, err
    return out


def same(a, b):
    assert a.best.cut_value == b.best.cut_value
    assert np.array_equal(a.best.assignment, b.best.assignment)
    assert a.best.member_index == b.best.member_index and a.best.batch_index == b.best.batch_index
    assert a.batch_trace == b.batch_trace and a.phase_trace == b.phase_trace
    assert a.search_trace == b.search_trace


@pytest.mark.parametrize("algo", [lc.Algorithm.pQUCO, lc.Algorithm.pDECO])
def test_two_ranks_equal_one_rank_with_double_batch(algo):
    cg = O.generate_er(400, 0.03, 5)
    g = pg(cg)
    B = 24
    cfg = lc.SolverConfig(algorithm=algo, batch_size=2 * B, lift_dim=2, num_batches=3,
                          ascent=lc.AscentParams(0.05, 120, 0.9, True), deco_alternations=2)
    fn = {lc.Algorithm.pQUCO: lc.pquco, lc.Algorithm.pDECO: lc.pdeco}[algo]
    one = fn(g, cfg, 7, opts=lc.RunOptions(precision=LCB_FP64))
    half = lc.SolverConfig(**{**cfg.__dict__, "batch_size": B})
    two = sharded(lambda r, c: fn(g, half, 7, opts=lc.RunOptions(precision=LCB_FP64, comm=c)), 2)
    for t in two:
        same(t, one)
    # and the reference solve with the full batch
    ref = O.solve(cg, O.default_config(algorithm=int(algo), batch_size=2 * B, num_batches=3, iterations=120,
                                       l_iterations=120), 7)
    assert one.best.cut_value == ref.cut_value and one.best.assignment.tolist() == ref.assignment.tolist()


def test_two_ranks_with_search_and_lifted():
    cg = O.generate_er(250, 0.05, 9)
    g = pg(cg)
    cfg = lc.SolverConfig(algorithm=lc.Algorithm.pLUCO, batch_size=32, lift_dim=2, num_batches=2,
                          ascent=lc.AscentParams(0.05, 60, 0.9, True),
                          search=lc.SearchConfig(20, 70, -3.0, -1.0, 4, 2))
    one = lc.pluco(g, cfg, 3, opts=lc.RunOptions(precision=LCB_FP64))
    half = lc.SolverConfig(**{**cfg.__dict__, "batch_size": 16})
    two = sharded(lambda r, c: lc.pluco(g, half, 3, opts=lc.RunOptions(precision=LCB_FP64, comm=c)), 2)
    for t in two:
        same(t, one)


def test_two_ranks_per_component_shards_members_within_each_component():
    # three components plus isolated nodes (solve_per_component, solver.cpp:314-364)
    a = O.generate_er(120, 0.08, 1)
    b = O.generate_er(90, 0.1, 2)
    eu, ev = [], []
    for off, cg in ((0, a), (120, b)):
        u, v = cg.edges()
        eu += list(u + off)
        ev += list(v + off)
    eu += [215, 216, 217]
    ev += [216, 217, 218]
    cg = O.csr_from_edges(230, eu, ev)
    g = pg(cg)
    cfg = lc.SolverConfig(batch_size=20, num_batches=2, ascent=lc.AscentParams(0.05, 80, 0.9, True))
    one = lc.solve_per_component(g, cfg, 5, opts=lc.RunOptions(precision=LCB_FP64))
    half = lc.SolverConfig(**{**cfg.__dict__, "batch_size": 10})
    two = sharded(lambda r, c: lc.solve_per_component(g, half, 5, opts=lc.RunOptions(precision=LCB_FP64, comm=c)), 2)
    for t in two:
        assert t.best.cut_value == one.best.cut_value
        assert np.array_equal(t.best.assignment, one.best.assignment)
        assert t.batch_trace == one.batch_trace
    ref = O.solve(cg, O.default_config(batch_size=20, num_batches=2, iterations=80), 5, per_component=True)
    assert one.best.cut_value == ref.cut_value


@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_solve_runs_sharded_over_ranks(nranks):
    cg = O.generate_er(300, 0.04, 4)
    g = pg(cg)
    cfg = lc.SolverConfig(batch_size=16, num_batches=2, ascent=lc.AscentParams(0.05, 60, 0.9, True))
    seeds = [11, 12, 13, 14, 15]
    singles = [lc.solve_per_component(g, cfg, s, opts=lc.RunOptions(precision=LCB_FP64)) for s in seeds]
    want = [s.best.cut_value for s in singles]
    res = sharded(lambda r, c: lc.solve_runs(g, cfg, seeds, opts=lc.RunOptions(precision=LCB_FP64, comm=c)),
                  nranks)
    best = int(np.argmax(want))
    for r in res:
        assert r.run_cuts.tolist() == want
        assert r.best_run == best and r.best.cut_value == want[best]
        assert np.array_equal(r.best.assignment, singles[best].best.assignment)
        assert lc.cut_value(g, r.best.assignment) == want[best]
