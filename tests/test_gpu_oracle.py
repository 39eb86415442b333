"""Device exhaustive MaxCut (lcb_brute_force_maxcut) against the CPU oracle, which is
pinned to the compiled reference in test_oracle_golden.py.  Cases follow
test_oracle.cpp:36-120: known optima, tie counting, the smallest-encoding witness,
the n <= 26 guard.  Bit-exact: optimum, count and witness must all agree."""
import numpy as np
import pytest

import oracle as O
from paper_2509_18612_b200 import liftcut as lc

pytestmark = pytest.mark.gpu


def _pair(n, eu, ev):
    eu = np.asarray(eu, dtype=np.int64)
    ev = np.asarray(ev, dtype=np.int64)
    cg = O.csr_from_edges(n, eu, ev)
    return cg, lc.Graph.from_csr(cg.n, cg.off, cg.adj)


def _check(cg, g):
    best, w, cnt = O.brute_force_maxcut(cg)
    r = lc.brute_force_maxcut(g)
    assert (r.optimum, r.count_optimal, r.witness.tolist()) == (best, cnt, w.tolist())
    assert lc.cut_value(g, r.witness) == r.optimum


def test_known_optima():
    # complete graphs: floor(n^2 / 4)
    for n in range(2, 11):
        eu, ev = np.triu_indices(n, 1)
        cg, g = _pair(n, eu, ev)
        r = lc.brute_force_maxcut(g)
        assert r.optimum == (n * n) // 4
        _check(cg, g)
    # Petersen graph: 12
    eu = list(range(5)) + [5 + v for v in range(5)] + list(range(5))
    ev = [(v + 1) % 5 for v in range(5)] + [5 + (v + 2) % 5 for v in range(5)] + [5 + v for v in range(5)]
    cg, g = _pair(10, eu, ev)
    assert lc.brute_force_maxcut(g).optimum == 12
    _check(cg, g)
    # two disjoint triangles: 2 + 2
    cg, g = _pair(6, [0, 1, 0, 3, 4, 3], [1, 2, 2, 4, 5, 5])
    assert lc.brute_force_maxcut(g).optimum == 4
    _check(cg, g)


def test_triangle_tie_rule():  # smallest encoding among optimal (z, ~z) pairs
    cg, g = _pair(3, [0, 1, 0], [1, 2, 2])
    r = lc.brute_force_maxcut(g)
    assert (r.optimum, "".join(map(str, r.witness)), r.count_optimal) == (2, "100", 6)


def test_edgeless_and_single_node():
    cg, g = _pair(5, [0], [1])
    _check(cg, g)
    # edgeless: every assignment is optimal (cut 0), 2^n of them
    cg = O.CSR(4, np.zeros(5, dtype=np.int64), np.zeros(0, dtype=np.uint32))
    g = lc.Graph.from_csr(4, cg.off, cg.adj)
    r = lc.brute_force_maxcut(g)
    assert (r.optimum, r.count_optimal, r.witness.tolist()) == (0, 16, [0, 0, 0, 0])
    one = lc.Graph.from_csr(1, np.zeros(2, dtype=np.int64), np.zeros(0, dtype=np.uint32))
    r = lc.brute_force_maxcut(one)
    assert (r.optimum, r.count_optimal, r.witness.tolist()) == (0, 2, [0])


@pytest.mark.parametrize("n", [4, 9, 13, 17, 20, 22])
def test_random_graphs_bitwise(n):
    rng = np.random.default_rng(n)
    for p in (0.15, 0.5, 0.85):
        eu, ev = np.triu_indices(n, 1)
        keep = rng.random(len(eu)) < p
        cg, g = _pair(n, eu[keep], ev[keep])
        _check(cg, g)


def test_ragged_csr_with_repeated_entries():
    # a raw CSR may repeat a neighbour; the Gray update then counts it with multiplicity
    # (oracle.cpp:72-77), exactly as the oracle's full recount does
    off = np.array([0, 3, 5, 7, 8], dtype=np.int64)
    adj = np.array([1, 1, 2, 0, 0, 0, 3, 2], dtype=np.uint32)
    cg = O.CSR(4, off, adj)
    g = lc.Graph.from_csr(4, off, adj)
    _check(cg, g)


def test_guard_and_extended_scan():
    with pytest.raises(lc.ValidationError, match="exceeds the exhaustive-scan guard"):
        lc.brute_force_maxcut(_pair(27, [0], [1])[1])
    # lifted guard: a 32-node bipartite graph (cycle of even length) cuts every edge
    n = 32
    cg, g = _pair(n, list(range(n)), [(v + 1) % n for v in range(n)])
    r = lc.brute_force_maxcut(g, max_nodes=32)
    assert r.optimum == n and r.count_optimal == 2
    # min(z, ~z) by integer encoding: the alternating pattern with node 0 on side 1
    assert lc.cut_value(g, r.witness) == n and r.witness.tolist() == [1, 0] * (n // 2)
    # odd cycle C_31: optimum m - 1, one uncut edge anywhere (x 2 orientations)
    n = 31
    cg, g = _pair(n, list(range(n)), [(v + 1) % n for v in range(n)])
    r = lc.brute_force_maxcut(g, max_nodes=31)
    assert r.optimum == n - 1 and r.count_optimal == 2 * n
    assert lc.cut_value(g, r.witness) == n - 1
    with pytest.raises(lc.ValidationError):
        lc.brute_force_maxcut(g, max_nodes=41)
