"""Device graph ingest (lcb_graph_from_edges) against the CSR build of
the CPU oracle (orc_csr_build, pinned to graph.cpp:15-50 in test_oracle_golden.py) and the
host constructor: identical offsets and adjacency, the reference's errors."""
import numpy as np
import pytest

import oracle as O
from paper_2509_18612_b200 import liftcut as lc

pytestmark = pytest.mark.gpu


def _same(n, e):
    e = np.asarray(e, dtype=np.int64).reshape(-1, 2)
    want = O.csr_from_edges(n, e[:, 0], e[:, 1])
    g = lc.Graph.from_edges_device(n, e)
    assert np.array_equal(g.offsets, want.off) and np.array_equal(g.adjacency, want.adj)
    h = lc.Graph(n, e)
    assert np.array_equal(h.offsets, g.offsets) and np.array_equal(h.adjacency, g.adjacency)
    return g


@pytest.mark.parametrize("seed", range(3))
def test_random_multigraph_edge_lists(seed):
    rng = np.random.default_rng(seed)
    for n, m in ((1, 0), (2, 1), (7, 30), (300, 2000), (20000, 150000)):
        u = rng.integers(0, n, size=m)
        v = rng.integers(0, n, size=m)
        keep = u != v
        e = np.stack([u[keep], v[keep]], 1)
        if len(e) > 4:
            e = np.concatenate([e, e[: len(e) // 3, ::-1], e[: 5]])  # duplicates, both orientations
        _same(n, e)


def test_large_ingest_and_solve_uses_the_built_handle():
    g = lc.generate_er(3000, 0.01, 1)
    e = np.array(g.edges(), dtype=np.int64)
    d = _same(3000, e[np.random.default_rng(0).permutation(len(e))])
    cfg = lc.SolverConfig(batch_size=32, ascent=lc.AscentParams(0.05, 50), num_batches=1)
    assert lc.pquco(d, cfg, 3).best.cut_value == lc.pquco(g, cfg, 3).best.cut_value


def test_errors_match_the_reference():
    with pytest.raises(lc.ValidationError, match="at least one node"):
        lc.Graph.from_edges_device(0, [])
    with pytest.raises(lc.ValidationError, match=r"edge endpoint out of range: \(1, 5\) with n=5"):
        lc.Graph.from_edges_device(5, [[0, 1], [1, 5], [2, 2]])
    # the first offending edge decides: a self-loop before an out-of-range edge
    with pytest.raises(lc.ValidationError, match="self-loop at node 2"):
        lc.Graph.from_edges_device(5, [[0, 1], [2, 2], [1, 9]])
    with pytest.raises(lc.ValidationError, match="self-loop at node 2"):
        lc.Graph(5, [[0, 1], [2, 2], [1, 9]])
