"""Rounding on the device (lcb_round: objectives.cpp:81-96) against the oracle, with the
ties on purpose: round_unlifted maps exact zeros (either sign) to 0 (strict), round_lifted
maps a zero row sum to 1 (inclusive), the lifted row sum runs in column order."""
import numpy as np
import pytest

import oracle as O
from paper_2509_18612_b200 import liftcut as lc

pytestmark = pytest.mark.gpu


def test_round_unlifted_strict_zero_ties():
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, 5000)
    x[::7] = 0.0
    x[3::11] = -0.0
    x[5::13] = 1e-300
    got = lc.round_unlifted(x)
    assert got.dtype == np.uint8 and np.array_equal(got, O.round_unlifted(x))
    assert got[0] == 0 and got[3] == 0


@pytest.mark.parametrize("l", [2, 3, 5])
def test_round_lifted_inclusive_and_column_order(l):
    rng = np.random.default_rng(l)
    n, B = 3000, 4
    s = lc.DenseState(n, l, B)
    s.values[:] = rng.choice([-1.0, -0.5, 0.0, 0.5, 1.0], n * l * B)
    # rows whose sum is zero only in a particular order: 1e16 + 1 - 1e16
    if l == 3:
        m = s.member(2).reshape(l, n)
        m[0, :10], m[1, :10], m[2, :10] = 1e16, 1.0, -1e16
    for j in range(B):
        want = O.round_lifted(s.member(j), n, l)
        assert np.array_equal(lc.round_lifted(s, j), want), j


@pytest.mark.parametrize("p", [0.02, 0.5])
def test_cut_counts_dense_warp_rows_vs_oracle(p):
    """Cut counting on a dense graph (average degree > 64: one row per warp, lanes striding
    over the neighbours) and a sparse one (one row per thread): every count equals the
    oracle's, through lcb_cut_values and through the fused epilogue (round_cut_batch)."""
    cg = O.generate_er(700, p, 3)
    g = lc.Graph.from_csr(cg.n, cg.off, cg.adj)
    rng = np.random.default_rng(int(p * 100))
    Z = rng.integers(0, 2, (70, cg.n), dtype=np.uint8)
    got = lc.cut_values(g, Z)
    want = [O.cut_value(cg, z) for z in Z]
    assert got.tolist() == want
    B = 70
    s = lc.DenseState(cg.n, 1, B)
    s.values[:] = rng.normal(0, 1, B * cg.n)
    cuts, _, _, _ = lc.round_cut_batch(g, s, lifted=False)
    zz = (s.values.reshape(B, cg.n) > 0).astype(np.uint8)
    assert cuts.tolist() == [O.cut_value(cg, row) for row in zz]
