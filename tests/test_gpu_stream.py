"""K1s (lcb_stream.cu, the warp-specialised streaming step) against the oracle.

K1s runs every HBM-streaming iteration (configs 4 and 5, and any batch K2 does not
take).  Forced here with the library knobs resident=0 (no K2) and stream=1.
* fp64: bit-exact states vs the oracle (CSR-order sums, FMA-free epilogue), through the
  saturation codes once the iterate reaches the box corners, with and without early
  exit, lifted, ragged last slab, isolated rows, hubs beyond the staged column buffer.
* fp32: ||dx||_inf / ||x||_inf <= 1e-5 per member before saturation (T <= 6 on these BA
  graphs), >= 99 % identical cuts at full T.
* the batched-search path (per-member alpha / T, shrinking live width) bit-exact.
* one iterate larger than L2 (126 MB) in fp64, bit-exact.
* x-code mode (row slabs on the box corners stored as sign codes only, X completed after
  the last iteration) on and off: fp64 bit-exact with the oracle either way, fp32 on ==
  off bit for bit.
"""
import numpy as np
import pytest

import oracle as O
from paper_2509_18612_b200 import LCB_FP32, LCB_FP64
from paper_2509_18612_b200 import liftcut as lc

pytestmark = pytest.mark.gpu

FP32_NORM_TOL = 1e-5


def pg(c):
    return lc.Graph.from_csr(c.n, c.off, c.adj)


def run(g, x, n, l, B, alpha, T, mu, ee, prec, slab_outer=-1, xcode=1):
    s = lc.DenseState(n, l, B)
    s.values[:] = x
    with lc.options(resident=0, stream=1, chunk=0, slab_outer=slab_outer, xcode=xcode):
        lc.ascend(g, s, lc.AscentParams(alpha, T, mu, ee), precision=prec)
    return s.values


def ba_like(n, m, seed):
    rng = np.random.default_rng(seed)
    us, vs = [], []
    rep = list(range(m))
    for v in range(m, n):
        chosen = set()
        while len(chosen) < m:
            chosen.add(int(rep[rng.integers(0, len(rep))]))
        for u in chosen:
            us.append(u)
            vs.append(v)
        rep += list(chosen) + [v] * m
    return O.csr_from_edges(n, us, vs)


def start(rng, n, l, B):
    return rng.choice([-1e-4, 1e-4], B * l * n) + rng.normal(0, 9e-5, B * l * n)


@pytest.mark.parametrize("xcode", [1, 0])
@pytest.mark.parametrize("slab_outer", [0, 1])
@pytest.mark.parametrize("l,B,ee", [(1, 100, False), (1, 100, True), (2, 70, False), (2, 70, True),
                                    (3, 45, False), (3, 45, True), (1, 300, False), (1, 256, True)])
def test_stream_fp64_bitwise_through_saturation(l, B, ee, slab_outer, xcode):
    cg = ba_like(2600, 4, 3)          # hubs (degree > 100), BA skew
    rng = np.random.default_rng(l * 100 + B)
    x = start(rng, cg.n, l, B)
    for T in (1, 7, 60):              # 60: well past saturation -> code path
        want, _ = O.ascend(cg, x, l, B, 0.05, T, 0.9, ee)
        got = run(pg(cg), x, cg.n, l, B, 0.05, T, 0.9, ee, LCB_FP64, slab_outer, xcode)
        assert np.array_equal(got, want), (l, B, ee, T)


@pytest.mark.parametrize("slab_outer", [0, 1])
def test_stream_xcode_fp32_on_equals_off(slab_outer):
    """fp32, full slabs (no padding columns): most row slabs reach the corners and are
    stored as codes only; the final X (after the fill) equals the fully stored run bit for
    bit at every T, odd and even."""
    rng = np.random.default_rng(21)
    n = 30_000
    u, v = rng.integers(0, n, 150_000), rng.integers(0, n, 150_000)
    keep = u != v
    cg = O.csr_from_edges(n, u[keep], v[keep])
    g = pg(cg)
    B = 512
    x = start(rng, n, 1, B)
    for T in (1, 2, 41, 120):
        on = run(g, x, n, 1, B, 0.05, T, 0.9, False, LCB_FP32, slab_outer, 1)
        off = run(g, x, n, 1, B, 0.05, T, 0.9, False, LCB_FP32, slab_outer, 0)
        assert np.array_equal(on, off), T
    assert np.mean(np.abs(on) == 1.0) > 0.9  # the code-only path was exercised


def test_stream_fp64_low_skew_natural_order_and_isolated_rows():
    rng = np.random.default_rng(9)
    n = 5000
    u = rng.integers(0, 4200, 16000)
    v = rng.integers(0, 4200, 16000)
    keep = u != v
    cg = O.csr_from_edges(n, u[keep], v[keep])   # rows 4200.. isolated
    B = 129                                      # two fp64 slabs + one ragged column
    x = start(rng, n, 1, B)
    for ee in (False, True):
        want, _ = O.ascend(cg, x, 1, B, 0.05, 50, 0.9, ee)
        assert np.array_equal(run(pg(cg), x, n, 1, B, 0.05, 50, 0.9, ee, LCB_FP64), want), ee


@pytest.mark.parametrize("prec", [LCB_FP64, LCB_FP32])
@pytest.mark.parametrize("l,B,ee", [(2, 32, False), (2, 32, True), (1, 70, False)])
def test_stream_small_graph_single_partial_slab(prec, l, B, ee):
    """n = 250 (code buffers whose size is not a multiple of 16 bytes), one partial slab."""
    cg = O.generate_er(250, 0.05, 9)
    rng = np.random.default_rng(l + B)
    x = rng.normal(0, 1e-4, B * l * cg.n)
    want, _ = O.ascend(cg, x, l, B, 0.05, 60, 0.9, ee)
    got = run(pg(cg), x, cg.n, l, B, 0.05, 60, 0.9, ee, prec)
    if prec == LCB_FP64:
        assert np.array_equal(got, want)
    else:  # the same CSR-order sums and epilogue as K1: bit for bit
        s = lc.DenseState(cg.n, l, B)
        s.values[:] = x
        with lc.options(resident=0, stream=0, chunk=0):
            lc.ascend(pg(cg), s, lc.AscentParams(0.05, 60, 0.9, ee), precision=prec)
        assert np.array_equal(got, s.values)


def test_stream_fp64_hub_beyond_staged_columns():
    # one row with 3000 neighbours: its column list does not fit the stage buffer and is
    # read from global memory; a second hub row in the same tile
    n = 3200
    u = [0] * 3000 + [1] * 700 + list(range(2, 3199))
    v = list(range(1, 3001)) + list(range(2400, 3100)) + list(range(3, 3200))
    cg = O.csr_from_edges(n, u, v)
    rng = np.random.default_rng(4)
    x = start(rng, n, 1, 33)
    want, _ = O.ascend(cg, x, 1, 33, 0.02, 40, 0.9, False)
    assert np.array_equal(run(pg(cg), x, n, 1, 33, 0.02, 40, 0.9, False, LCB_FP64), want)


@pytest.mark.parametrize("l,B", [(1, 256), (2, 128)])
def test_stream_fp32_tolerance_and_cuts(l, B):
    cg = ba_like(4000, 4, 8)
    g = pg(cg)
    rng = np.random.default_rng(l)
    x = start(rng, cg.n, l, B)
    for T in (3, 6):  # pre-saturation on this BA graph (41 % of entries are on the box at T=10)
        want, _ = O.ascend(cg, x, l, B, 0.05, T, 0.9, False)
        got = run(g, x, cg.n, l, B, 0.05, T, 0.9, False, LCB_FP32)
        for j in range(B):
            a, b = got[j * l * cg.n:(j + 1) * l * cg.n], want[j * l * cg.n:(j + 1) * l * cg.n]
            assert np.max(np.abs(a - b)) / np.max(np.abs(b)) <= FP32_NORM_TOL, (j, T)
    T = 300
    want, _ = O.ascend(cg, x, l, B, 0.05, T, 0.9, False)
    got = run(g, x, cg.n, l, B, 0.05, T, 0.9, False, LCB_FP32)
    s32, s64 = lc.DenseState(cg.n, l, B), lc.DenseState(cg.n, l, B)
    s32.values[:], s64.values[:] = got, want
    c32, _, _, _ = lc.round_cut_batch(g, s32, lifted=l > 1)
    c64, _, _, _ = lc.round_cut_batch(g, s64, lifted=l > 1)
    assert np.mean(c32 == c64) >= 0.99
    assert int(c32.max()) >= int(c64.max()) - 2


@pytest.mark.parametrize("slab_outer", [0, 1])
def test_stream_batched_search_bitwise(slab_outer):
    """Per-member alpha / T and the shrinking live width of batched evolve() rounds
    (GEN variant, early exit on) through K1s: sequential == batched == oracle."""
    cg = O.generate_er(300, 0.03, 3)
    cfg = lc.SolverConfig(batch_size=64, num_batches=2, ascent=lc.AscentParams(0.05, 60),
                          search=lc.SearchConfig(20, 80, -3.0, -1.0, 6, 3))
    with lc.options(resident=0, stream=1, slab_outer=slab_outer):
        a = lc.pquco(pg(cg), cfg, 11, opts=lc.RunOptions(precision=LCB_FP64, batched_search=False))
        b = lc.pquco(pg(cg), cfg, 11, opts=lc.RunOptions(precision=LCB_FP64, batched_search=True))
    assert a.kernel_stats["k_stream"][1] > 0 and a.kernel_stats["k_resident"][1] == 0
    assert a.best.cut_value == b.best.cut_value and a.batch_trace == b.batch_trace
    assert a.search_trace == b.search_trace and np.array_equal(a.best.assignment, b.best.assignment)
    w = O.solve(cg, O.default_config(batch_size=64, num_batches=2, iterations=60, has_search=1, t_lower=20,
                                     t_upper=80, e_lower=-3.0, e_upper=-1.0, population_size=6, rounds=3), 11)
    assert b.best.cut_value == w.cut_value and b.best.assignment.tolist() == w.assignment.tolist()


def test_stream_fp64_iterate_larger_than_l2():
    # ER n=250k, B=72 fp64: the padded iterate is 250k x 128 x 8 B = 256 MB per buffer
    rng = np.random.default_rng(1)
    n, m = 250_000, 1_250_000
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    keep = u != v
    cg = O.csr_from_edges(n, u[keep], v[keep])
    B, T = 72, 25
    x = start(rng, n, 1, B)
    want, _ = O.ascend(cg, x, 1, B, 0.05, T, 0.9, False)
    got = run(pg(cg), x, n, 1, B, 0.05, T, 0.9, False, LCB_FP64)
    assert np.array_equal(got, want)
