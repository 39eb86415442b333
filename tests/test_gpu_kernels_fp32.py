"""The fp32 variants the benchmark numbers come from, against the oracle, and fp32
batch / rank invariance.

* K2 (member-resident) at config-2 scale (BA n=10k, networkx seed 0): K=2 packed
  columns with the bank-balanced neighbour order, wave-tail split on and off, l=1 and
  l=2: ||dx||_inf / ||x||_inf <= 1e-5 per member before saturation, and
  >= 99 % identical rounded cuts at T=500 against the fp64 path (itself bit-exact with
  the oracle, test_gpu_parity.py).
* the refined neighbour order is a per-row permutation of the CSR row (layout hook).
* K1 with saturation codes (signrec=1, stream=0): fp64 bit-exact through saturation and
  for an iterate larger than L2; fp32 within tolerance.
* fp32 invariance: a member's trajectory does not depend on the batch width (the kernel
  is chosen from the graph, not from W; one epilogue op sequence for every kernel), K1 ==
  K1s bit for bit, and K=1 == K=2 columns per CTA.
"""
import ctypes as C
import os
import sys

import numpy as np
import pytest

import oracle as O
from paper_2509_18612_b200 import LCB_FP32, LCB_FP64, _abi
from paper_2509_18612_b200 import liftcut as lc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def c2():
    from bench import ba_edges

    u, v = ba_edges(10_000, 4, 0)
    cg = O.csr_from_edges(10_000, u, v)
    return cg, lc.Graph.from_csr(cg.n, cg.off, cg.adj)


def start(rng, n, l, B):
    return rng.choice([-1e-4, 1e-4], B * l * n) + rng.normal(0, 9e-5, B * l * n)


def run(g, x, n, l, B, T, prec, alpha=0.05, ee=False, **opts):
    s = lc.DenseState(n, l, B)
    s.values[:] = x
    with lc.options(**opts):
        lc.ascend(g, s, lc.AscentParams(alpha, T, 0.9, ee), precision=prec)
    return s.values


def norm_err(got, want, n, l, B):
    return max(float(np.max(np.abs(got[j * l * n:(j + 1) * l * n] - want[j * l * n:(j + 1) * l * n])) /
                     np.max(np.abs(want[j * l * n:(j + 1) * l * n]))) for j in range(B))


def cuts(g, x, n, l, B):
    s = lc.DenseState(n, l, B)
    s.values[:] = x
    c, _, _, _ = lc.round_cut_batch(g, s, lifted=l > 1)
    return c


@pytest.mark.parametrize("l,B,split", [(1, 1024, 1), (1, 1024, 0), (2, 512, 1)])
def test_k2_packed_config2_vs_oracle(c2, l, B, split):
    cg, g = c2
    rng = np.random.default_rng(l * 7 + split)
    x = start(rng, cg.n, l, B)
    for T in (2, 4):  # before saturation on BA 10k (hubs of degree 280 saturate from T ~ 5)
        want, _ = O.ascend(cg, x, l, B, 0.05, T, 0.9, False)
        got = run(g, x, cg.n, l, B, T, LCB_FP32, resident=1, res_split=split)
        assert norm_err(got, want, cg.n, l, B) <= TOL, T
    T = 500
    x32 = run(g, x, cg.n, l, B, T, LCB_FP32, resident=1, res_split=split)
    x64 = run(g, x, cg.n, l, B, T, LCB_FP64, resident=1)
    c32, c64 = cuts(g, x32, cg.n, l, B), cuts(g, x64, cg.n, l, B)
    assert np.mean(c32 == c64) >= 0.99, np.mean(c32 == c64)
    assert int(c32.max()) >= int(c64.max()) - 2


def test_k2_refined_order_is_a_row_permutation(c2):
    cg, g = c2
    L = _abi.lib()
    ln = C.c_int64()
    assert L.lcb_debug_resident_layout(g.handle(), C.byref(ln), None, None, None, None) == 0
    col = np.zeros(ln.value, dtype=np.uint16)
    fast = np.zeros(ln.value, dtype=np.uint16)
    rw = np.zeros((cg.n, 2), dtype=np.int64)
    perm = np.zeros(cg.n, dtype=np.int32)
    assert L.lcb_debug_resident_layout(g.handle(), C.byref(ln), col.ctypes.data, fast.ctypes.data,
                                       rw.ctypes.data, perm.ctypes.data) == 0
    assert not np.all(fast == 0xFFFF)
    assert sorted(perm.tolist()) == list(range(cg.n))
    for r in range(cg.n):
        w, d = int(rw[r, 0]), int(rw[r, 1])
        seg = slice(4 * w, 4 * w + ((d + 3) & ~3))
        a, b = col[seg], fast[seg]
        assert sorted(a.tolist()) == sorted(b.tolist())                  # a permutation, pads included
        assert (a[d:] == cg.n).all() and int((b == cg.n).sum()) == len(a) - d  # pads = zero row n
        orig = np.sort(perm[a[:d].astype(np.int64)])
        v = int(perm[r])
        assert np.array_equal(orig, cg.adj[cg.off[v]:cg.off[v + 1]])       # the CSR row of perm[r]


def test_fp32_member_independent_of_batch_width(c2):
    """test_ascent.cpp:110-136 in fp32: members 0..199 of a W=1024 batch equal the same
    members run alone (W=200), and the same holds on a graph K2 does not take (K1s)."""
    cg, g = c2
    rng = np.random.default_rng(3)
    x = start(rng, cg.n, 1, 1024)
    wide = run(g, x, cg.n, 1, 1024, 80, LCB_FP32)
    narrow = run(g, x[:200 * cg.n], cg.n, 1, 200, 80, LCB_FP32)
    assert np.array_equal(wide[:200 * cg.n], narrow)
    # lifted with early exit: K = 2 per CTA at any width
    x2 = start(rng, cg.n, 2, 300)
    wide = run(g, x2, cg.n, 2, 300, 60, LCB_FP32, ee=True)
    narrow = run(g, x2[:40 * 2 * cg.n], cg.n, 2, 40, 60, LCB_FP32, ee=True)
    assert np.array_equal(wide[:40 * 2 * cg.n], narrow)
    # large graph (no K2): K1s at W=512 vs W=136
    rng2 = np.random.default_rng(8)
    n = 20_000
    u, v = rng2.integers(0, n, 100_000), rng2.integers(0, n, 100_000)
    keep = u != v
    big = O.csr_from_edges(n, u[keep], v[keep])
    gb = lc.Graph.from_csr(big.n, big.off, big.adj)
    xb = start(rng2, n, 1, 512)
    wide = run(gb, xb, n, 1, 512, 70, LCB_FP32)
    narrow = run(gb, xb[:136 * n], n, 1, 136, 70, LCB_FP32)
    assert np.array_equal(wide[:136 * n], narrow)


@pytest.mark.parametrize("ee,l,B", [(False, 1, 384), (True, 1, 384), (True, 2, 150)])
def test_k1_and_k1s_bitwise_equal_fp32(c2, ee, l, B):
    """K1 (saturation codes on / off) and K1s (x-code mode, slab-major and iteration-major)
    give the same fp32 iterate bit for bit, with and without early exit, unlifted and lifted
    with a ragged last slab."""
    cg, g = c2
    rng = np.random.default_rng(4 + l)
    x = start(rng, cg.n, l, B)
    a = run(g, x, cg.n, l, B, 70, LCB_FP32, ee=ee, resident=0, stream=0, signrec=1)
    b = run(g, x, cg.n, l, B, 70, LCB_FP32, ee=ee, resident=0, stream=1)
    c = run(g, x, cg.n, l, B, 70, LCB_FP32, ee=ee, resident=0, stream=0, signrec=0)
    d = run(g, x, cg.n, l, B, 70, LCB_FP32, ee=ee, resident=0, stream=1, slab_outer=1)
    assert np.array_equal(a, b) and np.array_equal(a, c) and np.array_equal(a, d)


@pytest.mark.parametrize("ee", [False, True])
def test_k1_saturation_codes_vs_oracle(ee):
    rng = np.random.default_rng(11)
    n = 3000
    u, v = rng.integers(0, n, 15000), rng.integers(0, n, 15000)
    u = np.concatenate([u, np.zeros(300, dtype=np.int64)])
    v = np.concatenate([v, rng.integers(1, n, 300)])
    keep = u != v
    cg = O.csr_from_edges(n, u[keep], v[keep])
    g = lc.Graph.from_csr(cg.n, cg.off, cg.adj)
    B = 200
    x = start(rng, n, 1, B)
    for T in (1, 10, 60):
        want, _ = O.ascend(cg, x, 1, B, 0.05, T, 0.9, ee)
        got = run(g, x, n, 1, B, T, LCB_FP64, ee=ee, resident=0, stream=0, signrec=1)
        assert np.array_equal(got, want), T
    for T in (3, 6):
        want, _ = O.ascend(cg, x, 1, B, 0.05, T, 0.9, ee)
        got = run(g, x, n, 1, B, T, LCB_FP32, ee=ee, resident=0, stream=0, signrec=1)
        assert norm_err(got, want, n, 1, B) <= TOL


def test_k1_saturation_codes_iterate_larger_than_l2():
    rng = np.random.default_rng(2)
    n, m = 250_000, 1_250_000
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    keep = u != v
    cg = O.csr_from_edges(n, u[keep], v[keep])
    g = lc.Graph.from_csr(cg.n, cg.off, cg.adj)
    B, T = 72, 25   # padded iterate 250k x 128 x 8 B = 256 MB per buffer
    x = start(rng, n, 1, B)
    want, _ = O.ascend(cg, x, 1, B, 0.05, T, 0.9, False)
    got = run(g, x, n, 1, B, T, LCB_FP64, resident=0, stream=0, signrec=-1)  # auto: on (> L2)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("opts,ee,want", [
    (dict(resident=1), False, "k_resident"),
    (dict(resident=1, res_split=0), False, "k_resident"),
    (dict(resident=0, stream=1), False, "k_stream"),
    (dict(resident=0, stream=1), True, "k_stream"),
    (dict(resident=0, stream=1, slab_outer=1), False, "k_stream"),
    (dict(resident=0, stream=0, signrec=1), True, "k_step"),
    (dict(resident=0, stream=0, signrec=0), False, "k_step"),
])
def test_options_route_to_the_named_kernel(c2, opts, ee, want):
    """The option sets the tests above use select the kernel they are named after (the
    solver's per-kernel launch counts on the same graph and batch shape), so a test of
    "K2" or "K1s" cannot pass on another kernel."""
    _, g = c2
    cfg = lc.SolverConfig(batch_size=384, num_batches=1, ascent=lc.AscentParams(0.05, 20, 0.9, ee))
    with lc.options(**opts):
        out = lc.pquco(g, cfg, 1, opts=lc.RunOptions(precision=LCB_FP32))
    ks = {k: v[1] for k, v in out.kernel_stats.items()}
    assert ks[want] > 0, ks
    assert all(v == 0 for k, v in ks.items() if k != want), ks
