"""Parity of the CUDA path (through the C ABI) with the oracle and the golden vectors.

fp64 (LCB_FP64): bit-exact states, cuts, assignments and solver records.
fp32 (LCB_FP32): ||dx||_inf / ||x||_inf <= 1e-5 at T <= 10 (pre-saturation),
identical rounded cuts on >= 99% of members at full T, integer parts exact.
"""
import hashlib

import numpy as np
import pytest

import oracle as O
from conftest import oracle_config, product_config
from paper_2509_18612_b200 import LCB_FP32, LCB_FP64
from paper_2509_18612_b200 import liftcut as lc

pytestmark = pytest.mark.gpu

FP32_NORM_TOL = 1e-5


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def pg(c: O.CSR) -> lc.Graph:
    return lc.Graph.from_csr(c.n, c.off, c.adj)


def state_of(x, n, l, B):
    s = lc.DenseState(n, l, B)
    s.values[:] = x
    return s


def run_ascend(g, x, n, l, B, alpha, T, mu, ee, prec=LCB_FP64):
    s = state_of(x, n, l, B)
    lc.ascend(g, s, lc.AscentParams(alpha, T, mu, ee), precision=prec)
    return s.values


# --------------------------------------------------------------------------- ascend
def test_ascent_golden_bitwise(golden):
    meta, arr = golden("ascent_states.json"), golden("ascent_states.npz")
    for c in meta:
        g = pg(O.CSR(c["n"], arr[c["name"] + "/off"], arr[c["name"] + "/adj"]))
        x0 = arr[c["name"] + "/x0"]
        for T in c["horizons"]:
            got = run_ascend(g, x0, c["n"], c["l"], c["B"], c["alpha"], T, c["mu"], c["early_exit"])
            assert np.array_equal(got, arr[f"{c['name']}/x{T}"]), (c["name"], T)


@pytest.mark.parametrize("seed", range(6))
def test_ascent_random_vs_oracle_bitwise(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 400))
    cg = O.generate_er(n, float(rng.uniform(0.01, 0.3)), seed)
    if cg.m == 0:
        return
    l, B = int(rng.integers(1, 4)), int(rng.integers(1, 70))
    x = rng.uniform(-1, 1, B * l * n) * (10.0 ** -rng.integers(0, 5))
    alpha, mu, T = float(rng.uniform(0.001, 0.3)), float(rng.choice([0.0, 0.5, 0.9])), int(rng.integers(1, 120))
    for ee in (False, True):
        want, _ = O.ascend(cg, x, l, B, alpha, T, mu, ee)
        got = run_ascend(pg(cg), x, n, l, B, alpha, T, mu, ee)
        assert np.array_equal(got, want), (seed, ee)


def test_ascent_degree_skew_bitwise():
    # star + hub rows exercise long CSR rows (BA-like degree skew)
    n = 700
    u = [0] * 600 + list(range(1, 699))
    v = list(range(1, 601)) + list(range(2, 700))
    cg = O.csr_from_edges(n, u, v)
    rng = np.random.default_rng(7)
    x = rng.uniform(-1e-3, 1e-3, 37 * n)
    want, _ = O.ascend(cg, x, 1, 37, 0.01, 40, 0.9, False)
    assert np.array_equal(run_ascend(pg(cg), x, n, 1, 37, 0.01, 40, 0.9, False), want)


def test_c1_er800_golden(golden):
    c1 = golden("c1_er800.json")
    cg = O.generate_er(800, 0.015, 0)
    g = pg(cg)
    mean = O.lifted_init_mean(cg, 1, 0.2, 1, O.split(0, 0x696E, 0, 0)) / 1e4
    x0 = O.gaussian_batch(mean, 800, 1, 0.8e-8, 64, int(c1["gauss_key"]))
    for T in (10, 500):
        xt = run_ascend(g, x0, 800, 1, 64, 0.05, T, 0.9, False)
        assert sha(xt) == c1[f"x{T}_sha"]
        cuts, bm, bc, _ = lc.round_cut_batch(g, state_of(xt, 800, 1, 64), lifted=False)
        assert cuts.tolist() == c1[f"cuts{T}"]
        assert bc == max(c1[f"cuts{T}"]) and bm == c1[f"cuts{T}"].index(bc)
    # fp32 fast path: norm-wise early, identical cuts late
    x10 = run_ascend(g, x0, 800, 1, 64, 0.05, 10, 0.9, False, LCB_FP32)
    ref10, _ = O.ascend(cg, x0, 1, 64, 0.05, 10, 0.9, False)
    for j in range(64):
        a, b = x10[j * 800:(j + 1) * 800], ref10[j * 800:(j + 1) * 800]
        assert np.max(np.abs(a - b)) / np.max(np.abs(b)) <= FP32_NORM_TOL
    x500 = run_ascend(g, x0, 800, 1, 64, 0.05, 500, 0.9, False, LCB_FP32)
    cuts32, _, _, _ = lc.round_cut_batch(g, state_of(x500, 800, 1, 64), lifted=False)
    same = sum(int(a == b) for a, b in zip(cuts32.tolist(), c1["cuts500"]))
    assert same >= 0.99 * 64


def test_ascent_fp32_lifted_tolerance():
    cg = O.generate_er(300, 0.05, 5)
    rng = np.random.default_rng(3)
    x = rng.uniform(-1e-4, 1e-4, 20 * 2 * 300)
    want, _ = O.ascend(cg, x, 2, 20, 0.05, 8, 0.9, False)
    got = run_ascend(pg(cg), x, 300, 2, 20, 0.05, 8, 0.9, False, LCB_FP32)
    for j in range(20):
        a, b = got[j * 600:(j + 1) * 600], want[j * 600:(j + 1) * 600]
        assert np.max(np.abs(a - b)) / np.max(np.abs(b)) <= FP32_NORM_TOL


def test_ascent_errors():
    g = lc.Graph(2, [(0, 1)])
    s = state_of([0.1, -0.1], 2, 1, 1)
    with pytest.raises(lc.NumericError) as e:
        lc.ascend(g, s, lc.AscentParams(1e308, 5, 0.0))
    assert "iteration" in str(e.value) and "member" in str(e.value)
    with pytest.raises(lc.ShapeError):
        lc.ascend(g, lc.DenseState(3, 1, 1), lc.AscentParams())
    with pytest.raises(lc.ValidationError):
        lc.ascend(g, s, lc.AscentParams(alpha=0.0))


def test_ascent_trace_counts_every_step():  # test_ascent.cpp:208-223
    g = lc.Graph(3, [(0, 1), (1, 2), (0, 2)])
    rng = np.random.default_rng(15)
    s = state_of(rng.uniform(-0.5, 0.5, 6), 3, 1, 2)
    seen = []
    lc.ascend(g, s, lc.AscentParams(0.05, 7, 0.0), trace=lambda it, m, obj: seen.append((it, m, obj)))
    assert len(seen) == 14 and all(o >= -1e-12 for _, _, o in seen)
    cg = O.csr_from_edges(3, [0, 1, 0], [1, 2, 2])
    _, tr = O.ascend(cg, state_of(rng.uniform(-0.5, 0.5, 6), 3, 1, 2).values, 1, 2, 0.05, 7, 0.0, trace=True)
    assert tr.shape == (7, 2)


@pytest.mark.parametrize("l,prec", [(1, LCB_FP64), (2, LCB_FP64), (2, LCB_FP32)])
def test_ascent_trace_values_vs_oracle(l, prec):
    """Objective trace values (ascent.cpp:78-88: x'Lx summed over the lift columns after
    every step) against the oracle's sequential fp64 sums: the device reduction order
    differs, so equal to 1e-12 relative in fp64 (the states themselves bitwise), 1e-5 in fp32."""
    cg = O.generate_er(1500, 0.006, 5)
    g = lc.Graph.from_csr(cg.n, cg.off, cg.adj)
    rng = np.random.default_rng(l)
    B, T = 12, 25
    x = rng.uniform(-0.3, 0.3, B * l * cg.n)
    s = lc.DenseState(cg.n, l, B)
    s.values[:] = x
    seen = np.full((T, B), np.nan)
    lc.ascend(g, s, lc.AscentParams(0.05, T, 0.9), precision=prec,
              trace=lambda it, m, obj: seen.__setitem__((it, m), obj))
    want_x, want = O.ascend(cg, x, l, B, 0.05, T, 0.9, False, trace=True)
    assert not np.isnan(seen).any()
    tol = 1e-12 if prec == LCB_FP64 else 1e-5
    assert np.max(np.abs(seen - want) / np.maximum(np.abs(want), 1.0)) <= tol
    if prec == LCB_FP64:
        assert np.array_equal(s.values, want_x)


# --------------------------------------------------------------- objectives / epilogue
def test_laplacian_apply():
    g = lc.Graph(2, [(0, 1)])
    assert np.array_equal(g.laplacian_apply([1.0, -1.0]), [2.0, -2.0])
    cg = O.generate_er(500, 0.02, 9)
    x = np.random.default_rng(1).uniform(-1, 1, (5, 500))
    want = np.stack([O.laplacian(cg, r) for r in x])
    assert np.array_equal(pg(cg).laplacian_apply(x), want)


@pytest.mark.parametrize("count", [1, 31, 32, 33, 100, 1030])
def test_cut_values_vs_oracle(count):
    cg = O.generate_er(333, 0.04, count)
    Z = np.random.default_rng(count).integers(0, 2, (count, 333)).astype(np.uint8)
    got = lc.cut_values(pg(cg), Z)
    assert got.tolist() == [O.cut_value(cg, z) for z in Z]
    with pytest.raises(lc.ValidationError):
        lc.cut_value(pg(cg), np.full(333, 2, dtype=np.uint8))


@pytest.mark.parametrize("l", [1, 2, 3])
def test_round_cut_argmax_vs_oracle(l):
    n, B = 257, 70
    cg = O.generate_er(n, 0.05, l)
    rng = np.random.default_rng(l)
    x = rng.choice([-1.0, 0.0, 1.0, 0.25, -0.25], size=B * l * n)  # ties on purpose
    cuts, bm, bc, z = lc.round_cut_batch(pg(cg), state_of(x, n, l, B), lifted=l > 1)
    want = []
    for j in range(B):
        mv = x[j * l * n:(j + 1) * l * n]
        zz = O.round_lifted(mv, n, l) if l > 1 else O.round_unlifted(mv)
        want.append(O.cut_value(cg, zz))
    assert cuts.tolist() == want
    assert bc == max(want) and bm == want.index(max(want))
    mv = x[bm * l * n:(bm + 1) * l * n]
    assert np.array_equal(z, O.round_lifted(mv, n, l) if l > 1 else O.round_unlifted(mv))


# --------------------------------------------------------------------------- init
def test_init_golden_bitwise(golden):
    d = golden("init_vectors.json")
    g = lc.Graph.from_csr(len(d["off"]) - 1, d["off"], d["adj"])
    for c in d["cases"]:
        st = lc.RngStream(int(c["key"]))
        assert np.array_equal(lc.dui_init(g, st), np.array(c["dui"]))
        assert np.array_equal(lc.idi_init(g, 0.2, st), np.array(c["idi"]))
        m = lc.lifted_init_mean(g, lc.InitConfig(beta=0.35), 3, st)
        assert np.array_equal(m, np.array(c["lifted_idi3"]))


def test_gaussian_batch_close_to_glibc():
    n, l, B = 300, 2, 50
    mean = np.random.default_rng(2).choice([-1e-4, 1e-4], n * l)
    key = 987654321
    got = lc.gaussian_batch(mean, n, l, 0.8e-8, B, lc.RngStream(key), exact=False).values
    want = O.gaussian_batch(mean, n, l, 0.8e-8, B, key)
    # the exact variant (the fp64 default and the drop-in's) is the reference's bits
    assert np.array_equal(lc.gaussian_batch(mean, n, l, 0.8e-8, B, lc.RngStream(key), exact=True).values, want)
    # CUDA log/cos vs glibc: a few ulp in the normal, i.e. |dx| <= 8 eps (|mean| + |noise|)
    scale = np.abs(mean.reshape(1, -1)).repeat(B, 0).ravel() + np.sqrt(0.8e-8) * 6.0
    assert np.all(np.abs(got - want) <= 8 * np.finfo(float).eps * scale)
    assert np.mean(got == want) > 0.5
    big = lc.gaussian_batch(np.zeros(n), n, 1, 4.0, B, lc.RngStream(1), exact=False).values
    assert big.min() >= -1.0 and big.max() <= 1.0  # projected onto the box


# --------------------------------------------------------------------------- solver
def test_solver_golden_records_bitwise(golden):
    d = golden("solver_records.json")
    for c in d["cases"]:
        off, adj = d["graphs"][c["graph"]]
        g = lc.Graph.from_csr(len(off) - 1, off, adj)
        cfg = product_config(c["config"])
        fn = lc.solve_per_component if c["per_component"] else {0: lc.pquco, 1: lc.pluco, 2: lc.pdeco}[cfg.algorithm]
        r = fn(g, cfg, c["seed"], opts=lc.RunOptions(precision=LCB_FP64))
        assert r.best.cut_value == c["cut"], c
        assert (r.best.batch_index, r.best.member_index, r.batches_run) == (
            c["batch_index"], c["member_index"], c["batches_run"])
        assert r.best.assignment.tolist() == c["assignment"]
        assert [[e.serial, 0 if e.kind == "main" else 1, e.alpha, e.iterations, e.batch_best, e.best_so_far]
                for e in r.batch_trace] == c["batch_trace"]
        assert [[e.phase, 0 if e.kind == "quco" else 1, e.best_after] for e in r.phase_trace] == c["phase_trace"]
        assert [[e.round, e.exponent, e.iterations, e.fitness] for e in r.search_trace] == c["search_trace"]


@pytest.mark.parametrize("prec", [LCB_FP64, LCB_FP32])
@pytest.mark.parametrize("algo", [0, 1, 2])
def test_solver_device_init_quality(prec, algo):
    cg = O.generate_er(150, 0.06, 21)
    cfg_o = O.default_config(algorithm=algo, batch_size=48, iterations=300)
    want = O.solve(cg, cfg_o, 4)
    g = pg(cg)
    cfg = lc.SolverConfig(algorithm=lc.Algorithm(algo), batch_size=48,
                          ascent=lc.AscentParams(iterations=300))
    fn = {0: lc.pquco, 1: lc.pluco, 2: lc.pdeco}[algo]
    r = fn(g, cfg, 4, opts=lc.RunOptions(precision=prec, host_init=0))
    assert lc.cut_value(g, r.best.assignment) == r.best.cut_value
    assert r.batches_run == want.batches_run
    assert r.best.cut_value >= want.cut_value - 2  # same algorithm, ulp-level different draws


def test_solver_kats_from_reference_suite():  # test_solver.cpp:46-141, 189-224
    edge = lc.Graph(2, [(0, 1)])
    out = lc.pquco(edge, lc.SolverConfig(batch_size=4, ascent=lc.AscentParams(0.1, 50)), 1)
    assert out.best.cut_value == 1 and 0 <= out.best.member_index < 4
    star = lc.Graph(4, [(0, 1), (0, 2), (0, 3)])
    out = lc.pquco(star, lc.SolverConfig(), 0)
    assert out.best.cut_value == 3 and out.batch_trace[0].batch_best == 3
    k4 = lc.Graph(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)])
    cfg = lc.SolverConfig(batch_size=32, ascent=lc.AscentParams(iterations=200),
                          init=lc.InitConfig(method=lc.InitMethod.DUI))
    assert lc.pquco(k4, cfg, 0).best.cut_value == 4
    assert lc.pluco(k4, lc.SolverConfig(algorithm=lc.Algorithm.pLUCO), 0).best.cut_value == 4
    c5 = lc.Graph(5, [(0, 1), (1, 2), (2, 3), (3, 4), (0, 4)])
    cyc = lc.pdeco(c5, lc.SolverConfig(algorithm=lc.Algorithm.pDECO), 0)
    assert cyc.best.cut_value == 4 and [p.kind for p in cyc.phase_trace] == ["quco", "luco"] * 2
    two = lc.Graph(4, [(0, 1), (2, 3)])
    a = lc.solve_per_component(two, lc.SolverConfig(batch_size=16), 1)
    assert a.best.cut_value == 2 and a.best.batch_index == -1
    iso = lc.Graph(3, [(0, 1)])
    b = lc.solve_per_component(iso, lc.SolverConfig(batch_size=16), 1)
    assert b.best.cut_value == 1 and b.best.assignment[2] == 0 and b.best.batch_index >= 0
    with pytest.raises(lc.ValidationError):
        lc.pquco(lc.Graph(3, []), lc.SolverConfig(), 0)


# ------------------------------------------------------- member-resident fp32 kernel (K2)
def _ba_like(n, m, seed):
    rng = np.random.default_rng(seed)
    us, vs, targets = [], [], list(range(m))
    repeated = []
    for v in range(m, n):
        chosen = set()
        while len(chosen) < m:
            chosen.add(int(rng.choice(repeated)) if repeated and rng.random() < 0.9 else int(rng.integers(0, v)))
        for u in chosen:
            us.append(u)
            vs.append(v)
        repeated += list(chosen) + [v] * m
    return O.csr_from_edges(n, us, vs)


@pytest.mark.parametrize("l,B,ee", [(1, 400, False), (2, 200, False), (1, 400, True), (2, 200, True), (3, 110, False)])
def test_resident_fp32_tolerance_and_cuts(l, B, ee):
    cg = _ba_like(3000, 4, 11)
    g = pg(cg)
    rng = np.random.default_rng(l * 10 + B)
    x = rng.choice([-1e-4, 1e-4], B * l * cg.n) + rng.normal(0, 9e-5, B * l * cg.n)
    for T in (6,):
        want, _ = O.ascend(cg, x, l, B, 0.05, T, 0.9, ee)
        got = run_ascend(g, x, cg.n, l, B, 0.05, T, 0.9, ee, LCB_FP32)
        for j in range(B):
            a, b = got[j * l * cg.n:(j + 1) * l * cg.n], want[j * l * cg.n:(j + 1) * l * cg.n]
            assert np.max(np.abs(a - b)) / np.max(np.abs(b)) <= FP32_NORM_TOL, (j, T)
    T = 300
    want, _ = O.ascend(cg, x, l, B, 0.05, T, 0.9, ee)
    got = run_ascend(g, x, cg.n, l, B, 0.05, T, 0.9, ee, LCB_FP32)
    c32, _, _, _ = lc.round_cut_batch(g, state_of(got, cg.n, l, B), lifted=l > 1)
    c64, _, _, _ = lc.round_cut_batch(g, state_of(want, cg.n, l, B), lifted=l > 1)
    assert np.mean(c32 == c64) >= 0.97
    assert abs(int(c32.max()) - int(c64.max())) <= 2


def test_global_step_kernel_bitwise_when_resident_disabled(tmp_path):
    """The HBM-streaming k_step path (used when the slab does not fit on chip) stays
    bit-exact too: rerun the golden ascent states with LCB_RESIDENT=0."""
    import os
    import subprocess
    import sys

    code = (
        "import numpy as np, json, oracle as O\n"
        "from paper_2509_18612_b200 import liftcut as lc, LCB_FP64\n"
        "meta=json.load(open('tests/golden/ascent_states.json')); arr=np.load('tests/golden/ascent_states.npz')\n"
        "for c in meta:\n"
        "  g=lc.Graph.from_csr(c['n'],arr[c['name']+'/off'],arr[c['name']+'/adj'])\n"
        "  for T in c['horizons']:\n"
        "    s=lc.DenseState(c['n'],c['l'],c['B']); s.values[:]=arr[c['name']+'/x0']\n"
        "    lc.ascend(g,s,lc.AscentParams(c['alpha'],T,c['mu'],c['early_exit']),precision=LCB_FP64)\n"
        "    assert np.array_equal(s.values,arr[c['name']+'/x%d'%T]),(c['name'],T)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       env={**os.environ, "LCB_RESIDENT": "0"}, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_resident_isolated_and_heavy_rows_fp64_bitwise():
    # isolated nodes (degree 0), > 32-degree hubs and > 1024 rows in one graph
    n = 2500
    rng = np.random.default_rng(5)
    u = list(rng.integers(0, 2000, 4000)) + [0] * 300 + [1] * 120
    v = list(rng.integers(0, 2000, 4000)) + list(range(1000, 1300)) + list(range(1500, 1620))
    keep = [(a, b) for a, b in zip(u, v) if a != b]
    cg = O.csr_from_edges(n, [a for a, _ in keep], [b for _, b in keep])
    assert (np.diff(cg.off) == 0).sum() >= 400 and np.diff(cg.off).max() > 32
    x = rng.uniform(-1e-3, 1e-3, 40 * n)
    for ee in (False, True):
        want, _ = O.ascend(cg, x, 1, 40, 0.03, 60, 0.9, ee)
        assert np.array_equal(run_ascend(pg(cg), x, n, 1, 40, 0.03, 60, 0.9, ee), want)
        got32 = run_ascend(pg(cg), x, n, 1, 40, 0.03, 5, 0.9, ee, LCB_FP32)
        w5, _ = O.ascend(cg, x, 1, 40, 0.03, 5, 0.9, ee)
        for j in range(40):
            a_, b_ = got32[j * n:(j + 1) * n], w5[j * n:(j + 1) * n]
            assert np.max(np.abs(a_ - b_)) / np.max(np.abs(b_)) <= FP32_NORM_TOL


def test_batched_search_rounds_match_sequential_and_reference(golden):
    """evolve() rounds evaluated as one multi-candidate launch keep every serial,
    stream, fitness and trace of the sequential order (no time budget)."""
    d = golden("solver_records.json")
    n_search = 0
    for c in d["cases"]:
        if not c["config"]["has_search"]:
            continue
        n_search += 1
        off, adj = d["graphs"][c["graph"]]
        g = lc.Graph.from_csr(len(off) - 1, off, adj)
        cfg = product_config(c["config"])
        fn = {0: lc.pquco, 1: lc.pluco, 2: lc.pdeco}[cfg.algorithm]
        r = fn(g, cfg, c["seed"], opts=lc.RunOptions(precision=LCB_FP64, batched_search=True))
        assert r.best.cut_value == c["cut"] and r.best.assignment.tolist() == c["assignment"]
        assert [[e.serial, 0 if e.kind == "main" else 1, e.alpha, e.iterations, e.batch_best, e.best_so_far]
                for e in r.batch_trace] == c["batch_trace"]
        assert [[e.round, e.exponent, e.iterations, e.fitness] for e in r.search_trace] == c["search_trace"]
    assert n_search >= 2
    # a larger population through both paths
    cg = O.generate_er(300, 0.03, 3)
    cfg = lc.SolverConfig(batch_size=64, num_batches=2, ascent=lc.AscentParams(0.05, 60),
                          search=lc.SearchConfig(20, 80, -3.0, -1.0, 6, 3))
    a = lc.pquco(pg(cg), cfg, 11, opts=lc.RunOptions(precision=LCB_FP64, batched_search=False))
    b = lc.pquco(pg(cg), cfg, 11, opts=lc.RunOptions(precision=LCB_FP64, batched_search=True))
    assert a.best.cut_value == b.best.cut_value and a.batch_trace == b.batch_trace
    assert a.search_trace == b.search_trace and np.array_equal(a.best.assignment, b.best.assignment)
    w = O.solve(cg, O.default_config(batch_size=64, num_batches=2, iterations=60, has_search=1, t_lower=20,
                                     t_upper=80, e_lower=-3.0, e_upper=-1.0, population_size=6, rounds=3), 11)
    assert b.best.cut_value == w.cut_value and b.best.assignment.tolist() == w.assignment.tolist()


def test_l2_panel_chunked_driver_bitwise(tmp_path):
    """The L2-panel path (K1n, forced with LCB_CHUNK=1) gives the same fp64 bits, fp32 within
    tolerance, and the same solver records (early tlim segments inside a panel)."""
    import os
    import subprocess
    import sys

    code = (
        "import numpy as np, oracle as O\n"
        "from paper_2509_18612_b200 import liftcut as lc, LCB_FP64, LCB_FP32\n"
        "cg = O.generate_er(20000, 0.0004, 5)\n"
        "g = lc.Graph.from_csr(cg.n, cg.off, cg.adj)\n"
        "rng = np.random.default_rng(1)\n"
        "for l, B in ((1, 80), (2, 41)):\n"
        "    x = rng.uniform(-1e-3, 1e-3, B * l * cg.n)\n"
        "    want, _ = O.ascend(cg, x, l, B, 0.05, 12, 0.9, False)\n"
        "    s = lc.DenseState(cg.n, l, B); s.values[:] = x\n"
        "    lc.ascend(g, s, lc.AscentParams(0.05, 12, 0.9, False), precision=LCB_FP64)\n"
        "    assert np.array_equal(s.values, want), (l, B)\n"
        "    s32 = lc.DenseState(cg.n, l, B); s32.values[:] = x\n"
        "    lc.ascend(g, s32, lc.AscentParams(0.05, 12, 0.9, False), precision=LCB_FP32)\n"
        "    assert np.linalg.norm(s32.values - want) <= 1e-5 * np.linalg.norm(want), (l, B)\n"
        "cg2 = O.generate_er(300, 0.03, 3)\n"
        "g2 = lc.Graph.from_csr(cg2.n, cg2.off, cg2.adj)\n"
        "cfg = lc.SolverConfig(batch_size=64, num_batches=2, ascent=lc.AscentParams(0.05, 60),\n"
        "                      search=lc.SearchConfig(20, 80, -3.0, -1.0, 6, 3))\n"
        "w = O.solve(cg2, O.default_config(batch_size=64, num_batches=2, iterations=60, has_search=1, t_lower=20,\n"
        "            t_upper=80, e_lower=-3.0, e_upper=-1.0, population_size=6, rounds=3), 11)\n"
        "for bs in (False, True):\n"
        "    b = lc.pquco(g2, cfg, 11, opts=lc.RunOptions(precision=LCB_FP64, batched_search=bs))\n"
        "    assert b.best.cut_value == w.cut_value and b.best.assignment.tolist() == w.assignment.tolist(), bs\n"
        "    ks = b.kernel_stats\n"
        "    assert ks['k_step'][1] + ks['k_stream'][1] > 0 and ks['k_resident'][1] == 0\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "LCB_CHUNK": "1", "LCB_RESIDENT": "0"})
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-2000:]


def test_adjacency_range_checked_on_both_ingest_paths():
    """Entries >= n are rejected (graph.cpp:18-21 semantics): on the host for graphs the
    host relabels (n <= 14336), on the device after the upload for larger ones."""
    for n in (100, 20000):
        off = np.zeros(n + 1, dtype=np.int64)
        off[1:] = 2
        off[1] = 1
        adj = np.array([1, 0], dtype=np.uint32)
        lc.Graph.from_csr(n, off, adj).handle()  # fine
        with pytest.raises(lc.ValidationError, match="out of range"):
            lc.Graph.from_csr(n, off, np.array([n, 0], dtype=np.uint32)).handle()


def test_release_workspaces_then_solve_again():
    """lcb_release_workspaces frees the pooled workspaces and trims the graph pools; the
    next graph build and solve allocate afresh and still match the oracle."""
    from paper_2509_18612_b200 import _abi

    cg = O.generate_er(300, 0.05, 2)
    rng = np.random.default_rng(6)
    x = rng.uniform(-0.1, 0.1, 8 * cg.n)
    want, _ = O.ascend(cg, x, 1, 8, 0.05, 20, 0.9, False)
    for _ in range(2):
        g = lc.Graph.from_csr(cg.n, cg.off, cg.adj)
        s = lc.DenseState(cg.n, 1, 8)
        s.values[:] = x
        lc.ascend(g, s, lc.AscentParams(0.05, 20, 0.9, False), precision=LCB_FP64)
        assert np.array_equal(s.values, want)
        g.release()
        _abi.lib().lcb_release_workspaces()
