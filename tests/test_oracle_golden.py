"""Pins the CPU oracle (oracle/lc_oracle.c) to the reference.

1. golden vectors produced by the unmodified reference (tests/golden, generator
   tests/golden/make_golden.py);
2. the reference's own known-answer tests (proj/tests/test_*.cpp), restated;
3. a randomized cross-check against the compiled reference (oracle/_ref) when it
   is present.
"""
import hashlib

import numpy as np
import pytest

import oracle as O
from conftest import oracle_config


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# -- 1. golden vectors --------------------------------------------------------
def test_ascent_states_bitwise(golden):
    meta, arr = golden("ascent_states.json"), golden("ascent_states.npz")
    for c in meta:
        g = O.CSR(c["n"], arr[c["name"] + "/off"], arr[c["name"] + "/adj"])
        x0 = arr[c["name"] + "/x0"]
        for T in c["horizons"]:
            xt, _ = O.ascend(g, x0, c["l"], c["B"], c["alpha"], T, c["mu"], c["early_exit"])
            assert np.array_equal(xt, arr[f"{c['name']}/x{T}"]), (c["name"], T)


def test_gaussian_batch_bitwise(golden):
    meta, arr = golden("ascent_states.json"), golden("ascent_states.npz")
    for c in meta:
        g = O.CSR(c["n"], arr[c["name"] + "/off"], arr[c["name"] + "/adj"])
        mean = O.lifted_init_mean(g, 1, 0.2, c["l"], int(c["mean_key"])) / 1e4
        x0 = O.gaussian_batch(mean, g.n, c["l"], 0.8e-8, c["B"], int(c["gauss_key"]))
        assert np.array_equal(x0, arr[c["name"] + "/x0"]), c["name"]


def test_c1_er800_hashes(golden):
    c1 = golden("c1_er800.json")
    g = O.generate_er(800, 0.015, 0)
    assert g.m == c1["m"]
    mean = O.lifted_init_mean(g, 1, 0.2, 1, O.split(0, 0x696E, 0, 0)) / 1e4
    assert sha(mean) == c1["mean_sha"]
    x0 = O.gaussian_batch(mean, g.n, 1, 0.8e-8, 64, int(c1["gauss_key"]))
    assert sha(x0) == c1["x0_sha"]
    x10, _ = O.ascend(g, x0, 1, 64, 0.05, 10, 0.9, False)
    assert sha(x10) == c1["x10_sha"]
    cuts = [O.cut_value(g, O.round_unlifted(x10[j * 800:(j + 1) * 800])) for j in range(64)]
    assert cuts == c1["cuts10"]


def test_init_vectors_bitwise(golden):
    d = golden("init_vectors.json")
    g = O.CSR(len(d["off"]) - 1, np.array(d["off"], dtype=np.int64), np.array(d["adj"], dtype=np.uint32))
    for c in d["cases"]:
        key = int(c["key"])
        assert np.array_equal(O.dui_init(g, key), np.array(c["dui"]))
        assert np.array_equal(O.idi_init(g, 0.2, key), np.array(c["idi"]))
        assert np.array_equal(O.lifted_init_mean(g, 1, 0.35, 3, key), np.array(c["lifted_idi3"]))


def test_solver_records_bitwise(golden):
    d = golden("solver_records.json")
    for c in d["cases"]:
        off, adj = d["graphs"][c["graph"]]
        g = O.CSR(len(off) - 1, np.array(off, dtype=np.int64), np.array(adj, dtype=np.uint32))
        r = O.solve(g, oracle_config(c["config"]), c["seed"], per_component=c["per_component"])
        assert r.cut_value == c["cut"]
        assert r.batch_index == c["batch_index"] and r.member_index == c["member_index"]
        assert r.batches_run == c["batches_run"]
        assert r.assignment.tolist() == c["assignment"]
        assert [list(e) for e in r.batch_trace] == c["batch_trace"]
        assert [list(e) for e in r.phase_trace] == c["phase_trace"]
        assert [list(e) for e in r.search_trace] == c["search_trace"]


# -- 2. the reference's known-answer tests, restated on the oracle -------------
def edge():
    return O.csr_from_edges(2, [0], [1])


def test_kat_laplacian():  # test_graph.cpp:211-238
    assert np.array_equal(O.laplacian(edge(), [1.0, -1.0]), [2.0, -2.0])
    k3 = O.csr_from_edges(3, [0, 1, 0], [1, 2, 2])
    assert np.array_equal(O.laplacian(k3, [1.0, 0.0, 0.0]), [2.0, -1.0, -1.0])
    assert np.array_equal(O.laplacian(k3, np.ones(3)), np.zeros(3))


def test_kat_ascent_steps():  # test_ascent.cpp:28-65
    x, _ = O.ascend(edge(), [0.1, -0.1], 1, 1, 0.5, 1, 0.0)
    assert np.allclose(x, [0.2, -0.2])
    x, _ = O.ascend(edge(), [0.1, -0.1], 1, 1, 10.0, 3, 0.0)
    assert x.tolist() == [1.0, -1.0]
    g = O.generate_er(10, 0.5, 3)
    for mu in (0.0, 0.9):
        x, _ = O.ascend(g, np.full(10, 1e-4), 1, 1, 0.7, 25, mu, False)
        assert np.all(x == 1e-4)


def test_kat_numeric_error():  # test_ascent.cpp:225-240
    with pytest.raises(O.OracleError) as e:
        O.ascend(edge(), [0.1, -0.1], 1, 1, 1e308, 5, 0.0)
    assert e.value.status == 3 and "iteration" in str(e.value) and "member" in str(e.value)


def test_kat_rounding_and_cut():  # test_objectives.cpp:28-56,197-213
    tri = O.csr_from_edges(3, [0, 1, 0], [1, 2, 2])
    assert O.cut_value(tri, [1, 0, 0]) == 2 and O.cut_value(tri, [0, 0, 0]) == 0
    assert O.round_unlifted([0.0, 1e-300, -0.5]).tolist() == [0, 1, 0]
    assert O.round_lifted([0.5, -0.5, -0.5, 0.25], 2, 2).tolist() == [1, 0]
    with pytest.raises(O.OracleError):
        O.cut_value(tri, [2, 0, 0])


def test_kat_idi_star():  # test_init.cpp:55-63
    star = O.csr_from_edges(4, [0, 0, 0], [1, 2, 3])
    for key in range(5):
        x = O.idi_init(star, 0.2, key)
        assert all(x[v] == -x[0] for v in (1, 2, 3))


def test_kat_solver_small_graphs():  # test_solver.cpp:46-141
    pet_e = ([v for v in range(5)] + [5 + v for v in range(5)] + list(range(5)),
             [(v + 1) % 5 for v in range(5)] + [5 + (v + 2) % 5 for v in range(5)] + [5 + v for v in range(5)])
    pet = O.csr_from_edges(10, *pet_e)
    assert O.solve(pet, O.default_config(algorithm=2, batch_size=64), 0).cut_value == 12
    c5 = O.csr_from_edges(5, [0, 1, 2, 3, 0], [1, 2, 3, 4, 4])
    assert O.solve(c5, O.default_config(algorithm=1, batch_size=64), 0).cut_value == 4
    k4 = O.csr_from_edges(4, [0, 0, 0, 1, 1, 2], [1, 2, 3, 2, 3, 3])
    assert O.solve(k4, O.default_config(batch_size=32, iterations=200, init_method=0), 0).cut_value == 4


def test_brute_force_triangle():  # tests/CMakeLists.txt:36-37
    tri = O.csr_from_edges(3, [0, 1, 0], [1, 2, 2])
    best, w, cnt = O.brute_force_maxcut(tri)
    assert (best, "".join(map(str, w)), cnt) == (2, "100", 6)


# -- 3. randomized cross-check against the compiled reference -----------------
needs_ref = pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("seed", range(4))
def test_random_against_reference(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 50))
    rg = O.RefGraph.er(n, float(rng.uniform(0.05, 0.4)), seed)
    g = rg.csr()
    if g.m == 0:
        return
    l, B = int(rng.integers(1, 4)), int(rng.integers(1, 9))
    x = rng.uniform(-1, 1, B * l * n)
    ee = bool(seed % 2)
    a, _ = O.ascend(g, x, l, B, 0.1, 150, 0.9, ee)
    b, _ = O.ref_ascend(rg, x, l, B, 0.1, 150, 0.9, ee, workers=3)
    assert np.array_equal(a, b)
    for algo in (0, 1, 2):
        cfg = O.default_config(algorithm=algo, batch_size=8, iterations=60, has_search=seed % 2,
                               t_lower=10, t_upper=30, population_size=2, rounds=2)
        r1, r2 = O.solve(g, cfg, seed), O.ref_solve(rg, cfg, seed)
        assert (r1.cut_value, r1.batch_index, r1.member_index) == (r2.cut_value, r2.batch_index, r2.member_index)
        assert np.array_equal(r1.assignment, r2.assignment) and r1.batch_trace == r2.batch_trace


@needs_ref
def test_brute_force_against_reference():  # oracle.cpp:50-99, test_oracle.cpp:36-120
    rng = np.random.default_rng(7)
    for n in (1, 2, 3, 7, 11, 16):
        for p in (0.2, 0.5, 0.9):
            eu, ev = np.triu_indices(n, 1)
            keep = rng.random(len(eu)) < p
            cg = O.csr_from_edges(n, eu[keep], ev[keep])
            best, w, cnt = O.brute_force_maxcut(cg)
            rb, rw, rc = O.ref_brute_force_maxcut(O.RefGraph.from_edges(n, eu[keep], ev[keep]))
            assert (best, w.tolist(), cnt) == (rb, rw.tolist(), rc), (n, p)
    with pytest.raises(O.OracleError):
        O.ref_brute_force_maxcut(O.RefGraph.from_edges(27, [0], [1]))

