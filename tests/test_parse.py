"""parse_edge_list (graph.cpp:136-172): the golden outcomes of the UNMODIFIED reference
(tests/golden/parse_cases.json, tests/golden/make_parse_golden.py) against

* the host restatement `liftcut.parse_edge_list` and the fast reader `load_graph_file`
  (CPU);
* the device parser `liftcut.parse_edge_list_device` / `lcb_graph_parse` (GPU): the same
  CSR, the same error class and message, the weight warning;
* the oracle's own reference build, when present (pins the fixtures).
"""
import hashlib
import json
import os
import sys
import warnings

import numpy as np
import pytest

import oracle as O
from paper_2509_18612_b200 import liftcut as lc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from make_parse_golden import random_gset  # noqa: E402

GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "parse_cases.json")))
CASES = GOLD["cases"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(fn, text):
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        try:
            g = fn(text)
        except lc.ParseError as e:
            return {"status": 6, "message": str(e)}, w
        except lc.ValidationError as e:
            return {"status": 1, "message": str(e)}, w
    off = np.asarray(g.offsets, dtype=np.int64)
    adj = np.asarray(g.adjacency, dtype=np.uint32)[: 2 * g.edge_count()]
    return {"status": 0, "n": g.node_count(), "m": g.edge_count(), "off_sha": sha(off), "adj_sha": sha(adj)}, w


def check(got, want):
    assert got["status"] == want["status"], (got, want)
    if want["status"]:
        assert got["message"] == want["message"]
    else:
        for k in ("n", "m", "off_sha", "adj_sha"):
            assert got[k] == want[k], k


@pytest.mark.parametrize("name", sorted(CASES))
def test_host_parse_matches_reference(name):
    got, w = outcome(lc.parse_edge_list, CASES[name]["text"])
    check(got, CASES[name])
    if CASES[name]["status"] == 0:
        assert bool(w) == ("weights" in name)


@pytest.mark.parametrize("name", sorted(CASES))
def test_fast_file_reader_matches_reference(tmp_path, name):
    p = tmp_path / "g.txt"
    p.write_bytes(CASES[name]["text"].encode())
    got, _ = outcome(lambda _: lc.load_graph_file(str(p)), None)
    check(got, CASES[name])


@pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_pinned_by_reference_build(name):
    c = CASES[name]
    try:
        rg = O.RefGraph.parse(c["text"].encode())
    except O.OracleError as e:
        assert e.status == c["status"] and str(e).split(": ", 1)[1] == c["message"]
        return
    assert c["status"] == 0 and (rg.n, rg.m) == (c["n"], c["m"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_device_parse_matches_reference(name):
    got, w = outcome(lc.parse_edge_list_device, CASES[name]["text"])
    check(got, CASES[name])
    if CASES[name]["status"] == 0:
        assert bool(w) == ("weights" in name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD["random"]))
def test_device_parse_random_gset(name):
    r = GOLD["random"][name]
    text = random_gset(r["n"], r["lines"], r["seed"], r["weights"])
    got, w = outcome(lc.parse_edge_list_device, text)
    check(got, r)
    assert bool(w) == r["weights"]
    host, _ = outcome(lc.parse_edge_list, text.decode())
    check(host, r)


@pytest.mark.gpu
def test_device_parse_large_file_equals_device_ingest(tmp_path):
    """A 2M-edge Gset file (config-4 style ER) through load_graph_file_device equals the
    device edge-list ingest of the same edges; the handle is kept for the solve."""
    rng = np.random.default_rng(5)
    n, m = 400_000, 2_000_000
    u = rng.integers(0, n, m)
    v = rng.integers(0, n - 1, m)
    v = np.where(v >= u, v + 1, v)
    p = tmp_path / "big.txt"
    body = np.char.add(np.char.add((u + 1).astype(str), " "), (v + 1).astype(str))
    p.write_text(f"{n} {m}\n" + "\n".join(body.tolist()) + "\n")
    g = lc.load_graph_file_device(str(p))
    ref = lc.Graph.from_edges_device(n, np.stack([u, v], 1))
    assert g.node_count() == n and g.edge_count() == ref.edge_count()
    assert np.array_equal(g.offsets, ref.offsets) and np.array_equal(g.adjacency, ref.adjacency)
    s = lc.DenseState(n, 1, 4)
    s.values[:] = rng.uniform(-0.1, 0.1, 4 * n)
    lc.ascend(g, s, lc.AscentParams(0.05, 3, 0.9), precision=lc.LCB_FP64)
