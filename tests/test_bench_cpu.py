"""bench.py host logic on CPU: the graph generators both arms share and the reference
arm's independence from the B200 package."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


@pytest.mark.parametrize("n,p,seed", [(2000, 0.01, 0), (20000, 0.0007, 3), (3000, 0.2, 1)])
def test_fast_gnp_edges_equal_networkx(n, p, seed):
    import networkx as nx

    G = nx.fast_gnp_random_graph(n, p, seed=seed)
    want = np.array(sorted((max(a, b), min(a, b)) for a, b in G.edges()), dtype=np.int64).reshape(-1, 2)
    v, w = bench.fast_gnp_edges(n, p, seed)
    got = np.array(sorted(zip(v.tolist(), w.tolist())), dtype=np.int64).reshape(-1, 2)
    assert np.array_equal(got, want)


def test_config4_graph_matches_survey_edge_count():
    v, w = bench.fast_gnp_edges(1_000_000, 10.0 / 999_999, 0)
    assert len(v) == 4_999_707  # networkx fast_gnp(1M, 10/(n-1), seed 0)
    assert (w < v).all()


def test_config_dict_is_arm_independent():
    for name in bench.WORKLOADS:
        a = bench.config_dict(name, 1, "fp32")
        assert a["config_id"] == name and a["global_batch"] == a["members_per_gpu"]
        assert bench.config_dict(name, 4, "fp32")["global_batch"] == 4 * a["members_per_gpu"]
    f = bench.solver_fields("c2")
    assert bench.expected_updates(f, 10_000) == 92_160_000_000


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libliftcut_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_runs_without_the_product():
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--config','c1','--steps','1',"
            "'--warmup','0']\n"
            "import bench; bench.ref_sample=lambda name: (50, 2)\n"
            "rc=bench.main()\n"
            "assert 'paper_2509_18612_b200' not in sys.modules, 'reference arm imported the product'\n"
            "sys.exit(rc)\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["config"] == bench.config_dict("c1", 1, "fp32")
    assert line["cpu_baseline"]["kind"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
