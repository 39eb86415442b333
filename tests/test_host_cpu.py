"""CPU-only checks of the host side: the C ABI library loads and exports every
symbol include/liftcut_b200.h declares (no GPU calls), struct layouts agree with
the C compiler, and the host logic (CSR build, ER generator, RngStream, Gset
parsing, key packing, config validation) matches the oracle / reference."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

import oracle as O
from paper_2509_18612_b200 import _abi
from paper_2509_18612_b200 import liftcut as lc
from paper_2509_18612_b200.dist import pack_key, unpack_key

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "liftcut_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lcb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_abi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(syms) == set(_abi.SIGNATURES), set(syms) ^ set(_abi.SIGNATURES)
    assert _abi.lib().lcb_abi_version() == 3


def test_struct_layouts_match_the_c_header():
    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "liftcut_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(lcb_config), sizeof(lcb_outcome), sizeof(lcb_batch_trace),
         sizeof(lcb_phase_trace), sizeof(lcb_search_trace), sizeof(lcb_run_opts));
  printf("%zu %zu %zu\n", offsetof(lcb_config, deco_carry), offsetof(lcb_config, init_seed), offsetof(lcb_run_opts, kernel_stats));
  return 0;
}"""
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "t.c"), os.path.join(d, "t")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    want = [C.sizeof(_abi.Config), C.sizeof(_abi.Outcome), C.sizeof(_abi.BatchTrace), C.sizeof(_abi.PhaseTrace),
            C.sizeof(_abi.SearchTrace), C.sizeof(_abi.RunOpts), _abi.Config.deco_carry.offset,
            _abi.Config.init_seed.offset, _abi.RunOpts.kernel_stats.offset]
    assert [int(x) for x in out] == want
    assert C.sizeof(O.Config) == C.sizeof(_abi.Config)  # oracle shares the layout


def test_library_fails_loudly_without_a_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = lc.Graph(2, [(0, 1)])
    with pytest.raises(lc.Error):
        g.handle()


@pytest.mark.parametrize("seed", range(5))
def test_graph_construction_matches_reference_ctor(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 60))
    m = int(rng.integers(0, 3 * n))
    e = rng.integers(0, n, (m, 2))
    e = e[e[:, 0] != e[:, 1]]
    e = np.concatenate([e, e[: len(e) // 3, ::-1]])  # duplicates, reversed
    g = lc.Graph(n, e)
    c = O.csr_from_edges(n, e[:, 0], e[:, 1])
    assert np.array_equal(g.offsets, c.off) and np.array_equal(g.adjacency, c.adj)
    if O.ref is not None and len(e):
        r = O.RefGraph.from_edges(n, e[:, 0], e[:, 1]).csr()
        assert np.array_equal(r.off, c.off) and np.array_equal(r.adj, c.adj)
    st = g.degree_stats()
    mean, var, sd = C.c_double(), C.c_double(), C.c_double()
    O.orc.orc_degree_stats(n, O._ptr(c.off), C.byref(mean), C.byref(var), C.byref(sd))
    assert (st.mean, st.variance, st.std_dev) == (mean.value, var.value, sd.value)


def test_graph_validation_errors():
    with pytest.raises(lc.ValidationError):
        lc.Graph(3, [(0, 0)])
    with pytest.raises(lc.ValidationError):
        lc.Graph(3, [(0, 3)])
    with pytest.raises(lc.ValidationError):
        lc.Graph(0, [])


@pytest.mark.parametrize("n,p,seed", [(1, 0.5, 0), (30, 0.0, 1), (30, 1.0, 2), (200, 0.05, 3), (800, 0.015, 0)])
def test_generate_er_matches_reference_stream(n, p, seed):
    g = lc.generate_er(n, p, seed)
    c = O.generate_er(n, p, seed)
    assert np.array_equal(g.offsets, c.off) and np.array_equal(g.adjacency, c.adj)


def test_rng_stream_matches_oracle():
    for key in (0, 1, 2**64 - 1, 123456789):
        s = lc.RngStream(key)
        assert s.split([0x6261, 7]).key() == O.split(key, 0x6261, 7)
        for ctr in (0, 1, 99, 2**40):
            assert s.at(ctr) == O.orc.orc_at(key, ctr)
        t = lc.RngStream(key)
        for k in range(5):
            assert t.next_normal() == O.orc.orc_normal_at(key, k)


def test_parse_edge_list_semantics():
    g = lc.parse_edge_list("% comment\n3 3\n1 2\n2 3 5.0\n1 3\n")
    assert g.edge_count() == 3
    with pytest.raises(lc.ParseError, match="line 2"):
        lc.parse_edge_list("2 1\n1 x\n")
    with pytest.raises(lc.ValidationError):
        lc.parse_edge_list("2 1\n1 1\n")
    with pytest.raises(lc.ParseError):
        lc.parse_edge_list("3 1\n1 4\n")
    with pytest.raises(lc.ParseError):
        lc.parse_edge_list("# nothing\n")
    with tempfile.NamedTemporaryFile("w", suffix=".gset", delete=False) as f:
        f.write(lc.serialize_edge_list(lc.generate_er(50, 0.1, 4)))
    h = lc.load_graph_file(f.name)
    assert np.array_equal(h.adjacency, lc.generate_er(50, 0.1, 4).adjacency)
    os.unlink(f.name)


def test_packed_key_orders_first_max():
    assert unpack_key(pack_key(12, 5)) == (12, 5)
    # larger cut wins; on equal cuts the smaller member wins (solver.cpp:132-134)
    assert pack_key(13, 900) > pack_key(12, 0)
    assert pack_key(12, 3) > pack_key(12, 4)


def test_solver_config_validation():
    bad = [dict(batch_size=0), dict(num_batches=0), dict(time_budget_s=0.0), dict(search_refresh=-1),
           dict(deco_alternations=0)]
    for kw in bad:
        with pytest.raises(lc.ValidationError):
            lc.SolverConfig(**kw).validate()
    with pytest.raises(lc.ValidationError):
        lc.SolverConfig(init=lc.InitConfig(beta=1.0)).validate()
    with pytest.raises(lc.ValidationError):
        lc.SolverConfig(algorithm=lc.Algorithm.pLUCO, lift_dim=1).validate()
    with pytest.raises(lc.ValidationError):
        lc.AscentParams(momentum=1.0).validate()
    assert lc.algorithm_from_string("pQUCO") == lc.Algorithm.pQUCO
    with pytest.raises(lc.ValidationError):
        lc.algorithm_from_string("quco")


def test_presets_mirror_reference_table():
    cfg = lc.SolverConfig(algorithm=lc.Algorithm.pDECO)
    lc.apply_manual_preset(cfg, "gset-manual")
    assert (cfg.ascent.alpha, cfg.ascent.iterations) == (0.012, 80000)
    assert (cfg.lifted_ascent.alpha, cfg.lifted_ascent.iterations) == (0.001, 2000)
    with pytest.raises(lc.ValidationError):
        lc.apply_manual_preset(cfg, "nope")


def test_graph_constructor_first_offending_edge_decides():
    """graph.cpp:17-25 checks each edge in order, range before self-loop."""
    from paper_2509_18612_b200 import liftcut as lc
    with pytest.raises(lc.ValidationError, match="self-loop at node 2"):
        lc.Graph(5, [[0, 1], [2, 2], [1, 9]])
    with pytest.raises(lc.ValidationError, match=r"out of range: \(1, 9\)"):
        lc.Graph(5, [[0, 1], [1, 9], [2, 2]])


def test_every_documented_option_is_registered():
    """The kernel-selection knobs the header documents (lcb_set_option) exist, keep their
    documented defaults unless the LCB_<NAME> environment overrides them, round-trip
    through lc.options, and an unknown name is a ValidationError (no CUDA call)."""
    text = open(HEADER).read()
    block = text[text.index("Kernel-selection knobs"):text.index("int lcb_set_option")]
    names = re.findall(r'"([a-z_0-9]+)"', block)
    assert {"resident", "stream", "dense", "xcode", "dense_cut"} <= set(names)
    defaults = {"stream": 1, "xcode": 1, "dense_cut": 1, "dense": -1, "resident": -1}
    for k in names:
        v = lc.get_option(k)
        if k in defaults and f"LCB_{k.upper()}" not in os.environ:
            assert v == defaults[k], (k, v)
        with lc.options(**{k: 0}):
            assert lc.get_option(k) == 0
        assert lc.get_option(k) == v
    with pytest.raises(lc.ValidationError, match="unknown option"):
        lc.set_option("no_such_knob", 1)
