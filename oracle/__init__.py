"""TEST INFRASTRUCTURE ONLY — ctypes face of the CPU oracle.

Two CPU implementations of the liftcut hot path live behind this module:

* ``orc``  — ``liblc_oracle.so``, the plain-C restatement in ``lc_oracle.c``
  (each function cites the reference file:line it restates);
* ``ref``  — ``_ref/libliftcut_ref.so``, the UNMODIFIED reference library
  compiled from ``/root/reference/proj/src`` by ``oracle/Makefile`` with the
  thin ``ref_shim.cpp`` C face.  Present only where it was built (it travels to
  the GPU box as a prebuilt .so; the sources do not).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package.  The product (``paper_2509_18612_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liblc_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libliftcut_ref.so")

P = C.c_void_p
i64, u64, u32, i32, f64 = C.c_int64, C.c_uint64, C.c_uint32, C.c_int32, C.c_double


class Config(C.Structure):
    """Mirror of ``orc_config`` / ``lcb_config`` (one layout for both)."""

    _fields_ = [
        ("algorithm", i32), ("lift_dim", i32), ("batch_size", i64), ("num_batches", i64),
        ("alpha", f64), ("iterations", i64), ("momentum", f64), ("early_exit", i32),
        ("has_lifted_ascent", i32), ("l_alpha", f64), ("l_iterations", i64),
        ("l_momentum", f64), ("l_early_exit", i32), ("init_method", i32), ("beta", f64),
        ("eta", f64), ("init_scale", f64), ("init_seed", u64), ("resample_idi", i32),
        ("scale_noise", i32), ("time_budget_s", f64), ("has_search", i32),
        ("population_size", i32), ("t_lower", i64), ("t_upper", i64), ("e_lower", f64),
        ("e_upper", f64), ("rounds", i32), ("search_refresh", i32),
        ("deco_alternations", i32), ("deco_carry", i32),
    ]


class BatchTrace(C.Structure):
    _fields_ = [("serial", i64), ("kind", i32), ("pad_", i32), ("alpha", f64),
                ("iterations", i64), ("batch_best", i64), ("best_so_far", i64)]


class PhaseTrace(C.Structure):
    _fields_ = [("phase", i32), ("kind", i32), ("best_after", i64)]


class SearchTrace(C.Structure):
    _fields_ = [("round", i32), ("pad_", i32), ("exponent", f64), ("iterations", i64),
                ("fitness", f64)]


class Outcome(C.Structure):
    _fields_ = [("cut_value", i64), ("batch_index", i64), ("member_index", i64),
                ("batches_run", i64), ("n_batch_trace", i64), ("n_phase_trace", i64),
                ("n_search_trace", i64), ("init_s", f64), ("ascent_s", f64),
                ("rounding_s", f64), ("search_s", f64), ("wall_s", f64)]


def default_config(**kw) -> Config:
    """SolverConfig defaults (solver.hpp:26-41, ascent.hpp:12-19, init.hpp:15-26,
    evo_search.hpp:16-23)."""
    c = Config(algorithm=0, lift_dim=2, batch_size=64, num_batches=3, alpha=0.05,
               iterations=500, momentum=0.9, early_exit=1, has_lifted_ascent=0,
               l_alpha=0.05, l_iterations=500, l_momentum=0.9, l_early_exit=1,
               init_method=1, beta=0.2, eta=0.8, init_scale=1e4, init_seed=0,
               resample_idi=1, scale_noise=1, time_budget_s=0.0, has_search=0,
               population_size=6, t_lower=3000, t_upper=10000, e_lower=-4.0,
               e_upper=-1.0, rounds=5, search_refresh=0, deco_alternations=2, deco_carry=0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def _ptr(a):
    return a.ctypes.data_as(P) if a is not None else None


def _load_orc():
    if not os.path.exists(ORC_PATH):
        raise RuntimeError(f"oracle not built: run `make -C {HERE} oracle`")
    L = C.CDLL(ORC_PATH)
    sig = {
        "orc_mix64": (u64, [u64]), "orc_combine": (u64, [u64, u64]),
        "orc_split": (u64, [u64, P, C.c_int]), "orc_at": (u64, [u64, u64]),
        "orc_unit": (f64, [u64]), "orc_normal_at": (f64, [u64, u64]),
        "orc_csr_build": (i64, [u32, P, P, i64, P, P]),
        "orc_laplacian": (None, [u32, P, P, P, P]),
        "orc_degree_stats": (None, [u32, P, P, P, P]),
        "orc_generate_er": (i64, [u32, f64, u64, P, P, i64]),
        "orc_ascend": (C.c_int, [u32, P, P, P, C.c_int, i64, f64, i64, f64, C.c_int, P, P, P]),
        "orc_cut_value": (i64, [u32, P, P, P]),
        "orc_round_unlifted": (None, [i64, P, P]),
        "orc_round_lifted": (None, [i64, C.c_int, P, P]),
        "orc_project_box": (None, [P, i64]),
        "orc_dui_init": (C.c_int, [u32, P, u64, P]),
        "orc_idi_init": (None, [u32, P, P, f64, u64, P]),
        "orc_gaussian_batch": (None, [P, i64, C.c_int, f64, i64, u64, P]),
        "orc_gaussian_members": (None, [P, i64, C.c_int, f64, i64, i64, u64, P]),
        "orc_lifted_init_mean": (None, [u32, P, P, C.c_int, f64, C.c_int, u64, P]),
        "orc_solve": (C.c_int, [u32, P, P, P, u64, C.c_int, P, P, P, i64, P, i64, P, i64]),
        "orc_sample_population": (None, [i64, i64, f64, f64, C.c_int, u64, P, P, P]),
        "orc_perturb_exponent": (f64, [f64, u64, P]),
        "orc_perturb_iterations": (i64, [i64, u64, P]),
        "orc_brute_force_maxcut": (i64, [u32, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


def _load_ref():
    if not os.path.exists(REF_PATH):
        return None
    L = C.CDLL(REF_PATH)
    sig = {
        "ref_last_error": (C.c_char_p, []),
        "ref_graph_new": (C.c_int, [u32, P, P, i64, C.POINTER(P)]),
        "ref_graph_load": (C.c_int, [C.c_char_p, C.POINTER(P)]),
        "ref_graph_parse": (C.c_int, [C.c_char_p, i64, C.POINTER(P)]),
        "ref_graph_er": (C.c_int, [u32, f64, u64, C.POINTER(P)]),
        "ref_graph_free": (None, [P]),
        "ref_graph_shape": (None, [P, P, P, P]),
        "ref_graph_csr": (None, [P, P, P]),
        "ref_laplacian": (C.c_int, [P, P, P]),
        "ref_degree_stats": (None, [P, P, P, P]),
        "ref_ascend": (C.c_int, [P, P, i64, C.c_int, i64, f64, i64, f64, C.c_int, C.c_uint, P]),
        "ref_cut_value": (i64, [P, P]),
        "ref_round_unlifted": (None, [P, i64, P]),
        "ref_round_lifted": (None, [P, i64, C.c_int, i64, i64, P]),
        "ref_dui_init": (C.c_int, [P, u64, P]),
        "ref_idi_init": (None, [P, f64, u64, P]),
        "ref_gaussian_batch": (C.c_int, [P, i64, C.c_int, f64, i64, u64, C.c_uint, P]),
        "ref_lifted_init_mean": (None, [P, C.c_int, f64, C.c_int, u64, P]),
        "ref_split": (u64, [u64, P, C.c_int]),
        "ref_normal": (f64, [u64, u64]),
        "ref_solve": (C.c_int, [P, P, u64, C.c_int, C.c_uint, P, P, P, i64, P, i64, P, i64]),
        "ref_brute_force": (i64, [P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


orc = _load_orc()
ref = _load_ref()


class OracleError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"status {status}: {msg}")
        self.status = status


# --------------------------------------------------------------------------
# graph helpers (pure host arrays)
# --------------------------------------------------------------------------
@dataclass
class CSR:
    n: int
    off: np.ndarray  # int64[n+1]
    adj: np.ndarray  # uint32[2m]

    @property
    def m(self) -> int:
        return int(self.off[-1]) // 2

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.off)

    def edges(self):
        rows = np.repeat(np.arange(self.n, dtype=np.uint32), self.degrees)
        keep = rows < self.adj
        return rows[keep], self.adj[keep]


def csr_from_edges(n: int, eu, ev) -> CSR:
    eu = np.ascontiguousarray(eu, dtype=np.uint32)
    ev = np.ascontiguousarray(ev, dtype=np.uint32)
    off = np.zeros(n + 1, dtype=np.int64)
    adj = np.zeros(max(2 * len(eu), 1), dtype=np.uint32)
    m = orc.orc_csr_build(n, _ptr(eu), _ptr(ev), len(eu), _ptr(off), _ptr(adj))
    if m < 0:
        raise OracleError(1, "bad edge list")
    return CSR(n, off, adj[: 2 * m].copy())


def generate_er(n: int, p: float, seed: int) -> CSR:
    cap = int(p * n * (n - 1) / 2 * 1.1) + 64
    eu = np.zeros(cap, dtype=np.uint32)
    ev = np.zeros(cap, dtype=np.uint32)
    m = orc.orc_generate_er(n, p, seed, _ptr(eu), _ptr(ev), cap)
    if m < 0:
        raise OracleError(5, "edge capacity")
    return csr_from_edges(n, eu[:m], ev[:m])


# --------------------------------------------------------------------------
# oracle entry points (restated algorithm)
# --------------------------------------------------------------------------
def split(key: int, *path: int) -> int:
    arr = np.array(path, dtype=np.uint64)
    return int(orc.orc_split(key, _ptr(arr), len(path)))


def laplacian(g: CSR, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    orc.orc_laplacian(g.n, _ptr(g.off), _ptr(g.adj), _ptr(x), _ptr(y))
    return y


def ascend(g: CSR, values, l: int, B: int, alpha=0.05, T=500, mu=0.9, early_exit=True,
           trace=False):
    """In-place on a copy; returns (values, trace_or_None).  Raises OracleError(3)."""
    v = np.array(values, dtype=np.float64, copy=True).reshape(-1)
    tr = np.zeros((T, B), dtype=np.float64) if trace else None
    ei, ej = C.c_int64(-1), C.c_int64(-1)
    st = orc.orc_ascend(g.n, _ptr(g.off), _ptr(g.adj), _ptr(v), l, B, alpha, T, mu,
                        int(early_exit), _ptr(tr), C.byref(ei), C.byref(ej))
    if st != 0:
        e = OracleError(st, f"iteration {ei.value}, member {ej.value}")
        e.iteration, e.member = ei.value, ej.value
        raise e
    return v, tr


def cut_value(g: CSR, z) -> int:
    z = np.ascontiguousarray(z, dtype=np.uint8)
    r = orc.orc_cut_value(g.n, _ptr(g.off), _ptr(g.adj), _ptr(z))
    if r < 0:
        raise OracleError(1, "cut_value: assignment entries must be 0 or 1")
    return int(r)


def round_unlifted(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    z = np.empty(len(x), dtype=np.uint8)
    orc.orc_round_unlifted(len(x), _ptr(x), _ptr(z))
    return z


def round_lifted(member_values, n: int, l: int):
    mv = np.ascontiguousarray(member_values, dtype=np.float64)
    z = np.empty(n, dtype=np.uint8)
    orc.orc_round_lifted(n, l, _ptr(mv), _ptr(z))
    return z


def dui_init(g: CSR, key: int):
    x = np.empty(g.n, dtype=np.float64)
    if orc.orc_dui_init(g.n, _ptr(g.off), key, _ptr(x)) != 0:
        raise OracleError(1, "dui_init: graph has no edges")
    return x


def idi_init(g: CSR, beta: float, key: int):
    x = np.empty(g.n, dtype=np.float64)
    orc.orc_idi_init(g.n, _ptr(g.off), _ptr(g.adj), beta, key, _ptr(x))
    return x


def gaussian_batch(mean, n: int, l: int, eta: float, B: int, key: int):
    mean = np.ascontiguousarray(mean, dtype=np.float64)
    out = np.empty(B * l * n, dtype=np.float64)
    orc.orc_gaussian_batch(_ptr(mean), n, l, eta, B, key, _ptr(out))
    return out


def gaussian_members(mean, n: int, l: int, eta: float, first: int, count: int, key: int):
    mean = np.ascontiguousarray(mean, dtype=np.float64)
    out = np.empty(count * l * n, dtype=np.float64)
    orc.orc_gaussian_members(_ptr(mean), n, l, eta, first, count, key, _ptr(out))
    return out


def lifted_init_mean(g: CSR, method: int, beta: float, l: int, key: int):
    out = np.empty(g.n * l, dtype=np.float64)
    orc.orc_lifted_init_mean(g.n, _ptr(g.off), _ptr(g.adj), method, beta, l, key, _ptr(out))
    return out


@dataclass
class SolveResult:
    cut_value: int
    batch_index: int
    member_index: int
    batches_run: int
    assignment: np.ndarray
    batch_trace: list
    phase_trace: list
    search_trace: list
    stage_times: dict


def _collect(out, z, bt, pt, st):
    nb, npt, ns = out.n_batch_trace, out.n_phase_trace, out.n_search_trace
    return SolveResult(
        out.cut_value, out.batch_index, out.member_index, out.batches_run, z,
        [(e.serial, e.kind, e.alpha, e.iterations, e.batch_best, e.best_so_far)
         for e in bt[: min(nb, len(bt))]],
        [(e.phase, e.kind, e.best_after) for e in pt[: min(npt, len(pt))]],
        [(e.round, e.exponent, e.iterations, e.fitness) for e in st[: min(ns, len(st))]],
        dict(init_s=out.init_s, ascent_s=out.ascent_s, rounding_s=out.rounding_s,
             search_s=out.search_s, wall_s=out.wall_s),
    )


def solve(g: CSR, cfg: Config, seed: int, per_component=False, cap=4096) -> SolveResult:
    out = Outcome()
    z = np.zeros(g.n, dtype=np.uint8)
    bt, pt, st = (BatchTrace * cap)(), (PhaseTrace * cap)(), (SearchTrace * cap)()
    s = orc.orc_solve(g.n, _ptr(g.off), _ptr(g.adj), C.byref(cfg), seed, int(per_component),
                      C.byref(out), _ptr(z), bt, cap, pt, cap, st, cap)
    if s != 0:
        raise OracleError(s, "oracle solve failed")
    return _collect(out, z, bt, pt, st)


def brute_force_maxcut(g: CSR):
    w = np.zeros(g.n, dtype=np.uint8)
    cnt = C.c_int64(0)
    best = orc.orc_brute_force_maxcut(g.n, _ptr(g.off), _ptr(g.adj), _ptr(w), C.byref(cnt))
    return int(best), w, int(cnt.value)


# --------------------------------------------------------------------------
# the compiled reference itself (oracle/_ref), same calling conventions
# --------------------------------------------------------------------------
class RefGraph:
    """Reference ``liftcut::Graph`` built by the reference constructor."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)
        n, m, md = C.c_uint32(), C.c_int64(), C.c_int64()
        ref.ref_graph_shape(self.h, C.byref(n), C.byref(m), C.byref(md))
        self.n, self.m, self.max_degree = n.value, m.value, md.value

    @classmethod
    def from_edges(cls, n, eu, ev):
        eu = np.ascontiguousarray(eu, dtype=np.uint32)
        ev = np.ascontiguousarray(ev, dtype=np.uint32)
        h = C.c_void_p()
        s = ref.ref_graph_new(n, _ptr(eu), _ptr(ev), len(eu), C.byref(h))
        if s != 0:
            raise OracleError(s, ref.ref_last_error().decode())
        return cls(h.value)

    @classmethod
    def from_csr(cls, g: CSR):
        eu, ev = g.edges()
        return cls.from_edges(g.n, eu, ev)

    @classmethod
    def parse(cls, text: bytes):
        """The reference's parse_edge_list(text); OracleError(status 6 = ParseError, 1 =
        ValidationError) with the reference's message."""
        h = C.c_void_p()
        s = ref.ref_graph_parse(text, len(text), C.byref(h))
        if s != 0:
            raise OracleError(s, ref.ref_last_error().decode())
        return cls(h.value)

    @classmethod
    def er(cls, n, p, seed):
        h = C.c_void_p()
        s = ref.ref_graph_er(n, p, seed, C.byref(h))
        if s != 0:
            raise OracleError(s, ref.ref_last_error().decode())
        return cls(h.value)

    @classmethod
    def load(cls, path):
        h = C.c_void_p()
        s = ref.ref_graph_load(path.encode(), C.byref(h))
        if s != 0:
            raise OracleError(s, ref.ref_last_error().decode())
        return cls(h.value)

    def csr(self) -> CSR:
        off = np.zeros(self.n + 1, dtype=np.int64)
        adj = np.zeros(max(2 * self.m, 1), dtype=np.uint32)
        ref.ref_graph_csr(self.h, _ptr(off), _ptr(adj))
        return CSR(self.n, off, adj[: 2 * self.m].copy())

    def __del__(self):
        if ref is not None and getattr(self, "h", None):
            ref.ref_graph_free(self.h)
            self.h = None


def ref_brute_force_maxcut(rg: RefGraph):
    """The reference ``brute_force_maxcut`` (oracle.cpp:50-99) -> (optimum, witness, count)."""
    w = np.zeros(rg.n, dtype=np.uint8)
    cnt = C.c_int64(0)
    best = ref.ref_brute_force(rg.h, _ptr(w), C.byref(cnt))
    if best < 0:
        raise OracleError(1, ref.ref_last_error().decode())
    return int(best), w, int(cnt.value)


def ref_ascend(rg: RefGraph, values, l, B, alpha=0.05, T=500, mu=0.9, early_exit=True,
               workers=1, trace=False):
    v = np.array(values, dtype=np.float64, copy=True).reshape(-1)
    tr = np.zeros((T, B), dtype=np.float64) if trace else None
    s = ref.ref_ascend(rg.h, _ptr(v), rg.n, l, B, alpha, T, mu, int(early_exit), workers,
                       _ptr(tr))
    if s != 0:
        raise OracleError(s, ref.ref_last_error().decode())
    return v, tr


def ref_solve(rg: RefGraph, cfg: Config, seed: int, per_component=False, workers=1,
              cap=4096) -> SolveResult:
    out = Outcome()
    z = np.zeros(rg.n, dtype=np.uint8)
    bt, pt, st = (BatchTrace * cap)(), (PhaseTrace * cap)(), (SearchTrace * cap)()
    s = ref.ref_solve(rg.h, C.byref(cfg), seed, int(per_component), workers, C.byref(out),
                      _ptr(z), bt, cap, pt, cap, st, cap)
    if s != 0:
        raise OracleError(s, ref.ref_last_error().decode())
    return _collect(out, z, bt, pt, st)
