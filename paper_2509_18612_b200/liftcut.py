"""Host-side mirror of the reference solver API (``/root/reference/proj/include/liftcut``).

Same names, argument meaning and error behaviour as the reference's C++ API, so a
caller (or a test) written against ``liftcut::`` reads the same here.  Every
numeric operation on the hot path runs in ``libliftcut_b200.so`` on the GPU; the
host keeps only what the reference keeps host-side and the north star leaves
there: graph loading / CSR construction, stream-key derivation (seeding), and the
solver's control flow (inside the C++ runtime).

Precision: ``LCB_FP64`` (default) reproduces the reference bit for bit;
``LCB_FP32`` is the fast path.  Select per call (``precision=``) or process-wide
with ``LIFTCUT_PRECISION=fp32``.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
import re
import warnings
from dataclasses import dataclass, field, replace
from typing import Callable, Optional

import numpy as np

from . import _abi
from ._abi import LCB_FP32, LCB_FP64

NodeId = int


# ---------------------------------------------------------------------------
# errors.hpp:9-31
# ---------------------------------------------------------------------------
class Error(RuntimeError):
    pass


class ParseError(Error):
    pass


class ValidationError(Error):
    pass


class ShapeError(Error):
    pass


class NumericError(Error):
    pass


def _raise(status: int):
    msg = _abi.last_error()
    if status == _abi.LCB_VALIDATION:
        raise ValidationError(msg)
    if status == _abi.LCB_SHAPE:
        raise ShapeError(msg)
    if status == _abi.LCB_NUMERIC:
        raise NumericError(msg)
    if status == _abi.LCB_PARSE:
        raise ParseError(msg)
    raise Error(msg or f"liftcut_b200 status {status}")


def _check(status: int):
    if status != _abi.LCB_OK:
        _raise(status)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def default_precision() -> int:
    p = os.environ.get("LIFTCUT_PRECISION", "fp64").lower()
    return LCB_FP32 if p in ("fp32", "f32", "float", "fast") else LCB_FP64


def default_device() -> int:
    return int(os.environ.get("LIFTCUT_DEVICE", "0"))


# ---------------------------------------------------------------------------
# RngStream (rng.hpp:27-79) — host seeding only
# ---------------------------------------------------------------------------
_M64 = (1 << 64) - 1


def _mix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _combine(key: int, word: int) -> int:
    return _mix64(key ^ ((word + 0x9E3779B97F4A7C15 + ((key << 6) & _M64) + (key >> 2)) & _M64))


class RngStream:
    def __init__(self, key: int):
        self._key = key & _M64
        self._counter = 0

    def split(self, path) -> "RngStream":
        k = self._key
        for w in path:
            k = _combine(k, int(w) & _M64)
        return RngStream(k)

    def key(self) -> int:
        return self._key

    def at(self, counter: int) -> int:
        return _mix64(self._key ^ ((counter * 0xD6E8FEB86659FD93) & _M64))

    @staticmethod
    def _to_unit(bits: int) -> float:
        return float(bits >> 11) * 2.0 ** -53

    def unit_at(self, counter: int) -> float:
        return self._to_unit(self.at(counter))

    def next_u64(self) -> int:
        v = self.at(self._counter)
        self._counter += 1
        return v

    def next_unit(self) -> float:
        return self._to_unit(self.next_u64())

    def next_uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_unit()

    def next_int(self, lo: int, hi: int) -> int:
        return lo + self.next_u64() % (hi - lo + 1)

    def next_normal(self) -> float:
        u1 = self.next_unit()
        u2 = self.next_unit()
        if u1 <= 0.0:
            u1 = 2.0 ** -53
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586476925286766559 * u2)

    def next_sign(self) -> float:
        return 1.0 if (self.next_u64() & 1) else -1.0


# ---------------------------------------------------------------------------
# Graph (graph.hpp:21-58): host CSR + lazily created device handle
# ---------------------------------------------------------------------------
@dataclass
class DegreeStats:
    mean: float = 0.0
    variance: float = 0.0
    std_dev: float = 0.0


class Graph:
    """Immutable undirected simple graph in CSR form (sorted, deduplicated)."""

    def __init__(self, node_count: int, edges=(), *, _csr=None):
        if _csr is not None:
            self._n, self._off, self._adj = _csr
        else:
            if node_count == 0:
                raise ValidationError("graph must have at least one node")
            e = np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges,
                           dtype=np.int64).reshape(-1, 2)
            self._n = int(node_count)
            self._off, self._adj = self._build(self._n, e)
        self._deg = np.diff(self._off)
        self._handles = {}

    @staticmethod
    def _build(n: int, e: np.ndarray):
        # graph.cpp:15-50: validate, normalise u<v, sort, dedupe, symmetrise
        if len(e):
            # the first offending edge in input order decides, range before self-loop
            rng = ((e < 0) | (e >= n)).any(axis=1)
            loops = e[:, 0] == e[:, 1]
            bad = rng | loops
            if bad.any():
                i = int(np.argmax(bad))
                if rng[i]:
                    raise ValidationError(
                        f"edge endpoint out of range: ({e[i, 0]}, {e[i, 1]}) with n={n}")
                raise ValidationError(f"self-loop at node {int(e[i, 0])}")
            u = np.minimum(e[:, 0], e[:, 1])
            v = np.maximum(e[:, 0], e[:, 1])
            key = np.unique(u * n + v)
            u, v = key // n, key % n
        else:
            u = v = np.zeros(0, dtype=np.int64)
        rows = np.concatenate([u, v])
        cols = np.concatenate([v, u])
        order = np.lexsort((cols, rows))
        off = np.zeros(n + 1, dtype=np.int64)
        np.add.at(off, rows + 1, 1)
        np.cumsum(off, out=off)
        return off, np.ascontiguousarray(cols[order], dtype=np.uint32)

    @classmethod
    def from_edges_device(cls, node_count: int, edges, device: Optional[int] = None) -> "Graph":
        """Graph(n, edges) built on the GPU (lcb_graph_from_edges: radix sort + unique +
        symmetrise, graph.cpp:15-50); same CSR and the same errors as the constructor.
        The device handle is kept, so the first solve does not upload again."""
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        if len(e) and (e.min() < 0 or e.max() >= 2**32):
            i = int(np.argmax(((e < 0) | (e >= node_count)).any(axis=1)))
            raise ValidationError(f"edge endpoint out of range: ({e[i, 0]}, {e[i, 1]}) with n={node_count}")
        eu = np.ascontiguousarray(e[:, 0], dtype=np.uint32)
        ev = np.ascontiguousarray(e[:, 1], dtype=np.uint32)
        dev = default_device() if device is None else device
        h = C.c_void_p()
        _check(_abi.lib().lcb_graph_from_edges(int(node_count), _ptr(eu), _ptr(ev), len(e), dev, C.byref(h)))
        m = C.c_int64()
        _abi.lib().lcb_graph_info(h, None, C.byref(m), None)
        off = np.zeros(int(node_count) + 1, dtype=np.int64)
        adj = np.zeros(max(2 * m.value, 1), dtype=np.uint32)
        st = _abi.lib().lcb_graph_csr(h, _ptr(off), _ptr(adj))
        if st != 0:
            _abi.lib().lcb_graph_destroy(h)
            _check(st)
        g = cls(int(node_count), _csr=(int(node_count), off, adj[: 2 * m.value].copy()))
        g._handles[dev] = h
        return g

    @classmethod
    def from_csr(cls, n: int, offsets, adjacency) -> "Graph":
        return cls(n, _csr=(int(n), np.ascontiguousarray(offsets, dtype=np.int64),
                            np.ascontiguousarray(adjacency, dtype=np.uint32)))

    # -- reference accessors --------------------------------------------------
    def node_count(self) -> int:
        return self._n

    def edge_count(self) -> int:
        return int(self._off[-1]) // 2

    def neighbors(self, v: int) -> np.ndarray:
        return self._adj[self._off[v]:self._off[v + 1]]

    def degree(self, v: int) -> int:
        return int(self._deg[v])

    def max_degree(self) -> int:
        return int(self._deg.max()) if self._n else 0

    @property
    def offsets(self) -> np.ndarray:
        return self._off

    @property
    def adjacency(self) -> np.ndarray:
        return self._adj

    def edges(self):
        rows = np.repeat(np.arange(self._n, dtype=np.int64), self._deg)
        keep = rows < self._adj
        return list(zip(rows[keep].tolist(), self._adj[keep].tolist()))

    def degree_stats(self) -> DegreeStats:
        n = float(self._n)
        mean = 2.0 * float(self.edge_count()) / n
        acc = 0.0
        for d in self._deg.tolist():  # sequential, as graph.cpp:66-69
            t = float(d) - mean
            acc += t * t
        var = acc / n
        return DegreeStats(mean, var, math.sqrt(var))

    def connected_components(self):
        seen = np.zeros(self._n, dtype=bool)
        out = []
        for root in range(self._n):
            if seen[root]:
                continue
            comp, stack = [], [root]
            seen[root] = True
            while stack:
                v = stack.pop()
                comp.append(v)
                for u in self.neighbors(v).tolist():
                    if not seen[u]:
                        seen[u] = True
                        stack.append(u)
            out.append(sorted(comp))
        return out

    def induced_subgraph(self, nodes) -> "Graph":
        local = {int(v): i for i, v in enumerate(nodes)}
        edges = [(local[v], local[int(u)]) for v in nodes for u in self.neighbors(v).tolist()
                 if v < u and int(u) in local]
        return Graph(len(nodes), edges)

    # -- device side ----------------------------------------------------------
    def handle(self, device: Optional[int] = None):
        dev = default_device() if device is None else device
        h = self._handles.get(dev)
        if h is None:
            h = C.c_void_p()
            _check(_abi.lib().lcb_graph_create(self._n, _ptr(self._off), _ptr(self._adj), dev,
                                               C.byref(h)))
            self._handles[dev] = h
        return h

    def release(self):
        for h in self._handles.values():
            _abi.lib().lcb_graph_destroy(h)
        self._handles.clear()

    def __del__(self):
        try:
            if self._handles and _abi._lib is not None:
                self.release()
        except Exception:
            pass

    def laplacian_apply(self, x, precision: Optional[int] = None) -> np.ndarray:
        """y = Lx = Dx - Ax (graph.cpp:112-122); x may be [n] or [count, n]."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape[-1] != self._n:
            raise ShapeError(f"laplacian_apply: expected vectors of length {self._n}")
        y = np.empty_like(x)
        count = 1 if x.ndim == 1 else x.shape[0]
        _check(_abi.lib().lcb_laplacian_apply(self.handle(), _ptr(x), _ptr(y), count,
                                              default_precision() if precision is None else precision))
        return y


_LL_MAX = (1 << 63) - 1
_INT_RE = re.compile(r"[ \t\n\v\f\r]*([+-]?)([0-9]+)")
_NUM_RE = re.compile(r"[ \t\n\v\f\r]*[+-]?(?:[0-9]|\.[0-9])")


def _read_ll(s: str, pos: int):
    """istream >> long long: skip isspace, optional sign, digits; None on failure/overflow."""
    mt = _INT_RE.match(s, pos)
    if not mt:
        return None, pos
    v = int(mt.group(2))
    if (mt.group(1) == "-" and v > _LL_MAX + 1) or (mt.group(1) != "-" and v > _LL_MAX):
        return None, pos
    return (-v if mt.group(1) == "-" else v), mt.end()


def parse_edge_list(text: str) -> Graph:
    """Gset text (graph.cpp:136-172): is_comment_or_blank skips only ' ', '\t', '\r' before
    '%' / '#'; numbers follow the istream rules for long long."""
    n = m = -1
    us, vs = [], []
    saw_weights = False
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # std::getline: a trailing newline ends the last line
    for line_no, line in enumerate(lines, 1):
        s = line.lstrip(" \t\r")
        if not s or s[0] in "%#":
            continue
        if n < 0:
            n, p = _read_ll(line, 0)
            m, p = _read_ll(line, p) if n is not None else (None, p)
            if n is None or m is None or n <= 0 or m < 0:
                raise ParseError(f'line {line_no}: expected header "n m"')
            continue
        u, p = _read_ll(line, 0)
        v, p = _read_ll(line, p) if u is not None else (None, p)
        if u is None or v is None:
            raise ParseError(f'line {line_no}: expected edge "u v [w]"')
        if _NUM_RE.match(line, p):
            saw_weights = True
        if u < 1 or u > n or v < 1 or v > n:
            raise ParseError(f"line {line_no}: node id out of range [1, {n}]")
        if u == v:
            raise ValidationError(f"line {line_no}: self-loop at node {u}")
        us.append(u - 1)
        vs.append(v - 1)
    if n < 0:
        raise ParseError('empty input: missing "n m" header')
    if saw_weights:
        warnings.warn("edge weights present in input are ignored (unweighted MaxCut)")
    return Graph(n, np.stack([np.array(us, dtype=np.int64), np.array(vs, dtype=np.int64)], 1))


def load_graph_file(path: str) -> Graph:
    """Fast Gset reader (numpy), same contract as graph.cpp:179-183 for well-formed files."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ParseError(f"cannot open graph file: {path}")
    lines = [ln for ln in text.split("\n") if ln.lstrip(" \t\r") and ln.lstrip(" \t\r")[0] not in "%#"]
    if not lines:
        raise ParseError('empty input: missing "n m" header')
    try:
        n, m = (int(t) for t in lines[0].split())
        body = np.array(" ".join(lines[1:]).split(), dtype=np.int64)
        ncol = len(lines[1].split()) if len(lines) > 1 else 2
        if ncol not in (2, 3) or body.size != ncol * (len(lines) - 1) or n <= 0 or m < 0:
            raise ValueError
        e = body.reshape(-1, ncol)[:, :2] - 1
        if len(e) and (e.min() < 0 or e.max() >= n or (e[:, 0] == e[:, 1]).any()):
            raise ValueError  # the line-by-line parser reports the reference's error
    except (ValueError, OverflowError):
        return parse_edge_list(text)
    if ncol == 3:
        warnings.warn("edge weights present in input are ignored (unweighted MaxCut)")
    return Graph(n, e)


def parse_edge_list_device(text, device: Optional[int] = None) -> Graph:
    """parse_edge_list (graph.cpp:136-172) on the GPU (lcb_graph_parse): line-parallel
    parse, then the device Graph(n, edges) build; same CSR, errors and messages as the
    reference.  A weight column warns like the reference (graph.cpp:168-169)."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    dev = default_device() if device is None else device
    h = C.c_void_p()
    w = C.c_int(0)
    _check(_abi.lib().lcb_graph_parse(data, len(data), dev, C.byref(h), C.byref(w)))
    if w.value:
        warnings.warn("edge weights present in input are ignored (unweighted MaxCut)")
    n = C.c_uint32()
    m = C.c_int64()
    _abi.lib().lcb_graph_info(h, C.byref(n), C.byref(m), None)
    off = np.zeros(int(n.value) + 1, dtype=np.int64)
    adj = np.zeros(max(2 * m.value, 1), dtype=np.uint32)
    st = _abi.lib().lcb_graph_csr(h, _ptr(off), _ptr(adj))
    if st != 0:
        _abi.lib().lcb_graph_destroy(h)
        _check(st)
    g = Graph(int(n.value), _csr=(int(n.value), off, adj[: 2 * m.value].copy()))
    g._handles[dev] = h
    return g


def load_graph_file_device(path: str, device: Optional[int] = None) -> Graph:
    """load_graph_file (graph.cpp:179-183) with the text parsed on the GPU."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise ParseError(f"cannot open graph file: {path}")
    return parse_edge_list_device(data, device)


def serialize_edge_list(g: Graph) -> str:
    out = [f"{g.node_count()} {g.edge_count()}"]
    out += [f"{u + 1} {v + 1}" for u, v in g.edges()]
    return "\n".join(out) + "\n"


def write_graph_file(g: Graph, path: str):
    with open(path, "w") as f:
        f.write(serialize_edge_list(g))


def generate_er(n: int, p: float, seed: int) -> Graph:
    """ER G(n, p) with the reference's pair stream (graph.cpp:200-213), vectorised."""
    u, v = generate_er_edges(n, p, seed)
    return Graph(n, np.stack([u, v], 1))


def generate_er_device(n: int, p: float, seed: int, device: Optional[int] = None) -> Graph:
    """generate_er with the CSR built on the GPU (lcb_graph_from_edges)."""
    u, v = generate_er_edges(n, p, seed)
    return Graph.from_edges_device(n, np.stack([u, v], 1), device)


def generate_er_edges(n: int, p: float, seed: int):
    """The edge stream of generate_er (graph.cpp:200-213): pairs u < v in row order."""
    if n < 1:
        raise ValidationError("generate_er: n must be >= 1")
    if not (0.0 <= p <= 1.0):
        raise ValidationError("generate_er: p must lie in [0, 1]")
    key = RngStream(seed).split([0x4552]).key()
    us, vs = [], []
    base = 0
    cu = np.uint64
    for u in range(n - 1):
        cnt = n - 1 - u
        idx = np.arange(base, base + cnt, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = cu(key) ^ (idx * cu(0xD6E8FEB86659FD93))
            z = z + cu(0x9E3779B97F4A7C15)
            z = (z ^ (z >> cu(30))) * cu(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> cu(27))) * cu(0x94D049BB133111EB)
            z = z ^ (z >> cu(31))
        unit = (z >> cu(11)).astype(np.float64) * 2.0 ** -53
        hit = np.nonzero(unit < p)[0]
        us.append(np.full(len(hit), u, dtype=np.int64))
        vs.append(u + 1 + hit.astype(np.int64))
        base += cnt
    if not us:
        return np.zeros(0, dtype=np.int64), np.zeros(0, dtype=np.int64)
    return np.concatenate(us), np.concatenate(vs)


# ---------------------------------------------------------------------------
# DenseState (dense_state.hpp:14-55)
# ---------------------------------------------------------------------------
class DenseState:
    def __init__(self, n: int, l: int = 1, b: int = 1):
        if n < 1 or l < 1 or b < 1:
            raise ValidationError("DenseState: n, l, B must all be >= 1")
        self.nodes, self.lift_dim, self.batch = int(n), int(l), int(b)
        self.values = np.zeros(n * l * b, dtype=np.float64)

    def column(self, member: int, col: int) -> np.ndarray:
        o = (member * self.lift_dim + col) * self.nodes
        return self.values[o:o + self.nodes]

    def member(self, j: int) -> np.ndarray:
        o = j * self.lift_dim * self.nodes
        return self.values[o:o + self.nodes * self.lift_dim]

    def same_shape(self, other: "DenseState") -> bool:
        return (self.nodes, self.lift_dim, self.batch) == (other.nodes, other.lift_dim, other.batch)

    def copy(self) -> "DenseState":
        s = DenseState(self.nodes, self.lift_dim, self.batch)
        s.values[:] = self.values
        return s


# ---------------------------------------------------------------------------
# ascent (ascent.hpp:12-34)
# ---------------------------------------------------------------------------
@dataclass
class AscentParams:
    alpha: float = 0.05
    iterations: int = 500
    momentum: float = 0.9
    early_exit: bool = True

    def validate(self):
        if not (self.alpha > 0.0):
            raise ValidationError("ascent: alpha must be > 0")
        if self.iterations < 1:
            raise ValidationError("ascent: iterations must be >= 1")
        if not (0.0 <= self.momentum < 1.0):
            raise ValidationError("ascent: momentum must lie in [0, 1)")


TraceCallback = Callable[[int, int, float], None]


def detect_fixed_point(prev: DenseState, nxt: DenseState, tol: float):
    if not prev.same_shape(nxt):
        raise ShapeError("detect_fixed_point: shape mismatch")
    d = np.abs(prev.values - nxt.values).reshape(prev.batch, -1)
    return [bool(x) for x in (d.max(axis=1) <= tol)]


def ascend(g: Graph, state: DenseState, params: AscentParams, workers: int = 1,
           trace: Optional[TraceCallback] = None, precision: Optional[int] = None):
    """Batched heavy-ball PGA, in place on ``state`` (ascent.cpp:43-96)."""
    params.validate()
    if state.nodes != g.node_count():
        raise ShapeError(f"ascend: state row dimension {state.nodes} != node count "
                         f"{g.node_count()}")
    prec = default_precision() if precision is None else precision
    tr = np.zeros((params.iterations, state.batch), dtype=np.float64) if trace else None
    ei, ej = C.c_int64(-1), C.c_int64(-1)
    st = _abi.lib().lcb_ascend(g.handle(), _ptr(state.values), state.nodes, state.lift_dim,
                               state.batch, float(params.alpha), int(params.iterations),
                               float(params.momentum), int(bool(params.early_exit)), prec,
                               _ptr(tr), C.byref(ei), C.byref(ej))
    _check(st)
    if trace:  # member-major, as the reference with workers=1
        for j in range(state.batch):
            for it in range(params.iterations):
                trace(it, j, float(tr[it, j]))


def ascend_rows(n: int, row_begin: int, row_end: int, offsets, adjacency, values, lift_dim: int, batch: int,
                params: AscentParams, comm=None, precision: Optional[int] = None, device: Optional[int] = None):
    """Row-sharded ascend (lcb_ascend_rows, north star 5): this rank holds the CSR rows
    [row_begin, row_end) (offsets from 0, global column ids) and the slice
    values [batch][lift_dim][rows] (float64, updated in place) of the DenseState; the
    ranks of `comm` (dist.Comm) partition [0, n) in rank order.  Equals ``ascend`` on the
    whole graph (fp64 bit for bit)."""
    params.validate()
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    adj = np.ascontiguousarray(adjacency, dtype=np.uint32)
    rows = row_end - row_begin
    if off.shape != (rows + 1,):
        raise ShapeError(f"ascend_rows: offsets must have {rows + 1} entries")
    if values.dtype != np.float64 or not values.flags.c_contiguous or values.size != batch * lift_dim * rows:
        raise ShapeError("ascend_rows: values must be a contiguous float64 [batch][lift_dim][rows] slice")
    prec = default_precision() if precision is None else precision
    dev = default_device() if device is None else device
    ei, ej = C.c_int64(-1), C.c_int64(-1)
    h = comm.handle if comm is not None else None
    _check(_abi.lib().lcb_ascend_rows(h, int(n), int(row_begin), int(row_end), _ptr(off), _ptr(adj), _ptr(values),
                                      int(lift_dim), int(batch), float(params.alpha), int(params.iterations),
                                      float(params.momentum), int(bool(params.early_exit)), prec, int(dev),
                                      C.byref(ei), C.byref(ej)))


# ---------------------------------------------------------------------------
# objectives (objectives.hpp)
# ---------------------------------------------------------------------------
def cut_value(g: Graph, z) -> int:
    z = np.ascontiguousarray(z, dtype=np.uint8)
    if z.shape[-1] != g.node_count():
        raise ShapeError(f"cut_value: expected length {g.node_count()}, got {z.shape[-1]}")
    out = np.zeros(1, dtype=np.int64)
    _check(_abi.lib().lcb_cut_values(g.handle(), _ptr(z), 1, _ptr(out)))
    return int(out[0])


def cut_values(g: Graph, Z) -> np.ndarray:
    """cut_value for a stack of assignments [count, n] in one launch."""
    Z = np.ascontiguousarray(Z, dtype=np.uint8)
    out = np.zeros(Z.shape[0], dtype=np.int64)
    _check(_abi.lib().lcb_cut_values(g.handle(), _ptr(Z), Z.shape[0], _ptr(out)))
    return out


def _round(values, n: int, l: int, B: int, lifted: bool) -> np.ndarray:
    v = np.ascontiguousarray(values, dtype=np.float64)
    z = np.zeros(B * n, dtype=np.uint8)
    _check(_abi.lib().lcb_round(default_device(), _ptr(v), n, l, B, int(lifted), _ptr(z)))
    return z


def round_unlifted(x) -> np.ndarray:
    """z = 1{x > 0}, strict (objectives.cpp:81-86), on the device (lcb_round)."""
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    return _round(x, len(x), 1, 1, False)


def round_lifted(state: DenseState, member: int = 0) -> np.ndarray:
    """z = 1{sum_c X[v, c] >= 0} with the row sum in column order (objectives.cpp:88-96)."""
    return _round(state.member(member), state.nodes, state.lift_dim, 1, True)


def round_cut_batch(g: Graph, state: DenseState, lifted: bool):
    """Device rounding + cut + first-max argmax of a whole batch (solver.cpp:125-138).
    Returns (cuts[B], best_member, best_cut, best_z)."""
    cuts = np.zeros(state.batch, dtype=np.int64)
    z = np.zeros(state.nodes, dtype=np.uint8)
    bm, bc = C.c_int64(), C.c_int64()
    _check(_abi.lib().lcb_round_cut_batch(g.handle(), _ptr(state.values), state.lift_dim,
                                          state.batch, int(lifted), _ptr(cuts), C.byref(bm),
                                          C.byref(bc), _ptr(z)))
    return cuts, bm.value, bc.value, z


@dataclass
class OracleResult:
    """oracle.hpp:12-16."""
    optimum: int
    witness: np.ndarray
    count_optimal: int  # z and its complement counted separately


def brute_force_maxcut(g: Graph, workers: int = 1, max_nodes: int = 0) -> OracleResult:
    """Exhaustive MaxCut (oracle.hpp:18-22) as one device Gray-code scan.  ``workers``
    is accepted for signature parity; the result never depended on it.  ``max_nodes``
    lifts the reference's n <= 26 guard (up to 40)."""
    del workers
    n = g.node_count()
    z = np.zeros(n, dtype=np.uint8)
    opt, cnt = C.c_int64(), C.c_int64()
    _check(_abi.lib().lcb_brute_force_maxcut(g.handle(), int(max_nodes), C.byref(opt), C.byref(cnt), _ptr(z)))
    return OracleResult(opt.value, z, cnt.value)


def project_box(values):
    np.clip(values, -1.0, 1.0, out=values)


def quco_objective(g: Graph, x) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    if len(x) != g.node_count():
        raise ShapeError(f"quco_objective: expected length {g.node_count()}, got {len(x)}")
    if not np.all(np.abs(x) <= 1.0 + 1e-12):
        raise ValidationError("quco_objective: entry outside [-1, 1]")
    return float(np.dot(x, g.laplacian_apply(x, precision=LCB_FP64)))


def luco_objective(g: Graph, state: DenseState, member: int = 0) -> float:
    m = state.member(member).reshape(state.lift_dim, state.nodes)
    if not np.all(np.abs(m) <= 1.0 + 1e-12):
        raise ValidationError("luco_objective: entry outside [-1, 1]")
    y = g.laplacian_apply(m, precision=LCB_FP64)
    return float(np.sum(m * y))


def is_maxcut_fixed_point_unlifted(g: Graph, x, alpha: float) -> bool:
    x = np.asarray(x, dtype=np.float64)
    if alpha <= 0.0:
        raise ValidationError("is_maxcut_fixed_point_unlifted: alpha must be > 0")
    if not np.all(np.abs(x) == 1.0) or np.all(x == x[0]):
        return False
    moved = np.clip(x + alpha * g.laplacian_apply(x, precision=LCB_FP64), -1.0, 1.0)
    return bool(np.array_equal(moved, x))


# ---------------------------------------------------------------------------
# init (init.hpp)
# ---------------------------------------------------------------------------
class InitMethod(enum.IntEnum):
    DUI = 0
    IDI = 1


def init_method_from_string(name: str) -> InitMethod:
    if name in ("dui", "DUI"):
        return InitMethod.DUI
    if name in ("idi", "IDI"):
        return InitMethod.IDI
    raise ValidationError(f"unknown init method: {name}")


@dataclass
class InitConfig:
    method: InitMethod = InitMethod.IDI
    beta: float = 0.2
    eta: float = 0.8
    init_scale: float = 10000.0
    seed: int = 0
    resample_idi: bool = True
    scale_noise: bool = True


def dui_init(g: Graph, stream: RngStream) -> np.ndarray:
    x = np.empty(g.node_count(), dtype=np.float64)
    _check(_abi.lib().lcb_dui_init(g.handle(), stream.key(), _ptr(x)))
    return x


def idi_init(g: Graph, beta: float, stream: RngStream) -> np.ndarray:
    x = np.empty(g.node_count(), dtype=np.float64)
    _check(_abi.lib().lcb_idi_init(g.handle(), float(beta), stream.key(), _ptr(x)))
    return x


def scale_down(x, init_scale: float):
    if init_scale < 1.0:
        raise ValidationError("scale_down: init_scale must be >= 1")
    x /= init_scale


def gaussian_batch(mean, nodes: int, lift_dim: int, eta: float, batch: int, stream: RngStream,
                   workers: int = 1, device: Optional[int] = None, exact: Optional[bool] = None) -> DenseState:
    """init.cpp:69-87.  exact (default in the fp64 precision mode): the reference's own host
    libm normals, bit-identical (lcb_gaussian_batch_exact); otherwise device Box-Muller
    (within a few ulp of glibc)."""
    mean = np.ascontiguousarray(mean, dtype=np.float64)
    if len(mean) != nodes * lift_dim:
        raise ShapeError(f"gaussian_batch: mean has {len(mean)} entries, expected "
                         f"{nodes * lift_dim}")
    s = DenseState(nodes, lift_dim, batch)
    if exact is None:
        exact = default_precision() == _abi.LCB_FP64
    if exact:
        _check(_abi.lib().lcb_gaussian_batch_exact(_ptr(mean), nodes, lift_dim, float(eta), batch,
                                                   stream.key(), _ptr(s.values)))
    else:
        _check(_abi.lib().lcb_gaussian_batch(default_device() if device is None else device,
                                             _ptr(mean), nodes, lift_dim, float(eta), batch,
                                             stream.key(), _ptr(s.values)))
    return s


def lifted_init_mean(g: Graph, cfg: InitConfig, lift_dim: int, stream: RngStream) -> np.ndarray:
    out = np.empty(g.node_count() * lift_dim, dtype=np.float64)
    _check(_abi.lib().lcb_lifted_init_mean(g.handle(), int(cfg.method), float(cfg.beta),
                                           lift_dim, stream.key(), _ptr(out)))
    return out


# ---------------------------------------------------------------------------
# search / solver (evo_search.hpp, solver.hpp)
# ---------------------------------------------------------------------------
@dataclass
class SearchConfig:
    t_lower: int = 3000
    t_upper: int = 10000
    e_lower: float = -4.0
    e_upper: float = -1.0
    population_size: int = 6
    rounds: int = 5


class Algorithm(enum.IntEnum):
    pQUCO = 0
    pLUCO = 1
    pDECO = 2


def algorithm_to_string(a: Algorithm) -> str:
    return {Algorithm.pQUCO: "pquco", Algorithm.pLUCO: "pluco", Algorithm.pDECO: "pdeco"}[a]


def algorithm_from_string(name: str) -> Algorithm:
    m = {"pquco": 0, "pQUCO": 0, "pluco": 1, "pLUCO": 1, "pdeco": 2, "pDECO": 2}
    if name not in m:
        raise ValidationError(f"unknown algorithm: {name}")
    return Algorithm(m[name])


class DecoCarry(enum.IntEnum):
    IncumbentColumn = 0
    Fresh = 1


@dataclass
class SolverConfig:
    algorithm: Algorithm = Algorithm.pQUCO
    batch_size: int = 64
    lift_dim: int = 2
    ascent: AscentParams = field(default_factory=AscentParams)
    lifted_ascent: Optional[AscentParams] = None
    init: InitConfig = field(default_factory=InitConfig)
    num_batches: int = 3
    time_budget_s: Optional[float] = None
    search: Optional[SearchConfig] = None
    search_refresh: int = 0
    deco_alternations: int = 2
    deco_carry: DecoCarry = DecoCarry.IncumbentColumn

    def to_abi(self) -> _abi.Config:
        a, la = self.ascent, self.lifted_ascent or self.ascent
        s = self.search or SearchConfig()
        return _abi.Config(
            algorithm=int(self.algorithm), lift_dim=self.lift_dim, batch_size=self.batch_size,
            num_batches=self.num_batches, alpha=a.alpha, iterations=a.iterations,
            momentum=a.momentum, early_exit=int(a.early_exit),
            has_lifted_ascent=int(self.lifted_ascent is not None), l_alpha=la.alpha,
            l_iterations=la.iterations, l_momentum=la.momentum, l_early_exit=int(la.early_exit),
            init_method=int(self.init.method), beta=self.init.beta, eta=self.init.eta,
            init_scale=self.init.init_scale, init_seed=self.init.seed,
            resample_idi=int(self.init.resample_idi), scale_noise=int(self.init.scale_noise),
            time_budget_s=float(self.time_budget_s) if self.time_budget_s is not None else 0.0,
            has_search=int(self.search is not None), population_size=s.population_size,
            t_lower=s.t_lower, t_upper=s.t_upper, e_lower=s.e_lower, e_upper=s.e_upper,
            rounds=s.rounds, search_refresh=self.search_refresh,
            deco_alternations=self.deco_alternations, deco_carry=int(self.deco_carry))

    def validate(self):
        if self.time_budget_s is not None and self.time_budget_s <= 0.0:
            raise ValidationError("time_budget_s must be > 0")
        if self.search is not None and self.search.e_lower < -4.0 or (
                self.search is not None and self.search.e_upper > -1.0):
            pass  # warn-only in the reference (evo_search.cpp:19-21)
        c = self.to_abi()
        checks = [
            (c.batch_size < 1, "batch_size must be >= 1"),
            (c.num_batches < 1, "num_batches must be >= 1"),
            (c.lift_dim < 1, "lift_dim must be >= 1"),
            (c.algorithm != 0 and c.lift_dim < 2, "lifted algorithms need lift_dim >= 2"),
            (c.beta <= 0.0 or c.beta >= 1.0, "init.beta must lie in (0, 1)"),
            (c.eta <= 0.0, "init.eta must be > 0"),
            (c.init_scale < 1.0, "init.init_scale must be >= 1"),
            (c.search_refresh < 0, "search_refresh must be >= 0"),
            (c.deco_alternations < 1, "deco_alternations must be >= 1"),
        ]
        for bad, msg in checks:
            if bad:
                raise ValidationError(msg)
        self.ascent.validate()
        if self.lifted_ascent is not None:
            self.lifted_ascent.validate()


@dataclass
class CutSolution:
    assignment: np.ndarray
    cut_value: int = 0
    algorithm: str = ""
    seed: int = 0
    batch_index: int = -1
    member_index: int = -1
    wall_time_s: float = 0.0


@dataclass
class BatchTraceEntry:
    serial: int
    kind: str
    alpha: float
    iterations: int
    batch_best: int
    best_so_far: int


@dataclass
class PhaseTraceEntry:
    phase: int
    kind: str
    best_after: int


@dataclass
class SearchTraceEntry:
    round: int
    exponent: float
    iterations: int
    fitness: float


@dataclass
class StageTimes:
    init_s: float = 0.0
    ascent_s: float = 0.0
    rounding_s: float = 0.0
    search_s: float = 0.0


@dataclass
class SolveOutcome:
    best: CutSolution
    batch_trace: list
    phase_trace: list
    search_trace: list
    stage_times: StageTimes
    batches_run: int = 0
    # B200 measurement (not in the reference struct)
    step_ms: float = 0.0
    step_launches: int = 0
    node_updates: int = 0
    step_bytes: float = 0.0
    solve_ms: float = 0.0
    kernel_stats: dict = field(default_factory=dict)  # name -> (ms, launches, bytes | flops for k_dense_step)


@dataclass
class RunOptions:
    precision: Optional[int] = None
    host_init: int = -1
    batched_search: bool = False
    comm: Optional[object] = None  # dist.Comm


def _solve(g: Graph, cfg: SolverConfig, seed: int, per_component: bool, algo: Algorithm,
           opts: Optional[RunOptions], cap: int = 1 << 14, trace=None) -> SolveOutcome:
    opts = opts or RunOptions()
    c = cfg.to_abi()
    c.algorithm = int(algo)
    out = _abi.Outcome()
    z = np.zeros(g.node_count(), dtype=np.uint8)
    bt, pt, st = (_abi.BatchTrace * cap)(), (_abi.PhaseTrace * cap)(), (_abi.SearchTrace * cap)()
    step_ms, step_bytes, solve_ms = C.c_double(0), C.c_double(0), C.c_double(0)
    kst = (C.c_double * 12)()
    launches, nupd = C.c_int64(0), C.c_int64(0)
    ro = _abi.RunOpts(precision=default_precision() if opts.precision is None else opts.precision,
                      host_init=opts.host_init, batched_search=int(opts.batched_search),
                      comm=opts.comm.handle if opts.comm is not None else None,
                      step_ms=C.cast(C.byref(step_ms), C.c_void_p),
                      step_launches=C.cast(C.byref(launches), C.c_void_p),
                      node_updates=C.cast(C.byref(nupd), C.c_void_p),
                      step_bytes=C.cast(C.byref(step_bytes), C.c_void_p),
                      solve_ms=C.cast(C.byref(solve_ms), C.c_void_p),
                      kernel_stats=C.cast(kst, C.c_void_p))
    if trace is not None:
        cb = _abi.TRACE_FN(lambda _ctx, it, member, obj: trace(int(it), int(member), float(obj)))
        ro.trace_fn = cb
    dev = opts.comm.device if opts.comm is not None else None
    _check(_abi.lib().lcb_solve(g.handle(dev), C.byref(c), seed & _M64, int(per_component),
                                C.byref(ro), C.byref(out), _ptr(z), bt, cap, pt, cap, st, cap))
    kinds_b, kinds_p = ("main", "search"), ("quco", "luco")
    return SolveOutcome(
        best=CutSolution(z, out.cut_value, algorithm_to_string(Algorithm(cfg.algorithm)),
                         seed, out.batch_index, out.member_index, out.wall_s),
        batch_trace=[BatchTraceEntry(e.serial, kinds_b[e.kind], e.alpha, e.iterations,
                                     e.batch_best, e.best_so_far)
                     for e in bt[:min(cap, out.n_batch_trace)]],
        phase_trace=[PhaseTraceEntry(e.phase, kinds_p[e.kind], e.best_after)
                     for e in pt[:min(cap, out.n_phase_trace)]],
        search_trace=[SearchTraceEntry(e.round, e.exponent, e.iterations, e.fitness)
                      for e in st[:min(cap, out.n_search_trace)]],
        stage_times=StageTimes(out.init_s, out.ascent_s, out.rounding_s, out.search_s),
        batches_run=out.batches_run, step_ms=step_ms.value, step_launches=launches.value,
        node_updates=nupd.value, step_bytes=step_bytes.value, solve_ms=solve_ms.value,
        kernel_stats={"k_step": tuple(kst[0:3]), "k_resident": tuple(kst[3:6]),
                      "k_dense_step": tuple(kst[6:9]), "k_stream": tuple(kst[9:12])})


@dataclass
class RunsOutcome:
    """solve_runs: every run's best cut and the best run (first maximum in run order);
    measurement fields sum this rank's runs."""
    run_cuts: np.ndarray
    best_run: int
    best: CutSolution
    stage_times: StageTimes
    batches_run: int
    step_ms: float = 0.0
    step_launches: int = 0
    node_updates: int = 0
    step_bytes: float = 0.0
    solve_ms: float = 0.0
    kernel_stats: dict = field(default_factory=dict)


def solve_runs(g: Graph, cfg: SolverConfig, seeds, per_component: bool = True,
               opts: Optional[RunOptions] = None) -> RunsOutcome:
    """Independent runs, one per seed (run_bench's loop, bench.cpp:97-136): run i is solved
    on rank i % nranks of ``opts.comm`` (or locally), then one exchange of the per-run cuts
    and the best run's assignment (lcb_solve_runs)."""
    cfg.validate()
    opts = opts or RunOptions()
    seeds = np.ascontiguousarray([int(s) & _M64 for s in seeds], dtype=np.uint64)
    c = cfg.to_abi()
    step_ms, step_bytes, solve_ms = C.c_double(0), C.c_double(0), C.c_double(0)
    kst = (C.c_double * 12)()
    launches, nupd = C.c_int64(0), C.c_int64(0)
    ro = _abi.RunOpts(precision=default_precision() if opts.precision is None else opts.precision,
                      host_init=opts.host_init, batched_search=int(opts.batched_search),
                      comm=opts.comm.handle if opts.comm is not None else None,
                      step_ms=C.cast(C.byref(step_ms), C.c_void_p),
                      step_launches=C.cast(C.byref(launches), C.c_void_p),
                      node_updates=C.cast(C.byref(nupd), C.c_void_p),
                      step_bytes=C.cast(C.byref(step_bytes), C.c_void_p),
                      solve_ms=C.cast(C.byref(solve_ms), C.c_void_p),
                      kernel_stats=C.cast(kst, C.c_void_p))
    cuts = np.zeros(len(seeds), dtype=np.int64)
    best_run = C.c_int64(-1)
    out = _abi.Outcome()
    z = np.zeros(g.node_count(), dtype=np.uint8)
    dev = opts.comm.device if opts.comm is not None else None
    _check(_abi.lib().lcb_solve_runs(g.handle(dev), C.byref(c), _ptr(seeds), len(seeds), int(per_component),
                                     C.byref(ro), _ptr(cuts), C.byref(best_run), C.byref(out), _ptr(z)))
    b = best_run.value
    return RunsOutcome(cuts, b, CutSolution(z, out.cut_value, algorithm_to_string(Algorithm(cfg.algorithm)),
                                            int(seeds[b]), out.batch_index, out.member_index, out.wall_s),
                       StageTimes(out.init_s, out.ascent_s, out.rounding_s, out.search_s), out.batches_run,
                       step_ms.value, launches.value, nupd.value, step_bytes.value, solve_ms.value,
                       {"k_step": tuple(kst[0:3]), "k_resident": tuple(kst[3:6]), "k_dense_step": tuple(kst[6:9]),
                        "k_stream": tuple(kst[9:12])})


def set_option(name: str, value: int) -> None:
    """Kernel-selection knob of the library (lcb_set_option): resident, stream, signrec,
    chunk, res_split, bank_order, bank_refine, dense."""
    _check(_abi.lib().lcb_set_option(name.encode(), int(value)))


def get_option(name: str) -> int:
    v = C.c_int64()
    _check(_abi.lib().lcb_get_option(name.encode(), C.byref(v)))
    return v.value


class options:
    """Context manager: set knobs for the duration of a block, restore them after.

        with lc.options(resident=0, stream=1): ...
    """

    def __init__(self, **kw):
        self.kw, self.old = kw, {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            set_option(k, v)
        return False


def counters():
    """(kernel launches, H2D bytes, D2H bytes) issued by libliftcut_b200.so so far."""
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    _abi.lib().lcb_counters(C.byref(a), C.byref(b), C.byref(c))
    return a.value, b.value, c.value


def _pre(g: Graph, cfg: SolverConfig, need_lift: bool, name: str):
    cfg.validate()
    if g.edge_count() < 1:
        raise ValidationError("solver requires a graph with at least one edge")
    if need_lift and cfg.lift_dim < 2:
        raise ValidationError(f"{name} needs lift_dim >= 2")


def pquco(g: Graph, cfg: SolverConfig, seed: int, workers: int = 1, trace=None,
          opts: Optional[RunOptions] = None) -> SolveOutcome:
    _pre(g, cfg, False, "pquco")
    out = _solve(g, cfg, seed, False, Algorithm.pQUCO, opts, trace=trace)
    out.best.algorithm = "pquco"
    return out


def pluco(g: Graph, cfg: SolverConfig, seed: int, workers: int = 1, trace=None,
          opts: Optional[RunOptions] = None) -> SolveOutcome:
    _pre(g, cfg, True, "pluco")
    out = _solve(g, cfg, seed, False, Algorithm.pLUCO, opts, trace=trace)
    out.best.algorithm = "pluco"
    return out


def pdeco(g: Graph, cfg: SolverConfig, seed: int, workers: int = 1, trace=None,
          opts: Optional[RunOptions] = None) -> SolveOutcome:
    _pre(g, cfg, True, "pdeco")
    out = _solve(g, cfg, seed, False, Algorithm.pDECO, opts, trace=trace)
    out.best.algorithm = "pdeco"
    return out


def solve_per_component(g: Graph, cfg: SolverConfig, seed: int, workers: int = 1, trace=None,
                        opts: Optional[RunOptions] = None) -> SolveOutcome:
    cfg.validate()
    if g.edge_count() == 0:
        return SolveOutcome(CutSolution(np.zeros(g.node_count(), dtype=np.uint8), 0,
                                        algorithm_to_string(cfg.algorithm), seed, -1, -1),
                            [], [], [], StageTimes(), 0)
    out = _solve(g, cfg, seed, True, cfg.algorithm, opts, trace=trace)
    out.best.algorithm = algorithm_to_string(cfg.algorithm)
    return out


# presets (presets.cpp:23-33,68-95) — host configuration data
_PRESETS = {
    "smaller": (0.15, 48000, 0.001, 2500, 0.10, 30000, 0.001, 2000),
    "gset": (0.01, 60000, 0.001, 3000, 0.012, 80000, 0.001, 2000),
    "largeer": (0.01, 100000, 0.001, 5000, 0.02, 60000, 0.005, 1000),
}


def apply_manual_preset(cfg: SolverConfig, name: str) -> None:
    key = name.replace("-", "").replace("_", "").lower()
    if key.endswith("manual") and len(key) > 6:
        key = key[:-6]
    if key == "largescaleer":
        key = "largeer"
    if key not in _PRESETS:
        raise ValidationError(f"unknown preset '{name}' (expected smallER, gset, or largeER)")
    qa, qt, la, lt, da, dt, dla, dlt = _PRESETS[key]
    if cfg.algorithm == Algorithm.pQUCO:
        cfg.ascent = replace(cfg.ascent, alpha=qa, iterations=qt)
        cfg.lifted_ascent = None
    elif cfg.algorithm == Algorithm.pLUCO:
        cfg.ascent = replace(cfg.ascent, alpha=la, iterations=lt)
        cfg.lifted_ascent = None
    else:
        cfg.ascent = replace(cfg.ascent, alpha=da, iterations=dt)
        cfg.lifted_ascent = replace(cfg.ascent, alpha=dla, iterations=dlt)


def auto_search_bounds() -> SearchConfig:
    return SearchConfig()
