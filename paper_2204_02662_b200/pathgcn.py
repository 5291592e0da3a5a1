"""Host-side mirror of the reference's ``pathgcn`` operator API for the
backward-aggregation path, over the C ABI (include/pathgcn_b200.h).

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/core/include/pathgcn/*.hpp): graph load
(``build_undirected_csr``, ``assign_edge_weights``, ``sample_training_set``),
execution-path build (``compute_frontiers``, ``extract_execution_path``,
``prepare_all_paths``, ``path_fingerprint``), group partition
(``group_neighbors``, ``regression_gs``, ``oracle_gs``, ``grouping_cost``,
``default_gs_candidates``) and backward aggregate (``aggregate_pull``,
``backward_aggregation`` = engine.hpp:331-338, ``backward_epp``).
All compute runs in libpathgcn_b200.so on the GPU; there is no CPU path.
Host data is numpy; device data is torch CUDA tensors (plumbing only).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import f32p, f64p, u32p, u64p

DETERMINISTIC = "deterministic"
FAST = "fast"
GROUPED = "grouped"  # Fast on the group-partitioned kernel (PG_AGG_GROUPED)
AGG_FAST = 1
AGG_OVERWRITE = 2
AGG_GROUPED = 4


class Error(RuntimeError):
    """error.hpp:10-12"""


class ConfigError(Error):
    """error.hpp:14-16 (ShapeError / StalenessError derive from it)."""


class ShapeError(ConfigError):
    pass


class ParseError(ConfigError):
    """error.hpp:18-22: carries the 1-based line number."""

    def __init__(self, msg, line_number=None):
        super().__init__(msg)
        self.line_number = line_number


class StalenessError(ConfigError):
    pass


class IoError(Error):
    pass


class NumericError(Error):
    pass


class DeviceError(Error):
    """CUDA runtime / device failure (status 5)."""


_CODES = {2: ConfigError, 3: IoError, 4: NumericError, 5: DeviceError}


def _lib_():
    return _lib.load()


# PG_KIND_* (pathgcn_b200.h): the exact reference exception type of a failure
_KINDS = {1: "ConfigError", 2: "ShapeError", 3: "StalenessError", 4: "ParseError", 5: "IoError",
          6: "NumericError", 7: "DeviceError"}


def _check(rc):
    if rc:
        buf = C.create_string_buffer(2048)
        _lib_().pg_last_error(buf, 2048)
        msg = buf.value.decode(errors="replace")
        line = C.c_uint64(0)
        kind = _lib_().pg_last_error_kind(C.byref(line))
        name = _KINDS.get(kind)
        if name == "ParseError":
            raise ParseError(msg, int(line.value))
        cls = globals()[name] if name else _CODES.get(rc, Error)
        raise cls(msg)


def _p(a, t):
    return a.ctypes.data_as(t)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


# ---------------------------------------------------------------- inputs ---

def gen_rmat(n, m, a=0.57, b=0.19, c=0.19, d=0.05, seed=0):
    """rmat.cpp:10-44. Returns (pairs[m, 2] u32, n_pad)."""
    pairs = np.empty((m, 2), np.uint32)
    n_pad = C.c_uint32()
    _check(_lib_().pg_gen_rmat(n, m, a, b, c, d, seed, _p(pairs, u32p), C.byref(n_pad)))
    return pairs, n_pad.value


def sample_training_set(n, ratio, seed):
    """training_set.cpp:28-49: sorted u32 ids."""
    k = C.c_uint64()
    _check(_lib_().pg_training_set_size(n, ratio, C.byref(k)))
    out = np.empty(k.value, np.uint32)
    _check(_lib_().pg_sample_training_set(n, ratio, seed, _p(out, u32p)))
    return out


# ------------------------------------------------------------ graph load ---

class CsrGraph:
    """csr_graph.hpp:19-38, device resident."""

    def __init__(self, handle, device):
        self._h = C.c_void_p(handle)
        self.device = device
        n, m, md = C.c_uint32(), C.c_uint64(), C.c_uint32()
        _check(_lib_().pg_graph_info(self._h, C.byref(n), C.byref(m), C.byref(md), None))
        self.n, self.m, self._max_degree = n.value, m.value, md.value

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            try:
                _lib_().pg_graph_destroy(self._h)
            except Exception:
                pass
            self._h = C.c_void_p(None)

    def max_degree(self):
        return self._max_degree

    def fingerprint(self):
        fp = C.c_uint64()
        _check(_lib_().pg_graph_info(self._h, None, None, None, C.byref(fp)))
        return fp.value

    def export(self):
        offs = np.empty(self.n + 1, np.uint64)
        nb = np.empty(max(self.m, 1), np.uint32)
        w = np.empty(max(self.m, 1), np.float64)
        _check(_lib_().pg_graph_export(self._h, _p(offs, u64p), _p(nb, u32p), _p(w, f64p)))
        return offs, nb[: self.m], w[: self.m]

    def assign_edge_weights(self, mode):
        _check(_lib_().pg_graph_assign_weights(self._h, _weight_mode(mode)))


def _weight_mode(mode):
    if mode in (1, "symnorm", "sym-norm", "SymNorm"):
        return 1
    if mode in (0, "unit", "Unit"):
        return 0
    raise ConfigError(f"unknown weight mode {mode!r}")


def build_undirected_csr(pairs, n_hint=None, weights="unit", device=0) -> CsrGraph:
    """csr_graph.cpp:33-63 + assign_edge_weights (:65-77), on device."""
    pairs = _u32(pairs).reshape(-1, 2)
    h = C.c_void_p()
    _check(_lib_().pg_graph_build(device, -1 if n_hint is None else int(n_hint), _p(pairs, u32p), len(pairs),
                                  _weight_mode(weights), C.byref(h)))
    return CsrGraph(h.value, device)


@dataclass
class EdgeList:
    """edge_list.hpp:14-18"""
    pairs: np.ndarray  # [m, 2] u32
    n_hint: int | None = None
    self_loops_dropped: int = 0


def load_edge_list_file(path) -> EdgeList:
    """edge_list.cpp:34-68 (ParseError with line_number, IoError)."""
    h = C.c_void_p()
    _check(_lib_().pg_edge_list_load(str(path).encode(), C.byref(h)))
    try:
        n, sl = C.c_uint64(), C.c_uint64()
        _check(_lib_().pg_edge_list_info(h, C.byref(n), C.byref(sl)))
        pairs = np.empty((n.value, 2), np.uint32)
        _check(_lib_().pg_edge_list_export(h, _p(pairs, u32p)))
    finally:
        _lib_().pg_edge_list_destroy(h)
    return EdgeList(pairs, None, sl.value)


def write_edge_list(path, pairs):
    """edge_list.cpp:70-73"""
    pairs = _u32(pairs).reshape(-1, 2)
    _check(_lib_().pg_edge_list_write(str(path).encode(), _p(pairs, u32p), len(pairs)))


def load_graph_file(path, weights="unit", device=0) -> CsrGraph:
    """load_edge_list_file + build_undirected_csr + assign_edge_weights."""
    h = C.c_void_p()
    _check(_lib_().pg_graph_load_file(device, str(path).encode(), _weight_mode(weights), C.byref(h)))
    return CsrGraph(h.value, device)


def load_training_set_file(path, n):
    """training_set.cpp:51-79: sorted unique u32 ids."""
    k = C.c_uint64()
    _check(_lib_().pg_training_set_load(str(path).encode(), n, None, 0, C.byref(k)))
    out = np.empty(max(k.value, 1), np.uint32)
    _check(_lib_().pg_training_set_load(str(path).encode(), n, _p(out, u32p), len(out), C.byref(k)))
    return out[: k.value]


def write_training_set(path, vt):
    """training_set.cpp:81-83"""
    vt = _u32(vt)
    _check(_lib_().pg_training_set_write(str(path).encode(), _p(vt, u32p), len(vt)))


def graph_from_csr(n, offsets, neighbors, weights, device=0, validate=True) -> CsrGraph:
    offsets = np.ascontiguousarray(offsets, np.uint64)
    neighbors = np.ascontiguousarray(neighbors, np.uint32)
    weights = np.ascontiguousarray(weights, np.float64)
    h = C.c_void_p()
    _check(_lib_().pg_graph_create(device, n, _p(offsets, u64p), _p(neighbors, u32p), _p(weights, f64p),
                                   int(validate), C.byref(h)))
    return CsrGraph(h.value, device)


def assign_edge_weights(g: CsrGraph, mode):
    g.assign_edge_weights(mode)


def path_fingerprint(g: CsrGraph, vt, layers):
    """execution_path.cpp:17-22"""
    vt = _u32(vt)
    fp = C.c_uint64()
    _check(_lib_().pg_path_fingerprint(g._h, _p(vt, u32p), len(vt), layers, C.byref(fp)))
    return fp.value


# ------------------------------------------------------------ path build ---

class FrontierSets:
    """frontier.hpp:14-18"""

    def __init__(self, handle, graph, L):
        self._h = C.c_void_p(handle)
        self.graph = graph  # keeps the graph alive
        self.L = L

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            try:
                _lib_().pg_frontiers_destroy(self._h)
            except Exception:
                pass
            self._h = C.c_void_p(None)

    def depth(self):
        return self.L

    def size(self, level):
        s = C.c_uint64()
        _check(_lib_().pg_frontiers_size(self._h, level, C.byref(s)))
        return s.value

    def level(self, k):
        out = np.empty(max(self.size(k), 1), np.uint32)
        _check(_lib_().pg_frontiers_export(self._h, k, _p(out, u32p)))
        return out[: self.size(k)]

    @property
    def levels(self):
        return [self.level(k) for k in range(self.L + 1)]


def compute_frontiers(g: CsrGraph, vt, layers) -> FrontierSets:
    """frontier.cpp:7-26"""
    vt = _u32(vt)
    h = C.c_void_p()
    _check(_lib_().pg_frontiers_compute(g._h, _p(vt, u32p), len(vt), layers, C.byref(h)))
    return FrontierSets(h.value, g, layers)


class ExecutionPath:
    """execution_path.hpp:16-33"""

    def __init__(self, handle, frontiers):
        self._h = C.c_void_p(handle)
        self.frontiers = frontiers
        layer, D, S, E, P, md = C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_uint64(), C.c_uint32(), C.c_uint32()
        _check(_lib_().pg_path_info(self._h, C.byref(layer), C.byref(D), C.byref(S), C.byref(E), C.byref(P),
                                    C.byref(md)))
        self.layer, self.D, self.S, self.E, self.P, self.max_degree = (layer.value, D.value, S.value, E.value,
                                                                      P.value, md.value)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            try:
                _lib_().pg_path_destroy(self._h)
            except Exception:
                pass
            self._h = C.c_void_p(None)

    def dest_count(self):
        return self.D

    def src_count(self):
        return self.S

    def edge_count(self):
        return self.E

    @property
    def fingerprint(self):
        fp = C.c_uint64()
        _check(_lib_().pg_path_get_fingerprint(self._h, C.byref(fp)))
        return fp.value

    @fingerprint.setter
    def fingerprint(self, v):
        _check(_lib_().pg_path_set_fingerprint(self._h, int(v)))

    def export(self):
        """dict of the reference ExecutionPath arrays (host copies)."""
        D, S, E = self.D, self.S, self.E
        dest = np.empty(max(D, 1), np.uint32)
        src = np.empty(max(S, 1), np.uint32)
        pos = np.empty(max(S, 1), np.uint32)
        offs = np.empty(D + 1, np.uint64)
        nb = np.empty(max(E, 1), np.uint32)
        w = np.empty(max(E, 1), np.float64)
        _check(_lib_().pg_path_export(self._h, _p(dest, u32p), _p(src, u32p), _p(pos, u32p), _p(offs, u64p),
                                      _p(nb, u32p), _p(w, f64p)))
        return dict(dest=dest[:D], src=src[:S], srcpos=pos[:S], offsets=offs, neighbors=nb[:E], weights=w[:E])

    def shard_bounds(self, world):
        b = np.empty(world + 1, np.uint32)
        _check(_lib_().pg_path_shard_bounds(self._h, world, _p(b, u32p)))
        return b


def extract_execution_path(g: CsrGraph, frontiers: FrontierSets, layer) -> ExecutionPath:
    """execution_path.cpp:24-88"""
    h = C.c_void_p()
    _check(_lib_().pg_path_extract(g._h, frontiers._h, layer, C.byref(h)))
    return ExecutionPath(h.value, frontiers)


def prepare_all_paths(g: CsrGraph, frontiers: FrontierSets):
    """execution_path.cpp:90-96: SG_{L-1} first."""
    return [extract_execution_path(g, frontiers, l) for l in range(frontiers.L - 1, -1, -1)]


# -------------------------------------------------------- group partition ---

def regression_gs(n_vertices, n_edges, avg_degree, beta=None):
    """gs_model.cpp:68-74"""
    b = None if beta is None else _p(np.asarray(beta, np.float64), f64p)
    gs = C.c_uint32()
    _check(_lib_().pg_gs_regression_stats(n_vertices, n_edges, avg_degree, b, C.byref(gs)))
    return gs.value


def path_regression_gs(path: ExecutionPath, beta=None):
    """regression_gs(path_stats(path)) (train.hpp:16-24, :63-64)"""
    b = None if beta is None else _p(np.asarray(beta, np.float64), f64p)
    gs = C.c_uint32()
    _check(_lib_().pg_gs_regression(path._h, b, C.byref(gs)))
    return gs.value


def default_gs_candidates(max_degree):
    """group_cost.cpp:30-34"""
    out = np.empty(40, np.uint32)
    k = C.c_uint64()
    _check(_lib_().pg_gs_default_candidates(max_degree, _p(out, u32p), C.byref(k)))
    return out[: k.value].copy()


def oracle_gs(path: ExecutionPath, dim, workers, atomic_penalty=0.25, candidates=None):
    """group_cost.cpp:36-53 with the cost-model evaluator; (best_gs, [(gs, cost)])."""
    if candidates is None:
        candidates = default_gs_candidates(path.max_degree)
    cands = _u32(candidates)
    table = np.empty(max(len(cands), 1), np.float64)
    best = C.c_uint32()
    n = C.c_uint64()
    _check(_lib_().pg_gs_oracle_cost(path._h, dim, workers, atomic_penalty, _p(cands, u32p), len(cands),
                                     C.byref(best), _p(table, f64p), C.byref(n)))
    return best.value, list(zip(cands.tolist(), table[: n.value].tolist()))


def oracle_gs_measured(path: ExecutionPath, dim, repeats=5, seed=42, candidates=None):
    """train.hpp:35-54 + group_cost.cpp:36-53 on the device: each candidate's
    grouped (Fast) aggregation timed, median of repeats; (best_gs,
    [(gs, seconds)]). Timing based — not bit-reproducible."""
    if candidates is None:
        candidates = default_gs_candidates(path.max_degree)
    cands = _u32(candidates)
    table = np.empty(max(len(cands), 1), np.float64)
    best = C.c_uint32()
    n = C.c_uint64()
    _check(_lib_().pg_gs_oracle_measured(path._h, dim, repeats, seed, _p(cands, u32p), len(cands), C.byref(best),
                                         _p(table, f64p), C.byref(n)))
    return best.value, list(zip(cands.tolist(), table[: n.value].tolist()))


class GroupedCsr:
    """grouping.hpp:14-28 (borrows its base)."""

    def __init__(self, handle, base):
        self._h = C.c_void_p(handle)
        self.base = base
        gs, cnt, D = C.c_uint32(), C.c_uint64(), C.c_uint32()
        _check(_lib_().pg_groups_info(self._h, C.byref(gs), C.byref(cnt), C.byref(D)))
        self.gs, self.count, self.D = gs.value, cnt.value, D.value

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            try:
                _lib_().pg_groups_destroy(self._h)
            except Exception:
                pass
            self._h = C.c_void_p(None)

    def group_count(self):
        return self.count

    def export(self):
        G, D = self.count, self.D
        gd = np.empty(max(G, 1), np.uint32)
        gb = np.empty(max(G, 1), np.uint64)
        ge = np.empty(max(G, 1), np.uint64)
        dg = np.empty(D + 1, np.uint64)
        _check(_lib_().pg_groups_export(self._h, _p(gd, u32p), _p(gb, u64p), _p(ge, u64p), _p(dg, u64p)))
        return dict(dest=gd[:G], begin=gb[:G], end=ge[:G], dest_groups=dg)

    remap_rows = None

    def remap_sources(self, mapping, new_rows):
        """Multi-GPU: parent row p of y_grad lives at row mapping[p] of a
        new_rows-row (padded allgather) buffer. None removes the map."""
        if mapping is None:
            _check(_lib_().pg_groups_remap_sources(self._h, None, 0, 0))
            self.remap_rows = None
            return
        m = _u32(mapping)
        _check(_lib_().pg_groups_remap_sources(self._h, _p(m, u32p), len(m), int(new_rows)))
        self.remap_rows = int(new_rows)

    def set_segments(self, cuts):
        """Source-row segments (cuts[0] = 0 ... cuts[-1] = input rows); run
        them in order with backward_aggregation(..., segment=k)."""
        if cuts is None:
            _check(_lib_().pg_groups_set_segments(self._h, None, 0))
            self.nseg = 0
            return
        c = np.ascontiguousarray(cuts, np.uint64)
        _check(_lib_().pg_groups_set_segments(self._h, _p(c, u64p), len(c) - 1))
        self.nseg = len(c) - 1

    def counters(self, dim, mode=DETERMINISTIC):
        c = np.zeros(3, np.uint64)
        _check(_lib_().pg_stage_counters(self._h, dim, _flags(mode), _p(c, u64p)))
        return dict(edges_traversed=int(c[0]), groups_executed=int(c[1]), atomic_commits=int(c[2]))


def group_neighbors(base, gs) -> GroupedCsr:
    """grouping.cpp:7-27 over an ExecutionPath or a CsrGraph."""
    h = C.c_void_p()
    if isinstance(base, ExecutionPath):
        _check(_lib_().pg_group(base._h, gs, C.byref(h)))
    else:
        _check(_lib_().pg_group_graph(base._h, gs, C.byref(h)))
    return GroupedCsr(h.value, base)


def grouping_cost(grouped: GroupedCsr, dim, workers, atomic_penalty=0.25):
    """group_cost.cpp:9-24"""
    c = C.c_double()
    _check(_lib_().pg_grouping_cost(grouped._h, dim, workers, atomic_penalty, C.byref(c)))
    return c.value


# ------------------------------------------------------ backward aggregate ---

def _flags(mode, overwrite=False):
    f = 0
    if mode in (FAST, "Fast", AGG_FAST):
        f |= AGG_FAST
    elif mode in (GROUPED, AGG_GROUPED):
        f |= AGG_FAST | AGG_GROUPED
    elif mode not in (DETERMINISTIC, "Deterministic", 0, None):
        raise ConfigError(f"unknown commit mode {mode!r}")
    if overwrite:
        f |= AGG_OVERWRITE
    return f


def _dev(t, name, rows=None, cols=None, dtype=None):
    import torch

    dtype = dtype or torch.float32
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dtype:
        raise ShapeError(f"{name}: expected a {str(dtype).replace('torch.', '')} CUDA tensor")
    if t.dim() != 2 or t.stride(1) != 1:
        raise ShapeError(f"{name}: expected a row-major 2-D tensor")
    if rows is not None and t.shape[0] != rows:
        raise ShapeError(f"{name}: {t.shape[0]} rows, expected {rows}")
    if cols is not None and t.shape[1] != cols:
        raise ShapeError(f"{name}: {t.shape[1]} cols, expected {cols}")
    return t


def _stream(stream):
    import torch

    if stream is None:
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def aggregate_pull(grouped: GroupedCsr, inp, out, mode=DETERMINISTIC, counters=None, overwrite=False,
                   stream=None):
    """aggregate.hpp:56-122: out (+)= A * inp.

    numpy float32 in/out: host DenseMatrix drop-in (copies in, runs, copies
    out, in place on ``out``). torch CUDA tensors: asynchronous on ``stream``.
    Input rows are the base's local source ids.
    """
    flags = _flags(mode, overwrite)
    if _is_f64(inp):  # aggregate_pull<double>, the reference's default precision
        _pull_f64(grouped, inp, out, flags, stream, backward=False)
        if counters is not None:
            for k, v in grouped.counters(inp.shape[1], mode).items():
                counters[k] = counters.get(k, 0) + v
        return out
    if isinstance(inp, np.ndarray):
        if inp.dtype != np.float32 or out.dtype != np.float32:
            raise ShapeError("aggregate_pull: float32 matrices expected")
        if out.shape[1] != inp.shape[1]:
            raise ShapeError("aggregate_pull: input/output dims differ")
        if out.shape[0] != grouped.D:
            raise ShapeError("aggregate_pull: output rows != dest count")
        inp = np.ascontiguousarray(inp)
        if not out.flags.c_contiguous:
            raise ShapeError("aggregate_pull: output must be contiguous")
        c = np.zeros(3, np.uint64)
        _check(_lib_().pg_aggregate_pull_host(grouped._h, _p(inp, f32p), inp.shape[0], inp.shape[1],
                                              _p(out, f32p), flags, _p(c, u64p)))
    else:
        _dev(inp, "input")
        _dev(out, "output", rows=grouped.D, cols=inp.shape[1])
        _check(_lib_().pg_aggregate_pull(grouped._h, C.c_void_p(inp.data_ptr()), inp.shape[0], inp.stride(0),
                                         C.c_void_p(out.data_ptr()), out.stride(0), inp.shape[1], flags,
                                         _stream(stream)))
        c = None
    if counters is not None:
        cc = grouped.counters(inp.shape[1], mode)
        for k, v in cc.items():
            counters[k] = counters.get(k, 0) + v
    return out


def _is_f64(a):
    if isinstance(a, np.ndarray):
        return a.dtype == np.float64
    import torch

    return isinstance(a, torch.Tensor) and a.dtype == torch.float64


def _pull_f64(grouped, inp, out, flags, stream, backward):
    """aggregate.hpp:56-122 with T = double: numpy (host DenseMatrix<double>
    drop-in, synchronous) or float64 CUDA tensors (rows with an even pitch)."""
    import torch

    base = grouped.base
    rows_in = (base.P if backward else (base.S if isinstance(base, ExecutionPath) else base.n))
    if isinstance(inp, np.ndarray):
        x = np.ascontiguousarray(inp, np.float64)
        if x.shape[0] != rows_in:
            raise ShapeError("aggregate_pull: input rows != source count of the grouping's base")
        if out.shape != (grouped.D, x.shape[1]) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ShapeError("aggregate_pull: output must be a C-contiguous float64 D x dim array")
        fn = _lib_().pg_backward_aggregate_host_f64 if backward else _lib_().pg_aggregate_pull_host_f64
        c = np.zeros(3, np.uint64)
        _check(fn(grouped._h, _p(x, f64p), x.shape[0], x.shape[1], _p(out, f64p), flags, _p(c, u64p)))
        return out
    _dev(inp, "input", rows=rows_in, dtype=torch.float64)
    _dev(out, "output", rows=grouped.D, cols=inp.shape[1], dtype=torch.float64)
    fn = _lib_().pg_backward_aggregate_f64 if backward else _lib_().pg_aggregate_pull_f64
    _check(fn(grouped._h, C.c_void_p(inp.data_ptr()), inp.shape[0], inp.stride(0), C.c_void_p(out.data_ptr()),
              out.stride(0), inp.shape[1], flags, _stream(stream)))
    return out


def backward_aggregation(grouped: GroupedCsr, y_grad, x_grad, mode=DETERMINISTIC, overwrite=False, stream=None,
                         rows=None, segment=None):
    """The reference's timed stage engine.hpp:331-338 (gather_rows over
    src_pos_in_parent + aggregate_pull), gather folded into the edge stream.
    y_grad rows follow the parent frontier. ``rows=(b, e)`` computes only
    destination rows [b, e) into x_grad (e-b rows) for row sharding."""
    path = grouped.base
    if not isinstance(path, ExecutionPath):
        raise ConfigError("backward_aggregation: grouping is not over an execution path")
    flags = _flags(mode, overwrite)
    if _is_f64(y_grad):  # aggregate_pull<double>, the reference's default precision
        if rows is not None or segment is not None:
            raise ConfigError("backward_aggregation<double>: whole paths only")
        return _pull_f64(grouped, y_grad, x_grad, flags, stream, backward=True)
    if isinstance(y_grad, np.ndarray):
        y = np.ascontiguousarray(y_grad, np.float32)
        if x_grad.shape != (path.D, y.shape[1]) or x_grad.dtype != np.float32:
            raise ShapeError("backward_aggregation: x_grad shape mismatch")
        if not (x_grad.flags.c_contiguous and x_grad.flags.writeable):
            raise ShapeError("backward_aggregation: host x_grad must be a writeable C-contiguous float32 array")
        c = np.zeros(3, np.uint64)
        _check(_lib_().pg_backward_aggregate_host(grouped._h, _p(y, f32p), y.shape[0], y.shape[1],
                                                  _p(x_grad, f32p), flags, _p(c, u64p)))
        return x_grad
    _dev(y_grad, "y_grad", rows=path.P if grouped.remap_rows is None else grouped.remap_rows)
    if segment is not None:
        b, e = (0, path.D) if rows is None else (int(rows[0]), int(rows[1]))
        _dev(x_grad, "x_grad", rows=e - b, cols=y_grad.shape[1])
        _check(_lib_().pg_backward_aggregate_segment(grouped._h, int(segment), b, e, C.c_void_p(y_grad.data_ptr()),
                                                     y_grad.shape[0], y_grad.stride(0), C.c_void_p(x_grad.data_ptr()),
                                                     x_grad.stride(0), y_grad.shape[1], flags, _stream(stream)))
        return x_grad
    if rows is None:
        _dev(x_grad, "x_grad", rows=path.D, cols=y_grad.shape[1])
        _check(_lib_().pg_backward_aggregate(grouped._h, C.c_void_p(y_grad.data_ptr()), y_grad.shape[0],
                                             y_grad.stride(0), C.c_void_p(x_grad.data_ptr()), x_grad.stride(0),
                                             y_grad.shape[1], flags, _stream(stream)))
    else:
        b, e = int(rows[0]), int(rows[1])
        _dev(x_grad, "x_grad", rows=e - b, cols=y_grad.shape[1])
        _check(_lib_().pg_backward_aggregate_rows(grouped._h, b, e, C.c_void_p(y_grad.data_ptr()),
                                                  y_grad.shape[0], y_grad.stride(0), C.c_void_p(x_grad.data_ptr()),
                                                  x_grad.stride(0), y_grad.shape[1], flags, _stream(stream)))
    return x_grad


PG_GEMM_TF32X3 = 1


def gemm_a_bt(a, b, out, stream=None, tensor_cores=False):
    """dense_matrix.hpp:78-95: out = a * b^T. Default: fp32, ascending k,
    unfused (bit-exact). tensor_cores=True: tcgen05 kind::tf32 with 3xTF32
    operand splitting (PG_GEMM_TF32X3) — within the fp32 tolerance, not
    bit-exact."""
    _dev(a, "a")
    _dev(b, "b", cols=a.shape[1])
    _dev(out, "out", rows=a.shape[0], cols=b.shape[0])
    _check(_lib_().pg_gemm_a_bt_ex(C.c_void_p(a.data_ptr()), a.stride(0), C.c_void_p(b.data_ptr()), b.stride(0),
                                   C.c_void_p(out.data_ptr()), out.stride(0), a.shape[0], b.shape[0], a.shape[1],
                                   PG_GEMM_TF32X3 if tensor_cores else 0, _stream(stream)))
    return out


def relu_backward(grad, pre, out, stream=None):
    """dense_matrix.hpp:114-121"""
    _dev(grad, "grad")
    _dev(pre, "pre", rows=grad.shape[0], cols=grad.shape[1])
    _dev(out, "out", rows=grad.shape[0], cols=grad.shape[1])
    _check(_lib_().pg_relu_backward(C.c_void_p(grad.data_ptr()), grad.stride(0), C.c_void_p(pre.data_ptr()),
                                    pre.stride(0), C.c_void_p(out.data_ptr()), out.stride(0), grad.shape[0],
                                    grad.shape[1], _stream(stream)))
    return out


def gather_rows(src, ids, out, stream=None):
    """engine.hpp:162-169 (ids: int32/uint32 CUDA tensor)."""
    _dev(src, "src")
    _dev(out, "out", rows=ids.shape[0], cols=src.shape[1])
    _check(_lib_().pg_gather_rows(C.c_void_p(src.data_ptr()), src.stride(0), C.c_void_p(ids.data_ptr()),
                                  ids.shape[0], C.c_void_p(out.data_ptr()), out.stride(0), src.shape[1],
                                  _stream(stream)))
    return out


def set_heavy_min_degree(min_degree=None):
    """Scheduling knob: destinations with >= min_degree edges run on the
    heavy-destination kernel (0 disables, None restores the width-dependent
    default). Never changes results."""
    _check(_lib_().pg_set_heavy_min_degree(2**64 - 1 if min_degree is None else int(min_degree)))


def set_tuning(key, value=None):
    """Scheduling knob of the SpMM kernels by name (see pg_set_tuning in
    include/pathgcn_b200.h; None restores the default). Never changes
    results except "grouped_seg" (a Fast-mode association order)."""
    _check(_lib_().pg_set_tuning(key.encode(), -1 if value is None else int(value)))


def padded_ld(cols):
    """Device row pitch for gradient matrices: 16-B rows for narrow widths,
    whole 128-B lines (32 floats) beyond 32 columns, so every row gather is
    sector aligned (e.g. 602 -> 608: 19 full lines instead of 76-77 sectors)."""
    return (cols + 3) // 4 * 4 if cols <= 32 else (cols + 31) // 32 * 32


def empty_rows(rows, cols, device="cuda"):
    """A rows x cols fp32 view over a 128-B-pitched allocation."""
    import torch

    buf = torch.empty((rows, padded_ld(cols)), dtype=torch.float32, device=device)
    return buf[:, :cols]


@dataclass
class PreparedPaths:
    """train.hpp:94-99 detail::PreparedPaths."""
    frontiers: FrontierSets
    paths: list
    groups: list
    gs: list
    fingerprint: int = 0
    graph: "CsrGraph | None" = None  # the graph and training set the paths were built from
    vt: "np.ndarray | None" = None

    def current_fingerprint(self):
        """path_fingerprint of the graph and training set as they are now
        (the caller-side expected_fingerprint of engine.hpp:280-283)."""
        if self.graph is None or self.vt is None:
            raise ConfigError("PreparedPaths without its graph/training set: pass expected_fingerprint")
        return path_fingerprint(self.graph, self.vt, self.frontiers.L)


def choose_gs(strategy, path: ExecutionPath, dim, workers=8, atomic_penalty=0.25):
    """train.hpp:56-82 for the deterministic strategies: ("fixed", k),
    "regression", "oracle:cost". (oracle:measured is timing-based and not
    bit-reproducible.)"""
    if isinstance(strategy, tuple) and strategy[0] == "fixed":
        return int(strategy[1])
    if strategy == "regression":
        return path_regression_gs(path)
    if strategy in ("oracle:cost", "oracle"):
        return oracle_gs(path, dim, workers, atomic_penalty)[0]
    if strategy == "oracle:measured":
        return oracle_gs_measured(path, dim)[0]
    raise ConfigError(f"unknown gs strategy {strategy!r}")


def prepare_paths(g: CsrGraph, vt, layers, agg_dims, gs_strategy="regression", workers=8,
                  atomic_penalty=0.25) -> PreparedPaths:
    """train.hpp:101-123: frontiers -> paths (SG_{L-1} first) -> fingerprint
    stamp -> per-path gs -> grouping. agg_dims[i] = aggregation width of
    path i (in_dim of layer L-1-i)."""
    F = compute_frontiers(g, vt, layers)
    paths = prepare_all_paths(g, F)
    stamp = path_fingerprint(g, vt, layers)
    groups, gss = [], []
    for i, p in enumerate(paths):
        p.fingerprint = stamp
        gs = choose_gs(gs_strategy, p, agg_dims[i], workers, atomic_penalty)
        gss.append(gs)
        groups.append(group_neighbors(p, gs))
    return PreparedPaths(F, paths, groups, gss, stamp, g, vt)


# ------------------------------------------------- the chain (engine.hpp) ---
# Device-resident forward / backward variants, bit-exact with the
# reference's f32 build. Matrices are float32 CUDA tensors (row-major,
# unit column stride; any row pitch — empty_rows() gives the 16-byte rows
# the SpMM's 128-bit gathers want).

def _mat(t, name, rows=None, cols=None):
    _dev(t, name, rows, cols)
    return _lib.PgMat(t.data_ptr(), t.shape[0], t.shape[1], t.stride(0))


def _mats(ts, name):
    arr = (_lib.PgMat * max(len(ts), 1))()
    for i, t in enumerate(ts):
        arr[i] = _mat(t, f"{name}[{i}]")
    return arr


def gemm(a, b, out, stream=None):
    """dense_matrix.hpp:40-55: out = a * b."""
    _check(_lib_().pg_gemm(_mat(a, "a"), _mat(b, "b"), 0, _mat(out, "out"), _stream(stream)))
    return out


def gemm_at_b(a, b, out, a_rows=None, stream=None, tensor_cores=False):
    """dense_matrix.hpp:57-76: out = a^T * b; with a_rows (int32/uint32 CUDA
    tensor of b.rows ids) out = gather_rows(a, a_rows)^T * b. Default:
    bit-exact serial chains. tensor_cores=True: split-K tcgen05 3xTF32
    (PG_GEMM_TF32X3) — within the fp32 tolerance, not bit-exact."""
    rows = None if a_rows is None else C.c_void_p(a_rows.data_ptr())
    _check(_lib_().pg_gemm_at_b_ex(_mat(a, "a"), rows, _mat(b, "b"), _mat(out, "out"),
                                   PG_GEMM_TF32X3 if tensor_cores else 0, _stream(stream)))
    return out


def relu(x, out, stream=None):
    """dense_matrix.hpp:98-104"""
    _check(_lib_().pg_relu(_mat(x, "x"), _mat(out, "out"), _stream(stream)))
    return out


def row_softmax(x, out, stream=None):
    """dense_matrix.hpp:116-135 (expf bit-exact with glibc)."""
    _check(_lib_().pg_row_softmax(_mat(x, "x"), _mat(out, "out"), _stream(stream)))
    return out


def top_grad_from_probs(probs, ref, vt_dev, out, stream=None):
    """engine.hpp:146-156 (vt_dev: int32/uint32 CUDA tensor of V_t)."""
    _check(_lib_().pg_top_grad_from_probs(_mat(probs, "probs"), _mat(ref, "ref"), C.c_void_p(vt_dev.data_ptr()),
                                          vt_dev.shape[0], _mat(out, "out"), _stream(stream)))
    return out


def aggregate_pull_filtered(grouped: GroupedCsr, frontiers: FrontierSets, dest_level, src_level, inp, out,
                            overwrite=False, counters=None, stream=None):
    """aggregate.hpp:127-210 (Deterministic): destinations outside frontier
    level dest_level keep their rows, sources outside src_level are
    skipped. ``counters`` (dict) receives the reference's StageCounters."""
    _dev(inp, "input")
    _dev(out, "output", cols=inp.shape[1])
    c = np.zeros(4, np.uint64) if counters is not None else None
    _check(_lib_().pg_aggregate_pull_filtered(grouped._h, frontiers._h, dest_level, src_level,
                                              C.c_void_p(inp.data_ptr()), inp.shape[0], inp.stride(0),
                                              C.c_void_p(out.data_ptr()), out.stride(0), inp.shape[1],
                                              _flags(DETERMINISTIC, overwrite),
                                              None if c is None else _p(c, u64p), _stream(stream)))
    if counters is not None:
        for k, v in zip(("edges_traversed", "groups_executed", "edges_skipped", "groups_skipped"), c.tolist()):
            counters[k] = counters.get(k, 0) + int(v)
    return out


@dataclass
class EpochArtifacts:
    """engine.hpp:27-31: x[0..L], y[0..L-1], pre_act[0..L-1] (device)."""
    x: list
    y: list
    pre_act: list


def forward(graph_grouped: GroupedCsr, x0, weights, stream=None) -> EpochArtifacts:
    """engine.hpp:114-140 over a full-graph grouping."""
    import torch

    n = x0.shape[0]
    y, pre, xs = [], [], []
    cur = x0.shape[1]
    for w in weights:
        y.append(empty_rows(n, cur, device=x0.device))
        pre.append(empty_rows(n, w.shape[1], device=x0.device))
        xs.append(empty_rows(n, w.shape[1], device=x0.device))
        cur = w.shape[1]
    _check(_lib_().pg_forward(graph_grouped._h, _mat(x0, "x0"), _mats(weights, "w"), len(weights), _mats(y, "y"),
                              _mats(pre, "pre"), _mats(xs, "x"), _stream(stream)))
    del torch
    return EpochArtifacts([x0] + xs, y, pre)


def _wgrads(weights):
    return [empty_rows(w.shape[0], w.shape[1], device=w.device) for w in weights]


def backward_epp(prepared: PreparedPaths, arts: EpochArtifacts, top_grad, weights, gather="local",
                 expected_fingerprint=None, x_grads_out=None, counters=None, stream=None):
    """engine.hpp:267-349. Returns W' per layer. ``x_grads_out`` (list)
    receives X^(l)' per path (Local mode); ``counters`` (dict) gets
    backward_edges_per_layer."""
    L = len(weights)
    if len(prepared.groups) != L or prepared.frontiers.L != L:  # engine.hpp:278-279
        raise StalenessError("epp backward: paths were prepared for a different layer count")
    # engine.hpp:280-283: the stamp on the paths must match the fingerprint of
    # the CURRENT graph and training set (recomputed here when not given)
    fp = prepared.current_fingerprint() if expected_fingerprint is None else expected_fingerprint
    hs = (C.c_void_p * max(L, 1))(*[g._h.value for g in prepared.groups])
    wg = _wgrads(weights)
    xg = None
    if x_grads_out is not None:
        xg = [empty_rows(prepared.paths[i].D, weights[L - 1 - i].shape[0], device=top_grad.device) for i in range(L)]
    e = np.zeros(max(L, 1), np.uint64)
    _check(_lib_().pg_backward_epp(hs, prepared.frontiers._h, L, _mats(arts.y, "y"), _mats(arts.pre_act, "pre"),
                                   _mat(top_grad, "top_grad"), _mats(weights, "w"), fp,
                                   {"local": 0, "global": 1}[gather], _mats(wg, "w_grads"),
                                   None if xg is None else _mats(xg, "x_grads"), _p(e, u64p), _stream(stream)))
    if x_grads_out is not None:
        x_grads_out.extend(xg)
    if counters is not None:
        counters["backward_edges_per_layer"] = e[:L].tolist()
    return wg


def backward_all_active(graph_grouped: GroupedCsr, arts: EpochArtifacts, top_grad, weights, x_grads_out=None,
                        counters=None, stream=None):
    """engine.hpp:177-214 (Alg. 1 over the full graph)."""
    L = len(weights)
    n = top_grad.shape[0]
    wg = _wgrads(weights)
    xg = None
    if x_grads_out is not None:
        xg = [empty_rows(n, weights[L - 1 - i].shape[0], device=top_grad.device) for i in range(L)]
    e = np.zeros(max(L, 1), np.uint64)
    _check(_lib_().pg_backward_all_active(graph_grouped._h, L, _mats(arts.y, "y"), _mats(arts.pre_act, "pre"),
                                          _mat(top_grad, "top_grad"), _mats(weights, "w"), _mats(wg, "w_grads"),
                                          None if xg is None else _mats(xg, "x_grads"), _p(e, u64p),
                                          _stream(stream)))
    if x_grads_out is not None:
        x_grads_out.extend(xg)
    if counters is not None:
        counters["backward_edges_per_layer"] = e[:L].tolist()
    return wg


def backward_ifelse(graph_grouped: GroupedCsr, frontiers: FrontierSets, arts: EpochArtifacts, top_grad, weights,
                    x_grads_out=None, counters=None, stream=None):
    """engine.hpp:218-257 (full graph with the frontier activity tests)."""
    L = len(weights)
    n = top_grad.shape[0]
    wg = _wgrads(weights)
    xg = None
    if x_grads_out is not None:
        xg = [empty_rows(n, weights[L - 1 - i].shape[0], device=top_grad.device) for i in range(L)]
    e = np.zeros(max(L, 1), np.uint64)
    _check(_lib_().pg_backward_ifelse(graph_grouped._h, frontiers._h, L, _mats(arts.y, "y"),
                                      _mats(arts.pre_act, "pre"), _mat(top_grad, "top_grad"), _mats(weights, "w"),
                                      _mats(wg, "w_grads"), None if xg is None else _mats(xg, "x_grads"),
                                      None if counters is None else _p(e, u64p), _stream(stream)))
    if x_grads_out is not None:
        x_grads_out.extend(xg)
    if counters is not None:
        counters["backward_edges_per_layer"] = e[:L].tolist()
    return wg
