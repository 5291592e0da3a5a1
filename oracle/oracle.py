"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product path.

ctypes views of
  * ``Oracle``: the plain-C restatement (oracle/pathgcn_oracle.c -> liboracle.so);
  * ``Ref``: the reference implementation compiled from its own sources
    (oracle/_ref/libpathgcn_ref.so, see oracle/Makefile and ref_capi.cpp).

Both expose the same numpy-level methods so tests can compare them 1:1 and
compare the CUDA product path (paper_2204_02662_b200) against either. Only
tests/, ``__graft_entry__.smoke()`` and bench.py's reference / cpu_baseline
leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpathgcn_ref.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


def _p(a, t):
    return a.ctypes.data_as(t)


@dataclass
class Csr:
    """The reference CsrGraph (csr_graph.hpp:19-38) as numpy arrays."""
    n: int
    offsets: np.ndarray  # u64[n+1]
    neighbors: np.ndarray  # u32[m]
    weights: np.ndarray  # f64[m]

    @property
    def m(self) -> int:
        return int(self.offsets[-1]) if len(self.offsets) else 0

    def max_degree(self) -> int:
        return int(np.diff(self.offsets).max()) if self.n else 0


@dataclass
class Path:
    """The reference ExecutionPath (execution_path.hpp:16-33) as numpy arrays."""
    layer: int
    dest: np.ndarray  # u32[D] dest_local_to_global
    src: np.ndarray  # u32[S] src_local_to_global
    srcpos: np.ndarray  # u32[S] src_pos_in_parent
    offsets: np.ndarray  # u64[D+1]
    neighbors: np.ndarray  # u32[E] local source ids
    weights: np.ndarray  # f64[E]

    @property
    def D(self):
        return len(self.dest)

    @property
    def S(self):
        return len(self.src)

    @property
    def E(self):
        return int(self.offsets[-1])


@dataclass
class Groups:
    """The reference GroupedCsr (grouping.hpp:14-28), SoA."""
    gs: int
    dest: np.ndarray  # u32[G]
    begin: np.ndarray  # u64[G]
    end: np.ndarray  # u64[G]
    dest_groups: np.ndarray  # u64[D+1]


def build_oracle(force=False):
    if force or not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Oracle:
    """The C restatement (pathgcn_oracle.c)."""

    def __init__(self):
        build_oracle()
        L = C.CDLL(ORACLE_SO)
        self.L = L
        L.orc_gen_rmat.restype = C.c_uint32
        L.orc_gen_rmat.argtypes = [C.c_uint32, C.c_uint64] + [C.c_double] * 4 + [C.c_uint64, u32p]
        L.orc_training_set_size.restype = C.c_uint64
        L.orc_training_set_size.argtypes = [C.c_uint32, C.c_double]
        L.orc_sample_training_set.argtypes = [C.c_uint32, C.c_double, C.c_uint64, u32p]
        L.orc_random_matrix_f32.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_double, f32p]
        L.orc_build_undirected_csr.argtypes = [C.c_int64, u32p, C.c_uint64, u32p, u64p,
                                               C.POINTER(u64p), C.POINTER(u32p)]
        L.orc_assign_edge_weights.argtypes = [C.c_uint32, u64p, u32p, C.c_int, f64p]
        L.orc_free.argtypes = [vp]
        L.orc_graph_fingerprint.restype = C.c_uint64
        L.orc_graph_fingerprint.argtypes = [C.c_uint32, u64p, u32p]
        L.orc_training_fingerprint.restype = C.c_uint64
        L.orc_training_fingerprint.argtypes = [u32p, C.c_uint64]
        L.orc_path_fingerprint.restype = C.c_uint64
        L.orc_path_fingerprint.argtypes = [C.c_uint64] * 3
        L.orc_compute_frontiers.argtypes = [C.c_uint32, u64p, u32p, u32p, C.c_uint64, C.c_uint64, u32p, u64p]
        L.orc_extract_path.argtypes = [C.c_uint32, u64p, u32p, f64p, u32p, C.c_uint32, u32p, C.c_uint32,
                                       u64p, u32p, f64p, u32p, u32p, u64p, u32p]
        L.orc_group_count.restype = C.c_uint64
        L.orc_group_count.argtypes = [C.c_uint32, u64p, C.c_uint32]
        L.orc_group_neighbors.argtypes = [C.c_uint32, u64p, C.c_uint32, u32p, u64p, u64p, u64p]
        L.orc_regression_gs.restype = C.c_uint32
        L.orc_regression_gs.argtypes = [C.c_uint32, C.c_uint64, C.c_double, f64p]
        L.orc_path_regression_gs.restype = C.c_uint32
        L.orc_path_regression_gs.argtypes = [C.c_uint32, C.c_uint64]
        L.orc_grouping_cost.restype = C.c_double
        L.orc_grouping_cost.argtypes = [C.c_uint32, u64p, C.c_uint32, C.c_uint64, C.c_int, C.c_double]
        L.orc_default_candidates.restype = C.c_uint64
        L.orc_default_candidates.argtypes = [C.c_uint32, u32p]
        L.orc_oracle_gs_cost.argtypes = [C.c_uint32, u64p, u32p, C.c_uint64, C.c_uint64, C.c_int,
                                         C.c_double, u32p, f64p]
        L.orc_fast_atomic_commits.restype = C.c_uint64
        L.orc_fast_atomic_commits.argtypes = [C.c_uint32, u64p, C.c_uint32, C.c_uint64]
        L.orc_aggregate_pull_f32.argtypes = [C.c_uint32, u64p, u32p, f64p, f32p, C.c_uint64, f32p]
        L.orc_aggregate_pull_f64.argtypes = [C.c_uint32, u64p, u32p, f64p, f64p, C.c_uint64, f64p]
        L.orc_gemm_a_bt_f32.argtypes = [f32p, C.c_uint64, C.c_uint64, f32p, C.c_uint64, f32p]
        L.orc_gemm_a_bt_f64.argtypes = [f64p, C.c_uint64, C.c_uint64, f64p, C.c_uint64, f64p]
        L.orc_relu_backward_f32.argtypes = [f32p, f32p, C.c_uint64, f32p]
        L.orc_gemm_f32.argtypes = [f32p, C.c_uint64, C.c_uint64, f32p, C.c_uint64, f32p]
        L.orc_gemm_at_b_f32.argtypes = [f32p, C.c_uint64, C.c_uint64, f32p, C.c_uint64, f32p]
        L.orc_relu_f32.argtypes = [f32p, C.c_uint64, f32p]
        L.orc_row_softmax_f32.argtypes = [f32p, C.c_uint64, C.c_uint64, f32p]
        L.orc_top_grad_f32.argtypes = [f32p, f32p, C.c_uint64, C.c_uint64, u32p, C.c_uint64, f32p]
        L.orc_aggregate_pull_filtered_f32.argtypes = [C.c_uint32, u64p, u32p, f64p, f32p, C.c_uint64,
                                                      C.POINTER(C.c_uint8), C.POINTER(C.c_uint8), C.c_uint32,
                                                      f32p, u64p]

    # -- inputs --
    def gen_rmat(self, n, m, a=0.45, b=0.22, c=0.22, d=0.11, seed=7):
        pairs = np.empty((m, 2), np.uint32)
        n_pad = self.L.orc_gen_rmat(n, m, a, b, c, d, seed, _p(pairs, u32p))
        return pairs, int(n_pad)

    def sample_training_set(self, n, ratio, seed):
        k = self.L.orc_training_set_size(n, ratio)
        out = np.empty(k, np.uint32)
        rc = self.L.orc_sample_training_set(n, ratio, seed, _p(out, u32p))
        if rc:
            raise ValueError("training set: bad arguments")
        return out

    def random_matrix_f32(self, rows, cols, seed, lo=-1.0, hi=1.0):
        out = np.empty((rows, cols), np.float32)
        self.L.orc_random_matrix_f32(rows, cols, seed, lo, hi, _p(out, f32p))
        return out

    # -- graph load --
    def build_graph(self, pairs, n_hint=None, symnorm=False) -> Csr:
        pairs = np.ascontiguousarray(pairs, np.uint32).reshape(-1, 2)
        n = C.c_uint32()
        m = C.c_uint64()
        po = u64p()
        pn = u32p()
        rc = self.L.orc_build_undirected_csr(-1 if n_hint is None else n_hint, _p(pairs, u32p),
                                             len(pairs), C.byref(n), C.byref(m), C.byref(po), C.byref(pn))
        if rc:
            raise ValueError("cannot build a graph from an empty edge list without a vertex-count hint")
        offsets = np.ctypeslib.as_array(po, (n.value + 1,)).copy()
        nbrs = np.ctypeslib.as_array(pn, (max(m.value, 1),))[: m.value].copy()
        self.L.orc_free(C.cast(po, vp))
        self.L.orc_free(C.cast(pn, vp))
        w = np.empty(m.value, np.float64)
        self.L.orc_assign_edge_weights(n.value, _p(offsets, u64p), _p(nbrs, u32p), int(symnorm), _p(w, f64p))
        return Csr(n.value, offsets, nbrs, w)

    def graph_fingerprint(self, g: Csr) -> int:
        return self.L.orc_graph_fingerprint(g.n, _p(g.offsets, u64p), _p(g.neighbors, u32p))

    def training_fingerprint(self, vt) -> int:
        vt = np.ascontiguousarray(vt, np.uint32)
        return self.L.orc_training_fingerprint(_p(vt, u32p), len(vt))

    def path_fingerprint(self, g: Csr, vt, L) -> int:
        return self.L.orc_path_fingerprint(self.graph_fingerprint(g), self.training_fingerprint(vt), L)

    # -- execution-path build --
    def compute_frontiers(self, g: Csr, vt, L):
        vt = np.ascontiguousarray(vt, np.uint32)
        cap = max(g.n, len(vt), 1)
        levels = np.empty((L + 1, cap), np.uint32)
        sizes = np.zeros(L + 1, np.uint64)
        rc = self.L.orc_compute_frontiers(g.n, _p(g.offsets, u64p), _p(g.neighbors, u32p), _p(vt, u32p),
                                          len(vt), L, _p(levels, u32p), _p(sizes, u64p))
        if rc:
            raise ValueError("frontiers: layer count must be >= 1 and training set non-empty")
        return [levels[k, : int(sizes[k])].copy() for k in range(L + 1)]

    def extract_path(self, g: Csr, levels, layer) -> Path:
        L = len(levels) - 1
        if layer >= L:
            raise ValueError("execution path: layer index out of range")
        dests = np.ascontiguousarray(levels[L - layer], np.uint32)
        parent = np.ascontiguousarray(levels[L - layer - 1], np.uint32)
        deg = np.diff(g.offsets)
        cap = int(deg[dests].sum()) if len(dests) else 0
        offs = np.empty(len(dests) + 1, np.uint64)
        nb = np.empty(max(cap, 1), np.uint32)
        w = np.empty(max(cap, 1), np.float64)
        src = np.empty(max(len(parent), 1), np.uint32)
        pos = np.empty(max(len(parent), 1), np.uint32)
        E = C.c_uint64()
        S = C.c_uint32()
        self.L.orc_extract_path(g.n, _p(g.offsets, u64p), _p(g.neighbors, u32p), _p(g.weights, f64p),
                                _p(dests, u32p), len(dests), _p(parent, u32p), len(parent), _p(offs, u64p),
                                _p(nb, u32p), _p(w, f64p), _p(src, u32p), _p(pos, u32p), C.byref(E), C.byref(S))
        return Path(layer, dests.copy(), src[: S.value].copy(), pos[: S.value].copy(), offs,
                    nb[: E.value].copy(), w[: E.value].copy())

    def prepare_all_paths(self, g: Csr, levels):
        L = len(levels) - 1
        return [self.extract_path(g, levels, l) for l in range(L - 1, -1, -1)]

    # -- groups / gs --
    def group_neighbors(self, offsets, gs) -> Groups:
        offsets = np.ascontiguousarray(offsets, np.uint64)
        D = len(offsets) - 1
        if gs == 0:
            raise ValueError("group size must be at least 1")
        G = self.L.orc_group_count(D, _p(offsets, u64p), gs)
        gd = np.empty(max(G, 1), np.uint32)
        gb = np.empty(max(G, 1), np.uint64)
        ge = np.empty(max(G, 1), np.uint64)
        dg = np.empty(D + 1, np.uint64)
        self.L.orc_group_neighbors(D, _p(offsets, u64p), gs, _p(gd, u32p), _p(gb, u64p), _p(ge, u64p), _p(dg, u64p))
        return Groups(gs, gd[:G], gb[:G], ge[:G], dg)

    def regression_gs(self, n_vertices, n_edges, avg_degree, beta=None):
        b = None if beta is None else _p(np.asarray(beta, np.float64), f64p)
        return self.L.orc_regression_gs(n_vertices, n_edges, avg_degree, b)

    def path_regression_gs(self, D, E):
        return self.L.orc_path_regression_gs(D, E)

    def grouping_cost(self, offsets, gs, dim, workers, lam):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        return self.L.orc_grouping_cost(len(offsets) - 1, _p(offsets, u64p), gs, dim, workers, lam)

    def default_candidates(self, max_degree):
        out = np.empty(40, np.uint32)
        k = self.L.orc_default_candidates(max_degree, _p(out, u32p))
        return out[:k].copy()

    def oracle_gs_cost(self, offsets, cands, dim, workers, lam):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        cands = np.ascontiguousarray(cands, np.uint32)
        best = C.c_uint32()
        table = np.empty(len(cands), np.float64)
        rc = self.L.orc_oracle_gs_cost(len(offsets) - 1, _p(offsets, u64p), _p(cands, u32p), len(cands), dim,
                                       workers, lam, C.byref(best), _p(table, f64p))
        if rc:
            raise ValueError("oracle_gs: bad arguments")
        return best.value, table

    def fast_atomic_commits(self, offsets, gs, dim):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        return self.L.orc_fast_atomic_commits(len(offsets) - 1, _p(offsets, u64p), gs, dim)

    # -- aggregation / dense --
    def aggregate_pull_f32(self, offsets, nbrs, w, inp, out=None):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        nbrs = np.ascontiguousarray(nbrs, np.uint32)
        w = np.ascontiguousarray(w, np.float64)
        inp = np.ascontiguousarray(inp, np.float32)
        D = len(offsets) - 1
        dim = inp.shape[1]
        out = np.zeros((D, dim), np.float32) if out is None else np.ascontiguousarray(out, np.float32).copy()
        self.L.orc_aggregate_pull_f32(D, _p(offsets, u64p), _p(nbrs, u32p), _p(w, f64p), _p(inp, f32p), dim,
                                      _p(out, f32p))
        return out

    def aggregate_pull_f64(self, offsets, nbrs, w, inp, out=None):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        nbrs = np.ascontiguousarray(nbrs, np.uint32)
        w = np.ascontiguousarray(w, np.float64)
        inp = np.ascontiguousarray(inp, np.float64)
        D = len(offsets) - 1
        dim = inp.shape[1]
        out = np.zeros((D, dim), np.float64) if out is None else np.ascontiguousarray(out, np.float64).copy()
        self.L.orc_aggregate_pull_f64(D, _p(offsets, u64p), _p(nbrs, u32p), _p(w, f64p), _p(inp, f64p), dim,
                                      _p(out, f64p))
        return out

    def gemm_a_bt_f32(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.empty((a.shape[0], b.shape[0]), np.float32)
        self.L.orc_gemm_a_bt_f32(_p(a, f32p), a.shape[0], a.shape[1], _p(b, f32p), b.shape[0], _p(out, f32p))
        return out

    def gemm_a_bt_f64(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.empty((a.shape[0], b.shape[0]), np.float64)
        self.L.orc_gemm_a_bt_f64(_p(a, f64p), a.shape[0], a.shape[1], _p(b, f64p), b.shape[0], _p(out, f64p))
        return out

    def relu_backward_f32(self, grad, pre):
        grad = np.ascontiguousarray(grad, np.float32)
        pre = np.ascontiguousarray(pre, np.float32)
        out = np.empty_like(grad)
        self.L.orc_relu_backward_f32(_p(grad, f32p), _p(pre, f32p), grad.size, _p(out, f32p))
        return out


    # -- the GCN chain (engine.hpp), compositions of the C kernels --
    def gemm_f32(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.empty((a.shape[0], b.shape[1]), np.float32)
        self.L.orc_gemm_f32(_p(a, f32p), a.shape[0], a.shape[1], _p(b, f32p), b.shape[1], _p(out, f32p))
        return out

    def gemm_at_b_f32(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.empty((a.shape[1], b.shape[1]), np.float32)
        self.L.orc_gemm_at_b_f32(_p(a, f32p), a.shape[0], a.shape[1], _p(b, f32p), b.shape[1], _p(out, f32p))
        return out

    def relu_f32(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.L.orc_relu_f32(_p(x, f32p), x.size, _p(out, f32p))
        return out

    def row_softmax_f32(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.L.orc_row_softmax_f32(_p(x, f32p), x.shape[0], x.shape[1], _p(out, f32p))
        return out

    def top_grad_f32(self, probs, ref, vt):
        probs = np.ascontiguousarray(probs, np.float32)
        ref = np.ascontiguousarray(ref, np.float32)
        vt = np.ascontiguousarray(vt, np.uint32)
        out = np.empty_like(probs)
        self.L.orc_top_grad_f32(_p(probs, f32p), _p(ref, f32p), probs.shape[0], probs.shape[1], _p(vt, u32p),
                                len(vt), _p(out, f32p))
        return out

    def aggregate_pull_filtered_f32(self, offsets, nbrs, w, inp, dest_active, src_active, gs):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        nbrs = np.ascontiguousarray(nbrs, np.uint32)
        w = np.ascontiguousarray(w, np.float64)
        inp = np.ascontiguousarray(inp, np.float32)
        da = np.ascontiguousarray(dest_active, np.uint8)
        sa = np.ascontiguousarray(src_active, np.uint8)
        D = len(offsets) - 1
        out = np.zeros((D, inp.shape[1]), np.float32)
        c = np.zeros(4, np.uint64)
        u8p = C.POINTER(C.c_uint8)
        self.L.orc_aggregate_pull_filtered_f32(D, _p(offsets, u64p), _p(nbrs, u32p), _p(w, f64p), _p(inp, f32p),
                                               inp.shape[1], _p(da, u8p), _p(sa, u8p), gs, _p(out, f32p),
                                               _p(c, u64p))
        return out, dict(edges_traversed=int(c[0]), groups_executed=int(c[1]), edges_skipped=int(c[2]),
                         groups_skipped=int(c[3]))

    def forward(self, g: Csr, x0, weights):
        """engine.hpp:114-140 (Deterministic pull over the full graph)."""
        x, y, pre = [np.ascontiguousarray(x0, np.float32)], [], []
        L = len(weights)
        for l, w in enumerate(weights):
            yl = self.aggregate_pull_f32(g.offsets, g.neighbors, g.weights, x[-1])
            p = self.gemm_f32(yl, w)
            x.append(self.relu_f32(p) if l + 1 < L else self.row_softmax_f32(p))
            y.append(yl)
            pre.append(p)
        return dict(x=x, y=y, pre=pre)

    def backward_full(self, g: Csr, arts, top_grad, weights, levels=None, gs=1):
        """engine.hpp:177-214 backward_all_active, or with ``levels`` (the
        frontier arrays) :218-257 backward_ifelse. Returns (w_grads, x_grads
        layer L-1 first, backward_edges_per_layer)."""
        L = len(weights)
        n = len(g.offsets) - 1
        wg, xg, edges = [None] * L, [], []
        gm = np.ascontiguousarray(top_grad, np.float32)
        for l in range(L - 1, -1, -1):
            wg[l] = self.gemm_at_b_f32(arts["y"][l], gm)
            yg = self.gemm_a_bt_f32(gm, weights[l])
            if levels is None:
                x = self.aggregate_pull_f32(g.offsets, g.neighbors, g.weights, yg)
                edges.append(int(g.offsets[-1]))
            else:
                da = np.zeros(n, np.uint8)
                da[levels[L - l]] = 1
                sa = np.zeros(n, np.uint8)
                sa[levels[L - l - 1]] = 1
                x, c = self.aggregate_pull_filtered_f32(g.offsets, g.neighbors, g.weights, yg, da, sa, gs)
                edges.append(c["edges_traversed"])
            xg.append(x)
            if l > 0:
                gm = self.relu_backward_f32(x, arts["pre"][l - 1])
        return wg, xg, edges

    def backward_epp(self, paths, levels, arts, top_grad, weights, gather="local"):
        """engine.hpp:267-349 (paths[i] = SG of layer L-1-i, oracle Path
        objects). Returns (w_grads, x_grads per path (Local), edges)."""
        L = len(weights)
        wg, xg, edges = [None] * L, [], []
        if gather == "global":
            n = top_grad.shape[0]
            gm = np.ascontiguousarray(top_grad, np.float32)
            for i in range(L):
                l = L - 1 - i
                p = paths[i]
                wg[l] = self.gemm_at_b_f32(arts["y"][l], gm)
                yg = self.gemm_a_bt_f32(gm, weights[l])
                x = np.zeros((n, yg.shape[1]), np.float32)
                # aggregate_pull_path_global (engine.hpp:352-376), Deterministic
                xr = self.aggregate_pull_f32(p.offsets, p.src[p.neighbors], p.weights, yg)
                x[p.dest] = xr
                edges.append(int(p.offsets[-1]))
                if l > 0:
                    gm = self.relu_backward_f32(x, arts["pre"][l - 1])
            return wg, xg, edges
        gm = np.ascontiguousarray(top_grad[levels[0]], np.float32)
        for i in range(L):
            l = L - 1 - i
            p = paths[i]
            wg[l] = self.gemm_at_b_f32(arts["y"][l][levels[L - l - 1]], gm)
            yg = self.gemm_a_bt_f32(gm, weights[l])
            x = self.aggregate_pull_f32(p.offsets, p.neighbors, p.weights, yg[p.srcpos])
            xg.append(x)
            edges.append(int(p.offsets[-1]))
            if l > 0:
                gm = self.relu_backward_f32(x, arts["pre"][l - 1][levels[L - l]])
        return wg, xg, edges


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Ref:
    """The reference itself, compiled from /root/reference sources (oracle/_ref)."""

    def __init__(self):
        if not ref_available():
            raise FileNotFoundError(REF_SO + " missing (make -C oracle ref with /root/reference present)")
        L = C.CDLL(REF_SO)
        self.L = L
        L.ref_last_error.argtypes = [C.c_char_p, C.c_uint64]
        for f in ("ref_free_graph", "ref_free_front", "ref_free_path", "ref_free_groups"):
            getattr(L, f).argtypes = [vp]
        L.ref_gen_rmat.restype = C.c_uint32
        L.ref_gen_rmat.argtypes = [C.c_uint32, C.c_uint64] + [C.c_double] * 4 + [C.c_uint64, u32p]
        L.ref_graph_build.argtypes = [C.c_int64, u32p, C.c_uint64, C.c_int, C.POINTER(vp)]
        L.ref_graph_load_file.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
        L.ref_graph_from_csr.argtypes = [C.c_uint32, u64p, u32p, f64p, C.POINTER(vp)]
        L.ref_graph_info.argtypes = [vp, u32p, u64p, u32p, u64p]
        L.ref_graph_export.argtypes = [vp, u64p, u32p, f64p]
        L.ref_training_set_size.restype = C.c_uint64
        L.ref_training_set_size.argtypes = [C.c_uint32, C.c_double]
        L.ref_sample_training_set.argtypes = [C.c_uint32, C.c_double, C.c_uint64, u32p]
        L.ref_training_fingerprint.restype = C.c_uint64
        L.ref_training_fingerprint.argtypes = [u32p, C.c_uint64]
        L.ref_path_fingerprint.restype = C.c_uint64
        L.ref_path_fingerprint.argtypes = [vp, u32p, C.c_uint64, C.c_uint64]
        L.ref_frontiers.argtypes = [vp, u32p, C.c_uint64, C.c_uint64, C.POINTER(vp)]
        L.ref_frontier_size.restype = C.c_uint64
        L.ref_frontier_size.argtypes = [vp, C.c_uint64]
        L.ref_frontier_export.argtypes = [vp, C.c_uint64, u32p]
        L.ref_path.argtypes = [vp, vp, C.c_uint64, C.POINTER(vp)]
        L.ref_path_info.argtypes = [vp, u32p, u32p, u64p]
        L.ref_path_export.argtypes = [vp, u32p, u32p, u32p, u64p, u32p, f64p]
        L.ref_path_sample.argtypes = [vp, C.c_uint32, C.POINTER(vp)]
        L.ref_path_from_arrays.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, u32p, u32p, u32p, u64p, u32p, f64p,
                                           C.POINTER(vp)]
        L.ref_group.argtypes = [vp, C.c_int, C.c_uint32, C.POINTER(vp)]
        L.ref_group_count.restype = C.c_uint64
        L.ref_group_count.argtypes = [vp]
        L.ref_group_export.argtypes = [vp, u32p, u64p, u64p, u64p]
        L.ref_regression_gs.restype = C.c_uint32
        L.ref_regression_gs.argtypes = [C.c_uint32, C.c_uint64, C.c_double, f64p]
        L.ref_path_regression_gs.restype = C.c_uint32
        L.ref_path_regression_gs.argtypes = [vp]
        L.ref_default_candidates.restype = C.c_uint64
        L.ref_default_candidates.argtypes = [C.c_uint32, u32p]
        L.ref_grouping_cost.restype = C.c_double
        L.ref_grouping_cost.argtypes = [vp, C.c_uint64, C.c_int, C.c_double]
        L.ref_oracle_gs_cost.argtypes = [vp, C.c_int, u32p, C.c_uint64, C.c_uint64, C.c_int, C.c_double,
                                         u32p, f64p]
        L.ref_aggregate_pull_f32.argtypes = [vp, f32p, C.c_uint64, C.c_uint64, f32p, C.c_int, C.c_int, u64p]
        L.ref_aggregate_pull_f64.argtypes = [vp, f64p, C.c_uint64, C.c_uint64, f64p, C.c_int, C.c_int, u64p]
        L.ref_gemm_a_bt_f32.argtypes = [f32p, C.c_uint64, C.c_uint64, f32p, C.c_uint64, f32p]
        L.ref_gemm_a_bt_f64.argtypes = [f64p, C.c_uint64, C.c_uint64, f64p, C.c_uint64, f64p]
        L.ref_backward_aggregation_f32.argtypes = [vp, vp, f32p, C.c_uint64, C.c_uint64, f32p, C.c_int,
                                                   C.c_int, f64p]
        L.ref_epp_chain_f32.argtypes = [vp, u32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.c_uint64, C.c_uint32, C.c_uint32, f32p, C.POINTER(f32p),
                                        C.POINTER(f32p), C.POINTER(f32p), C.POINTER(f32p)]
        L.ref_chain_f32.argtypes = [vp, u32p, C.c_uint64, C.c_uint64, C.c_uint64, u64p, f32p, C.POINTER(f32p),
                                    f32p, C.c_uint32, C.c_uint32, C.c_int, C.POINTER(f32p), C.POINTER(f32p),
                                    C.POINTER(f32p), f32p, C.POINTER(f32p), C.POINTER(f32p), u64p]

    def _check(self, rc):
        if rc:
            buf = C.create_string_buffer(1024)
            self.L.ref_last_error(buf, 1024)
            raise RefError(rc, buf.value.decode())

    def max_threads(self):
        return self.L.ref_max_threads()

    # handles ------------------------------------------------------------
    def graph_handle(self, g: Csr):
        h = vp()
        self._check(self.L.ref_graph_from_csr(g.n, _p(g.offsets, u64p), _p(g.neighbors, u32p),
                                              _p(g.weights, f64p), C.byref(h)))
        return h

    def _export_graph(self, h) -> Csr:
        n = C.c_uint32()
        m = C.c_uint64()
        md = C.c_uint32()
        fp = C.c_uint64()
        self.L.ref_graph_info(h, C.byref(n), C.byref(m), C.byref(md), C.byref(fp))
        offs = np.empty(n.value + 1, np.uint64)
        nb = np.empty(max(m.value, 1), np.uint32)
        w = np.empty(max(m.value, 1), np.float64)
        self.L.ref_graph_export(h, _p(offs, u64p), _p(nb, u32p), _p(w, f64p))
        return Csr(n.value, offs, nb[: m.value].copy(), w[: m.value].copy())

    # inputs -------------------------------------------------------------
    def gen_rmat(self, n, m, a=0.45, b=0.22, c=0.22, d=0.11, seed=7):
        pairs = np.empty((m, 2), np.uint32)
        n_pad = self.L.ref_gen_rmat(n, m, a, b, c, d, seed, _p(pairs, u32p))
        return pairs, int(n_pad)

    def sample_training_set(self, n, ratio, seed):
        k = self.L.ref_training_set_size(n, ratio)
        out = np.empty(k, np.uint32)
        self._check(self.L.ref_sample_training_set(n, ratio, seed, _p(out, u32p)))
        return out

    def build_graph(self, pairs, n_hint=None, symnorm=False) -> Csr:
        pairs = np.ascontiguousarray(pairs, np.uint32).reshape(-1, 2)
        h = vp()
        self._check(self.L.ref_graph_build(-1 if n_hint is None else n_hint, _p(pairs, u32p), len(pairs),
                                           int(symnorm), C.byref(h)))
        try:
            return self._export_graph(h)
        finally:
            self.L.ref_free_graph(h)

    def load_graph_file(self, path, symnorm=False) -> Csr:
        h = vp()
        self._check(self.L.ref_graph_load_file(path.encode(), int(symnorm), C.byref(h)))
        try:
            return self._export_graph(h)
        finally:
            self.L.ref_free_graph(h)

    def graph_fingerprint(self, g: Csr) -> int:
        h = self.graph_handle(g)
        n = C.c_uint32()
        m = C.c_uint64()
        md = C.c_uint32()
        fp = C.c_uint64()
        self.L.ref_graph_info(h, C.byref(n), C.byref(m), C.byref(md), C.byref(fp))
        self.L.ref_free_graph(h)
        return fp.value

    def training_fingerprint(self, vt) -> int:
        vt = np.ascontiguousarray(vt, np.uint32)
        return self.L.ref_training_fingerprint(_p(vt, u32p), len(vt))

    def path_fingerprint(self, g: Csr, vt, L) -> int:
        vt = np.ascontiguousarray(vt, np.uint32)
        h = self.graph_handle(g)
        r = self.L.ref_path_fingerprint(h, _p(vt, u32p), len(vt), L)
        self.L.ref_free_graph(h)
        return r

    # path build ---------------------------------------------------------
    def frontier_handle(self, hg, vt, L):
        vt = np.ascontiguousarray(vt, np.uint32)
        hf = vp()
        self._check(self.L.ref_frontiers(hg, _p(vt, u32p), len(vt), L, C.byref(hf)))
        return hf

    def compute_frontiers(self, g: Csr, vt, L):
        hg = self.graph_handle(g)
        try:
            hf = self.frontier_handle(hg, vt, L)
        finally:
            self.L.ref_free_graph(hg)
        out = []
        for k in range(L + 1):
            a = np.empty(max(self.L.ref_frontier_size(hf, k), 1), np.uint32)
            self.L.ref_frontier_export(hf, k, _p(a, u32p))
            out.append(a[: self.L.ref_frontier_size(hf, k)].copy())
        self.L.ref_free_front(hf)
        return out

    def export_path(self, hp, layer) -> Path:
        D = C.c_uint32()
        S = C.c_uint32()
        E = C.c_uint64()
        self.L.ref_path_info(hp, C.byref(D), C.byref(S), C.byref(E))
        dest = np.empty(max(D.value, 1), np.uint32)
        src = np.empty(max(S.value, 1), np.uint32)
        pos = np.empty(max(S.value, 1), np.uint32)
        offs = np.empty(D.value + 1, np.uint64)
        nb = np.empty(max(E.value, 1), np.uint32)
        w = np.empty(max(E.value, 1), np.float64)
        self.L.ref_path_export(hp, _p(dest, u32p), _p(src, u32p), _p(pos, u32p), _p(offs, u64p), _p(nb, u32p),
                               _p(w, f64p))
        return Path(layer, dest[: D.value].copy(), src[: S.value].copy(), pos[: S.value].copy(), offs,
                    nb[: E.value].copy(), w[: E.value].copy())

    def prepare_all_paths(self, g: Csr, vt, L):
        """frontiers + prepare_all_paths (execution_path.cpp:90-96), SG_{L-1} first."""
        hg = self.graph_handle(g)
        hf = self.frontier_handle(hg, vt, L)
        paths = []
        try:
            for layer in range(L - 1, -1, -1):
                hp = vp()
                self._check(self.L.ref_path(hg, hf, layer, C.byref(hp)))
                paths.append(self.export_path(hp, layer))
                self.L.ref_free_path(hp)
        finally:
            self.L.ref_free_front(hf)
            self.L.ref_free_graph(hg)
        return paths

    def _csr_handle(self, offsets, nbrs, w):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        nbrs = np.ascontiguousarray(nbrs, np.uint32)
        w = np.ascontiguousarray(w, np.float64)
        h = vp()
        self._check(self.L.ref_graph_from_csr(len(offsets) - 1, _p(offsets, u64p), _p(nbrs, u32p), _p(w, f64p),
                                              C.byref(h)))
        return h, (offsets, nbrs, w)

    def group_neighbors(self, offsets, gs) -> Groups:
        offsets = np.ascontiguousarray(offsets, np.uint64)
        E = int(offsets[-1])
        h, keep = self._csr_handle(offsets, np.zeros(max(E, 1), np.uint32), np.zeros(max(E, 1)))
        hgr = vp()
        try:
            self._check(self.L.ref_group(h, 0, gs, C.byref(hgr)))
            G = self.L.ref_group_count(hgr)
            gd = np.empty(max(G, 1), np.uint32)
            gb = np.empty(max(G, 1), np.uint64)
            ge = np.empty(max(G, 1), np.uint64)
            dg = np.empty(len(offsets), np.uint64)
            self.L.ref_group_export(hgr, _p(gd, u32p), _p(gb, u64p), _p(ge, u64p), _p(dg, u64p))
            self.L.ref_free_groups(hgr)
        finally:
            self.L.ref_free_graph(h)
        return Groups(gs, gd[:G], gb[:G], ge[:G], dg)

    def regression_gs(self, n_vertices, n_edges, avg_degree, beta=None):
        b = None if beta is None else _p(np.asarray(beta, np.float64), f64p)
        return self.L.ref_regression_gs(n_vertices, n_edges, avg_degree, b)

    def default_candidates(self, max_degree):
        out = np.empty(40, np.uint32)
        k = self.L.ref_default_candidates(max_degree, _p(out, u32p))
        return out[:k].copy()

    def grouping_cost(self, offsets, gs, dim, workers, lam):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        E = int(offsets[-1])
        h, keep = self._csr_handle(offsets, np.zeros(max(E, 1), np.uint32), np.zeros(max(E, 1)))
        hgr = vp()
        try:
            self._check(self.L.ref_group(h, 0, gs, C.byref(hgr)))
            c = self.L.ref_grouping_cost(hgr, dim, workers, lam)
            self.L.ref_free_groups(hgr)
        finally:
            self.L.ref_free_graph(h)
        return c

    def oracle_gs_cost(self, offsets, cands, dim, workers, lam):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        cands = np.ascontiguousarray(cands, np.uint32)
        E = int(offsets[-1])
        h, keep = self._csr_handle(offsets, np.zeros(max(E, 1), np.uint32), np.zeros(max(E, 1)))
        best = C.c_uint32()
        table = np.empty(len(cands), np.float64)
        try:
            self._check(self.L.ref_oracle_gs_cost(h, 0, _p(cands, u32p), len(cands), dim, workers, lam,
                                                  C.byref(best), _p(table, f64p)))
        finally:
            self.L.ref_free_graph(h)
        return best.value, table

    def aggregate_pull(self, offsets, nbrs, w, inp, gs=1, fast=False, workers=0, out=None):
        """aggregate_pull<T> (aggregate.hpp:56-122); T from inp.dtype (f32/f64)."""
        f64 = inp.dtype == np.float64
        dt = np.float64 if f64 else np.float32
        inp = np.ascontiguousarray(inp, dt)
        h, keep = self._csr_handle(offsets, nbrs, w)
        D = len(keep[0]) - 1
        out = np.zeros((D, inp.shape[1]), dt) if out is None else np.ascontiguousarray(out, dt).copy()
        counters = np.zeros(3, np.uint64)
        hgr = vp()
        try:
            self._check(self.L.ref_group(h, 0, gs, C.byref(hgr)))
            fn = self.L.ref_aggregate_pull_f64 if f64 else self.L.ref_aggregate_pull_f32
            pt = f64p if f64 else f32p
            self._check(fn(hgr, _p(inp, pt), inp.shape[0], inp.shape[1], _p(out, pt), int(fast), workers,
                           _p(counters, u64p)))
            self.L.ref_free_groups(hgr)
        finally:
            self.L.ref_free_graph(h)
        return out, counters

    def gemm_a_bt(self, a, b):
        f64 = a.dtype == np.float64
        dt = np.float64 if f64 else np.float32
        a = np.ascontiguousarray(a, dt)
        b = np.ascontiguousarray(b, dt)
        out = np.empty((a.shape[0], b.shape[0]), dt)
        pt = f64p if f64 else f32p
        fn = self.L.ref_gemm_a_bt_f64 if f64 else self.L.ref_gemm_a_bt_f32
        self._check(fn(_p(a, pt), a.shape[0], a.shape[1], _p(b, pt), b.shape[0], _p(out, pt)))
        return out

    def epp_chain_f32(self, g: Csr, vt, L, f, dim0, classes, seed, graph_gs=4, path_gs=2):
        """Real gradient chain operands (see ref_capi.cpp ref_epp_chain_f32)."""
        vt = np.ascontiguousarray(vt, np.uint32)
        levels = self.compute_frontiers(g, vt, L)
        dims = [dim0] * L
        dims[-1] = classes
        in_dims = [f] + dims[:-1]
        top = np.empty((len(levels[0]), classes), np.float32)
        w = [np.empty((in_dims[l], dims[l]), np.float32) for l in range(L)]
        pre, yg, xg = [], [], []
        for i in range(L):
            l = L - 1 - i
            yg.append(np.empty((len(levels[i]), in_dims[l]), np.float32))
            xg.append(np.empty((len(levels[i + 1]), in_dims[l]), np.float32))
            pre.append(np.empty((len(levels[i + 1]), dims[l - 1]) if l > 0 else (1, 1), np.float32))
        arr = lambda lst: (f32p * len(lst))(*[_p(x, f32p) for x in lst])
        hg = self.graph_handle(g)
        try:
            self._check(self.L.ref_epp_chain_f32(hg, _p(vt, u32p), len(vt), L, f, dim0, classes, seed, graph_gs,
                                                 path_gs, _p(top, f32p), arr(w), arr(pre), arr(yg), arr(xg)))
        finally:
            self.L.ref_free_graph(hg)
        return dict(levels=levels, top_g=top, w=w, pre_c=pre, y_grad=yg, x_grad=xg)

    # the reference's timed stage (engine.hpp:331-338) on a sub-sampled path
    def backward_stage_handles(self, g: Csr, vt, L, gs_list=None, sample_stride=1):
        """Build reference handles for all paths (optionally stride-sampled) + groupings."""
        hg = self.graph_handle(g)
        hf = self.frontier_handle(hg, vt, L)
        items = []
        for i, layer in enumerate(range(L - 1, -1, -1)):
            hp = vp()
            self._check(self.L.ref_path(hg, hf, layer, C.byref(hp)))
            # gs of the full path (train.hpp:63-64), kept for its sample
            gs = self.L.ref_path_regression_gs(hp) if gs_list is None else gs_list[i]
            if sample_stride > 1:
                hs = vp()
                self._check(self.L.ref_path_sample(hp, sample_stride, C.byref(hs)))
                self.L.ref_free_path(hp)
                hp = hs
            hgr = vp()
            self._check(self.L.ref_group(hp, 1, gs, C.byref(hgr)))
            D = C.c_uint32()
            S = C.c_uint32()
            E = C.c_uint64()
            self.L.ref_path_info(hp, C.byref(D), C.byref(S), C.byref(E))
            items.append(dict(hp=hp, hgr=hgr, layer=layer, gs=gs, D=D.value, S=S.value, E=E.value))
        self.L.ref_free_front(hf)
        self.L.ref_free_graph(hg)
        return items

    def stage_items_from_arrays(self, paths, sample_stride=1, gs_list=None):
        """Reference handles for paths given as dicts of ExecutionPath arrays
        (dest, src, srcpos, offsets, neighbors, weights, layer), optionally
        stride-sampled (ref_path_sample), grouped with regression gs."""
        items = []
        for i, p in enumerate(paths):
            arr = {k: np.ascontiguousarray(p[k]) for k in ("dest", "src", "srcpos", "offsets", "neighbors", "weights")}
            hp = vp()
            self._check(self.L.ref_path_from_arrays(
                p["layer"], len(arr["dest"]), len(arr["src"]), _p(arr["dest"], u32p), _p(arr["src"], u32p),
                _p(arr["srcpos"], u32p), _p(arr["offsets"], u64p), _p(arr["neighbors"], u32p),
                _p(arr["weights"], f64p), C.byref(hp)))
            gs = self.L.ref_path_regression_gs(hp) if gs_list is None else gs_list[i]
            if sample_stride > 1:
                hs = vp()
                self._check(self.L.ref_path_sample(hp, sample_stride, C.byref(hs)))
                self.L.ref_free_path(hp)
                hp = hs
            hgr = vp()
            self._check(self.L.ref_group(hp, 1, gs, C.byref(hgr)))
            D = C.c_uint32()
            S = C.c_uint32()
            E = C.c_uint64()
            self.L.ref_path_info(hp, C.byref(D), C.byref(S), C.byref(E))
            items.append(dict(hp=hp, hgr=hgr, layer=p["layer"], gs=gs, D=D.value, S=S.value, E=E.value))
        return items

    def run_backward_stage(self, item, y_grad, fast=False, workers=0, want_out=False):
        y_grad = np.ascontiguousarray(y_grad, np.float32)
        secs = C.c_double()
        out = np.empty((item["D"], y_grad.shape[1]), np.float32) if want_out else None
        self._check(self.L.ref_backward_aggregation_f32(item["hp"], item["hgr"], _p(y_grad, f32p), y_grad.shape[0],
                                                        y_grad.shape[1], None if out is None else _p(out, f32p),
                                                        int(fast), workers, C.byref(secs)))
        return secs.value, out

    def chain_f32(self, g: Csr, vt, x0, weights, rmat, mode, graph_gs=4, path_gs=2):
        """The reference's forward + top_grad_from_probs + backward variant
        on given inputs (ref_capi.cpp ref_chain_f32). mode: 0 all-active,
        1 ifelse, 2 epp local, 3 epp global."""
        vt = np.ascontiguousarray(vt, np.uint32)
        x0 = np.ascontiguousarray(x0, np.float32)
        L = len(weights)
        n = g.n
        f = x0.shape[1]
        dims = np.array([w.shape[1] for w in weights], np.uint64)
        in_dims = [f] + dims[:-1].tolist()
        ws = [np.ascontiguousarray(w, np.float32) for w in weights]
        rmat = np.ascontiguousarray(rmat, np.float32)
        y = [np.empty((n, in_dims[l]), np.float32) for l in range(L)]
        pre = [np.empty((n, int(dims[l])), np.float32) for l in range(L)]
        x = [np.empty((n, int(dims[l])), np.float32) for l in range(L)]
        top = np.empty((n, int(dims[-1])), np.float32)
        wg = [np.empty_like(w) for w in ws]
        xg = [np.empty((n, in_dims[L - 1 - i]), np.float32) for i in range(L)] if mode == 0 else None
        edges = np.zeros(L, np.uint64)
        arr = lambda lst: (f32p * len(lst))(*[_p(a, f32p) for a in lst])
        hg = self.graph_handle(g)
        try:
            self._check(self.L.ref_chain_f32(hg, _p(vt, u32p), len(vt), L, f, _p(dims, u64p), _p(x0, f32p), arr(ws),
                                             _p(rmat, f32p), graph_gs, path_gs, mode, arr(y), arr(pre), arr(x),
                                             _p(top, f32p), arr(wg), None if xg is None else arr(xg),
                                             _p(edges, u64p)))
        finally:
            self.L.ref_free_graph(hg)
        return dict(y=y, pre=pre, x=[x0] + x, top=top, w_grads=wg, x_grads=xg, edges=edges.tolist())

    def free_stage_handles(self, items):
        for it in items:
            self.L.ref_free_groups(it["hgr"])
            self.L.ref_free_path(it["hp"])
