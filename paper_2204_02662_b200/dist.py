"""Multi-GPU destination-row sharding of the execution paths.

Each rank holds the full graph and all paths (replicated, built on device),
owns an edge-balanced slice of every path's destination rows
(pg_path_shard_bounds) and computes only those rows of X'. The rows of
y_grad entering path i follow the parent frontier levels[i]; they are
produced in the previous path's destination partition (path i-1), or an
equal split of V_t for the top path. Before each path's SpMM one NCCL
all_gather of the padded y_grad row shards gives every rank the full
matrix; the SpMM reads it in place through a remapped edge stream
(parent row p -> rank(p) * max_rows + (p - start(rank(p)))), so no unpad
copy is needed. Only host-side planning lives here; the exchange is
torch.distributed (NCCL on GPU, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def equal_bounds(rows: int, world: int) -> np.ndarray:
    return np.array([(rows * r) // world for r in range(world + 1)], np.int64)


def edge_balanced_bounds(offsets: np.ndarray, world: int) -> np.ndarray:
    """Host restatement of pg_path_shard_bounds: cut dest rows at E*r/world."""
    E = int(offsets[-1])
    D = len(offsets) - 1
    b = [0]
    for r in range(1, world):
        target = (E * r) // world
        row = int(np.searchsorted(offsets[:-1], target, side="left"))
        b.append(max(b[-1], min(row, D)))
    b.append(D)
    return np.array(b, np.int64)


@dataclass
class LayerShard:
    """Row ownership of one path on one rank."""
    parent_bounds: np.ndarray  # world+1 cuts of the parent frontier (y_grad rows)
    dest_bounds: np.ndarray  # world+1 cuts of the destination rows (x_grad rows)
    max_rows: int  # padded y_grad shard rows (allgather unit)
    source_map: np.ndarray  # parent row -> row of the padded allgather buffer

    def my_parent_rows(self, rank):
        return int(self.parent_bounds[rank]), int(self.parent_bounds[rank + 1])

    def my_dest_rows(self, rank):
        return int(self.dest_bounds[rank]), int(self.dest_bounds[rank + 1])

    @property
    def gathered_rows(self):
        return self.max_rows * (len(self.parent_bounds) - 1)


def padded_source_map(parent_bounds: np.ndarray) -> tuple[np.ndarray, int]:
    world = len(parent_bounds) - 1
    sizes = np.diff(parent_bounds)
    max_rows = int(max(sizes.max(initial=0), 1))
    P = int(parent_bounds[-1])
    owner = np.searchsorted(parent_bounds[1:], np.arange(P), side="right")
    local = np.arange(P) - parent_bounds[owner]
    m = (owner * max_rows + local).astype(np.uint32)
    assert owner.max(initial=0) < world
    return m, max_rows


def plan(path_offsets: list, parent_rows: list, world: int, dest_bounds: list | None = None) -> list:
    """LayerShard per path (SG_{L-1} first). path_offsets[i]: u64[D_i+1];
    parent_rows[i] = |levels[i]|; dest_bounds[i] optional precomputed cuts
    (from the device, pg_path_shard_bounds); path_offsets may then be None."""
    out = []
    prev_dest = None
    for i, offs in enumerate(path_offsets):
        db = np.asarray(dest_bounds[i], np.int64) if dest_bounds is not None else edge_balanced_bounds(offs, world)
        if i == 0 or prev_dest is None:
            pb = equal_bounds(parent_rows[i], world)
        else:
            pb = prev_dest
        if int(pb[-1]) != parent_rows[i]:
            raise ValueError("path chain: parent frontier of path i must be the destinations of path i-1")
        smap, mr = padded_source_map(pb)
        out.append(LayerShard(pb, db, mr, smap))
        prev_dest = db
    return out


def whole_rows(t):
    """The contiguous (rows, pitch) tensor behind a pitched row view (an
    ``empty_rows`` matrix, or a column slice of one): NCCL point-to-point and
    broadcast copy ``numel`` elements from ``data_ptr``, so a view with
    ``stride(0) > shape[1]`` must be exchanged as whole padded rows. Returns
    ``t`` itself when it is already contiguous, else None when the pitch is
    not backed by storage (then the caller packs)."""
    if t.is_contiguous():
        return t
    if t.dim() != 2 or t.stride(1) != 1 or t.stride(0) < t.shape[1]:
        return None
    ld = t.stride(0)
    need = t.storage_offset() + t.shape[0] * ld
    if t.untyped_storage().nbytes() < need * t.element_size():
        return None
    w = t.as_strided((t.shape[0], ld), (ld, 1))
    assert w.is_contiguous()
    return w


def allgatherv_rows(full, bounds, rank, group=None):
    """Unpadded all-gather-v in place: rank r owns rows [bounds[r],
    bounds[r+1]) of `full` (frontier order); afterwards every rank holds all
    rows. One grouped NCCL call (batch_isend_irecv): each rank sends its rows
    to every peer and receives theirs straight into place, so uneven
    edge-balanced shards cost no padding and the SpMM needs no remap."""
    import torch.distributed as dist

    world = len(bounds) - 1
    if world == 1:
        return full
    if full.is_cuda and dist.get_backend(group) != "nccl":
        host = full.cpu()
        allgatherv_rows(host, bounds, rank, group)
        full.copy_(host)
        return full
    w = whole_rows(full)
    if w is None:  # pitch not backed by storage: exchange a packed copy
        packed = full.contiguous()
        allgatherv_rows(packed, bounds, rank, group)
        full.copy_(packed)
        return full
    full_rows = w
    b = [int(x) for x in bounds]
    mine = full_rows[b[rank]:b[rank + 1]]
    assert mine.is_contiguous()
    ops = []
    for r in range(world):
        if r == rank:
            continue
        if mine.shape[0]:
            ops.append(dist.P2POp(dist.isend, mine, r, group))
        theirs = full_rows[b[r]:b[r + 1]]
        if theirs.shape[0]:
            ops.append(dist.P2POp(dist.irecv, theirs, r, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return full


def bcast_rows_async(full, bounds, group=None):
    """Per-rank broadcasts of the row shards of `full` (frontier order),
    issued asynchronously in rank order; returns one work per rank (None when
    complete already or empty). Waiting on work s makes the current stream
    wait for rank s's rows only, so source segment s can be aggregated while
    later broadcasts are still in flight."""
    import torch.distributed as dist

    b = [int(x) for x in bounds]
    world = len(b) - 1
    if world == 1:
        return [None]
    if full.is_cuda and dist.get_backend(group) != "nccl":
        host = full.cpu()
        for s in range(world):
            if b[s + 1] > b[s]:
                dist.broadcast(host[b[s]:b[s + 1]], src=s, group=group)
        full.copy_(host)
        return [None] * world
    w = whole_rows(full)
    if w is None:
        raise ValueError("bcast_rows_async: the row pitch of `full` is not backed by storage (pass a contiguous "
                         "or empty_rows matrix)")
    works = []
    for s in range(world):
        works.append(dist.broadcast(w[b[s]:b[s + 1]], src=s, group=group, async_op=True)
                     if b[s + 1] > b[s] else None)
    return works


def allgather_rows(shard, out, group=None):
    """All-gather equal-sized padded row shards: out[world*max_rows, ...].
    NCCL gathers device buffers in place over NVLink; a gloo group (CPU tests,
    single-GPU rehearsal of the N>1 path) stages CUDA tensors through host."""
    import torch.distributed as dist

    if not (shard.is_contiguous() and out.is_contiguous()):
        raise ValueError("allgather_rows: shard and output must be contiguous (NCCL copies numel from data_ptr)")
    if shard.is_cuda and dist.get_backend(group) != "nccl":
        host = out.cpu()
        dist.all_gather_into_tensor(host, shard.cpu(), group=group)
        out.copy_(host)
        return out
    dist.all_gather_into_tensor(out, shard, group=group)
    return out


def backward_epp(prepared, arts, top_grad, weights, plan_, rank, group=None, expected_fingerprint=None, comm=None):
    """engine.hpp:316-346 (Local gather) row-sharded over the ranks of
    ``group``, bit-identical to the single-GPU ``backward_epp``.

    Every rank holds the forward artefacts, W and top_grad (replicated, as in
    data-parallel GCN training). Per path i (layer l = L-1-i):
      * W'[l] = gather_rows(Y[l], levels[i])^T g is computed on every rank
        from the full g — one serial ascending chain per entry, like the
        reference (a sum of per-rank partials + all-reduce would re-associate
        the chain and change the bits);
      * y_grad = g W[l]^T is also recomputed on every rank: it is the SpMM's
        source matrix and every rank gathers arbitrary rows of it, and the
        narrow g (dims[l] wide) is what travels — at Reddit layer 0 that is
        233K x 16 floats (15 MB) instead of the 602-wide y_grad (566 MB);
      * each rank aggregates its edge-balanced destination rows and applies
        relu_backward with the gathered pre-activation rows (engine.hpp:
        340-345), then one all-gather-v of the g row shards (NCCL P2P)
        assembles the next layer's g in frontier order.
    ``plan_`` is ``plan(...)`` over the paths (dest bounds per path).
    ``expected_fingerprint`` (default: recomputed from the graph and training
    set the paths were prepared from) must match every path's stamp, else
    StalenessError (engine.hpp:280-283). ``comm`` (a ``Comm``): the g row
    exchange runs inside the library (NCCL broadcasts), else torch.distributed.
    Returns W' per layer (full, identical on every rank)."""
    import torch

    from . import pathgcn as pg

    L = len(weights)
    if len(prepared.groups) != L or prepared.frontiers.L != L:
        raise pg.StalenessError("epp backward: paths were prepared for a different layer count")
    fp = prepared.current_fingerprint() if expected_fingerprint is None else expected_fingerprint
    for p in prepared.paths:
        if p.fingerprint != fp:
            raise pg.StalenessError("epp backward: execution paths are stale for this graph/training set")
    F = prepared.frontiers
    dev = top_grad.device
    lv = [torch.from_numpy(F.level(k).astype(np.int32)).to(dev) for k in range(L + 1)]
    c = top_grad.shape[1]
    g = pg.empty_rows(lv[0].shape[0], c, device=dev)
    pg.gather_rows(top_grad, lv[0], g)
    w_grads = [None] * L
    for i in range(L):
        l = L - 1 - i
        p, G = prepared.paths[i], prepared.groups[i]
        in_dim = weights[l].shape[0]
        wg = pg.empty_rows(in_dim, weights[l].shape[1], device=dev)
        pg.gemm_at_b(arts.y[l], g, wg, a_rows=lv[i])
        w_grads[l] = wg
        yg = pg.empty_rows(p.P, in_dim, device=dev)
        pg.gemm_a_bt(g, weights[l], yg)
        db, de = plan_[i].my_dest_rows(rank)
        x = pg.empty_rows(de - db, in_dim, device=dev)
        pg.backward_aggregation(G, yg, x, overwrite=True, rows=(db, de))
        if l == 0:
            break
        pre = pg.empty_rows(de - db, in_dim, device=dev)
        pg.gather_rows(arts.pre_act[l - 1], lv[i + 1][db:de], pre)
        g = pg.empty_rows(p.D, in_dim, device=dev)  # pitched: exchanged as whole padded rows
        pg.relu_backward(x, pre, g[db:de])
        if comm is not None:  # the exchange inside the library (NCCL broadcasts)
            comm.allgather_rows(g, plan_[i].dest_bounds)
        else:
            allgatherv_rows(g, plan_[i].dest_bounds, rank, group)
    return w_grads


# ------------------------------------------------ library communicator ----

class Comm:
    """The library's communicator (pg_comm, include/pathgcn_b200.h): one
    NCCL rank on this process's device. The row-sharded stage and the row
    all-gather run INSIDE the library (comm.cu): per-owner broadcasts on its
    communication stream, each source-segment pass of the SpMM starting as
    soon as its owner's rows have landed. torch.distributed only bootstraps
    the 128-byte NCCL id (``from_process_group``)."""

    SINGLE_PASS = 8  # PG_SHARD_SINGLE_PASS

    def __init__(self, device, world, rank, unique_id: bytes):
        import ctypes as C

        from . import _lib

        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self._L = _lib.load()
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        from .pathgcn import _check

        _check(self._L.pg_comm_init_rank(int(device), buf, int(world), int(rank), C.byref(h)))
        self._h = h
        self.world, self.rank, self.device = int(world), int(rank), int(device)

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C

        from . import _lib
        from .pathgcn import _check

        buf = (C.c_uint8 * 128)()
        _check(_lib.load().pg_comm_unique_id(buf))
        return bytes(buf)

    @classmethod
    def from_process_group(cls, device, group=None):
        """Rank 0 of ``group`` makes the id; torch.distributed ships it."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(device, world, rank, obj[0])

    def nccl_version(self):
        import ctypes as C

        from .pathgcn import _check

        v = C.c_int()
        _check(self._L.pg_comm_info(self._h, None, None, C.byref(v)))
        return v.value

    def allgather_rows(self, full, bounds, stream=None):
        """In place: rank s owns rows [bounds[s], bounds[s+1]) of ``full`` (a
        pitched row matrix, e.g. ``empty_rows``); whole padded rows move."""
        import ctypes as C

        from .pathgcn import _check, _p, _stream, u32p

        w = whole_rows(full)
        if w is None:
            raise ValueError("allgather_rows: the row pitch of `full` is not backed by storage")
        b = np.ascontiguousarray(bounds, np.uint32)
        _check(self._L.pg_comm_allgather_rows(self._h, C.c_void_p(w.data_ptr()), w.stride(0), _p(b, u32p),
                                              _stream(stream)))
        return full

    def backward_aggregation(self, grouped, y_full, x_rows, parent_bounds, dest_bounds, mode="deterministic",
                             overwrite=True, single_pass=False, stream=None):
        """pg_backward_aggregate_sharded: this rank's parent rows of ``y_full``
        are filled; the call completes it from the other ranks and aggregates
        this rank's destination rows into ``x_rows``."""
        import ctypes as C

        from .pathgcn import _check, _dev, _flags, _p, _stream, u32p

        pb = np.ascontiguousarray(parent_bounds, np.uint32)
        db = np.ascontiguousarray(dest_bounds, np.uint32)
        p = grouped.base
        _dev(y_full, "y_grad", rows=p.P)
        _dev(x_rows, "x_grad", rows=int(db[self.rank + 1] - db[self.rank]), cols=y_full.shape[1])
        flags = _flags(mode, overwrite) | (self.SINGLE_PASS if single_pass else 0)
        _check(self._L.pg_backward_aggregate_sharded(self._h, grouped._h, _p(pb, u32p), _p(db, u32p),
                                                     C.c_void_p(y_full.data_ptr()), y_full.shape[0],
                                                     y_full.stride(0), C.c_void_p(x_rows.data_ptr()),
                                                     x_rows.stride(0), y_full.shape[1], flags, _stream(stream)))
        return x_rows

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.pg_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def balance_bounds(offsets, bounds, times):
    """One re-balancing step of the destination-row cuts from measured
    per-shard times: inside current shard r every edge is assumed to cost
    times[r] / edges[r]; the new cuts split that piecewise-linear cost into
    equal parts (at destination-row granularity, cuts kept monotone). Edge-
    balanced cuts treat a hub's edges like any others, but a hub is a serial
    chain: the shard holding the biggest hubs runs longest."""
    offsets = np.asarray(offsets, np.int64)
    b = [int(x) for x in bounds]
    world = len(b) - 1
    D = len(offsets) - 1
    cost = np.zeros(D + 1, np.float64)  # cumulative cost at each destination row
    for r in range(world):
        e0, e1 = offsets[b[r]], offsets[b[r + 1]]
        rate = float(times[r]) / max(int(e1 - e0), 1)
        seg = offsets[b[r]:b[r + 1] + 1] - e0
        cost[b[r]:b[r + 1] + 1] = cost[b[r]] + seg * rate
    total = cost[-1]
    out = [0]
    for r in range(1, world):
        row = int(np.searchsorted(cost, total * r / world, side="left"))
        out.append(max(out[-1], min(row, D)))
    out.append(D)
    return np.array(out, np.int64)


def calibrate_bounds(time_shard, offsets, bounds, iters=2, group=None, rank=None):
    """Adjust the cuts until the measured shard times even out: ``time_shard
    (b, e)`` runs destination rows [b, e) and returns milliseconds. With
    ``rank`` set (N GPUs) each rank times its own shard and the times are
    all-gathered, so every rank derives the same cuts; without it (one GPU)
    all shards are timed in turn. Returns (bounds, times before, times after)."""
    import torch

    def measure(bb):
        world = len(bb) - 1
        if rank is None:
            return [time_shard(int(bb[r]), int(bb[r + 1])) for r in range(world)]
        import torch.distributed as dist

        on = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.zeros(world, dtype=torch.float64, device=on)
        t[rank] = time_shard(int(bb[rank]), int(bb[rank + 1]))
        dist.all_reduce(t, group=group)  # every other entry is 0
        return t.cpu().tolist()

    b = np.asarray(bounds, np.int64)
    first = measure(b)
    times = first
    for _ in range(iters):
        nb = balance_bounds(offsets, b, times)
        nt = measure(nb)
        if max(nt) < max(times):
            b, times = nb, nt
        else:
            break
    return b, first, times
