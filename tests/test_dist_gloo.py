"""Multi-GPU host logic on CPU (world_size 2, gloo): destination-row shards,
the padded y_grad all_gather and the parent-row source remap must reproduce
the single-process backward aggregation bit for bit. The CUDA
kernel is replaced by the oracle here; the GPU tests cover the kernel with
the same row ranges and remapped edge streams."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2204_02662_b200 import dist as pgd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle

        from conftest import rmat_pairs

        orc = Oracle()
        pairs, n_pad = rmat_pairs(orc, 2048, 2048 * 8, 5)
        g = orc.build_graph(pairs, n_hint=n_pad, symnorm=True)
        vt = orc.sample_training_set(g.n, 0.2, 3)
        paths = orc.prepare_all_paths(g, orc.compute_frontiers(g, vt, 2))
        dims = [16, 37]
        plan = pgd.plan([p.offsets for p in paths], [_parent_rows(p, vt, paths, i) for i, p in enumerate(paths)],
                        world)
        rng = np.random.default_rng(0)
        ok = True
        for i, p in enumerate(paths):
            sh = plan[i]
            P = int(sh.parent_bounds[-1])
            y_full = rng.uniform(-1, 1, size=(P, dims[i])).astype(np.float32)  # same on every rank
            pb, pe = sh.my_parent_rows(rank)
            shard = torch.zeros((sh.max_rows, dims[i]), dtype=torch.float32)
            shard[: pe - pb] = torch.from_numpy(y_full[pb:pe])
            gathered = torch.empty((sh.gathered_rows, dims[i]), dtype=torch.float32)
            pgd.allgather_rows(shard, gathered)
            # remapped edge stream reads the padded buffer in place
            assert np.array_equal(gathered.numpy()[sh.source_map], y_full)
            # unpadded all-gather-v straight into frontier order
            fv = torch.zeros((P, dims[i]), dtype=torch.float32)
            fv[pb:pe] = torch.from_numpy(y_full[pb:pe])
            pgd.allgatherv_rows(fv, sh.parent_bounds, rank)
            assert np.array_equal(fv.numpy(), y_full)
            # the same into a PITCHED view (empty_rows layout, ld > dim): the
            # exchange must move whole padded rows (NCCL copies numel from
            # data_ptr), or the tail rows of every peer shard stay stale
            ld = (dims[i] + 31) // 32 * 32 if dims[i] > 32 else (dims[i] + 3) // 4 * 4
            buf = torch.full((P, ld + 8), float("nan"), dtype=torch.float32)
            pv = buf[:, :dims[i]]
            pv[pb:pe] = torch.from_numpy(y_full[pb:pe])
            assert not pv.is_contiguous()
            pgd.allgatherv_rows(pv, sh.parent_bounds, rank)
            assert np.array_equal(pv.numpy(), y_full)
            bv = torch.full((P, ld + 8), float("nan"), dtype=torch.float32)[:, :dims[i]]
            bv[pb:pe] = torch.from_numpy(y_full[pb:pe])
            for w in pgd.bcast_rows_async(bv, sh.parent_bounds):
                if w is not None:
                    w.wait()
            assert np.array_equal(bv.numpy(), y_full)
            db, de = sh.my_dest_rows(rank)
            offs = p.offsets[db:de + 1]
            src_rows = sh.source_map[p.srcpos[p.neighbors]]  # gather folded + remapped
            mine = orc.aggregate_pull_f32(offs - offs[0], src_rows[offs[0]:offs[-1]], p.weights[offs[0]:offs[-1]],
                                          gathered.numpy())
            full = orc.aggregate_pull_f32(p.offsets, p.neighbors, p.weights, y_full[p.srcpos])
            ok = ok and np.array_equal(mine.view(np.uint32), full[db:de].view(np.uint32))
            # chain rule: this path's destination cut is the next path's parent cut
            if i + 1 < len(paths):
                assert np.array_equal(plan[i + 1].parent_bounds, sh.dest_bounds)
        result_q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def _parent_rows(p, vt, paths, i):
    # |levels[i]|: |V_t| for the top path, the previous path's destinations after
    return len(vt) if i == 0 else paths[i - 1].D


def test_two_rank_shards_match_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert res == {0: True, 1: True}


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_bounds_and_source_map(world):
    rng = np.random.default_rng(world)
    deg = rng.integers(0, 50, size=1000)
    deg[0] = 5000  # hub
    offs = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    b = pgd.edge_balanced_bounds(offs, world)
    assert b[0] == 0 and b[-1] == 1000 and (np.diff(b) >= 0).all()
    m, mr = pgd.padded_source_map(b)
    assert len(set(m.tolist())) == 1000 and m.max() < mr * world
    for r in range(world):
        assert np.array_equal(m[b[r]:b[r + 1]], r * mr + np.arange(b[r + 1] - b[r]))


def test_balance_bounds_moves_cuts_toward_the_slow_shard():
    """dist.balance_bounds: a shard measured slower than its edge share
    loses destination rows; cuts stay monotone and cover every row."""
    from paper_2204_02662_b200 import dist as pgd

    deg = np.array([500, 400, 300] + [10] * 300, np.int64)
    offs = np.concatenate([[0], np.cumsum(deg)])
    b = pgd.edge_balanced_bounds(offs, 4)
    t = [4.0, 1.0, 1.0, 1.0]  # shard 0 (the hubs) twice as slow per edge
    nb = pgd.balance_bounds(offs, b, t)
    assert nb[0] == 0 and nb[-1] == len(deg) and (np.diff(nb) >= 0).all()
    assert nb[1] <= b[1]
    # equal times leave edge-balanced cuts (up to row granularity) in place
    eq = pgd.balance_bounds(offs, b, [1.0] * 4)
    assert np.abs(eq - b).max() <= 1
    # calibrate_bounds on one process: a synthetic cost model
    rate = np.where(np.arange(len(deg)) < 3, 3.0, 1.0)
    cost = lambda b0, b1: float((deg[b0:b1] * rate[b0:b1]).sum())
    cb, t0, t1 = pgd.calibrate_bounds(cost, offs, b, iters=3)
    assert max(t1) <= max(t0)


def test_whole_rows_views():
    """dist.whole_rows: a pitched row view maps to its contiguous padded rows
    (a row slice of it stays contiguous); views whose pitch is not backed by
    storage are refused so the caller packs instead."""
    buf = torch.arange(10 * 12, dtype=torch.float32).reshape(10, 12)
    v = buf[:, :5]
    w = pgd.whole_rows(v)
    assert w.is_contiguous() and w.shape == (10, 12) and w.data_ptr() == v.data_ptr()
    assert w[3:7].is_contiguous() and torch.equal(w[3:7, :5], v[3:7])
    assert pgd.whole_rows(buf) is buf
    # a column slice starting past column 0 of the last row overruns storage
    assert pgd.whole_rows(buf[:, 8:]) is None
    assert pgd.whole_rows(buf.t()) is None
