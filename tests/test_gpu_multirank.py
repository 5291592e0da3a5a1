"""The multi-GPU data path with the real CUDA kernels: two ranks (gloo, both
on cuda:0 — this sandbox has one GPU) shard every path's destination rows,
all_gather their padded y_grad row shards, run the remapped row-range SpMM
and must reproduce the oracle bit for bit. Only NCCL itself is not covered
(the driver's multi-GPU bench runs it)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    import paper_2204_02662_b200 as pg
    from conftest import rmat_pairs
    from oracle.oracle import Oracle
    from paper_2204_02662_b200 import dist as pgd

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = True
    try:
        orc = Oracle()
        pairs, n_pad = rmat_pairs(orc, 8192, 8192 * 16, 23)
        vt = orc.sample_training_set(8192, 0.3, 2)
        g = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm")
        paths = pg.prepare_all_paths(g, pg.compute_frontiers(g, vt, 2))
        og = orc.build_graph(pairs, n_hint=n_pad, symnorm=True)
        ops = orc.prepare_all_paths(og, orc.compute_frontiers(og, vt, 2))
        plan = pgd.plan([None, None], [p.P for p in paths], world, [p.shard_bounds(world) for p in paths])
        dims = [16, 602]
        for i, (p, op) in enumerate(zip(paths, ops)):
            sh = plan[i]
            y = np.random.default_rng(i).uniform(-1, 1, size=(p.P, dims[i])).astype(np.float32)
            ld = pg.padded_ld(dims[i])
            ys = torch.zeros((sh.max_rows, ld), dtype=torch.float32, device="cuda")
            pb, pe = sh.my_parent_rows(rank)
            ys[: pe - pb, : dims[i]] = torch.from_numpy(y[pb:pe]).cuda()
            yf = torch.empty((sh.gathered_rows, ld), dtype=torch.float32, device="cuda")
            pgd.allgather_rows(ys, yf)
            G = pg.group_neighbors(p, 5)
            G.remap_sources(sh.source_map, sh.gathered_rows)
            db, de = sh.my_dest_rows(rank)
            x = pg.empty_rows(de - db, dims[i])
            pg.backward_aggregation(G, yf[:, : dims[i]], x, overwrite=True, rows=(db, de))
            torch.cuda.synchronize()
            want = orc.aggregate_pull_f32(op.offsets, op.neighbors, op.weights, y[op.srcpos])[db:de]
            ok = ok and np.array_equal(x.cpu().numpy().view(np.uint32), want.view(np.uint32))
            # the default exchange: unpadded all-gather-v, no remap
            G.remap_sources(None, 0)
            fv = torch.zeros((p.P, ld), dtype=torch.float32, device="cuda")
            fv[pb:pe, : dims[i]] = torch.from_numpy(y[pb:pe]).cuda()
            pgd.allgatherv_rows(fv, sh.parent_bounds, rank)
            x2 = pg.empty_rows(de - db, dims[i])
            pg.backward_aggregation(G, fv[:, : dims[i]], x2, overwrite=True, rows=(db, de))
            torch.cuda.synchronize()
            ok = ok and np.array_equal(x2.cpu().numpy().view(np.uint32), want.view(np.uint32))
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()
    q.put((rank, ok))


def test_two_ranks_on_device_match_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}, res
    assert all(p.exitcode == 0 for p in procs)
