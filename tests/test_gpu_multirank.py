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


def _chain_worker(rank, world, port, q):
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
        pairs, n_pad = rmat_pairs(orc, 4096, 4096 * 12, 31)
        vt = orc.sample_training_set(4096, 0.2, 5)
        g = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm")
        f, dims = 37, [19, 6]
        prep = pg.prepare_paths(g, vt, 2, [dims[0], f])
        rng = np.random.default_rng(9)  # identical inputs on every rank

        def dev(a):
            t = pg.empty_rows(a.shape[0], a.shape[1])
            t.copy_(torch.from_numpy(a))
            return t

        x0 = dev(rng.uniform(0, 1, (g.n, f)).astype(np.float32))
        ws = [dev(rng.uniform(-0.5, 0.5, (f, dims[0])).astype(np.float32)),
              dev(rng.uniform(-0.5, 0.5, (dims[0], dims[1])).astype(np.float32))]
        r = np.zeros((g.n, dims[1]), np.float32)
        r[vt, rng.integers(0, dims[1], len(vt))] = 1
        arts = pg.forward(pg.group_neighbors(g, 3), x0, ws)
        top = pg.empty_rows(g.n, dims[1])
        pg.top_grad_from_probs(arts.x[-1], dev(r), torch.from_numpy(vt.astype(np.int32)).cuda(), top)
        want = pg.backward_epp(prep, arts, top, ws)
        plan = pgd.plan([None, None], [p.P for p in prep.paths], world, [p.shard_bounds(world) for p in prep.paths])
        got = pgd.backward_epp(prep, arts, top, ws, plan, rank)
        torch.cuda.synchronize()
        for a, b in zip(got, want):
            ok = ok and torch.equal(a.view(torch.int32), b.view(torch.int32))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()
    q.put((rank, ok))


def test_sharded_backward_epp_chain_matches_single_gpu():
    """dist.backward_epp (row-sharded chain, narrow g all-gathered, W' and
    y_grad recomputed per rank) == the single-GPU chain, bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_chain_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}, res
    assert all(p.exitcode == 0 for p in procs)
