"""The library's communicator (pg_comm, comm.cu) and its row-sharded stage
(pg_backward_aggregate_sharded): NCCL inside the library, per-owner
broadcasts overlapping the source-segment passes. On one GPU the
communicator has one rank (the whole NCCL path still runs: id, init,
stream/event plumbing, segment passes); with >= 2 visible GPUs a 2-rank NCCL
job checks every rank's rows bit-exact against the single-GPU stage."""
import os
import socket

import numpy as np
import pytest

from conftest import rmat_pairs

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def _paths(pg, orc, n=8192, m=8192 * 40, seed=13, ratio=0.4):
    pairs, n_pad = rmat_pairs(orc, n, m, seed)
    g = pg.build_undirected_csr(pairs, n_hint=n_pad, weights="symnorm")
    vt = pg.sample_training_set(n_pad, ratio, 42)
    return g, pg.prepare_all_paths(g, pg.compute_frontiers(g, vt, 2))


def test_single_rank_comm_stage_bit_exact(pg, orc, cuda):
    import torch

    from paper_2204_02662_b200 import dist as pgd

    comm = pgd.Comm(0, 1, 0, pgd.Comm.unique_id())
    assert comm.nccl_version() >= 21800
    g, paths = _paths(pg, orc)
    for dim in (16, 602):
        for p in paths:
            G = pg.group_neighbors(p, 4)
            y = np.random.default_rng(dim).uniform(-1, 1, size=(p.P, dim)).astype(np.float32)
            yd = pg.empty_rows(p.P, dim)
            yd.copy_(torch.from_numpy(y))
            want = pg.empty_rows(p.D, dim)
            pg.backward_aggregation(G, yd, want, overwrite=True)
            for single in (False, True):
                x = pg.empty_rows(p.D, dim)
                x.fill_(float("nan"))
                comm.backward_aggregation(G, yd, x, [0, p.P], [0, p.D], single_pass=single)
                torch.cuda.synchronize()
                assert np.array_equal(bits(x.cpu().numpy()), bits(want.cpu().numpy()))
            comm.allgather_rows(yd, [0, p.P])
            torch.cuda.synchronize()
            assert np.array_equal(bits(yd.cpu().numpy()), bits(y))
    comm.close()


def test_comm_argument_errors(pg, orc, cuda):
    from paper_2204_02662_b200 import dist as pgd

    comm = pgd.Comm(0, 1, 0, pgd.Comm.unique_id())
    g, paths = _paths(pg, orc, n=1024, m=8192)
    p = paths[1]
    G = pg.group_neighbors(p, 2)
    y = pg.empty_rows(p.P, 8)
    x = pg.empty_rows(p.D, 8)
    with pytest.raises(pg.ConfigError):  # bounds must cover the frontier
        comm.backward_aggregation(G, y, x, [0, p.P - 1], [0, p.D])
    with pytest.raises(pg.ConfigError):
        comm.backward_aggregation(G, y, x, [0, p.P], [0, p.D], mode="grouped")
    with pytest.raises(ValueError):
        pgd.Comm(0, 1, 0, b"short")
    comm.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # bootstrap only
    try:
        import paper_2204_02662_b200 as pg
        from oracle.oracle import Oracle
        from paper_2204_02662_b200 import dist as pgd

        comm = pgd.Comm.from_process_group(rank)
        g, paths = _paths(pg, Oracle())
        ok = True
        prev = None
        for i, p in enumerate(paths):
            dim = 33 + 300 * i
            G = pg.group_neighbors(p, 4)
            db = p.shard_bounds(world)
            pb = pgd.equal_bounds(p.P, world) if prev is None else prev
            y = np.random.default_rng(i).uniform(-1, 1, size=(p.P, dim)).astype(np.float32)
            full = pg.empty_rows(p.P, dim, device=f"cuda:{rank}")
            full.copy_(torch.from_numpy(y))
            want = pg.empty_rows(p.D, dim, device=f"cuda:{rank}")
            pg.backward_aggregation(G, full, want, overwrite=True)
            mine = pg.empty_rows(p.P, dim, device=f"cuda:{rank}")
            mine.fill_(float("nan"))
            a, b = int(pb[rank]), int(pb[rank + 1])
            mine[a:b] = full[a:b]
            for single in (False, True):
                x = pg.empty_rows(int(db[rank + 1] - db[rank]), dim, device=f"cuda:{rank}")
                comm.backward_aggregation(G, mine, x, pb, db, single_pass=single)
                torch.cuda.synchronize()
                ok &= np.array_equal(bits(x.cpu().numpy()), bits(want.cpu().numpy()[db[rank]:db[rank + 1]]))
            prev = db
        comm.close()
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_two_rank_nccl_stage(pg, cuda):
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU visible: NCCL cannot put two ranks on one device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}
