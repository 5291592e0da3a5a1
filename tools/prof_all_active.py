"""Profiling driver: one backward_all_active (Alg. 1) on a bench config
after a warm-up, for `ncu --metrics gpu__time_duration.sum` launch lists."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2204_02662_b200 as pg  # noqa: E402


def main(config="products"):
    cfg = bench.CONFIGS[config]
    pairs = bench.make_pairs(cfg, pg.gen_rmat)
    g = pg.build_undirected_csr(pairs, n_hint=cfg["V"], weights="symnorm")
    n, f, dims = g.n, cfg["f"], cfg["dims"]
    ins = [f] + dims[:-1]
    x0 = pg.empty_rows(n, f)
    x0.uniform_(0, 1)
    ws = []
    for l in range(len(dims)):
        w = pg.empty_rows(ins[l], dims[l])
        w.uniform_(-0.1, 0.1)
        ws.append(w)
    G = pg.group_neighbors(g, 1)
    arts = pg.forward(G, x0, ws)
    top = pg.empty_rows(n, dims[-1])
    top.uniform_(-1e-3, 1e-3)
    pg.backward_all_active(G, arts, top, ws)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    pg.backward_all_active(G, arts, top, ws)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main(*sys.argv[1:])
