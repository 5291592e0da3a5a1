"""Profiling driver: one backward_epp (Local) on a bench config after a
warm-up, for `ncu --metrics gpu__time_duration.sum` launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2204_02662_b200 as pg  # noqa: E402


def main(config="reddit"):
    cfg = bench.CONFIGS[config]
    pairs = bench.make_pairs(cfg, pg.gen_rmat)
    vt = pg.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    g = pg.build_undirected_csr(pairs, n_hint=cfg["V"], weights="symnorm")
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), bench.agg_dims(cfg))
    n, f, dims = g.n, cfg["f"], cfg["dims"]
    ins = [f] + dims[:-1]
    x0 = pg.empty_rows(n, f)
    x0.uniform_(0, 1)
    ws = []
    for l in range(len(dims)):
        w = pg.empty_rows(ins[l], dims[l])
        w.uniform_(-0.1, 0.1)
        ws.append(w)
    arts = pg.forward(pg.group_neighbors(g, 1), x0, ws)
    top = pg.empty_rows(n, dims[-1])
    top.uniform_(-1e-3, 1e-3)
    pg.backward_epp(prep, arts, top, ws)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    pg.backward_epp(prep, arts, top, ws)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pg.backward_epp(prep, arts, top, ws)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"backward_epp {config}: median {sorted(ts)[2]:.3f} ms over 5", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
