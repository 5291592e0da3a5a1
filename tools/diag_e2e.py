"""Diagnostics: time the host-buffer drop-in (pg_backward_aggregate_host)
per path on the Reddit-shaped workload, against the device-only kernel."""
import os
import sys
import time

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
    dims = bench.agg_dims(cfg)
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), dims)
    for i, (p, G) in enumerate(zip(prep.paths, prep.groups)):
        dim = dims[i]
        yh = torch.empty((p.P, dim), dtype=torch.float32, pin_memory=True).numpy()
        yh[:] = np.random.default_rng(0).uniform(-1, 1, size=yh.shape)
        xh = torch.empty((p.D, dim), dtype=torch.float32, pin_memory=True).numpy()
        for rep in range(4):
            t = time.perf_counter()
            pg.backward_aggregation(G, yh, xh, overwrite=True)
            dt = time.perf_counter() - t
            print(f"path {i} dim {dim}: host call {dt * 1e3:.2f} ms (rep {rep})", flush=True)
        yd = pg.empty_rows(p.P, dim)
        yd.copy_(torch.from_numpy(yh))
        xd = pg.empty_rows(p.D, dim)
        for rep in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            pg.backward_aggregation(G, yd, xd, overwrite=True)
            torch.cuda.synchronize()
            print(f"path {i}: device call {(time.perf_counter() - t) * 1e3:.2f} ms", flush=True)
        assert np.array_equal(xd.cpu().numpy().view(np.uint32), xh.view(np.uint32))


if __name__ == "__main__":
    main(*sys.argv[1:])
