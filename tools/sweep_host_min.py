"""e2e of the Reddit epoch through the host-buffer drop-in (pinned) vs the
pipeline size floor (tuning host_min_mb) and the top path's chunking."""
import os
import statistics
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
    ys, xs = [], []
    for i, p in enumerate(prep.paths):
        yh = torch.empty((p.P, dims[i]), dtype=torch.float32, pin_memory=True).numpy()
        yh[:] = bench.grad_input(p.P, dims[i], i)
        ys.append(yh)
        xs.append(torch.empty((p.D, dims[i]), dtype=torch.float32, pin_memory=True).numpy())
    for mb in (32, 8, 4, 32, 8):
        pg.set_tuning("host_min_mb", mb)
        per_path = [[] for _ in prep.paths]
        for rep in range(8):
            for i in range(len(prep.paths)):
                t = time.perf_counter()
                pg.backward_aggregation(prep.groups[i], ys[i], xs[i], overwrite=True)
                per_path[i].append((time.perf_counter() - t) * 1e3)
        med = [statistics.median(v[2:]) for v in per_path]
        print(f"host_min_mb={mb:3d}: per-path host call ms {[round(m, 3) for m in med]} epoch {sum(med):.3f}",
              flush=True)
    pg.set_tuning("host_min_mb", None)


if __name__ == "__main__":
    main(*sys.argv[1:])
