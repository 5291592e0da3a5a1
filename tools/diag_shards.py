"""Diagnostics: per-rank SpMM time of each path's edge-balanced destination
shard (the N-GPU row split timed one shard at a time on one GPU), to see
shard imbalance. Usage: python tools/diag_shards.py [config] [world...]"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2204_02662_b200 as pg  # noqa: E402
from paper_2204_02662_b200 import dist as pgd  # noqa: E402


def main(config="reddit", *worlds):
    worlds = [int(w) for w in worlds] or [2, 4, 8]
    cfg = bench.CONFIGS[config]
    pairs = bench.make_pairs(cfg, pg.gen_rmat)
    vt = pg.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    g = pg.build_undirected_csr(pairs, n_hint=cfg["V"], weights="symnorm")
    dims = bench.agg_dims(cfg)
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), dims)
    for i, p in enumerate(prep.paths):
        y = pg.empty_rows(p.P, dims[i])
        y.uniform_(-1, 1)
        offs = p.export()["offsets"].astype(np.int64)
        for world in worlds:
            b = p.shard_bounds(world)
            ts = []
            for r in range(world):
                x = pg.empty_rows(int(b[r + 1] - b[r]), dims[i])
                rows = (int(b[r]), int(b[r + 1]))
                for _ in range(2):
                    pg.backward_aggregation(prep.groups[i], y, x, overwrite=True, rows=rows)
                ev = []
                for _ in range(5):
                    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    pg.backward_aggregation(prep.groups[i], y, x, overwrite=True, rows=rows)
                    z.record()
                    torch.cuda.synchronize()
                    ev.append(a.elapsed_time(z))
                ts.append(statistics.median(ev))
            edges = [int(offs[b[r + 1]] - offs[b[r]]) for r in range(world)]
            rowsn = [int(b[r + 1] - b[r]) for r in range(world)]
            maxdeg = [int(np.diff(offs[b[r]:b[r + 1] + 1]).max()) if b[r + 1] > b[r] else 0 for r in range(world)]
            print(f"path {i} dim {dims[i]} world {world}: ms {[round(t, 3) for t in ts]} max/mean "
                  f"{max(ts):.3f}/{statistics.mean(ts):.3f} rows {rowsn} maxdeg {maxdeg}", flush=True)

            def time_shard(b0, b1):
                x = pg.empty_rows(b1 - b0, dims[i])
                for _ in range(2):
                    pg.backward_aggregation(prep.groups[i], y, x, overwrite=True, rows=(b0, b1))
                ev = []
                for _ in range(5):
                    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    pg.backward_aggregation(prep.groups[i], y, x, overwrite=True, rows=(b0, b1))
                    z.record()
                    torch.cuda.synchronize()
                    ev.append(a.elapsed_time(z))
                return statistics.median(ev)

            nb, t0, t1 = pgd.calibrate_bounds(time_shard, offs, b, iters=3)
            print(f"    calibrated cuts: max/mean {max(t1):.3f}/{statistics.mean(t1):.3f} (was {max(t0):.3f}) "
                  f"ms {[round(t, 3) for t in t1]}", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
