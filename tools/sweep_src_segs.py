"""Whole-path L2-sized source segments of the layer-0 SpMM (Reddit shape):
segment count K (tuning src_segs) x cut balance (src_seg_balance: 0 = equal
source rows, 100 = equal edges), CUDA-event median of 9; every variant is
bit-identical (checked against K = 1)."""
import os
import statistics
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
    dims = bench.agg_dims(cfg)
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), dims)
    i = len(prep.paths) - 1
    p, G, dim = prep.paths[i], prep.groups[i], dims[i]
    y = pg.empty_rows(p.P, dim)
    y.copy_(torch.from_numpy(bench.grad_input(p.P, dim, i)))
    x = pg.empty_rows(p.D, dim)
    ref = None
    for K in (1, 2, 3, 4):
        for bal in ((0,) if K == 1 else (0, 25, 50, 100)):
            pg.set_tuning("src_segs", K)
            pg.set_tuning("src_seg_balance", bal)
            pg.backward_aggregation(G, y, x, overwrite=True)
            torch.cuda.synchronize()
            ts = []
            for _ in range(9):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                pg.backward_aggregation(G, y, x, overwrite=True)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            got = x.cpu().numpy().view(np.uint32)
            if ref is None:
                ref = got.copy()
            print(f"K={K} balance={bal:3d}: {statistics.median(ts):.3f} ms (min {min(ts):.3f}) "
                  f"bit-identical={np.array_equal(got, ref)}", flush=True)
    pg.set_tuning("src_segs", None)
    pg.set_tuning("src_seg_balance", None)


if __name__ == "__main__":
    main(*sys.argv[1:])
