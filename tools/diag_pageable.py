"""Diagnostics: the host-buffer drop-in with PAGEABLE buffers (plain numpy,
like a reference DenseMatrix's std::vector) vs pinned ones, Reddit layer-0
path; results checked bit-equal."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2204_02662_b200 as pg  # noqa: E402


def main():
    cfg = bench.CONFIGS["reddit"]
    pairs = bench.make_pairs(cfg, pg.gen_rmat)
    vt = pg.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    g = pg.build_undirected_csr(pairs, n_hint=cfg["V"], weights="symnorm")
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), bench.agg_dims(cfg))
    dims = bench.agg_dims(cfg)
    i = 1
    p, G, dim = prep.paths[i], prep.groups[i], dims[i]
    y = np.random.default_rng(0).uniform(-1, 1, size=(p.P, dim)).astype(np.float32)
    x = np.empty((p.D, dim), np.float32)
    yp = torch.from_numpy(y).pin_memory().numpy()
    xp = torch.empty((p.D, dim), dtype=torch.float32).pin_memory().numpy()
    for name, yy, xx in (("pinned", yp, xp), ("pageable", y, x)):
        ts = []
        for _ in range(5):
            t = time.perf_counter()
            pg.backward_aggregation(G, yy, xx, overwrite=True)
            ts.append((time.perf_counter() - t) * 1e3)
        print(f"{name}: host call {sorted(ts)[2]:.2f} ms (median of 5; all {[round(v, 1) for v in ts]})", flush=True)
    assert np.array_equal(x.view(np.uint32), xp.view(np.uint32))


if __name__ == "__main__":
    main()
