"""aggregate_pull<double> on a bench config's paths (the f64 stage of the
bench line), one warm-up then one timed execution per path, for ncu:
  ncu --set full -k regex:k_agg_f64 python tools/prof_f64.py [config]"""
import os
import sys

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
    for i, p in enumerate(prep.paths):
        dim = dims[i]
        ld = (dim + 15) // 16 * 16 if dim > 16 else dim + (dim & 1)
        y = torch.empty((p.P, ld), dtype=torch.float64, device="cuda")[:, :dim]
        y.uniform_(-1, 1)
        x = torch.zeros((p.D, ld), dtype=torch.float64, device="cuda")[:, :dim]
        for _ in range(2):
            pg.backward_aggregation(prep.groups[i], y, x, overwrite=True)
        torch.cuda.synchronize()
        print(f"[prof_f64] path {i} D={p.D} E={p.E} dim={dim}", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
