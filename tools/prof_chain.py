"""Profiling driver: the device-resident chain (forward + backward_epp +
backward_all_active + backward_ifelse) once after a warm-up on a bench
config, for `ncu --metrics gpu__time_duration.sum` launch lists."""
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
    out = bench.measure_chain(pg, torch, g, prep, cfg, vt, torch.device("cuda", 0), reps=1)
    print(out, flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
