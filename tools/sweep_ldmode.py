"""Gather load flavour of k_agg_vec4 (tuning ld_cg, see aggregate.cu ld_row)
on the Reddit-shaped epoch: per-path CUDA-event medians, bit-identity
checked against the default."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2204_02662_b200 as pg  # noqa: E402

NAMES = {0: "nc (default)", 2: "cg (L2 only)", 3: "nc.L1::no_allocate", 4: "plain ld.global", 5: "nc.L1::evict_last",
         6: "records L1::no_allocate"}


def main(config="reddit"):
    cfg = bench.CONFIGS[config]
    pairs = bench.make_pairs(cfg, pg.gen_rmat)
    vt = pg.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    g = pg.build_undirected_csr(pairs, n_hint=cfg["V"], weights="symnorm")
    dims = bench.agg_dims(cfg)
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), dims)
    ys, xs = [], []
    for i, p in enumerate(prep.paths):
        y = pg.empty_rows(p.P, dims[i])
        y.copy_(torch.from_numpy(bench.grad_input(p.P, dims[i], i)))
        ys.append(y)
        xs.append(pg.empty_rows(p.D, dims[i]))
    ref = None
    for rep in range(2):
        for m in (0, 2, 3, 4, 5, 6):
            pg.set_tuning("ld_cg", m)
            per = []
            for i, p in enumerate(prep.paths):
                pg.backward_aggregation(prep.groups[i], ys[i], xs[i], overwrite=True)
                torch.cuda.synchronize()
                ts = []
                for _ in range(9):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    pg.backward_aggregation(prep.groups[i], ys[i], xs[i], overwrite=True)
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                per.append(statistics.median(ts))
            got = [x.cpu().numpy().view(np.uint32).copy() for x in xs]
            if ref is None:
                ref = got
            same = all(np.array_equal(a, b) for a, b in zip(got, ref))
            print(f"[{rep}] ld mode {m} {NAMES[m]:24s}: per-path ms {[round(t, 3) for t in per]} total "
                  f"{sum(per):.3f} bit-identical={same}", flush=True)
    pg.set_tuning("ld_cg", None)


if __name__ == "__main__":
    main(*sys.argv[1:])
