"""Diagnostics: the layer-0 SpMM split into K source-row segments run as
accumulate passes (bit-identical to one pass) — does a smaller per-pass
source working set (S/K rows x 512 B per chunk pass) buy L2 hits?"""
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
    y.uniform_(-1, 1)
    ref = pg.empty_rows(p.D, dim)
    pg.backward_aggregation(G, y, ref, overwrite=True)
    x = pg.empty_rows(p.D, dim)
    offs = p.export()["offsets"]
    for K in (1, 2, 3, 4, 6):
        for mode in ("rows", "edges"):
            if mode == "rows":
                cuts = [p.P * k // K for k in range(K + 1)]
            else:  # cuts balancing the edges per segment (sources sorted by id)
                nb = p.export()["neighbors"]
                src = np.sort(p.export()["srcpos"][nb])
                cuts = [0] + [int(src[len(src) * k // K]) for k in range(1, K)] + [p.P]
            G.set_segments(cuts)

            def run():
                for k in range(K):
                    pg.backward_aggregation(G, y, x, overwrite=(k == 0), segment=k)

            run()
            torch.cuda.synchronize()
            ts = []
            for _ in range(7):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                run()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ok = torch.equal(x.view(torch.int32), ref.view(torch.int32))
            print(f"K={K} cuts by {mode}: {statistics.median(ts):.3f} ms (bit-equal: {ok})", flush=True)
            if K == 1:
                break
    G.set_segments(None)


if __name__ == "__main__":
    main(*sys.argv[1:])
