"""Diagnostics: the host pipeline's SpMM schedule on device-resident data,
without the copies (Reddit layer-0 path): auto device segments vs K
edge-balanced source segments as whole passes vs the same with the last
segment in R destination-row chunks — separates schedule overhead from DMA
contention in the host-buffer call."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2204_02662_b200 as pg  # noqa: E402


def timed(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts[1:])[reps // 2]


def main():
    cfg = bench.CONFIGS["reddit"]
    pairs = bench.make_pairs(cfg, pg.gen_rmat)
    vt = pg.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    g = pg.build_undirected_csr(pairs, n_hint=cfg["V"], weights="symnorm")
    dims = bench.agg_dims(cfg)
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), dims)
    p, G, dim = prep.paths[1], prep.groups[1], dims[1]
    x = p.export()
    src = x["neighbors"].astype(np.int64)  # local source ids = parent rows (identity path)
    cnt = np.bincount(x["srcpos"][src], minlength=p.P)
    csum = np.cumsum(cnt)
    y = pg.empty_rows(p.P, dim)
    y.uniform_(-1, 1)
    out = pg.empty_rows(p.D, dim)
    print(f"auto device call: {timed(lambda: pg.backward_aggregation(G, y, out, overwrite=True)):.2f} ms", flush=True)
    offs = x["offsets"].astype(np.int64)
    Ks = [int(v) for v in os.environ.get("DIAG_K", "2 3 4").split()]
    Rs = [int(v) for v in os.environ.get("DIAG_R", "1 16").split()]
    if os.environ.get("DIAG_HEAVY"):
        pg.set_heavy_min_degree(int(os.environ["DIAG_HEAVY"]))
    for K in Ks:
        cuts = np.array([0] + [int(np.searchsorted(csum, p.E * k / K)) + 1 for k in range(1, K)] + [p.P], np.uint64)
        cuts = np.maximum.accumulate(np.minimum(cuts, p.P))
        G.set_segments(cuts)

        def passes():
            for k in range(K):
                pg.backward_aggregation(G, y, out, overwrite=(k == 0), segment=k)
        for R in Rs:
            bnd = [0] + [int(np.searchsorted(offs[:-1], offs[-1] * r / R)) for r in range(1, R)] + [p.D]

            def chunked():
                for k in range(K - 1):
                    pg.backward_aggregation(G, y, out, overwrite=(k == 0), segment=k)
                for r in range(R - 1, -1, -1):
                    if bnd[r + 1] > bnd[r]:
                        pg.backward_aggregation(G, y, out[bnd[r]:bnd[r + 1]], segment=K - 1,
                                                rows=(bnd[r], bnd[r + 1]))
            fn = passes if R == 1 else chunked
            print(f"K={K} edge-balanced, last pass in R={R} chunks: {timed(fn):.2f} ms", flush=True)
        G.set_segments(None)


if __name__ == "__main__":
    main()
