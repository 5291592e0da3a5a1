"""PCIe copy rate alone vs beside the layer-0 SpMM (Reddit shape): is the
host pipeline's D2H (48 GB/s effective) slowed by the concurrent kernel?
  python tools/diag_copy_contention.py"""
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
    dims = bench.agg_dims(cfg)
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), dims)
    p, G, dim = prep.paths[1], prep.groups[1], dims[1]
    y = pg.empty_rows(p.P, dim)
    y.uniform_(-1, 1)
    x = pg.empty_rows(p.D, dim)
    nbytes = 560 << 20
    dsrc = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    hdst = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    hsrc = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    ddst = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    cs = torch.cuda.Stream()
    ks = torch.cuda.Stream()

    def copy_rate(kind, busy):
        for rep in range(3):
            if busy:
                with torch.cuda.stream(ks):
                    for _ in range(3):
                        pg.backward_aggregation(G, y, x, overwrite=True, stream=ks)
            torch.cuda.synchronize() if rep == 0 else None
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(cs):
                e0.record(cs)
                if kind == "d2h":
                    hdst.copy_(dsrc, non_blocking=True)
                else:
                    ddst.copy_(hsrc, non_blocking=True)
                e1.record(cs)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        return nbytes / ms / 1e6, ms

    for kind in ("d2h", "h2d"):
        for busy in (False, True, False):
            gbs, ms = copy_rate(kind, busy)
            print(f"{kind} {'beside the SpMM' if busy else 'alone'}: {gbs:.1f} GB/s ({ms:.2f} ms for 560 MiB)", flush=True)


if __name__ == "__main__":
    main()
