"""e2e of the Reddit epoch through the host-buffer drop-in vs host-pipeline
knobs: python tools/sweep_e2e.py '<json list of {knob: value}>' [pinned|pageable].
Each setting: 14 epochs, median of the last 12 per path (wall clock around the
synchronous C call, like bench.py's e2e)."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2204_02662_b200 as pg  # noqa: E402


def main(settings, mode="pinned", config="reddit"):
    cfg = bench.CONFIGS[config]
    pairs = bench.make_pairs(cfg, pg.gen_rmat)
    vt = pg.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    g = pg.build_undirected_csr(pairs, n_hint=cfg["V"], weights="symnorm")
    dims = bench.agg_dims(cfg)
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), dims)
    ys, xs = [], []
    for i, p in enumerate(prep.paths):
        if mode == "pinned":
            yh = torch.empty((p.P, dims[i]), dtype=torch.float32, pin_memory=True).numpy()
            xh = torch.empty((p.D, dims[i]), dtype=torch.float32, pin_memory=True).numpy()
        else:
            yh = np.empty((p.P, dims[i]), np.float32)
            xh = np.empty((p.D, dims[i]), np.float32)
        yh[:] = bench.grad_input(p.P, dims[i], i)
        ys.append(yh)
        xs.append(xh)
    for st in settings:
        for k, v in st.items():
            pg.set_tuning(k, v)
        per_path = [[] for _ in prep.paths]
        for rep in range(14):
            for i in range(len(prep.paths)):
                t = time.perf_counter()
                pg.backward_aggregation(prep.groups[i], ys[i], xs[i], overwrite=True)
                per_path[i].append((time.perf_counter() - t) * 1e3)
        par = bench.x_grad_parity([torch.from_numpy(x) for x in xs], dims, config)
        med = [statistics.median(v[2:]) for v in per_path]
        if os.environ.get("PG_SWEEP_VERBOSE"):
            print("  per-rep ms", [[round(x, 2) for x in v] for v in per_path], flush=True)
        print(f"[e2e {mode}] {json.dumps(st)} per-path ms {[round(m, 3) for m in med]} epoch {sum(med):.3f} "
              f"parity={par['all'] if par else None}", flush=True)
        for k in st:
            pg.set_tuning(k)


if __name__ == "__main__":
    main(json.loads(sys.argv[1]), *sys.argv[2:])
