"""Group-partitioned Fast aggregation (PG_AGG_GROUPED) on a config's paths:
the atomic-free kernel (grouped_seg 0: k_agg_grp + hub fixup) against the
atomic variants (1: CTA-segmented, 2: one atomic per extra group) and the
Deterministic kernel, per gs (CUDA events, median of 7 after a warm-up).
  python tools/prof_grouped.py [config] [gs ...]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2204_02662_b200 as pg  # noqa: E402


def timed(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    gss = [int(x) for x in sys.argv[2:]] or None
    cfg = bench.CONFIGS[name]
    pairs = bench.make_pairs(cfg, pg.gen_rmat)
    vt = pg.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    g = pg.build_undirected_csr(pairs, n_hint=cfg["V"], weights="symnorm")
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), bench.agg_dims(cfg))
    dims = bench.agg_dims(cfg)
    for i, p in enumerate(prep.paths):
        y = pg.empty_rows(p.P, dims[i])
        y.copy_(torch.from_numpy(bench.grad_input(p.P, dims[i], i)))
        x = pg.empty_rows(p.D, dims[i])
        det = timed(lambda: pg.backward_aggregation(prep.groups[i], y, x, overwrite=True))
        print(f"[{name}] path {i} D={p.D} E={p.E} dim={dims[i]} maxdeg={p.max_degree}: deterministic {det:.3f} ms",
              flush=True)
        cands = gss or sorted({prep.gs[i], 8, 32, 64, 128, 256, 512, 1024})
        for gs in cands:
            G = pg.group_neighbors(p, gs)
            row = []
            for seg in (0, 1, 2):
                pg.set_tuning("grouped_seg", seg)
                row.append(timed(lambda: pg.backward_aggregation(G, y, x, mode=pg.GROUPED, overwrite=True)))
            pg.set_tuning("grouped_seg", None)
            print(f"   gs={gs:5d} groups={G.count}: atomic-free {row[0]:.3f} ms | cta-seg+atomics {row[1]:.3f} | "
                  f"atomic/group {row[2]:.3f}  (det/af {det / row[0]:.2f}x)", flush=True)
            del G


if __name__ == "__main__":
    main()
