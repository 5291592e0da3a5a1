"""Digests of the REFERENCE's own outputs at the benchmarked sizes
(BASELINE.json configs[2..4]: arxiv-, Reddit- and products-shaped), for
tests/test_gpu_fullsize.py to compare the device path against bit for bit.

Runs the reference compiled from its sources (oracle/_ref/libpathgcn_ref.so,
oracle/Makefile) in the build container, on exactly bench.py's inputs:
  * graph:  gen_rmat + exact-V rejection (bench.make_pairs), build_undirected_csr
            + sym-norm assign_edge_weights          (csr_graph.cpp:33-77)
  * V_t:    sample_training_set(V, ratio, 42)        (training_set.cpp:28-49)
  * every frontier level                             (frontier.cpp:7-26)
  * every execution-path array, weights as bits      (execution_path.cpp:24-88)
  * the grouping at the path's regression gs         (grouping.cpp:7-27, gs_model.cpp:68-74)
  * the FULL x_grad of the timed stage, gather_rows + aggregate_pull<float>
    Deterministic (engine.hpp:331-338), for y_grad = fullsize.y_grad(P, dim, i)

usage: python tests/golden/make_fullsize_digests.py [config ...]   (default: all)
Writes tests/golden/fullsize_<config>.json. Reddit takes a few minutes.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import bench  # noqa: E402
import fullsize as fs  # noqa: E402
from oracle.oracle import Ref  # noqa: E402


def run(config):
    R = Ref()
    cfg = bench.CONFIGS[config]
    L = len(cfg["dims"])
    dims = bench.agg_dims(cfg)
    t0 = time.time()
    pairs = bench.make_pairs(cfg, R.gen_rmat)
    g = R.build_graph(pairs, n_hint=cfg["V"], symnorm=True)
    del pairs
    assert g.m == cfg["m"], (g.m, cfg["m"])
    vt = R.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    out = {"config": config, "V": cfg["V"], "m": int(g.m), "L": L, "agg_dims": dims,
           "generator": "tests/golden/make_fullsize_digests.py over oracle/_ref (the reference compiled from "
                        "/root/reference/proj/core/src)",
           "graph": {"offsets": fs.digest(g.offsets), "neighbors": fs.digest(g.neighbors),
                     "weights": fs.digest(g.weights.view(np.uint64))},
           "vt": fs.digest(vt), "graph_fingerprint": int(R.graph_fingerprint(g)),
           "path_fingerprint": int(R.path_fingerprint(g, vt, L))}
    print(f"[{config}] graph {time.time() - t0:.1f}s", flush=True)
    levels = R.compute_frontiers(g, vt, L)
    out["levels"] = [fs.digest(lv) for lv in levels]
    paths = R.prepare_all_paths(g, vt, L)
    print(f"[{config}] paths {time.time() - t0:.1f}s", flush=True)
    del g
    out["paths"] = []
    for i, p in enumerate(paths):
        D, E = len(p.dest), int(p.offsets[-1])
        gs = int(R.regression_gs(D, E, 0.0 if D == 0 else E / D))  # train.hpp:16-24 path_stats
        gr = R.group_neighbors(p.offsets, gs)
        rec = {"layer": p.layer, "D": len(p.dest), "S": len(p.src), "P": len(levels[i]), "E": int(p.offsets[-1]),
               "gs": gs, "dim": dims[i]}
        for f in ("dest", "src", "srcpos", "offsets", "neighbors"):
            rec[f] = fs.digest(getattr(p, f))
        rec["weights"] = fs.digest(p.weights.view(np.uint64))
        rec["groups"] = {"dest": fs.digest(gr.dest), "begin": fs.digest(gr.begin), "end": fs.digest(gr.end),
                         "dest_groups": fs.digest(gr.dest_groups)}
        del gr
        item = R.stage_items_from_arrays([{"dest": p.dest, "src": p.src, "srcpos": p.srcpos, "offsets": p.offsets,
                                           "neighbors": p.neighbors, "weights": p.weights, "layer": p.layer}],
                                          gs_list=[gs])[0]
        y = fs.y_grad(len(levels[i]), dims[i], i)
        rec["y_grad"] = fs.digest(y)
        sec, x = R.run_backward_stage(item, y, want_out=True)
        R.free_stage_handles([item])
        rec["x_grad"] = fs.digest(x)
        rec["x_grad_abs_sum"] = float(np.abs(x.astype(np.float64)).sum())
        rec["ref_stage_seconds"] = round(sec, 3)
        rec["ref_threads"] = R.max_threads()
        out["paths"].append(rec)
        print(f"[{config}] path {i}: D={rec['D']} E={rec['E']} gs={gs} stage {sec:.2f}s", flush=True)
        del x, y
    out["seconds"] = round(time.time() - t0, 1)
    with open(fs.digest_path(config), "w") as f:
        json.dump(out, f, indent=1)
    print(f"[{config}] wrote {fs.digest_path(config)} in {out['seconds']} s", flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:] or fs.CONFIGS:
        run(c)
