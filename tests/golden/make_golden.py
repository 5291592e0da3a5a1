"""Generates tests/golden/golden.npz from the REFERENCE itself
(oracle/_ref/libpathgcn_ref.so, compiled from /root/reference sources).
Run in the build container: python tests/golden/make_golden.py

Fixture: the reference's frozen RMAT graph rmat_graph(1024, 8192, 7)
(test_rmat.cpp:72-81) with sym-norm weights (csr_graph.cpp:65-77), training
set sample_training_set(1024, 0.1, 42), L = 2 (the survey's probe fixture).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Ref  # noqa: E402


def main():
    R = Ref()
    out = {}
    pairs, n_pad = R.gen_rmat(1024, 8192, 0.45, 0.22, 0.22, 0.11, 7)
    g = R.build_graph(pairs, n_hint=n_pad, symnorm=True)
    out.update(g_n=np.array([g.n]), g_offsets=g.offsets, g_neighbors=g.neighbors, g_weights=g.weights,
               g_fp=np.array([R.graph_fingerprint(g)], np.uint64))
    vt = R.sample_training_set(g.n, 0.1, 42)
    out["vt"] = vt
    out["path_fp"] = np.array([R.path_fingerprint(g, vt, 2)], np.uint64)
    lv = R.compute_frontiers(g, vt, 2)
    for k, x in enumerate(lv):
        out[f"level{k}"] = x
    paths = R.prepare_all_paths(g, vt, 2)
    for i, p in enumerate(paths):
        for f in ("dest", "src", "srcpos", "offsets", "neighbors", "weights"):
            out[f"p{i}_{f}"] = getattr(p, f)
        gs = (2, 9)[i]
        gr = R.group_neighbors(p.offsets, gs)
        for f in ("dest", "begin", "end", "dest_groups"):
            out[f"p{i}_g{gs}_{f}"] = getattr(gr, f)
        cands = R.default_candidates(int(np.diff(p.offsets).max()))
        out[f"p{i}_cands"] = cands
        for j, (dim, W, lam) in enumerate(((16, 8, 0.25), (602, 3, 0.1))):
            best, table = R.oracle_gs_cost(p.offsets, cands, dim, W, lam)
            out[f"p{i}_cost{j}_best"] = np.array([best])
            out[f"p{i}_cost{j}_table"] = table
        rng = np.random.default_rng(100 + i)
        x = rng.uniform(-1, 1, size=(p.S, 37)).astype(np.float32)
        y, _ = R.aggregate_pull(p.offsets, p.neighbors, p.weights, x, gs=gs)
        out[f"p{i}_agg_in"] = x
        out[f"p{i}_agg_out"] = y
    ch = R.epp_chain_f32(g, vt, 2, 16, 8, 4, 42)
    out["ch_top_g"] = ch["top_g"]
    for l in range(2):
        out[f"ch_w{l}"] = ch["w"][l]
    for i in range(2):
        out[f"ch_y{i}"] = ch["y_grad"][i]
        out[f"ch_x{i}"] = ch["x_grad"][i]
    out["ch_pre0"] = ch["pre_c"][0]
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
