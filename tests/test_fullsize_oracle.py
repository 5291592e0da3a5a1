"""The oracle (oracle/pathgcn_oracle.c, the plain-C restatement) against the
REFERENCE's committed full-size digests (tests/golden/fullsize_<config>.json,
made by tests/golden/make_fullsize_digests.py from oracle/_ref): graph,
V_t, frontiers, paths, groupings and the full x_grad of the timed stage —
the same digests the GPU tests hold the device to. arxiv-shaped by default
(seconds); PG_FULLSIZE_ORACLE=all adds the Reddit and products shapes
(minutes, single-threaded oracle)."""
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import fullsize as fs  # noqa: E402

CFGS = ["cora", "pubmed", "arxiv"] + (["products", "reddit"] if os.environ.get("PG_FULLSIZE_ORACLE") == "all" else [])


@pytest.mark.parametrize("config", CFGS)
def test_oracle_matches_reference_digests(orc, config):
    import bench

    want = json.load(open(fs.digest_path(config)))
    cfg = bench.CONFIGS[config]
    pairs = bench.make_pairs(cfg, orc.gen_rmat)
    g = orc.build_graph(pairs, n_hint=cfg["V"], symnorm=True)
    assert g.m == want["m"]
    errs = []

    def chk(name, w, a):
        e = fs.compare(name, w, a)
        if e:
            errs.append(e)

    chk("graph.offsets", want["graph"]["offsets"], g.offsets)
    chk("graph.neighbors", want["graph"]["neighbors"], g.neighbors)
    chk("graph.weights", want["graph"]["weights"], g.weights.view(np.uint64))
    vt = orc.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    chk("vt", want["vt"], vt)
    assert orc.path_fingerprint(g, vt, want["L"]) == want["path_fingerprint"]
    levels = orc.compute_frontiers(g, vt, want["L"])
    for k, lw in enumerate(want["levels"]):
        chk(f"level{k}", lw, levels[k])
    paths = orc.prepare_all_paths(g, levels)
    for i, (p, pw) in enumerate(zip(paths, want["paths"])):
        for f in ("dest", "src", "srcpos", "offsets", "neighbors"):
            chk(f"path{i}.{f}", pw[f], getattr(p, f))
        chk(f"path{i}.weights", pw["weights"], p.weights.view(np.uint64))
        D, E = len(p.dest), int(p.offsets[-1])
        assert orc.regression_gs(D, E, 0.0 if D == 0 else E / D) == pw["gs"]
        gr = orc.group_neighbors(p.offsets, pw["gs"])
        for f in ("dest", "begin", "end", "dest_groups"):
            chk(f"path{i}.groups.{f}", pw["groups"][f], getattr(gr, f))
        y = fs.y_grad(len(levels[i]), pw["dim"], i)
        chk(f"path{i}.y_grad", pw["y_grad"], y)
        x = orc.aggregate_pull_f32(p.offsets, p.neighbors, p.weights, y[p.srcpos])
        chk(f"path{i}.x_grad", pw["x_grad"], x)
    assert not errs, errs
