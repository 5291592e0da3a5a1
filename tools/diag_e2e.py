"""Diagnostics: the host-buffer drop-in (pg_backward_aggregate_host) on the
Reddit-shaped workload — per-path host-call time for each pipeline shape
(source segments K x last-pass row chunks R), a phase trace of the default,
raw pinned copy rates (one direction and both at once), and the device-only
kernel time for reference. Results are checked bit-equal to the device call."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2204_02662_b200 as pg  # noqa: E402


def copy_rates(nbytes=566 << 20):
    h = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    h2 = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    d = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    d2 = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h2.copy_(d2, non_blocking=True))]:
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 5
        print(f"[copy] {name}: {nbytes / dt / 1e9:.1f} GB/s ({dt * 1e3:.2f} ms)", flush=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"[copy] both directions at once: {2 * nbytes / dt / 1e9:.1f} GB/s total ({dt * 1e3:.2f} ms)", flush=True)


def main(config="reddit"):
    copy_rates()
    cfg = bench.CONFIGS[config]
    pairs = bench.make_pairs(cfg, pg.gen_rmat)
    vt = pg.sample_training_set(cfg["V"], bench.train_ratio(cfg), bench.TRAIN_SEED)
    g = pg.build_undirected_csr(pairs, n_hint=cfg["V"], weights="symnorm")
    dims = bench.agg_dims(cfg)
    prep = pg.prepare_paths(g, vt, len(cfg["dims"]), dims)
    for i, (p, G) in enumerate(zip(prep.paths, prep.groups)):
        dim = dims[i]
        yh = torch.empty((p.P, dim), dtype=torch.float32, pin_memory=True).numpy()
        yh[:] = np.random.default_rng(0).uniform(-1, 1, size=yh.shape)
        xh = torch.empty((p.D, dim), dtype=torch.float32, pin_memory=True).numpy()
        yd = pg.empty_rows(p.P, dim)
        yd.copy_(torch.from_numpy(yh))
        xd = pg.empty_rows(p.D, dim)
        for rep in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            pg.backward_aggregation(G, yd, xd, overwrite=True)
            torch.cuda.synchronize()
            dev_ms = (time.perf_counter() - t) * 1e3
        print(f"path {i} dim {dim}: device call {dev_ms:.2f} ms", flush=True)
        want = xd.cpu().numpy().view(np.uint32)
        # (K source segments, F of them in the chunked last pass, R row chunks, reversed order)
        shapes = [(2, 1, 4, 1)] if i == 0 else [
            (1, 1, 16, 1), (2, 1, 16, 1), (3, 1, 16, 1), (4, 1, 16, 1), (3, 1, 16, 0),
            (3, 2, 16, 1), (4, 2, 16, 1), (5, 2, 16, 1), (5, 3, 16, 1), (6, 3, 16, 1), (6, 2, 16, 1),
            (8, 3, 16, 1), (8, 4, 16, 1), (4, 3, 16, 1)]
        if os.environ.get("DIAG_SHAPES"):
            shapes = [tuple(int(v) for v in t.split(",")) for t in os.environ["DIAG_SHAPES"].split()]
        for K, F, R, order in shapes:
            pg.set_tuning("host_segs", K)
            pg.set_tuning("host_final_segs", F)
            pg.set_tuning("host_chunks", R)
            pg.set_tuning("host_chunk_order", order)
            ts = []
            for rep in range(4):
                t = time.perf_counter()
                pg.backward_aggregation(G, yh, xh, overwrite=True)
                ts.append((time.perf_counter() - t) * 1e3)
            assert np.array_equal(xh.view(np.uint32), want), (K, F, R)
            print(f"path {i} dim {dim}: host call K={K} F={F} R={R} reversed={order}: {min(ts[1:]):.2f} ms "
                  f"(min of 3)", flush=True)
        for key in ("host_segs", "host_final_segs", "host_chunks", "host_chunk_order"):
            pg.set_tuning(key)
        pg.set_tuning("host_trace", 1)
        for rep in range(3):
            t = time.perf_counter()
            pg.backward_aggregation(G, yh, xh, overwrite=True)
            print(f"path {i}: traced host call wall {(time.perf_counter() - t) * 1e3:.2f} ms", flush=True)
        pg.set_tuning("host_trace", 0)
        import ctypes
        from paper_2204_02662_b200 import _lib
        lib = _lib.load()
        c = np.zeros(3, np.uint64)
        for rep in range(3):
            t = time.perf_counter()
            lib.pg_backward_aggregate_host(G._h, yh.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), yh.shape[0],
                                           yh.shape[1], xh.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), 2,
                                           c.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
            print(f"path {i}: raw C call wall {(time.perf_counter() - t) * 1e3:.2f} ms", flush=True)
        pg.set_tuning("host_segs")
        pg.set_tuning("host_final_segs")
        pg.set_tuning("host_chunks")
        pg.set_tuning("host_chunk_order")


if __name__ == "__main__":
    main(*sys.argv[1:])
