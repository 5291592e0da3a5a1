"""gemm_a_bt (y_grad = g W^T) at the configs' shapes: the bit-exact FFMA2
kernel vs the tcgen05 3xTF32 tensor-core kernel, CUDA-event timed (median of
10 after warm-up), with the HBM bytes each moves (A read + output written).
  python tools/prof_gemm_tc.py [--ncu] [--only=products]   (--ncu: 2 launches each, for ncu)"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2204_02662_b200 as pg  # noqa: E402

# (name, n rows of g, m = out cols (W rows), K = g cols)
SHAPES = [("products layer0 y_grad", 2_177_454, 100, 256), ("products top y_grad", 1_198_008, 256, 47),
          ("reddit layer0 y_grad", 232_898, 602, 16), ("reddit top y_grad", 232_756, 16, 41),
          ("arxiv layer0 y_grad", 131_584, 128, 256)]


def main():
    ncu = "--ncu" in sys.argv
    only = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--only=")]
    for name, n, m, k in SHAPES:
        if only and not any(o in name for o in only):
            continue
        a = pg.empty_rows(n, k)
        a.uniform_(-1, 1)
        b = torch.empty((m, k), dtype=torch.float32, device="cuda").uniform_(-1, 1)
        o = pg.empty_rows(n, m)
        res = {}
        for tc in (False, True):
            reps = 2 if ncu else 10
            pg.gemm_a_bt(a, b, o, tensor_cores=tc)
            torch.cuda.synchronize()
            ts = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                pg.gemm_a_bt(a, b, o, tensor_cores=tc)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[tc] = statistics.median(ts)
        byt = n * k * 4 + n * m * 4
        print(f"{name:26s} n={n} m={m} K={k}: ffma2 {res[False]:.3f} ms, tcgen05 3xTF32 {res[True]:.3f} ms "
              f"({res[False] / res[True]:.2f}x); tc {byt / res[True] / 1e6:.0f} GB/s of A+out, "
              f"{3 * 2 * n * m * k / res[True] / 1e9:.0f} TFLOP/s (3 passes)", flush=True)
        del a, b, o
        torch.cuda.empty_cache()


# W' = gather_rows(Y, rows)^T g: (name, n rows of g, rows of Y, in_dim, out_dim)
ATB = [("products layer0 W'", 1_198_008, 2_449_029, 100, 256), ("products top W'", 195_922, 2_449_029, 256, 47),
       ("reddit layer0 W'", 232_756, 232_965, 602, 16), ("reddit top W'", 153_756, 232_965, 16, 41),
       ("arxiv layer0 W'", 113_323, 169_343, 128, 256)]


def main_atb():
    only = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--only=")]
    for name, n, ry, ind, outd in ATB:
        if only and not any(o in name for o in only):
            continue
        y = pg.empty_rows(ry, ind)
        y.uniform_(-1, 1)
        g = pg.empty_rows(n, outd)
        g.uniform_(-1, 1)
        ids = torch.sort(torch.randperm(ry, device="cuda")[:n].to(torch.int32))[0]
        o = pg.empty_rows(ind, outd)
        res = {}
        for tc in (False, True):
            pg.gemm_at_b(y, g, o, a_rows=ids, tensor_cores=tc)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                pg.gemm_at_b(y, g, o, a_rows=ids, tensor_cores=tc)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[tc] = statistics.median(ts)
        byt = n * ind * 4 + n * outd * 4
        print(f"{name:22s} n={n} {ind}x{outd}: serial chains {res[False]:.3f} ms, tcgen05 split-K 3xTF32 "
              f"{res[True]:.3f} ms ({res[False] / res[True]:.1f}x); tc {byt / res[True] / 1e6:.0f} GB/s of Y rows + g",
              flush=True)
        del y, g, o, ids
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
    main_atb()
