"""W' = gather_rows(Y, rows)^T g (gemm_at_b, bit-exact serial chains) at the
configs' shapes for each setting of tuning atb_depth, CUDA-event timed,
outputs compared bit for bit across settings.
  python tools/prof_atb.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2204_02662_b200 as pg  # noqa: E402

ATB = [("products layer0 W'", 1_198_008, 2_449_029, 100, 256), ("products top W'", 195_922, 2_449_029, 256, 47),
       ("reddit layer0 W'", 232_756, 232_965, 602, 16), ("reddit top W'", 153_756, 232_965, 16, 41),
       ("arxiv layer0 W'", 113_323, 169_343, 128, 256)]


def main():
    for name, n, ry, ind, outd in ATB:
        y = pg.empty_rows(ry, ind)
        y.uniform_(-1, 1)
        g = pg.empty_rows(n, outd)
        g.uniform_(-1, 1)
        ids = torch.sort(torch.randperm(ry, device="cuda")[:n].to(torch.int32))[0]
        res, outs = {}, {}
        for depth in (0, 1, 2, 3, 4):
            pg.set_tuning("atb_depth", depth if depth < 3 else 0)
            pg.set_tuning("atb_quad", 0 if depth < 3 else depth - 2)
            o = pg.empty_rows(ind, outd)
            pg.gemm_at_b(y, g, o, a_rows=ids)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                pg.gemm_at_b(y, g, o, a_rows=ids)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[depth] = statistics.median(ts)
            outs[depth] = o
        pg.set_tuning("atb_depth", None)
        pg.set_tuning("atb_quad", None)
        same = all(torch.equal(outs[0].view(torch.int32), o.view(torch.int32)) for o in outs.values())
        print(f"{name:22s} n={n} {ind}x{outd}: row per lane 4/2 {res[0]:.3f} ms, 7/5 {res[1]:.3f} ms, "
              f"rows shared by lanes {res[2]:.3f} ms, 4 chain + 4 copy warps per block 6/4 {res[3]:.3f} ms, "
              f"10/8 {res[4]:.3f} ms ({res[4] * 1e6 * 1.95 / n:.1f} cycles per row); "
              f"bit-identical: {same}", flush=True)
        del y, g, ids, outs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
