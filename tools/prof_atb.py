"""W' = gather_rows(Y, rows)^T g (gemm_at_b, bit-exact serial chains) at the
configs' shapes for each setting of tuning atb_depth, CUDA-event timed,
outputs compared bit for bit across settings.
  python tools/prof_atb.py"""
import json
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


# tuning settings compared (atb_pairs 0: one A column per lane; 1: two;
# atb_depth 0 = 4/2, 1 = 7/5, 2 = rows shared by lanes 4/2)
SETTINGS = json.loads(os.environ.get("ATB_SETTINGS", "null")) or [
    {}, {"atb_depth": 1}, {"atb_depth": 2}, {"atb_pairs": 0}, {"atb_pairs": 0, "atb_depth": 1},
    {"atb_pairs": 0, "atb_depth": 2}, {"atb_quad": 1}, {"atb_quad": 2}]


def main():
    for name, n, ry, ind, outd in ATB:
        y = pg.empty_rows(ry, ind)
        y.uniform_(-1, 1)
        g = pg.empty_rows(n, outd)
        g.uniform_(-1, 1)
        ids = torch.sort(torch.randperm(ry, device="cuda")[:n].to(torch.int32))[0]
        res, outs = {}, {}
        for si, st in enumerate(SETTINGS):
            for k, v in st.items():
                pg.set_tuning(k, v)
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
            res[si] = statistics.median(ts)
            outs[si] = o
            for k in st:
                pg.set_tuning(k, None)
        same = all(torch.equal(outs[0].view(torch.int32), o.view(torch.int32)) for o in outs.values())
        print(f"{name:22s} n={n} {ind}x{outd}: bit-identical {same}", flush=True)
        for si, st in enumerate(SETTINGS):
            print(f"    {json.dumps(st):48s} {res[si]:8.3f} ms  ({res[si] * 1e6 * 1.95 / n:5.1f} cycles per row)",
                  flush=True)
        del y, g, ids, outs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
