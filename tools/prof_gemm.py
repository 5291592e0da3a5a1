"""The bit-exact dense products of the chain at the configs' shapes:
k_gemm3 (8x8 register tiles, tuning gemm_packed = 2) vs k_gemm2 (FFMA2 column
pairs, 1) vs k_gemm (scalar, 0), CUDA-event timed (median of 10 after
warm-up), each output compared bit for bit with the k_gemm one.
  python tools/prof_gemm.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2204_02662_b200 as pg  # noqa: E402

# (name, kind, n, m, K): a_bt = g W^T (W m x K), ab = X W (W K x m)
SHAPES = [("products layer0 y_grad", "a_bt", 2_177_454, 100, 256), ("products top y_grad", "a_bt", 1_198_008, 256, 47),
          ("reddit layer0 y_grad", "a_bt", 232_898, 602, 16), ("arxiv layer0 y_grad", "a_bt", 131_584, 128, 256),
          ("products forward X W0", "ab", 2_449_029, 256, 100), ("arxiv forward X W0", "ab", 169_343, 256, 128),
          ("products forward H W1", "ab", 2_449_029, 47, 256)]
# unfused multiply + add on the FP32 pipe: the pipe retires 32 fp32 lane-ops per
# SMSP per cycle (an FFMA2 / FADD2 occupies it two cycles: ncu
# sm__pipe_fma_cycles_active ~1.84x sm__inst_executed_pipe_fma), and an
# unfused multiply-add is 2 lane-ops: 64 multiply-adds = 128 flops per SM-cycle
FP32_UNFUSED_TFLOPS = 148 * 128 * 1.965e9 / 1e12


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    for name, kind, n, m, k in SHAPES:
        a = pg.empty_rows(n, k)
        a.uniform_(-1, 1)
        if kind == "a_bt":
            b = torch.empty((m, k), dtype=torch.float32, device="cuda").uniform_(-1, 1)
        else:
            b = pg.empty_rows(k, m)
            b.uniform_(-1, 1)
        outs, res = {}, {}
        for key, packed, rows in (("k_gemm", 0, 8), ("k_gemm2", 1, 8), ("k_gemm3<8>", 2, 8), ("k_gemm3<16>", 2, 16)):
            pg.set_tuning("gemm_packed", packed)
            pg.set_tuning("gemm3_rows", rows)
            o = pg.empty_rows(n, m)
            f = (lambda: pg.gemm_a_bt(a, b, o)) if kind == "a_bt" else (lambda: pg.gemm(a, b, o))
            res[key] = timed(f)
            outs[key] = o
        pg.set_tuning("gemm_packed", None)
        pg.set_tuning("gemm3_rows", None)
        same = all(torch.equal(o.view(torch.int32), outs["k_gemm"].view(torch.int32)) for o in outs.values())
        fl = 2 * n * m * k
        best = min(res, key=res.get)
        print(f"{name:24s} n={n} m={m} K={k}: " + ", ".join(f"{key} {t:.3f} ms" for key, t in res.items()) +
              f"; best {best} {fl / res[best] / 1e9:.1f} TFLOP/s = {fl / res[best] / 1e9 / FP32_UNFUSED_TFLOPS:.2f} "
              f"of the unfused FP32 peak {FP32_UNFUSED_TFLOPS:.0f}; bit-identical: {same}", flush=True)
        del a, b, outs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
