"""Layout probe for the tensor-core W' kernel: structured inputs whose
products identify which (row, column) each output element picked up."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_02662_b200 as pg  # noqa: E402


def run(y, g):
    yd = pg.empty_rows(y.shape[0], y.shape[1])
    yd.copy_(torch.from_numpy(y))
    gd = pg.empty_rows(g.shape[0], g.shape[1])
    gd.copy_(torch.from_numpy(g))
    o = pg.empty_rows(y.shape[1], g.shape[1])
    o.fill_(float("nan"))
    pg.gemm_at_b(yd, gd, o, tensor_cores=True)
    torch.cuda.synchronize()
    return o.cpu().numpy()


np.set_printoptions(linewidth=220, threshold=100000)
n, ind, outd = 16, 128, 32
# 1: Y = [I_16 | 0], g[r][j] = 100 r + j  ->  out[i][j] = 100 i + j (i < 16)
y = np.zeros((n, ind), np.float32)
for r in range(n):
    y[r, r] = 1
g = (100 * np.arange(n)[:, None] + np.arange(outd)[None, :]).astype(np.float32)
o = run(y, g)
print("probe 1 (expect row i = 100 i + j):")
print(o[:20, :8])
# 2: only row r=0 of Y nonzero: Y[0][i] = i + 1; g[0][j] = (j == 0)
y = np.zeros((n, ind), np.float32)
y[0] = np.arange(ind) + 1
g = np.zeros((n, outd), np.float32)
g[0, 0] = 1
o = run(y, g)
print("probe 2 (expect column 0 = i + 1, rest 0):")
print(o[:, :4].T)
# 3: only g[0][j] = j + 1, Y[0][0] = 1
y = np.zeros((n, ind), np.float32)
y[0, 0] = 1
g = np.zeros((n, outd), np.float32)
g[0] = np.arange(outd) + 1
o = run(y, g)
print("probe 3 (expect row 0 = j + 1):")
print(o[:4, :])
