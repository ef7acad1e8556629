import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2104_11385_b200 import device, pic
nz = nx = int(sys.argv[1]) if len(sys.argv) > 1 else 512
fast = len(sys.argv) <= 2 or sys.argv[2] == "fast"
ppc = 8
rng = np.random.default_rng(42)
cell = np.repeat(np.arange(nz * nx, dtype=np.int64), ppc)
off = rng.random((cell.size, 2))
pos = np.column_stack([(cell // nx) + off[:, 0], (cell % nx) + off[:, 1]])
u = rng.normal(0.0, 0.05, size=(cell.size, 3))
ctx = device.Context(capacity=pos.shape[0])
st = pic.PicState.create(pos, u, nz, nx)
pic.pic_sort(ctx, st)
for s in range(3):
    out = pic.pic_step(ctx, st, 128 if nz >= 128 else 16, -1.0, -1e-4, 0.5, clock=True, fast=fast, gather="quad")
    torch.cuda.synchronize()
    print(s, out["n"], flush=True)
