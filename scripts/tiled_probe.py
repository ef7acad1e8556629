"""Uniform plasma: tiled in-place step times after 1 vs 2 consecutive tile sorts."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_11385_b200 import device, pic  # noqa: E402

dev = torch.device("cuda:0")
nz = nx = 4096
ppc = 8
rng = np.random.default_rng(42)
cell = np.repeat(np.arange(nz * nx, dtype=np.int64), ppc)
off = rng.random((cell.size, 2))
pos0 = np.column_stack([(cell // nx) + off[:, 0], (cell % nx) + off[:, 1]])
u0 = rng.normal(0.0, 0.05, size=(cell.size, 3))
del cell, off
n = pos0.shape[0]
ctx = device.Context(dev, capacity=n)
for nsorts, shuffle in ((1, False),):
    st = pic.PicState.create(pos0[:1], u0[:1], nz, nx, device=dev)
    for k, col in zip(("z", "x", "uz", "ux", "uy"), (pos0[:, 0], pos0[:, 1], u0[:, 0], u0[:, 1], u0[:, 2])):
        t = torch.zeros(n + 2, dtype=torch.float64, device=dev)
        t[:n].copy_(torch.from_numpy(np.ascontiguousarray(col)).to(dev))
        setattr(st, k, t)
    st.n = n
    if shuffle:   # random input order
        perm = torch.randperm(n, device=dev)
        for k in ("z", "x", "uz", "ux", "uy"):
            getattr(st, k)[:n] = getattr(st, k)[:n][perm]
    for _ in range(nsorts):
        pic.pic_sort(ctx, st, tiled=True)
    times = []
    for step in range(24):
        if step in (10, 20):
            pic.pic_sort(ctx, st, tiled=True)
            if step == 20:
                pic.pic_sort(ctx, st, tiled=True)
            torch.cuda.synchronize()
            m = st.n
            zi = st.z[:m].floor().long(); xi = st.x[:m].floor().long()
            key = (((zi >> 4) * (nx // 16) + (xi >> 4)) << 8) | ((zi & 15) << 4) | (xi & 15)
            d = key[1:] - key[:-1]
            print("step", step, "n", m, "descents", int((d < 0).sum()), "distinct keys", int(torch.unique(key).numel()), flush=True)
            vz = st.uz[:m]
            print("  corr(frac z, uz) in sorted order:", float(torch.corrcoef(torch.stack([st.z[:m] - zi, vz]))[0, 1]), flush=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pic.pic_step(ctx, st, 128, -1.0, -1e-4, 0.5, clock=True, field_solve=False, tiled=True)
        e1.record()
        torch.cuda.synchronize()
        times.append(round(e0.elapsed_time(e1), 2))
    print("sorts", nsorts, "shuffled", shuffle, times, flush=True)
    del st
