"""Time lbx_pic_sort(tiled) and the tiled step after it separately on the
sparse plasma (4096^2 x 8 ppc): where does a sorting step's time go?"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2104_11385_b200 import device, pic

dev = torch.device("cuda:0")
nz = nx = 4096
ppc = 8
rng = np.random.default_rng(42)
cell = np.repeat(np.arange(nz * nx, dtype=np.int64), ppc)
off = rng.random((cell.size, 2))
pos0 = np.column_stack([(cell // nx) + off[:, 0], (cell % nx) + off[:, 1]])
u0 = rng.normal(0.0, 0.05, size=(cell.size, 3))
n = pos0.shape[0]
ctx = device.Context(dev, capacity=n)
st = pic.PicState.create(pos0[:1], u0[:1], nz, nx, device=dev)
for name, col in (("z", pos0[:, 0]), ("x", pos0[:, 1]), ("uz", u0[:, 0]), ("ux", u0[:, 1]), ("uy", u0[:, 2])):
    t = torch.zeros(n + 2, dtype=torch.float64, device=dev)
    t[:n].copy_(torch.from_numpy(np.ascontiguousarray(col)).to(dev))
    setattr(st, name, t)
st.n = n
init = {k: getattr(st, k).clone() for k in ("z", "x", "uz", "ux", "uy")}
for name in ("Ex", "Ey", "Ez", "Bx", "By", "Bz"):
    if hasattr(st, name):
        getattr(st, name).normal_(0.0, 1e-3)
stream = torch.cuda.current_stream(dev)

import os
try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:   # noqa: BLE001
    _h = None
SLEEP = float(os.environ.get("PROBE_SLEEP", "0"))

def clk():
    if _h is None:
        return None
    return (pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM),
            hex(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(_h)))

def ev(fn):
    torch.cuda.synchronize(dev)
    if SLEEP:
        time.sleep(SLEEP)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record(stream)
    fn()
    e1.record(stream)
    h1 = time.perf_counter()
    c = clk()
    torch.cuda.synchronize(dev)
    return round(e0.elapsed_time(e1), 3), round((h1 - h0) * 1e3, 3), c

step = lambda: pic.pic_step(ctx, st, 128, -1.0, -1e-4, 0.5, clock=True, field_solve=False,
                            sort=False, tiled=True, fast=True)
sort = lambda: pic.pic_sort(ctx, st, tiled=True)
print("initial sort (gpu ms, host ms)", ev(sort))
print("sort again, no step between", ev(sort), "again", ev(sort))
for k in range(3):
    print("step", ev(step))
# which part of the state makes it slow?
def restore(shift=0.0, seed=None):
    for k in ("z", "x", "uz", "ux", "uy"):
        getattr(st, k).copy_(init[k])
    st.n = n
    if shift:
        st.z[:n].add_(shift)
        st.x[:n].add_(shift)
        st.z[:n].clamp_(0.0, nz - 1e-6)
        st.x[:n].clamp_(0.0, nx - 1e-6)
    if seed is not None:   # random sub-cell jitter (cells kept)
        g = torch.Generator(device=dev).manual_seed(seed)
        for k in ("z", "x"):
            t = getattr(st, k)[:n]
            t.copy_(torch.floor(t) + torch.rand(n, device=dev, dtype=torch.float64, generator=g))
restore()
print("fresh: sort", ev(sort)[:2], "step", ev(step)[:2], "step", ev(step)[:2], "step", ev(step)[:2])
print("evolved: sort", ev(sort)[:2], "sort", ev(sort)[:2], "step", ev(step)[:2])
for sh in (0.01, 0.3):
    restore(shift=sh)
    print("shift", sh, "sort", ev(sort)[:2], "sort", ev(sort)[:2], "step", ev(step)[:2])
restore(seed=1)
print("jitter: sort", ev(sort)[:2], "sort", ev(sort)[:2], "step", ev(step)[:2])
restore()
st.uz[:n].mul_(0.0); st.ux[:n].mul_(0.0); st.uy[:n].mul_(0.0)
print("u=0: sort", ev(sort)[:2], "step", ev(step)[:2], "step", ev(step)[:2], "step", ev(step)[:2], "sort", ev(sort)[:2], "step", ev(step)[:2])
# is it the layout?  key order of the state right after a re-sort
torch.cuda.synchronize(dev)
print("sort", ev(sort))
z = st.z[:st.n].cpu().numpy(); x = st.x[:st.n].cpu().numpy()
iz, ix = z.astype(np.int64), x.astype(np.int64)
key = ((iz >> 4) * (nx >> 4) + (ix >> 4)) * 256 + (iz & 15) * 16 + (ix & 15)
d = np.diff(key)
print("keys non-decreasing:", bool((d >= 0).all()), "descents:", int((d < 0).sum()), "n", st.n)
same = (d == 0).mean()
print("fraction of neighbours in the same cell:", round(float(same), 4))
