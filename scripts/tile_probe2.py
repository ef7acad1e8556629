"""ncu target: fresh (8 per cell) state -> sort -> step, then the state
shifted by 0.01 cells -> sort -> step (tile kernels 2 and 4 of the run)."""
import runpy, sys
from pathlib import Path
sys.argv = ["x"]
import os
os.environ["PROBE_MINIMAL"] = "1"
exec(open(Path(__file__).with_name("tile_sort_probe.py")).read().split("# which part of the state makes it slow?")[0].replace('print("initial sort (gpu ms, host ms)", ev(sort))', 'ev(sort)').split('print("sort again')[0])
def restore(shift):
    for k in ("z", "x", "uz", "ux", "uy"):
        getattr(st, k).copy_(init[k])
    st.n = n
    if shift:
        st.z[:n].add_(shift); st.x[:n].add_(shift)
        st.z[:n].clamp_(0.0, nz - 1e-6); st.x[:n].clamp_(0.0, nx - 1e-6)
for sh in (0.0, 0.01):
    restore(sh)
    ev(sort)
    print("shift", sh, "step", ev(step)[:2])
