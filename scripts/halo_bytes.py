"""Per-step guard-exchange bytes of the box-decomposed PIC (parallel.PicHalo
plans) for the C2 geometry at 8 ranks, against the round-1 scheme (all-reduce
of the 16 x int64 current rows of the union deposit box + replicated fields)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import lbsim_oracle as O  # noqa: E402
from paper_2104_11385_b200.parallel import cell_owner_map, halo_plan  # noqa: E402

nz = nx = 960
M, R = 32, 8
nbz = nbx = nz // M
pos, counts = O.init_scenario((nz, nx), M, (480.0, 480.0), 64.0, 4.0, 55.0, 7)
work = O.true_work(counts, M, (0.75, 0.25))
maps = {"slab": O.slab_mapping(nbz * nbx, R), "knapsack": O.knapsack_assign(work, R),
        "sfc": O.sfc_assign(work, O.morton_order(nbz, nbx), R)}
fa, fb = O.interior_faces(nbz, nbx)
out = {"grid": [nz, nx], "box": M, "ranks": R}
# round 1: union deposit box of the blob (rows) x 16 int64, all-reduced by every rank
rows = np.flatnonzero(counts.reshape(nbz, nbx).sum(axis=1) > 0)
union_rows = (rows[-1] - rows[0] + 1) * M + 2
out["round1_allreduce_bytes_per_rank"] = int(union_rows * nx * 16 * 8)
for name, owner in maps.items():
    cells = cell_owner_map(owner, (nbz, nbx), M)
    per = []
    for r in range(R):
        js, _ = halo_plan(cells, cells, r, R, 1, 1)
        fs, _ = halo_plan(cells, cells, r, R, 0, 2)
        per.append(16 * 8 * sum(a.size for a in js) + 6 * 4 * sum(a.size for a in fs))
    off = int(np.sum(owner[fa] != owner[fb]))
    out[name] = {"off_rank_faces": off, "bytes_per_step_max_rank": int(max(per)),
                 "bytes_per_step_total": int(sum(per)),
                 "bytes_per_off_rank_face": float(sum(per) / max(off, 1))}
print(json.dumps(out, indent=1))
