#!/usr/bin/env python
"""Summarise one kernel of an .ncu-rep (raw page) into a short text block for profiles/."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_atom.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def main(rep, label=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print(f"# {label} {d.get('Kernel Name', '')}  grid {d.get('Grid Size', '')} block {d.get('Block Size', '')}")
        for k in KEYS:
            if k in d:
                print(f"{k:60s} {d[k]:>20s} {u.get(k, '')}")
        st = sorted(((float(d[k]), k) for k in d if k.startswith("smsp__average_warps_issue_stalled")
                     and k.endswith("per_issue_active.ratio") and d[k] not in ("", "n/a")), reverse=True)
        print("top stalls (warps per issue):", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, k in st[:6]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
