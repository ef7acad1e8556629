#!/usr/bin/env python
"""Per-source-line instruction and stall attribution for one kernel of an
.ncu-rep: correlates the report's SASS listing with `nvdisasm -g` of the
locally built cubin (same sources/flags => same instruction order).
usage: ncu_lines.py REP CUBIN KERNEL_SUBSTRING N_PARTICLES [top]"""
import collections
import csv
import io
import re
import subprocess
import sys


def main(rep, cubin, kname, npart, top=40):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h, data = rows[1], rows[2:]
    sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
    start = [i for i, l in enumerate(sass) if l.startswith(".text.") and kname in l][0]
    cur, insts = None, []
    for l in sass[start + 1:]:
        if l.startswith(".text.") or l.startswith("//----"):
            break
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1), int(m.group(2)))
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+", l):
            insts.append(cur)
    assert len(insts) == len(data), (len(insts), len(data))
    ie, iS = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    il = h.index("stall_long_sb")
    agg, st, lsb = collections.Counter(), collections.Counter(), collections.Counter()
    for c, r in zip(insts, data):
        agg[c] += int(r[ie]); st[c] += int(r[iS]); lsb[c] += int(r[il])
    ts = sum(st.values())
    print(f"total inst/particle {sum(agg.values()) * 32 / npart:.1f}; samples {ts}")
    for c, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{c[0]}:{c[1]:<5d} inst/particle {v * 32 / npart:6.1f}  stall {100 * st[c] / ts:5.1f}%  long_sb {100 * lsb[c] / ts:5.1f}%")


if __name__ == "__main__":
    a = sys.argv
    main(a[1], a[2], a[3], float(a[4]), int(a[5]) if len(a) > 5 else 40)
