#!/usr/bin/env python
"""SASS opcode mix of one kernel in an .ncu-rep: warp instructions executed
per opcode (from the source page), per particle.
usage: ncu_opmix.py REP N_PARTICLES [top]"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, npart, top=30):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h, data = rows[1], rows[2:]
    ie, ia = h.index("Instructions Executed"), h.index("Source")
    mix = collections.Counter()
    for r in data:
        ins = r[ia].strip()
        if ins.startswith("@"):
            ins = ins.split(None, 1)[1] if " " in ins else ins
        op = ins.split()[0] if ins else "?"
        mix[op.split(".")[0]] += int(r[ie] or 0)
    tot = sum(mix.values())
    print(f"# {tot} warp instructions = {tot * 32 / npart:.1f} thread instructions per particle")
    for op, v in mix.most_common(top):
        print(f"{op:12s} {v:14d}  {100 * v / tot:5.1f} %  {v * 32 / npart:6.1f} /particle")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 30)
