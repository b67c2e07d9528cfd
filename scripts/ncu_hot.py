"""Top SASS instructions / CUDA lines by warp-stall samples from an ncu report.

usage: python scripts/ncu_hot.py report.ncu-rep [N] [sass|cuda] [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
mode = sys.argv[3] if len(sys.argv) > 3 else "sass"
kern = sys.argv[4] if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", mode]
                     + (["-k", "regex:" + kern] if kern else []),
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"') or l.startswith('"Line"') or l.startswith('"#"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
col = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
rows = [r for r in rows[1:] if len(r) > col and r[col] not in ("", None) and r[col] != hdr[col]]
tot = sum(float(r[col]) for r in rows)
top = sorted(rows, key=lambda r: -float(r[col]))[:n]
print("total samples", tot)
for r in top:
    print("%6.2f%%  %s  %s" % (100 * float(r[col]) / tot, r[0], r[src].strip()[:110]))
