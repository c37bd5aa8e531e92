"""Per-source-line instruction counts and stall samples of one kernel in an
ncu report (--import-source on, -lineinfo builds), plus its SASS opcode mix.
Usage: python tools/ncu_lines.py gpurun_out/X.ncu-rep [top_n]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines, ops = [], collections.Counter()
fname, tot = "?", 0
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        continue
    try:
        n, st = int(row[7]), int(row[4])
    except (ValueError, IndexError):
        continue
    if row[0]:  # a CUDA source line (aggregate of its SASS)
        lines.append((n, st, f"{fname}:{row[0]}", row[1].strip()[:90]))
        tot += n
    else:
        op = re.sub(r"^@!?U?P\w+\s+", "", row[3].strip()).split(" ")[0]
        ops[op] += n
print(f"total warp instructions {tot}")
for n, st, loc, src in sorted(lines, reverse=True)[:top]:
    print(f"{n / 1e6:7.2f}M {100 * n / tot:5.1f}% stall {st:5d}  {loc:22s} {src}")
print()
for o, n in ops.most_common(25):
    print(f"{o:22s} {n / 1e6:7.2f}M {100 * n / tot:5.1f}%")
