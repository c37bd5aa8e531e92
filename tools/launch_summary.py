"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel total / count / mean (us), divided by --passes."""
import collections
import csv
import sys

path = sys.argv[1]
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rows = list(csv.reader(open(path)))
hdr = None
tot = collections.defaultdict(float)
n = collections.Counter()
seq = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) < len(hdr):
        continue
    k = r[hdr.index("Kernel Name")][:80]
    v = float(r[hdr.index("Metric Value")].replace(",", ""))
    unit = r[hdr.index("Metric Unit")]
    v = v / 1e3 if unit == "nsecond" else v * 1e3 if unit == "msecond" else v
    tot[k] += v
    n[k] += 1
    seq.append((k, v))
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:15]:
    print(f"{v / passes:10.1f} us/pass {100 * v / s:5.1f}%  n={n[k] // passes:4d}  mean {v / n[k]:8.1f} us  {k}")
if "-v" in sys.argv:
    for k, v in seq[: len(seq) // passes]:
        print(f"{v:9.1f} {k[:60]}")
