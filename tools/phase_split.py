"""Split an ncu source-page CSV (--page source --csv --print-source sass)
into phases delimited by barriers / mbarrier waits / tcgen05 instructions,
with stall-sample shares and the dominant stall reasons per phase."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
rows = rows[2:]
si = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[si]) for r in rows)
marks = [i for i, r in enumerate(rows) if any(k in r[1] for k in ("BAR.SYNC", "TRYWAIT", "UTCHMMA", "UTCMMA", "LDTM", "STTM"))]
prev = 0
for m in marks + [len(rows) - 1]:
    seg = rows[prev:m + 1]
    s = sum(int(r[si]) for r in seg)
    if s > 0.01 * tot:
        rs = sorted(((sum(int(r[i]) for r in seg), hdr[i]) for i in reasons), reverse=True)[:3]
        print(f"{prev:5d}-{m:5d} {100 * s / tot:5.1f}%  {rows[m][1].strip()[:44]:44s} "
              + " ".join(f"{n[6:]}={100 * v / max(s, 1):.0f}%" for v, n in rs))
    prev = m + 1
