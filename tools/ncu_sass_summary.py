"""Summarise an `ncu --page source --csv --print-source sass` dump: stall
samples and executed instructions per SASS region (split at BAR / branch
targets), top instructions by stall samples."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot_samples = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
tot_inst = sum(float(r[ix["Instructions Executed"]] or 0) for r in data)
print(f"total samples {tot_samples:.0f}, warp instructions {tot_inst:.0f}")
# per-region: cut at BAR.SYNC
region, acc = 0, defaultdict(lambda: [0.0, 0.0, defaultdict(float), ""])
for r in data:
    src = r[ix["Source"]]
    a = acc[region]
    if not a[3]:
        a[3] = r[ix["Address"]]
    a[0] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    a[1] += float(r[ix["Instructions Executed"]] or 0)
    for s in stall_cols:
        a[2][s] += float(r[ix[s]] or 0)
    if "BAR.SYNC" in src or "BAR.RED" in src:
        region += 1
for k, (smp, ins, st, addr) in sorted(acc.items()):
    top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
    print(f"region {k} @{addr}: samples {100*smp/tot_samples:5.1f}%  inst {100*ins/tot_inst:5.1f}%  " +
          ", ".join(f"{n[6:]} {100*v/max(smp,1):.0f}%" for n, v in top))
print("top instructions by samples:")
for r in sorted(data, key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:25]:
    st = sorted(((s, float(r[ix[s]] or 0)) for s in stall_cols), key=lambda kv: -kv[1])[:2]
    print(f"  {r[ix['Address']]} {float(r[ix['Warp Stall Sampling (All Samples)']] or 0):6.0f} "
          f"{r[ix['Source']][:60]:60s} " + " ".join(f"{n[6:]}={v:.0f}" for n, v in st))
