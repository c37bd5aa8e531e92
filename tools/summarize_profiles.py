"""Summarise a round's ncu evidence into profiles/ (tracked):
  profiles/ncu_launches_<R>.md  per-kernel launch count, total / mean time and
                                share of the step from the launch list;
  profiles/ncu_full_<R>.json    per-kernel metrics of the --set full capture
                                (dram bytes per launch -> bench.py roofline
                                'traffic');
  profiles/ncu_summary_<R>.md   human-readable table of the above.
Usage: python tools/summarize_profiles.py r01
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1] if len(sys.argv) > 1 else "r01"
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
os.makedirs(PROF, exist_ok=True)


def short(name):
    m = re.match(r"(?:void )?(?:ccrd::)?([A-Za-z_0-9]+)", name)
    return m.group(1) if m else name


# ---- launch list
launch_md = []
lp = os.path.join(OUT, f"launches_{R}.csv")
if os.path.exists(lp):
    text = open(lp).read()
    text = text[text.index('"ID"'):] if '"ID"' in text else text
    rows = list(csv.DictReader(io.StringIO(text)))
    per = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "ns")
            ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}.get(unit, 1)
            per[short(r["Kernel Name"])].append(ns)
    tot = sum(sum(v) for v in per.values())
    launch_md.append(f"# ncu launch list ({R})\n")
    launch_md.append("`ncu --metrics gpu__time_duration.sum --clock-control none` over "
                     "`python bench.py --images 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline` "
                     "(cold-cache, serialised: compare shares, not absolutes).\n")
    launch_md.append("| kernel | launches | total us | mean us | share |")
    launch_md.append("|---|---|---|---|---|")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        launch_md.append(f"| {k} | {len(v)} | {sum(v)/1e3:.1f} | {sum(v)/len(v)/1e3:.2f} | {sum(v)/tot:.3f} |")
    open(os.path.join(PROF, f"ncu_launches_{R}.md"), "w").write("\n".join(launch_md) + "\n")

# ---- full capture
import glob
fps = sorted(glob.glob(os.path.join(OUT, f"full_{R}*.ncu-rep")))
want = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_active_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_inst_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}
kern = {}
for fp in fps:
    raw = subprocess.run(["ncu", "-i", fp, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = short(r[hdr.index("Kernel Name")])
        d = {}
        for m, key in want.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    val = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if key.startswith("dram_"):
                    val *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                if key == "duration":
                    val *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
                    key = "duration_us"
                if key == "sm_clock":
                    val *= {"hertz": 1e-9, "Khertz": 1e-6, "Mhertz": 1e-3, "Ghertz": 1, "cycle/nsecond": 1,
                            "cycle/second": 1e-9}.get(u, 1)
                    key = "sm_clock_ghz"
                d[key] = val
        d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
        kern.setdefault(name, d)
if kern:
    json.dump({"round": R, "source": f"ncu --set full --clock-control none captures full_{R}_<kernel>.ncu-rep "
                                     "(one launch per kernel, 2K image of the bench workload)",
               "kernels": kern}, open(os.path.join(PROF, f"ncu_full_{R}.json"), "w"), indent=1)

# ---- summary
bp = os.path.join(OUT, f"bench_{R}.json")
md = [f"# ncu summary ({R})\n"]
if os.path.exists(bp):
    b = json.loads(open(bp).read().strip().splitlines()[-1])
    md.append(f"bench: {b['value']:.4g} px/s, {b['ms_per_step']:.2f} ms/step, roofline frac "
              f"{b['roofline']['frac']:.3f} ({b['roofline']['kernel']}), whole step "
              f"{b['path_roofline']['frac']:.3f}, clocks {b['clocks']}\n")
md.append("| kernel | us | DRAM MB/launch | FMA pipe active % | FMA inst % | issue % | occupancy % | regs | SM GHz |")
md.append("|---|---|---|---|---|---|---|---|---|")
for k, d in kern.items():
    md.append(f"| {k} | {d.get('duration_us', 0):.1f} | {d['dram_bytes_per_launch']/1e6:.2f} | "
              f"{d.get('fma_pipe_active_pct', 0):.1f} | {d.get('fma_inst_pct', 0):.1f} | "
              f"{d.get('issue_active_pct', 0):.1f} | {d.get('occupancy_pct', 0):.1f} | {d.get('registers', 0):.0f} | "
              f"{d.get('sm_clock_ghz', 0):.3f} |")
md += [""] + launch_md[1:]
open(os.path.join(PROF, f"ncu_summary_{R}.md"), "w").write("\n".join(md) + "\n")
print("\n".join(md))
