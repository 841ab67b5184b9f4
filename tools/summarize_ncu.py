"""Summaries of the gpurun_out ncu artefacts for profiles/: launch list and the
search-kernel --set full capture.  usage: summarize_ncu.py TAG"""
import csv, json, subprocess, sys
from collections import defaultdict

tag = sys.argv[1]
rows = list(csv.reader(open("gpurun_out/launches.csv")))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
kn, mv = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(lambda: [0, 0.0])
for r in rows[i + 1:]:
    d[r[kn]][0] += 1
    d[r[kn]][1] += float(r[mv].replace(",", ""))
tot = sum(v[1] for v in d.values())
with open(f"profiles/{tag}_launches.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -- python bench.py --steps 2 "
            "--warmup 3 --no-cpu-baseline\n# (1 untimed MVC solve + 3 warm-up, 2 timed and 2 e2e PVC "
            "pairs = 15 solves; cold-cache, serialised)\n# count  total_ms  share  kernel\n")
    for k, v in sorted(d.items(), key=lambda x: -x[1][1]):
        f.write(f"{v[0]:5d} {v[1]/1e6:10.3f} {100*v[1]/tot:5.1f}%  {k[:110]}\n")
raw = subprocess.run(["ncu", "-i", "gpurun_out/prof_search.ncu-rep", "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
g = lambda n: v[h.index(n)]
stalls = {}
for j, x in enumerate(h):
    if x.startswith("smsp__average_warps_issue_stalled_") and x.endswith("_per_issue_active.ratio"):
        try:
            stalls[x[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v[j])
        except ValueError:
            pass
dr = float(g("dram__bytes_read.sum")) * 1e6
dw = float(g("dram__bytes_write.sum")) * 1e6
out = {
    "capture": "ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 4 -c 1 "
               "python bench.py --steps 1 --warmup 3 --no-cpu-baseline (rgg2000 PVC, parallel mode)",
    "kernel": g("Kernel Name"), "grid": g("Grid Size"), "block": g("Block Size"),
    "registers_per_thread": int(g("launch__registers_per_thread")),
    "duration_ms": float(g("gpu__time_duration.sum")),
    "dram_bytes_read": dr, "dram_bytes_write": dw, "dram_bytes_per_launch": dr + dw,
    "l2_hit_rate_pct": float(g("lts__t_sector_hit_rate.pct")),
    "sm_throughput_pct": float(g("sm__throughput.avg.pct_of_peak_sustained_elapsed")),
    "warps_active_pct_of_peak": float(g("sm__warps_active.avg.pct_of_peak_sustained_active")),
    "issue_active_pct": float(g("smsp__issue_active.avg.pct_of_peak_sustained_active")),
    "eligible_warps_per_cycle": float(g("smsp__warps_eligible.avg.per_cycle_active")),
    "instructions_executed": float(g("smsp__inst_executed.sum")),
    "top_stalls_per_issue": dict(sorted(stalls.items(), key=lambda x: -x[1])[:6]),
}
json.dump(out, open(f"profiles/{tag}_search_kernel_ncu.json", "w"), indent=1)
print(json.dumps(out, indent=1))
print(open(f"profiles/{tag}_launches.txt").read())
