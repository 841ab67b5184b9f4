"""Summaries of gpurun_out ncu artefacts for profiles/.

    summarize_ncu.py TAG                 launch list (gpurun_out/launches.csv)
                                         -> profiles/TAG_launches.txt
    summarize_ncu.py TAG REP NAME CMD    --set full capture gpurun_out/REP.ncu-rep
                                         -> profiles/TAG_NAME_ncu.json
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

tag = sys.argv[1]


def launches():
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
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -- python bench.py "
                "--steps 2 --warmup 3 --no-cpu-baseline --no-other-configs\n"
                "# (1 untimed + 3 warm-up + 2 timed + 2 e2e planted1m MVC solves; "
                "cold-cache, serialised)\n# count  total_ms  share  kernel\n")
        for k, v in sorted(d.items(), key=lambda x: -x[1][1]):
            f.write(f"{v[0]:5d} {v[1]/1e6:10.3f} {100*v[1]/tot:5.1f}%  {k[:110]}\n")
    print(open(f"profiles/{tag}_launches.txt").read())


def full(rep, name, cmd):
    raw = subprocess.run(["ncu", "-i", f"gpurun_out/{rep}.ncu-rep", "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]

    def g(n, scale=True):
        x = v[h.index(n)].replace(",", "")
        if not scale:
            return x
        u = units[h.index(n)]
        f = float(x)
        return f * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "ms": 1, "us": 1e-3,
                    "ns": 1e-6, "Tbyte/s": 1e12, "Gbyte/s": 1e9, "Mbyte/s": 1e6}.get(u, 1)

    stalls = {}
    for j, x in enumerate(h):
        if x.startswith("smsp__average_warps_issue_stalled_") and \
                x.endswith("_per_issue_active.ratio"):
            try:
                stalls[x[len("smsp__average_warps_issue_stalled_"):
                         -len("_per_issue_active.ratio")]] = float(v[j])
            except ValueError:
                pass
    opt = {}
    for key in ("lts__t_sectors.sum", "lts__t_requests.sum",
                "lts__t_requests_srcunit_tex_op_atom_dot_alu.sum",
                "lts__t_requests_srcunit_tex_op_atom_dot_cas.sum",
                "lts__t_requests_srcunit_tex_op_red.sum",
                "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
                "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
                "sm__warps_active.avg.pct_of_peak_sustained_active"):
        if key in h:
            try:
                opt[key] = g(key)
            except ValueError:
                pass
    dur_ms = g("gpu__time_duration.sum")
    dr, dw = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    out = {
        "capture": cmd,
        "kernel": g("Kernel Name", False), "grid": g("Grid Size", False),
        "block": g("Block Size", False),
        "registers_per_thread": int(g("launch__registers_per_thread")),
        "duration_ms": dur_ms,
        "dram_bytes_read": dr, "dram_bytes_write": dw, "dram_bytes_per_launch": dr + dw,
        "dram_gbs": (dr + dw) / (dur_ms * 1e-3) / 1e9,
        "l2_hit_rate_pct": float(g("lts__t_sector_hit_rate.pct")),
        "sm_throughput_pct": float(g("sm__throughput.avg.pct_of_peak_sustained_elapsed")),
        "issue_active_pct": float(g("smsp__issue_active.avg.pct_of_peak_sustained_active")),
        "eligible_warps_per_cycle": float(g("smsp__warps_eligible.avg.per_cycle_active")),
        "instructions_executed": float(g("smsp__inst_executed.sum")),
        "top_stalls_per_issue": dict(sorted(stalls.items(), key=lambda x: -x[1])[:6]),
    }
    if "lts__t_sectors.sum" in opt:
        out["l2_bytes"] = 32 * opt["lts__t_sectors.sum"]
        out["l2_gbs"] = out["l2_bytes"] / (dur_ms * 1e-3) / 1e9
        out["l2_sector_throughput_pct_of_peak"] = opt.get(
            "lts__t_sectors.avg.pct_of_peak_sustained_elapsed")
    at = sum(opt.get(k, 0.0) for k in ("lts__t_requests_srcunit_tex_op_atom_dot_alu.sum",
                                        "lts__t_requests_srcunit_tex_op_atom_dot_cas.sum",
                                        "lts__t_requests_srcunit_tex_op_red.sum"))
    if at:
        out["l2_atomic_requests"] = at
        out["l2_atomic_requests_per_s"] = at / (dur_ms * 1e-3)
        out["l2_atomic_unit_active_pct_of_peak"] = opt.get(
            "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed")
    if "sm__warps_active.avg.pct_of_peak_sustained_active" in opt:
        out["warps_active_pct_of_peak"] = opt["sm__warps_active.avg.pct_of_peak_sustained_active"]
    json.dump(out, open(f"profiles/{tag}_{name}_ncu.json", "w"), indent=1)
    print(json.dumps(out, indent=1))


if len(sys.argv) == 2:
    launches()
else:
    full(sys.argv[2], sys.argv[3], " ".join(sys.argv[4:]))
