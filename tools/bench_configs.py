"""All five BASELINE.json configs on one GPU vs the C restatement on the host.

Time-to-solution (end to end from host numpy buffers, median of reps) and
search-tree nodes/s; gnp400 / torus60 are beyond exact search within any
budget here, so both sides run a fixed time budget and report nodes/s and the
best bound reached.  Writes one JSON document to stdout.
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

BUDGET = float(os.environ.get("BUDGET_S", "10"))
CPU = os.environ.get("CPU", "1") == "1"
SKIP_CPU = set(os.environ.get("SKIP_CPU", "").split(","))


def gpu_solve(n, off, nbr, reps=3, **kw):
    """Median end-to-end time over `reps` solves after one untimed warm-up
    solve (first-call costs -- module load, pooled buffer growth -- excluded)."""
    times, r = [], None
    warm = dict(kw, timeout=0.2) if kw.get("timeout") else kw
    vc.solve(vc.StaticGraph(n, np.array(off), np.array(nbr)), vc.SolverConfig(**warm))
    for _ in range(reps):
        t = time.perf_counter()
        g = vc.StaticGraph(n, np.array(off), np.array(nbr))
        r = vc.solve(g, vc.SolverConfig(**kw))
        times.append(time.perf_counter() - t)
    return statistics.median(times), r


def cpu_solve(n, off, nbr, **kw):
    t = time.perf_counter()
    r = oracle.solve(n, off, nbr, **kw)
    return time.perf_counter() - t, r


out = {"budget_s": BUDGET, "host_cores": os.cpu_count(), "configs": {}}
for name, label in [("er200", "configs[0] MVC G(200, avg deg 4)"),
                    ("rgg2000", "configs[1] PVC pair RGG n=2000"),
                    ("ba100k", "configs[2] MVC BA n=100k m=3"),
                    ("planted1m", "configs[3] MVC planted n=1M"),
                    ("gnp400", "configs[4] G(400, 0.1), time budget"),
                    ("torus60", "configs[4] torus 60x60, time budget")]:
    n, off, nbr = synth.WORKLOADS[name]()
    e = {"label": label, "n": n, "m": int(off[-1] // 2)}
    bounded = name in ("gnp400", "torus60")
    if name == "rgg2000":
        opt = vc.solve(vc.StaticGraph(n, off, nbr), vc.SolverConfig()).cover_size
        tg, nodes = 0.0, 0
        for k in (opt, opt - 1):
            t, r = gpu_solve(n, off, nbr, mode="pvc", k=k)
            tg += t
            nodes += r.stats.tree_nodes_visited
        e.update(gpu_s=tg, gpu_nodes=nodes, answer={"opt": opt, "found_opt": True,
                                                      "found_opt_minus_1": False})
        if CPU:
            tc, nc = 0.0, 0
            for k, want in ((opt, True), (opt - 1, False)):
                t, r = cpu_solve(n, off, nbr, mode="pvc", k=k, deterministic=True)
                assert r["found"] == want
                tc += t
                nc += r["stats"]["tree_nodes_visited"]
            e.update(cpu_s=tc, cpu_nodes=nc)
    else:
        kw = dict(timeout=BUDGET) if bounded else {}
        tg, r = gpu_solve(n, off, nbr, reps=1 if bounded else 3, **kw)
        e.update(gpu_s=tg, gpu_nodes=r.stats.tree_nodes_visited, gpu_cover=r.cover_size,
                 gpu_exact=r.exact, gpu_search_ms=r.search_ms,
                 gpu_root_s=r.stats.phase_seconds["root_reduce"])
        if CPU and name not in SKIP_CPU:
            tc, rc = cpu_solve(n, off, nbr, deterministic=True, timeout=BUDGET if bounded else None)
            e.update(cpu_s=tc, cpu_nodes=rc["stats"]["tree_nodes_visited"], cpu_cover=rc["cover_size"],
                     cpu_exact=rc["exact"])
            if not bounded:
                assert rc["cover_size"] == r.cover_size, (name, rc["cover_size"], r.cover_size)
    if e.get("gpu_s"):
        e["gpu_nodes_per_s"] = e["gpu_nodes"] / e["gpu_s"]
    if e.get("cpu_s"):
        e["cpu_nodes_per_s"] = e["cpu_nodes"] / e["cpu_s"]
        e["speedup_time_to_solution"] = e["cpu_s"] / e["gpu_s"] if not bounded else None
    out["configs"][name] = e
    print(json.dumps({name: e}), file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
