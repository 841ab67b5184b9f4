"""PVC on the large configs (real root budget: the frontier kernel's
high-degree path): answers and times."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

for name, opt in (("planted1m", 243097), ("ba100k", 48591)):
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    for k in (opt, opt - 1, opt - 1000, opt + 1000):
        vc.solve(g, vc.SolverConfig(mode="pvc", k=k))
        t = time.perf_counter()
        r = vc.solve(g, vc.SolverConfig(mode="pvc", k=k))
        dt = time.perf_counter() - t
        print(f"{name} pvc k={k}: found={r.found} cover={r.cover_size} {dt*1e3:.3f} ms "
              f"root kernel {r.root_kernel} hd={r.stats.rule_counts['high_degree']}", flush=True)
