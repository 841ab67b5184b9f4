"""Candidate search-heavy instances for the strong-scaling line: exact MVC
time on one GPU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

cases = [("gnp%d_%.2f" % (n, p), (lambda n=n, p=p: synth.gnp(n, p, 1))) for n, p in
         ((150, 0.1), (160, 0.1), (180, 0.08), (250, 0.06), (300, 0.05), (400, 0.03))]
cases += [("rgg%d_%.3f" % (n, r), (lambda n=n, r=r: synth.rgg(n, r, 1))) for n, r in
          ((5000, 0.02), (5000, 0.025), (10000, 0.015), (20000, 0.01))]
cases += [("torus%d" % a, (lambda a=a: synth.torus(a, a))) for a in (16, 20, 24)]
cases += [("ba%d" % n, (lambda n=n: synth.ba(n, 3, 1, pendant=0.0))) for n in (300, 500, 800)]
for name, gen in cases:
    n, off, nbr = gen()
    g = vc.StaticGraph(n, off, nbr)
    t = time.perf_counter()
    try:
        r = vc.solve(g, vc.SolverConfig(timeout=15.0))
    except Exception as e:  # noqa: BLE001
        print(f"{name}: FAILED {e}", flush=True)
        continue
    dt = time.perf_counter() - t
    print(f"{name}: n={n} m={int(off[-1])//2} residual={r.stats.root_vertices_after} "
          f"mvc={r.cover_size} exact={r.exact} nodes={r.stats.tree_nodes_visited} {dt:.3f} s",
          flush=True)
