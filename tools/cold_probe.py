import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
for name in ("rgg2000", "torus60"):
    n, off, nbr = synth.WORKLOADS[name]()
    t = time.perf_counter()
    r = vc.solve(vc.StaticGraph(n, off, nbr), vc.SolverConfig(timeout=1.0))
    print(name, "cold wall", round(time.perf_counter() - t, 3), "s, search_ms", round(r.search_ms, 1), flush=True)
