import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
for i in range(6):
    t = time.perf_counter()
    pre = vc.root_reduce(g, bound=1281)
    t1 = time.perf_counter()
    r = vc.solve(g, vc.SolverConfig(mode="pvc", k=1282))
    t2 = time.perf_counter()
    print(f"root_reduce {1e3*(t1-t):.3f} ms  seconds={pre.seconds}  solve(pvc opt) {1e3*(t2-t1):.3f} ms phases={r.stats.phase_seconds} kern={r.search_ms:.3f}", file=sys.stderr, flush=True)
