"""PVC pair on rgg2000: sequential solve() vs solve_batch() wall time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
opt = vc.solve(g, vc.SolverConfig()).cover_size
cfgs = [vc.SolverConfig(mode="pvc", k=opt), vc.SolverConfig(mode="pvc", k=opt - 1)]
for label, fn in (("sequential", lambda: [vc.solve(g, c) for c in cfgs]),
                  ("batch", lambda: vc.solve_batch(g, cfgs))):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(20):
        t = time.perf_counter()
        rs = fn()
        ts.append(time.perf_counter() - t)
        assert rs[0].found and not rs[1].found
    ts.sort()
    print(f"{label}: median {ts[10]*1e3:.3f} ms  min {ts[0]*1e3:.3f} ms  nodes {sum(r.stats.tree_nodes_visited for r in rs)}"
          f"  blocks {[r.blocks for r in rs]} kern {[round(r.search_ms, 3) for r in rs]}", flush=True)
