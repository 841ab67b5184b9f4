"""Ad-hoc GPU sweep of search-kernel launch knobs on one workload."""
import itertools, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth

name = sys.argv[1] if len(sys.argv) > 1 else "rgg2000"
n, off, nbr = synth.WORKLOADS[name]()
g = vc.StaticGraph(n, off, nbr)
opt = vc.solve(g, vc.SolverConfig()).cover_size
print("opt", opt, flush=True)
for thr, threads, workers in itertools.product([0], [32, 64, 128, 256, 512], [0, 148 * 2, 148 * 4, 148 * 8]):
    tk = []
    for k in (opt, opt - 1):
        best = None
        for rep in range(3):
            t = time.perf_counter()
            r = vc.solve(g, vc.SolverConfig(mode="pvc", k=k, worklist_threshold=thr or None,
                                            threads=threads, workers=workers))
            wall = (time.perf_counter() - t) * 1e3
            if best is None or wall < best[0]:
                best = (wall, r.search_ms, r.stats.tree_nodes_visited, r.stats.worklist_pushes)
        tk.append(best)
    print(f"thr={thr:>10} threads={threads:3d} workers={workers:3d} | " +
          " | ".join(f"wall {w:6.1f} ms kern {k:6.2f} ms nodes {nd:6d} push {p:6d}" for w, k, nd, p in tk),
          flush=True)
