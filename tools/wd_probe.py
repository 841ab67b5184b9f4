import os, sys
sys.path.insert(0, os.getcwd())
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth, _lib
n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
for i in range(3):
    r = vc.solve(g, vc.SolverConfig())
    print("mvc", r.cover_size, "exact", r.exact, "search_ms", round(r.search_ms, 3), "nodes", r.stats.tree_nodes_visited, flush=True)
