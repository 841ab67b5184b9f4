"""Single parallel PVC(opt-1) solve on rgg2000 for an ncu capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1281
wl = int(os.environ.get("WL", "-1"))
for _ in range(2):
    r = vc.solve(g, vc.SolverConfig(mode="pvc", k=k, warp_limit=wl))
print("nodes", r.stats.tree_nodes_visited, "found", r.found, "kern", r.search_ms)
