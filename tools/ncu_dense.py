"""One parallel MVC solve of G(n, p) (default the strong instance G(180, 0.08)),
for an ncu capture of the wide warp tier."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

nn = int(sys.argv[1]) if len(sys.argv) > 1 else 180
p = float(sys.argv[2]) if len(sys.argv) > 2 else 0.08
n, off, nbr = synth.gnp(nn, p, 1)
g = vc.StaticGraph(n, off, nbr)
for _ in range(2):
    r = vc.solve(g, vc.SolverConfig(timeout=float(os.environ.get("BUDGET_S", "0")) or None))
print("mvc", r.cover_size, "nodes", r.stats.tree_nodes_visited, "warp", r.warp_nodes, "ms", r.search_ms)
