"""gnp400 / torus60 nodes/s (time budget) at warp limits 64 / 128 / auto."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

B = float(os.environ.get("BUDGET_S", "5"))
for name in sys.argv[1:] or ["gnp400", "torus60"]:
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    vc.solve(g, vc.SolverConfig(timeout=0.2))
    for wl in (64, 128, 256, -1):
        t = time.perf_counter()
        r = vc.solve(g, vc.SolverConfig(timeout=B, warp_limit=wl))
        dt = time.perf_counter() - t
        print(f"{name} wl={wl}: best={r.cover_size} nodes={r.stats.tree_nodes_visited} "
              f"warp_nodes={r.warp_nodes} {r.stats.tree_nodes_visited/dt/1e6:.1f} M/s "
              f"blocks={r.blocks}x{r.threads}", flush=True)
