"""Block size vs throughput on the wide-warp-tier instances."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

for (nn, p, budget) in ((180, 0.08, None), (400, 0.1, 3.0), (150, 0.1, None)):
    n, off, nbr = synth.gnp(nn, p, 1)
    g = vc.StaticGraph(n, off, nbr)
    vc.solve(g, vc.SolverConfig(timeout=0.3))
    for th in (0, 64, 128, 256):
        t = time.perf_counter()
        r = vc.solve(g, vc.SolverConfig(threads=th, timeout=budget))
        dt = time.perf_counter() - t
        print(f"gnp{nn}_{p} threads={th}: blocks={r.blocks}x{r.threads} mvc={r.cover_size} "
              f"exact={r.exact} {dt:.3f} s {r.stats.tree_nodes_visited/dt/1e6:.1f} M nodes/s "
              f"warp share {r.warp_nodes/max(1,r.stats.tree_nodes_visited):.3f}", flush=True)
