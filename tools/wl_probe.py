"""warp_limit 64 vs 128: rgg2000 PVC pair, gnp MVC instances."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
for wl in (64, 128):
    for k in (1282, 1281):
        ts = []
        for _ in range(7):
            t = time.perf_counter()
            r = vc.solve(g, vc.SolverConfig(mode="pvc", k=k, warp_limit=wl))
            ts.append((time.perf_counter() - t) * 1e3)
        ts.sort()
        print(f"rgg2000 wl={wl} k={k}: found={r.found} {ts[3]:.3f} ms nodes={r.stats.tree_nodes_visited} "
              f"warp_nodes={r.warp_nodes} search={r.search_ms:.3f} blocks={r.blocks}x{r.threads}", flush=True)
for (nn, p) in ((160, 0.1), (180, 0.08)):
    n, off, nbr = synth.gnp(nn, p, 1)
    g2 = vc.StaticGraph(n, off, nbr)
    for wl in (64, 128):
        t = time.perf_counter()
        r = vc.solve(g2, vc.SolverConfig(warp_limit=wl, timeout=30))
        dt = time.perf_counter() - t
        print(f"gnp{nn}_{p} wl={wl}: mvc={r.cover_size} exact={r.exact} nodes={r.stats.tree_nodes_visited} "
              f"warp_nodes={r.warp_nodes} {dt:.3f} s {r.stats.tree_nodes_visited/dt/1e6:.1f} M/s", flush=True)
