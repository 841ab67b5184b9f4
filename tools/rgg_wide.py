"""rgg2000 PVC queries with the wide warp tiers at explicit block sizes."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
for wl, th in ((64, 0), (128, 128), (128, 256), (256, 64), (256, 128)):
    for k in (1282, 1281):
        out = []
        for _ in range(8):
            r = vc.solve(g, vc.SolverConfig(mode="pvc", k=k, threads=th, warp_limit=wl))
            out.append(r.search_ms)
        print(f"wl={wl} threads={th} k={k}: search {statistics.median(out):.3f} ms "
              f"blocks={r.blocks}x{r.threads} warp share {r.warp_nodes/max(1,r.stats.tree_nodes_visited):.2f} "
              f"found={r.found}", flush=True)
