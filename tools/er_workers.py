"""configs[0] er200 MVC (and G(n, p) around it) at several worker counts."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

cases = [("er200", synth.WORKLOADS["er200"]), ("er250_d5", lambda: synth.er(250, 5.0, 3)),
         ("er120_d6", lambda: synth.er(120, 6.0, 2))]
for name, gen in cases:
    n, off, nbr = gen()
    g = vc.StaticGraph(n, off, nbr)
    for w in (0, 148, 296, 592, 1184):
        cfg = vc.SolverConfig(workers=w)
        vc.solve(g, cfg)
        sms = []
        for _ in range(15):
            r = vc.solve(g, cfg)
            sms.append(r.search_ms)
        print(f"{name} workers={w}: search kernel {statistics.median(sms):.3f} ms "
              f"n_red={r.stats.root_vertices_after} nodes={r.stats.tree_nodes_visited} "
              f"blocks={r.blocks}x{r.threads}", flush=True)
