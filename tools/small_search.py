"""Search-phase time of solves whose root reduction leaves a tiny residual
(ba100k, planted1m with 3x noise, er200) at several worker (block) counts."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

cases = [("ba100k", synth.WORKLOADS["ba100k"]), ("er200", synth.WORKLOADS["er200"]),
         ("planted_noisy", lambda: synth.planted(1_000_000, 50_000, 1, oo=1.0))]
for name, gen in cases:
    n, off, nbr = gen()
    g = vc.StaticGraph(n, off, nbr)
    for w in (0, 1, 8, 148):
        cfg = vc.SolverConfig(workers=w)
        vc.solve(g, cfg)
        tts, sms = [], []
        for _ in range(7):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = vc.solve(g, cfg)
            e1.record()
            torch.cuda.synchronize()
            tts.append(e0.elapsed_time(e1))
            sms.append(r.search_ms)
        print(f"{name} workers={w}: tts {statistics.median(tts):.3f} ms search kernel "
              f"{statistics.median(sms):.3f} ms reduced n={r.stats.root_vertices_after} "
              f"nodes={r.stats.tree_nodes_visited} blocks={r.blocks}x{r.threads}", flush=True)
