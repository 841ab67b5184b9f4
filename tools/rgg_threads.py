"""rgg2000 PVC query times vs block size."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
for th in (0, 128, 256, 512):
    for k in (1282, 1281):
        out = []
        for _ in range(12):
            r = vc.solve(g, vc.SolverConfig(mode="pvc", k=k, threads=th))
            out.append(r.search_ms)
        print(f"threads={th} k={k}: search {statistics.median(out):.3f} ms blocks={r.blocks}x{r.threads}",
              flush=True)
