"""Host-side cost of planted1m solve(): wall vs CUDA events vs root kernel,
and the Python profile of the call (cProfile, 30 solves)."""
import cProfile
import os
import pstats
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

n, off, nbr = synth.WORKLOADS["planted1m"]()
g = vc.StaticGraph(n, off, nbr)
for _ in range(3):
    vc.solve(g)
walls, evs, ks = [], [], []
for _ in range(30):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record()
    r = vc.solve(g)
    e1.record()
    torch.cuda.synchronize()
    walls.append((time.perf_counter() - t) * 1e3)
    evs.append(e0.elapsed_time(e1))
    ks.append(r.root_kernel.get("ms", 0.0))
print(f"wall {statistics.median(walls):.3f} ms, events {statistics.median(evs):.3f} ms, "
      f"root kernel {statistics.median(ks):.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(30):
    vc.solve(g)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
