"""Root pipeline + solve timing on the large configs (ba100k, planted1m):
device-resident input (value path) and from host buffers (e2e path).
VCG_TRACE=1 prints the library's host-side phase timings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

for name in sys.argv[1:] or ["ba100k", "planted1m"]:
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    g.device()
    for i in range(5):
        t = time.perf_counter()
        r = vc.solve(g, vc.SolverConfig())
        t1 = time.perf_counter()
        gh = vc.StaticGraph(n, np.array(off), np.array(nbr))
        r2 = vc.solve(gh, vc.SolverConfig())
        t2 = time.perf_counter()
        print(f"{name} mvc={r.cover_size} resident {1e3*(t1-t):.3f} ms  host {1e3*(t2-t1):.3f} ms "
              f"phases={ {k: round(v*1e3, 3) for k, v in r.stats.phase_seconds.items()} } "
              f"nodes={r.stats.tree_nodes_visited}", flush=True)
    pl = vc.root_reduce(g, ordered=False, lazy_greedy=True)
    print(f"{name} lazy root_reduce: forced={pl.forced_count} n'={pl.graph.num_vertices} "
          f"spec_need={pl.spec_need} kernel={pl.kernel}", flush=True)
    t = time.perf_counter()
    pre = vc.root_reduce(g)
    print(f"{name} ordered root_reduce {1e3*(time.perf_counter()-t):.3f} ms seconds={pre.seconds}",
          flush=True)
