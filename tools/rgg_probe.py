"""rgg5000 solves in a fresh process: python tools/rgg_probe.py N R"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

n, r = int(sys.argv[1]), float(sys.argv[2])
n, off, nbr = synth.rgg(n, r, 1)
g = vc.StaticGraph(n, off, nbr)
for i in range(3):
    t = time.perf_counter()
    res = vc.solve(g, vc.SolverConfig(timeout=15.0))
    print(f"rgg{n}_{r} [{os.environ.get('VCG_NO_RECLAIM', 'reclaim')}] run {i}: mvc={res.cover_size} "
          f"exact={res.exact} nodes={res.stats.tree_nodes_visited} residual={res.stats.root_vertices_after} "
          f"entries={len(res.registry)} {time.perf_counter()-t:.3f} s", flush=True)
