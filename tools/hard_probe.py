"""Probe config variants with a non-empty residual: planted(oo) and pure BA."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

cases = [("planted oo=%.2f" % oo, (lambda oo=oo: synth.planted(1_000_000, 50_000, 1, oo=oo)))
         for oo in (0.4, 0.5, 0.6, 0.8, 1.0)]
cases += [("planted n=1M cover=100k oo=0.5", lambda: synth.planted(1_000_000, 100_000, 1, oo=0.5)),
          ("ba100k pure", lambda: synth.ba(100_000, 3, 1, pendant=0.0)),
          ("ba100k pendant .05", lambda: synth.ba(100_000, 3, 1, pendant=0.05))]
for name, gen in cases:
    n, off, nbr = gen()
    g = vc.StaticGraph(n, off, nbr)
    t = time.perf_counter()
    pre = vc.root_reduce(g, ordered=False, lazy_greedy=True)
    tr = time.perf_counter() - t
    print(f"{name}: n={n} m={int(off[-1])//2} forced={pre.forced_count} residual n={pre.graph.num_vertices} "
          f"m={pre.graph.num_edges} root {tr*1e3:.1f} ms", flush=True)
    t = time.perf_counter()
    r = vc.solve(g, vc.SolverConfig(timeout=20.0))
    dt = time.perf_counter() - t
    print(f"   solve: mvc={r.cover_size} exact={r.exact} nodes={r.stats.tree_nodes_visited} "
          f"{dt:.3f} s  {r.stats.tree_nodes_visited/max(dt,1e-9)/1e6:.2f} M nodes/s", flush=True)
