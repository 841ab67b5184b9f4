"""Probe the large BASELINE configs: root pipeline size/time, time-bounded search."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
for name in sys.argv[1:]:
    t = time.perf_counter()
    n, off, nbr = synth.WORKLOADS[name]()
    tg = time.perf_counter() - t
    g = vc.StaticGraph(n, off, nbr)
    t = time.perf_counter()
    pre = vc.root_reduce(g)
    tr = time.perf_counter() - t
    rg = pre.graph
    import numpy as np
    md = int(np.diff(rg.offsets).max()) if rg.num_vertices else 0
    print(f"{name}: n={n} m={len(nbr)//2} gen={tg:.1f}s root_reduce={tr:.2f}s {pre.seconds} forced={pre.forced_count} "
          f"reduced n={rg.num_vertices} m={rg.num_edges} maxdeg={md} width={pre.width} greedy_orig={pre.greedy_original} greedy_red={pre.greedy_reduced}", flush=True)
    t = time.perf_counter()
    r = vc.solve(g, vc.SolverConfig(timeout=30))
    print(f"   solve: cover={r.cover_size} exact={r.exact} nodes={r.stats.tree_nodes_visited} splits={r.stats.component_branches} "
          f"kern={r.search_ms:.1f}ms wall={time.perf_counter()-t:.1f}s", flush=True)
