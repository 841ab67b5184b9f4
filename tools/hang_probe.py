import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
for label, kw in [("par", {}), ("det", dict(deterministic=True)), ("pvc", dict(mode="pvc", k=1282)), ("pvc-1", dict(mode="pvc", k=1281))]:
    t = time.time()
    print("start", label, flush=True)
    try:
        r = vc.solve(g, vc.SolverConfig(timeout=20, **kw))
        print(label, r.cover_size, r.found, r.exact, r.stats.tree_nodes_visited, f"{time.time()-t:.2f}s", flush=True)
    except Exception as e:
        print(label, "ERROR", e, flush=True)
