import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.WORKLOADS["torus60"]()
g = vc.StaticGraph(n, off, nbr)
for th in (64, 128, 256):
    t=time.time()
    r = vc.solve(g, vc.SolverConfig(threads=th, timeout=0.7))
    print(th, r.stats.tree_nodes_visited/r.search_ms*1e3/1e6, "Mn/s", time.time()-t, "s", flush=True)
