"""Slow warp tasks of the rgg2000 PVC(opt-1) query at warp_limit 128 (needs a
-DVCG_TASK_TRACE build: the device prints every task above 400k cycles)."""
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
vc.solve(g, vc.SolverConfig(mode="pvc", k=1281, warp_limit=128))
print("----", flush=True)
r = vc.solve(g, vc.SolverConfig(mode="pvc", k=1281, warp_limit=128))
print(r.search_ms, flush=True)
