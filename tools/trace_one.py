import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
for k in (1282, 1281, 1282, 1281, 1282, 1281):
    t = time.perf_counter()
    r = vc.solve(g, vc.SolverConfig(mode="pvc", k=k, threads=int(os.environ.get("TH", "0"))))
    print(f"k={k} wall={(time.perf_counter()-t)*1e3:.2f} ms kern={r.search_ms:.2f} phases={ {a: round(b*1e3, 2) for a, b in r.stats.phase_seconds.items()} }", file=sys.stderr, flush=True)
