import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
for name in sys.argv[1:]:
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    for i in range(5):
        t = time.perf_counter()
        r = vc.solve(g, vc.SolverConfig())
        print(f"{name}: solve {1e3*(time.perf_counter()-t):.1f} ms phases={r.stats.phase_seconds} cover={r.cover_size}", file=sys.stderr, flush=True)
