"""Host-side overhead of one rgg2000 PVC solve: wall vs device kernel time, cProfile top."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
opt = vc.solve(g, vc.SolverConfig()).cover_size
cfgs = [vc.SolverConfig(mode="pvc", k=opt), vc.SolverConfig(mode="pvc", k=opt - 1)]
for _ in range(3):
    for c in cfgs:
        vc.solve(g, c)
walls, kms = [], []
for _ in range(20):
    for c in cfgs:
        t = time.perf_counter()
        r = vc.solve(g, c)
        walls.append(time.perf_counter() - t)
        kms.append(r.search_ms)
print(f"pair wall {sum(walls)/10*1e3:.3f} ms, search kernels {sum(kms)/10:.3f} ms, phases {r.stats.phase_seconds}")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    for c in cfgs:
        vc.solve(g, c)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
