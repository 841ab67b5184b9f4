import os, sys, time, threading
sys.path.insert(0, os.getcwd())
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
from dataclasses import replace
n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
opt = vc.solve(g, vc.SolverConfig()).cover_size
cfgs = [vc.SolverConfig(mode="pvc", k=opt, gpu_share=2), vc.SolverConfig(mode="pvc", k=opt - 1, gpu_share=2)]
T0 = time.perf_counter()
def run(c, out, i):
    for rep in range(8):
        t = time.perf_counter()
        r = vc.solve(g, c)
        out.append((i, rep, round((t - T0) * 1e3, 2), round((time.perf_counter() - T0) * 1e3, 2), round(r.search_ms, 3),
                    {k: round(v * 1e3, 3) for k, v in r.stats.phase_seconds.items()}))
out = []
ths = [threading.Thread(target=run, args=(c, out, i)) for i, c in enumerate(cfgs)]
for t in ths: t.start()
for t in ths: t.join()
for o in sorted(out, key=lambda x: x[2]): print(o)
