import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
opt = vc.solve(g, vc.SolverConfig()).cover_size
for th in (0, 128, 512):
    for wl in (64, 32):
        cfgs = [vc.SolverConfig(mode="pvc", k=opt, threads=th, warp_limit=wl), vc.SolverConfig(mode="pvc", k=opt - 1, threads=th, warp_limit=wl)]
        for _ in range(3): vc.solve_batch(g, cfgs)
        ts = []
        for _ in range(15):
            t = time.perf_counter(); rs = vc.solve_batch(g, cfgs); ts.append(time.perf_counter() - t)
        ts.sort()
        print(f"threads={th} warp_limit={wl}: median {ts[7]*1e3:.3f} ms kern {[round(r.search_ms,3) for r in rs]} blocks {[r.blocks for r in rs]}", flush=True)
