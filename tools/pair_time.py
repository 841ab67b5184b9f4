"""rgg2000 PVC k=opt / opt-1 single-query and solve_batch pair times (CUDA events)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
opt = 1282


def timed(fn, reps=15):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


for k in (opt, opt - 1):
    timed(lambda: vc.solve(g, vc.SolverConfig(mode="pvc", k=k)), 3)
    sm = []
    t = timed(lambda: sm.append(vc.solve(g, vc.SolverConfig(mode='pvc', k=k))))
    print(f"[{os.environ.get('VCG_NO_RECLAIM', 'reclaim')}] k={k}: {t:.3f} ms  search kernel "
          f"{statistics.median(r.search_ms for r in sm):.3f} ms  root "
          f"{statistics.median(r.stats.phase_seconds['root_reduce'] for r in sm)*1e3:.3f} ms "
          f"nodes {statistics.median(r.stats.tree_nodes_visited for r in sm)}", flush=True)
cfgs = [vc.SolverConfig(mode="pvc", k=opt), vc.SolverConfig(mode="pvc", k=opt - 1)]
timed(lambda: vc.solve_batch(g, cfgs), 3)
print(f"[{os.environ.get('VCG_NO_RECLAIM', 'reclaim')}] pair: {timed(lambda: vc.solve_batch(g, cfgs)):.3f} ms")
