"""Default-launch-plan rates: rgg2000 PVC(opt-1) kernel ms, gnp400 / torus60 nodes/s."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
budget = float(os.environ.get("BUDGET", "1.0"))
for name in sys.argv[1:] or ["rgg2000", "gnp400", "torus60"]:
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    if name == "rgg2000":
        opt = vc.solve(g, vc.SolverConfig()).cover_size
        r = min((vc.solve(g, vc.SolverConfig(mode="pvc", k=opt - 1)) for _ in range(5)),
                key=lambda r: r.search_ms)
        print(f"{name} blocks={r.blocks} threads={r.threads} kern={r.search_ms:.3f} ms "
              f"nodes={r.stats.tree_nodes_visited}", flush=True)
    else:
        r = vc.solve(g, vc.SolverConfig(timeout=budget))
        print(f"{name} blocks={r.blocks} threads={r.threads} "
              f"{r.stats.tree_nodes_visited / r.search_ms * 1e3 / 1e6:.2f} Mnodes/s best={r.cover_size}",
              flush=True)
