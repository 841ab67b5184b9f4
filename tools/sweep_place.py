"""Sweep workspace / CSR placement and block size: rgg2000 PVC(opt-1) kernel ms,
gnp400 / torus60 / ba-like nodes/s under a time budget."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
tag = os.environ.get("TAG", "")
budget = float(os.environ.get("BUDGET", "0.7"))
for name in sys.argv[1:]:
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    opt = vc.solve(g, vc.SolverConfig()).cover_size if name == "rgg2000" else None
    for th in (64, 128, 256, 512):
        if opt is not None:
            best = min((vc.solve(g, vc.SolverConfig(mode="pvc", k=opt - 1, threads=th)) for _ in range(3)),
                       key=lambda r: r.search_ms)
            print(f"{tag} {name} th={th} kern={best.search_ms:.3f} ms nodes={best.stats.tree_nodes_visited}", flush=True)
        else:
            r = vc.solve(g, vc.SolverConfig(threads=th, timeout=budget))
            nodes = r.stats.tree_nodes_visited
            print(f"{tag} {name} th={th} {nodes/r.search_ms*1e3/1e6:.2f} Mnodes/s best={r.cover_size}", flush=True)
