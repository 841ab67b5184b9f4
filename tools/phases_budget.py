"""Phase breakdown of the search kernel on a time-budgeted MVC solve (gnp400, torus60)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
name = sys.argv[1]
budget = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
n, off, nbr = synth.WORKLOADS[name]()
g = vc.StaticGraph(n, off, nbr)
for th in (128, 256, 512):
    r = vc.solve(g, vc.SolverConfig(threads=th, timeout=budget))
    pc = {k: v for k, v in r.phase_cycles.items() if not k.startswith("fix_")}
    tot = sum(pc.values())
    nodes = r.stats.tree_nodes_visited
    print(f"{name} th={th} kern={r.search_ms:.0f} ms nodes={nodes} {nodes/r.search_ms*1e3/1e6:.2f} Mnodes/s best={r.cover_size} "
          f"busy-cyc/node={(tot-pc['idle'])/max(nodes,1):.0f} "
          + " ".join(f"{k}={v/tot*100:4.1f}%" for k, v in pc.items() if not k.startswith(("warp_", "t_"))), flush=True)
    fx = {k: v for k, v in r.phase_cycles.items() if k.startswith("fix_")}
    print("   fixpoint: " + " ".join(
        f"{nm}: {fx[f'fix_{nm}_count']/nodes:.2f}/node x {fx[f'fix_{nm}_cycles']/max(fx[f'fix_{nm}_count'],1):.0f} cyc"
        for nm in ("scan", "degree_one", "triangle", "high_degree")), flush=True)
