"""Per-phase block-time breakdown of the search kernel (clock64 counters)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
name = sys.argv[1] if len(sys.argv) > 1 else "rgg2000"
n, off, nbr = synth.WORKLOADS[name]()
g = vc.StaticGraph(n, off, nbr)
opt = vc.solve(g, vc.SolverConfig()).cover_size
for label, kw in [("det-mvc", dict(deterministic=True)), ("pvc-1 w296", dict(mode="pvc", k=opt - 1, workers=296)),
                  ("pvc-1 all", dict(mode="pvc", k=opt - 1))]:
    for th in (64, 128, 256):
        r = vc.solve(g, vc.SolverConfig(threads=th, **kw))
        pc = {k: v for k, v in r.phase_cycles.items() if not k.startswith("fix_")}
        fx = {k: v for k, v in r.phase_cycles.items() if k.startswith("fix_")}
        tot = sum(pc.values())
        nodes = r.stats.tree_nodes_visited
        busy = tot - pc["idle"]
        print(f"{label:11s} th={th:3d} kern={r.search_ms:8.2f} ms nodes={nodes} busy-cyc/node={busy/nodes:8.0f} "
              + " ".join(f"{k}={v/tot*100:4.1f}%" for k, v in pc.items()), flush=True)
        print("   fixpoint: " + " ".join(
            f"{nm}: {fx[f'fix_{nm}_count']/nodes:.2f}/node x {fx[f'fix_{nm}_cycles']/max(fx[f'fix_{nm}_count'],1):.0f} cyc"
            for nm in ("scan", "degree_one", "triangle", "high_degree")), flush=True)
