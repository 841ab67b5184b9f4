"""Block-tier node cost on rgg2000 PVC(opt-1): thread-0 cycles per block-level
node by phase (warp-tier nodes excluded)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
opt = vc.solve(g, vc.SolverConfig()).cover_size
for _ in range(2):
    r = vc.solve(g, vc.SolverConfig(mode="pvc", k=opt - 1, warp_limit=int(os.environ.get("WARP", "64"))))
    pc = r.phase_cycles
    bn = r.stats.tree_nodes_visited - r.warp_nodes
    names = ["load", "reduce", "label", "split", "select", "exclude", "include", "registry", "other"]
    tot = sum(pc[k] for k in names)
    print(f"block nodes {bn}, kernel {r.search_ms:.3f} ms, cycles/block-node {tot/bn:.0f}: " +
          " ".join(f"{k}={pc[k]/bn:.0f}" for k in names), flush=True)
    fx = {k: v for k, v in pc.items() if k.startswith("fix_")}
    print("   fixpoint per block node: " + " ".join(
        f"{nm}: {fx[f'fix_{nm}_count']/bn:.2f} x {fx[f'fix_{nm}_cycles']/max(fx[f'fix_{nm}_count'],1):.0f}"
        for nm in ("scan", "degree_one", "triangle", "high_degree")), flush=True)
