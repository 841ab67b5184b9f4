"""Strong-scaling instance on one GPU: plain solve vs solve_distributed
(world 1) at several subtree counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402
from paper_2512_18334_b200.distributed import solve_distributed  # noqa: E402

n, p = int(sys.argv[1]) if len(sys.argv) > 1 else 180, float(sys.argv[2]) if len(sys.argv) > 2 else 0.08
n, off, nbr = synth.gnp(n, p, 1)
g = vc.StaticGraph(n, off, nbr)
vc.solve(vc.StaticGraph(*synth.gnp(60, 0.1, 1)))
for label, fn in [("solve", lambda: vc.solve(g, vc.SolverConfig()))] + [
        (f"distributed per={k}", (lambda k=k: solve_distributed(g, vc.SolverConfig(), subtrees_per_rank=k)))
        for k in (8, 32, 128)]:
    t = time.perf_counter()
    r = fn()
    dt = time.perf_counter() - t
    print(f"{label}: mvc={r.cover_size} exact={r.exact} nodes={r.stats.tree_nodes_visited} {dt:.3f} s "
          f"{r.stats.tree_nodes_visited/dt/1e6:.1f} M nodes/s", flush=True)
