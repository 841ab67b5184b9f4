"""Node-rate sweep of block size / CSR placement on a time-budgeted MVC solve."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
budget = float(os.environ.get("BUDGET", "1.0"))
for name in sys.argv[1:]:
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    for th in (32, 64, 128, 256):
        r = vc.solve(g, vc.SolverConfig(threads=th, timeout=budget))
        nodes = r.stats.tree_nodes_visited
        print(f"{name} smemcsr={'0' if os.environ.get('VCG_NO_SMEM_CSR') else '1'} th={th} "
              f"{nodes/r.search_ms*1e3/1e6:.2f} Mnodes/s best={r.cover_size}", flush=True)
