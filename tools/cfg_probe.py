"""One time-budgeted MVC solve with a chosen block size (env TH, BUDGET) -- debugging aid."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
name = sys.argv[1]
n, off, nbr = synth.WORKLOADS[name]()
g = vc.StaticGraph(n, off, nbr)
th = int(os.environ.get("TH", "256"))
t = time.time()
r = vc.solve(g, vc.SolverConfig(threads=th, timeout=float(os.environ.get("BUDGET", "0.5")),
                                workers=int(os.environ.get("WORKERS", "0")),
                                warp_limit=int(os.environ.get("WARP", "64")),
                                use_components=os.environ.get("COMP", "1") == "1",
                                width=int(os.environ["WIDTH"]) if "WIDTH" in os.environ else None))
print(name, th, r.stats.tree_nodes_visited, r.cover_size, f"{time.time()-t:.2f}s", flush=True)
