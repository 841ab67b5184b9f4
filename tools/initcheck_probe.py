"""Small solves for compute-sanitizer initcheck (uninitialised device reads)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
from paper_2512_18334_b200.distributed import solve_distributed
from helpers import csr, golden
cases = golden("solve.json")
case = [c for c in cases if c["name"] == "mid_4"][0]
n, off, nbr = csr(case["n"], case["edges"])
g = vc.StaticGraph(n, off, nbr)
print("mid_4 dist", solve_distributed(g, vc.SolverConfig(workers=16), subtrees_per_rank=1).cover_size,
      case["runs"]["det"]["cover_size"], flush=True)
print("mid_4 par", vc.solve(g, vc.SolverConfig(workers=16)).cover_size, flush=True)
n, off, nbr = synth.WORKLOADS["er200"]()
g = vc.StaticGraph(n, off, nbr)
print("er200 par", vc.solve(g, vc.SolverConfig(workers=16)).cover_size, flush=True)
