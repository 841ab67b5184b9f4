"""solve_batch stress: mixed graphs / modes per batch, answers against goldens."""
import os, sys, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
from helpers import csr, golden
rng = random.Random(1)
cases = golden("solve.json")
items = []
for c in cases:
    n, off, nbr = csr(c["n"], c["edges"])
    items.append((vc.StaticGraph(n, off, nbr), c["runs"]["det"]["cover_size"]))
exp = golden("workloads.json")["rgg2000"]
n, off, nbr = synth.WORKLOADS["rgg2000"]()
items.append((vc.StaticGraph(n, off, nbr), exp["mvc"]))
bad = total = 0
for it in range(int(os.environ.get("ITERS", "150"))):
    k = rng.randint(2, 4)
    pick = [rng.choice(items) for _ in range(k)]
    cfgs = []
    for g, opt in pick:
        m = rng.randint(0, 2)
        kk = opt - (m - 1)
        cfgs.append(vc.SolverConfig() if m == 0 or kk < 0 else vc.SolverConfig(mode="pvc", k=kk))
    rs = vc.solve_batch([g for g, _ in pick], cfgs)
    for (g, opt), c, r in zip(pick, cfgs, rs):
        total += 1
        ok = (r.cover_size == opt) if c.mode == "mvc" else (r.found == (c.k >= opt))
        if not ok:
            bad += 1
            print("WRONG", c, r.cover_size, r.found, opt, flush=True)
print(f"batch stress: wrong {bad} of {total}", flush=True)
