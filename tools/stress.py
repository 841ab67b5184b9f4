"""Repeated parallel solves against known answers: counts wrong results (flaky-race hunting)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
from helpers import csr, golden
reps = int(os.environ.get("REPS", "30"))
bad = 0; total = 0
exp = golden("workloads.json")
for name in ("rgg2000", "er200"):
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    for i in range(reps):
        r = vc.solve(g, vc.SolverConfig())
        total += 1
        if r.cover_size != exp[name]["mvc"]:
            bad += 1
            print("WRONG", name, i, r.cover_size, exp[name]["mvc"], flush=True)
cases = golden("solve.json")
for i in range(reps // 3):
    for case in cases:
        n, off, nbr = csr(case["n"], case["edges"])
        g = vc.StaticGraph(n, off, nbr)
        r = vc.solve(g, vc.SolverConfig())
        total += 1
        if r.cover_size != case["runs"]["det"]["cover_size"]:
            bad += 1
            print("WRONG", case["name"], r.cover_size, case["runs"]["det"]["cover_size"], flush=True)
print(f"{os.environ.get('TAG','')} wrong {bad} of {total}", flush=True)
