"""Frontier root kernel (VCG_ROOT_GRID=2; BOUNDED=1 for real budgets) against the oracle's root reduction
on many random shapes: forced set, rule counts, vertex map, reduced CSR.
Prints the mismatches and a total (race hunting for the speculative
decrements and the one-phase degree-one decisions)."""
import os
import random
import sys
import time

os.environ["VCG_ROOT_GRID"] = "2"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2512_18334_b200 as vc  # noqa: E402
from helpers import csr  # noqa: E402

budget = float(os.environ.get("BUDGET_S", "240"))
rng = random.Random(int(os.environ.get("SEED", "11")))
t0 = time.time()
bad = total = 0
while time.time() - t0 < budget:
    n = rng.choice([300, 1000, 3000, 10000, 30000])
    kind = rng.choice(["sparse", "pendants", "hubs", "paths"])
    if kind == "sparse":
        m = int(n * rng.uniform(0.5, 2.5))
        e = {(rng.randrange(n), rng.randrange(n)) for _ in range(m)}
    elif kind == "pendants":
        core = max(4, n // rng.choice([4, 10, 30]))
        e = {(rng.randrange(core), rng.randrange(core)) for _ in range(core * 2)}
        e |= {(rng.randrange(core), v) for v in range(core, n) if rng.random() < 0.8}
    elif kind == "hubs":
        hubs = max(2, n // 200)
        e = {(rng.randrange(hubs), v) for v in range(hubs, n) for _ in range(rng.randint(1, 2))}
        e |= {(rng.randrange(n), rng.randrange(n)) for _ in range(n // 3)}
    else:
        e = {(i, i + 1) for i in range(n - 1) if rng.random() < 0.97}
        e |= {(i, i + 2) for i in range(0, n - 2, rng.randint(2, 7))}
    edges = sorted((min(a, b), max(a, b)) for a, b in e if a != b)
    nn, off, nbr = csr(n, edges)
    # BOUNDED=1: a real budget (the high-degree rule fires: the kernel's
    # block-level pass between its decode / re-encode of the degree words)
    bound = rng.randint(1, max(1, n // 8)) if os.environ.get("BOUNDED") else None
    want = oracle.root_reduce(nn, off, nbr, bound=bound)
    pre = vc.root_reduce(vc.StaticGraph(nn, off, nbr), ordered=False, bound=bound)
    total += 1
    ok = (pre.kernel["kind"] == "frontier" and pre.forced == sorted(want["forced"])
          and pre.rule_counts == want["rule_counts"]
          and pre.vertex_map.tolist() == want["vertex_map"]
          and np.array_equal(pre.graph.offsets, want["offsets"])
          and np.array_equal(pre.graph.neighbors, want["neighbors"]))
    if not ok:
        bad += 1
        print("MISMATCH", kind, n, len(edges), pre.rule_counts, want["rule_counts"], flush=True)
print(f"frontier stress: {bad} mismatches of {total} graphs in {time.time() - t0:.0f} s", flush=True)
