"""Repeated solves through the wide warp tiers (128 / 256-bit tasks, registry
splits of wide tasks) against pinned answers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_18334_b200 as vc  # noqa: E402
from helpers import golden  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

reps = int(os.environ.get("REPS", "20"))
bad = total = 0
exp = golden("workloads.json")["rgg2000"]
n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
for wl in (128, 256):
    for _ in range(reps):
        r = vc.solve(g, vc.SolverConfig(warp_limit=wl))
        total += 1
        bad += r.cover_size != exp["mvc"]
for nn, p, want in ((160, 0.1, 123), (150, 0.1, 113)):
    n, off, nbr = synth.gnp(nn, p, 1)
    g2 = vc.StaticGraph(n, off, nbr)
    for wl in (-1, 128, 256):
        for _ in range(reps):
            r = vc.solve(g2, vc.SolverConfig(warp_limit=wl))
            total += 1
            if r.cover_size != want:
                bad += 1
                print("WRONG", nn, p, wl, r.cover_size, flush=True)
print(f"wide stress: wrong {bad} of {total}", flush=True)
