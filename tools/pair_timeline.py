"""Device timeline of the rgg2000 PVC pair run as one solve_batch (k = opt and
opt - 1 on two host threads / streams): each search kernel's %globaltimer
start and drain end, and their overlap -- the evidence that the two
latency-bound searches run concurrently on the GPU (nsys is not in the
image; the kernels timestamp themselves).  Prints JSON."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
opt = 1282
cfgs = [vc.SolverConfig(mode="pvc", k=opt), vc.SolverConfig(mode="pvc", k=opt - 1)]
for _ in range(3):
    vc.solve_batch(g, cfgs)
runs = []
for _ in range(20):
    a, b = vc.solve_batch(g, cfgs)
    (a0, a1), (b0, b1) = a.kernel_interval_ns, b.kernel_interval_ns
    lo, hi = max(a0, b0), min(a1, b1)
    span = max(a1, b1) - min(a0, b0)
    runs.append({"k_opt": [0, a1 - a0], "k_opt_minus_1": [b0 - a0, b1 - a0],
                 "overlap_ns": max(0, hi - lo), "union_ns": span,
                 "sum_ns": (a1 - a0) + (b1 - b0), "blocks": [a.blocks, b.blocks]})
med = lambda k: statistics.median(r[k] for r in runs)  # noqa: E731
print(json.dumps({
    "what": "rgg2000 PVC pair (k=1282 yes, k=1281 no) as one solve_batch; per run, the two "
            "search kernels' device intervals (ns, relative to the k=1282 kernel's start)",
    "median_overlap_ns": med("overlap_ns"), "median_union_ns": med("union_ns"),
    "median_sum_ns": med("sum_ns"),
    "median_overlap_fraction_of_shorter": statistics.median(
        r["overlap_ns"] / max(1, min(r["k_opt"][1], r["k_opt_minus_1"][1] - r["k_opt_minus_1"][0]))
        for r in runs),
    "runs": runs[:5]}, indent=1))
