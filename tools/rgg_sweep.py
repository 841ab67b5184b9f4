"""rgg2000 PVC(opt-1 / opt) search time across the warp-tier knobs:
warp_limit, the export trigger (VCG_WEXPORT: nodes before a task may shed)
and the poll period (VCG_WCHECK mask)."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

n, off, nbr = synth.WORKLOADS["rgg2000"]()
g = vc.StaticGraph(n, off, nbr)
wls = [int(x) for x in os.environ.get("WLS", "64,128,256").split(",")]
exps = os.environ.get("EXPS", "4,1").split(",")
chks = os.environ.get("CHKS", "3,1").split(",")
thr = [int(x) for x in os.environ.get("THR", "0").split(",")]
for wl, ex, ck, th in itertools.product(wls, exps, chks, thr):
    os.environ["VCG_WEXPORT"] = ex
    os.environ["VCG_WCHECK"] = ck
    out = []
    for k in (1281, 1282):
        ms = []
        for _ in range(5):
            r = vc.solve(g, vc.SolverConfig(mode="pvc", k=k, warp_limit=wl, threads=th))
            ms.append(r.search_ms)
        ms.sort()
        out.append(f"k={k} {ms[2]:.3f} ms (nodes {r.stats.tree_nodes_visited}, warp {r.warp_nodes}, "
                   f"{r.blocks}x{r.threads})")
    print(f"wl={wl} export={ex} check={ck} threads={th}: " + " | ".join(out), flush=True)
