"""Per-warp-node cycle split (needs a -DVCG_WARP_PROFILE build, which reports
the fixpoint iterations in place of warp_task_max_nodes): fixpoint,
component test, splits, rest -- on the strong instance and rgg2000."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

for name, gen, cfg in (("gnp180_0.08", lambda: synth.gnp(180, 0.08, 1), vc.SolverConfig()),
                       ("rgg2000 pvc 1281", synth.WORKLOADS["rgg2000"],
                        vc.SolverConfig(mode="pvc", k=1281))):
    n, off, nbr = gen()
    g = vc.StaticGraph(n, off, nbr)
    vc.solve(g, cfg)
    r = vc.solve(g, cfg)
    pc = r.phase_cycles
    wn = max(r.warp_nodes, 1)
    print(f"{name}: warp nodes {r.warp_nodes}, per node: task {pc['warp_task_cycles']/wn:.0f} cyc = "
          f"fixpoint {pc['warp_fix_cycles']/wn:.0f} + components {pc['warp_comp_cycles']/wn:.0f} + "
          f"splits {pc['warp_split_cycles']/wn:.0f} + rest; fixpoint iterations/node "
          f"{pc['warp_task_max_nodes'] / wn:.2f}; rules {r.stats.rule_counts}", flush=True)
