"""GPU probe of the warp tier: PVC pair / MVC on the workloads at several
warp_limit values (kernel ms, nodes, warp tasks)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

names = sys.argv[1:] or ["er200", "rgg2000"]
for name in names:
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    opt = vc.solve(g, vc.SolverConfig(warp_limit=0)).cover_size
    for lim in (0, 64, 32):
        for label, kw in (("mvc", {}), ("pvc=opt", dict(mode="pvc", k=opt)),
                          ("pvc=opt-1", dict(mode="pvc", k=opt - 1))):
            best = None
            for _ in range(3):
                t = time.perf_counter()
                r = vc.solve(g, vc.SolverConfig(warp_limit=lim, **kw))
                dt = time.perf_counter() - t
                if best is None or r.search_ms < best[0].search_ms:
                    best = (r, dt)
            r, dt = best
            ph = r.phase_cycles
            print(f"{name} lim={lim} {label}: cover={r.cover_size} found={r.found} "
                  f"kernel={r.search_ms:.3f}ms wall={dt*1e3:.1f}ms nodes={r.stats.tree_nodes_visited} "
                  f"warp_tasks={r.warp_tasks} warp_nodes={r.warp_nodes} "
                  f"warp_cyc/node={ph['warp_task_cycles']/max(r.warp_nodes,1):.0f} "
                  f"pushes={r.stats.worklist_pushes}", flush=True)
            tot = sum(v for k, v in ph.items() if k in vc.engine._lib.PHASES) or 1
            print("    A-phases: " + " ".join(f"{k}={v/tot*100:.1f}%" for k, v in ph.items()
                                             if k in vc.engine._lib.PHASES and v),
                  f"wepoch/A-total={ph['warp_epoch_cycles']/tot:.2f} max_task_us={ph['warp_task_max_cycles']/1.9e3:.1f}",
                  f"(nodes={ph['warp_task_max_nodes']} n={ph['warp_task_max_n']}) "
                  f"t_node_last={ph['t_node_last_ns']/1e3:.0f}us t_task_first={ph['t_task_first_ns']/1e3:.0f}us "
                  f"t_task_last={ph['t_task_last_ns']/1e3:.0f}us", flush=True)
