"""Critical-path probe of the rgg2000 PVC pair: kernel time vs last node / last
warp task, longest warp task, node split between block and warp tiers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
name = sys.argv[1] if len(sys.argv) > 1 else "rgg2000"
n, off, nbr = synth.WORKLOADS[name]()
g = vc.StaticGraph(n, off, nbr)
opt = vc.solve(g, vc.SolverConfig()).cover_size
wl = int(os.environ.get("WL", "-1"))
for k in (opt, opt - 1):
    for rep in range(3):
        r = vc.solve(g, vc.SolverConfig(mode="pvc", k=k, warp_limit=wl))
        pc = r.phase_cycles
        print(f"wl={wl} k={k} kern={r.search_ms:.3f} ms nodes={r.stats.tree_nodes_visited} warp_nodes={r.warp_nodes} "
              f"tasks={r.warp_tasks} last_node={pc['t_node_last_ns']/1e6:.3f} ms task_first={pc['t_task_first_ns']/1e6:.3f} "
              f"task_last={pc['t_task_last_ns']/1e6:.3f} ms max_task={pc['warp_task_max_cycles']/1.9e6:.3f} ms "
              f"max_task_nodes={pc['warp_task_max_nodes']} max_task_n={pc['warp_task_max_n']} "
              f"pushes={r.stats.worklist_pushes} splits={r.stats.component_branches}", flush=True)
        wn = max(r.warp_nodes, 1)
        print(f"   per warp node: task {pc['warp_task_cycles']/wn:.0f} cyc = fixpoint {pc['warp_fix_cycles']/wn:.0f}"
              f" + component test {pc['warp_comp_cycles']/wn:.0f} + splits {pc['warp_split_cycles']/wn:.0f} + rest", flush=True)
