"""Ad-hoc GPU probe: time the solver on the synthetic workloads."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth

names = sys.argv[1:] or ["er200", "rgg2000"]
for name in names:
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    for label, cfg in [("det", dict(deterministic=True)), ("par", dict()),
                       ("par", dict()), ("pvc_opt", dict(mode="pvc", k=None)),
                       ("pvc_opt-1", dict(mode="pvc", k=None))]:
        if cfg.get("mode") == "pvc":
            cfg["k"] = mvc if label == "pvc_opt" else mvc - 1
        t = time.perf_counter()
        r = vc.solve(g, vc.SolverConfig(check_registry=True, **cfg))
        dt = time.perf_counter() - t
        if label == "det":
            mvc = r.cover_size
        s = r.stats
        print(f"{name} {label}: cover={r.cover_size} found={r.found} exact={r.exact} "
              f"wall={dt*1e3:.1f}ms search_kernel={r.search_ms:.2f}ms nodes={s.tree_nodes_visited} "
              f"nodes/s={s.tree_nodes_visited/max(r.search_ms,1e-9)*1e3:.3e} splits={s.component_branches} "
              f"pushes={s.worklist_pushes} pops={s.worklist_pops} reg_viol={r.registry.quiescence_violations() if r.registry else None} "
              f"phases={ {k: round(v*1e3,2) for k,v in s.phase_seconds.items()} }", flush=True)
