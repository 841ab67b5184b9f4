"""A/B of library builds, interleaved: medians over repeats of the strong
instance G(180, 0.08) MVC and nodes/s of a budgeted gnp400 run.  Each
variant runs in its own subprocess (VCG_LIB)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, time, json
sys.path.insert(0, %r)
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
out = {}
g = vc.StaticGraph(*synth.gnp(180, 0.08, 1))
vc.solve(vc.StaticGraph(*synth.gnp(60, 0.1, 1)))
ts = []
for _ in range(3):
    t = time.perf_counter(); r = vc.solve(g); ts.append(time.perf_counter() - t)
    assert r.cover_size == 136
out["strong_s"] = sorted(ts)[1]
g4 = vc.StaticGraph(*synth.WORKLOADS["gnp400"]())
t = time.perf_counter(); r = vc.solve(g4, vc.SolverConfig(timeout=2.0)); dt = time.perf_counter() - t
out["gnp400_Mnps"] = r.stats.tree_nodes_visited / dt / 1e6
rg = vc.StaticGraph(*synth.WORKLOADS["rgg2000"]())
ms = []
for _ in range(5):
    ms.append(vc.solve(rg, vc.SolverConfig(mode="pvc", k=1281)).search_ms)
out["rgg1281_ms"] = sorted(ms)[2]
print(json.dumps(out))
''' % ROOT
variants = sys.argv[1:] or ["_build_old", "_build"]
res = {v: [] for v in variants}
for rep in range(int(os.environ.get("REPS", "2"))):
    for v in variants:
        env = dict(os.environ, VCG_LIB=os.path.join(ROOT, "paper_2512_18334_b200", v, "libvcgpu.so"))
        o = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = [l for l in o.stdout.splitlines() if l.startswith("{")]
        res[v].append(json.loads(line[-1]) if line else {"error": o.stderr[-300:]})
        print(v, res[v][-1], flush=True)
