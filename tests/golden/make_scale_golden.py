"""Full-size expectations for the large BASELINE configs, from the C oracle
(oracle/vc_oracle.c, itself pinned to the reference by test_oracle_golden):
MVC size, forced count and reduced size of the root pipeline.

    python tests/golden/make_scale_golden.py      # writes tests/golden/scale.json
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

out = {}
for name in ("ba100k", "planted1m"):
    n, off, nbr = synth.WORKLOADS[name]()
    t = time.time()
    pre = oracle.root_reduce(n, off, nbr)
    t_root = time.time() - t
    t = time.time()
    r = oracle.solve(n, off, nbr, deterministic=True)
    out[name] = {"n": n, "m": int(off[-1] // 2), "mvc": r["cover_size"], "exact": r["exact"],
                 "forced": len(pre["forced"]), "reduced_n": len(pre["vertex_map"]),
                 "reduced_m": int(len(pre["neighbors"]) // 2),
                 "rule_counts": pre["rule_counts"], "greedy_original": pre["greedy_original"],
                 "stats": {k: v for k, v in r["stats"].items() if k != "phase_seconds"},
                 "oracle_seconds": {"root_reduce": t_root, "solve": time.time() - t}}
    print(name, out[name], flush=True)
with open(os.path.join(HERE, "scale.json"), "w") as f:
    json.dump(out, f, indent=1)
