"""Pin the strong-scaling instance (bench.py STRONG: G(n=180, p=0.08), seed 1)
with the C oracle's threaded engine (oracle/, itself pinned to the reference
by tests/test_oracle_golden.py).  ~6 min on 8 host threads; writes
tests/golden/strong.json.  Test infrastructure: run in the build container."""

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

out = {}
for n, p, seed in ((180, 0.08, 1),):
    nn, off, nbr = synth.gnp(n, p, seed)
    t = time.time()
    r = oracle.solve(nn, off, nbr, workers=os.cpu_count() or 1)
    out[f"gnp{n}_{p}_{seed}"] = {"n": nn, "m": int(off[-1]) // 2, "mvc": r["cover_size"],
                                 "exact": r["exact"], "oracle_nodes": r["stats"]["tree_nodes_visited"],
                                 "oracle_seconds": round(time.time() - t, 1),
                                 "oracle_threads": os.cpu_count()}
    print(out, flush=True)
with open(os.path.join(HERE, "strong.json"), "w") as f:
    json.dump(out, f, indent=1)
