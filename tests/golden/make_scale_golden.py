"""Full-size expectations for the large BASELINE configs, from the C oracle
(oracle/vc_oracle.c, itself pinned to the reference by test_oracle_golden):
the root pipeline's forced ids (count + sha256 of the int32 list in the
reference's forcing order), vertex map, reduced graph, rule counts, greedy
bounds, and the MVC with its deterministic-mode statistics.

    python tests/golden/make_scale_golden.py      # writes tests/golden/scale.json

The generators are loaded from synth.py by path (plain numpy), so this
script never loads the CUDA library.
"""
import hashlib
import importlib.util
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

_spec = importlib.util.spec_from_file_location(
    "vc_synth", os.path.join(ROOT, "paper_2512_18334_b200", "synth.py"))
synth = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(synth)


def digest(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=dtype)).tobytes()).hexdigest()


def main(names):
    path = os.path.join(HERE, "scale.json")
    out = {}
    if os.path.exists(path):
        with open(path) as f:
            out = json.load(f)
    for name in names:
        n, off, nbr = synth.WORKLOADS[name]()
        t = time.time()
        pre = oracle.root_reduce(n, off, nbr)
        t_root = time.time() - t
        t = time.time()
        r = oracle.solve(n, off, nbr, deterministic=True)
        t_solve = time.time() - t
        rn = len(pre["vertex_map"])
        out[name] = {
            "n": n, "m": int(off[-1] // 2),
            "graph_sha256": digest(np.concatenate([np.asarray(off, np.int64).view(np.int32),
                                                   np.asarray(nbr, np.int32)]), np.int32),
            "mvc": r["cover_size"], "exact": r["exact"],
            "forced_count": len(pre["forced"]),
            "forced_sha256": digest(pre["forced"], np.int32),
            "vertex_map_sha256": digest(pre["vertex_map"], np.int64),
            "reduced_n": rn, "reduced_m": int(len(pre["neighbors"]) // 2),
            "reduced_sha256": digest(np.concatenate([np.asarray(pre["offsets"], np.int64),
                                                     np.asarray(pre["neighbors"], np.int64)]),
                                     np.int64),
            "rule_counts": pre["rule_counts"],
            "greedy_original": pre["greedy_original"],
            "greedy_reduced": oracle.greedy_bound(rn, pre["offsets"], pre["neighbors"]),
            "stats": {k: v for k, v in r["stats"].items() if k != "phase_seconds"},
            "oracle_seconds": {"root_reduce": round(t_root, 3), "solve": round(t_solve, 3)},
        }
        print(name, {k: v for k, v in out[name].items() if "sha" not in k}, flush=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["ba100k", "planted1m"])
