"""Fixtures for the per-node reduction API (reductions.py), made by running
the REFERENCE: for seeded random graphs, each single rule (apply_*), the
fixpoint driver and the crown on the root node, with every outcome field and
the node's bookkeeping afterwards.

    python tests/golden/make_reductions_golden.py   # writes reductions.json
"""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("REF_SRC", "/root/reference/pkg/src"))

from vcsolver import build_csr  # noqa: E402
from vcsolver.graph import SearchNode  # noqa: E402
from vcsolver.reductions import (  # noqa: E402
    apply_degree_one,
    apply_degree_two_triangle,
    apply_high_degree,
    crown_reduce,
    reduce_to_fixpoint,
)


def make_graph(n, edges):
    canon = sorted({(min(u, v), max(u, v)) for u, v in edges if u != v})
    return build_csr(canon, n)


def node_state(node):
    return {"degrees": [int(d) for d in node.degrees], "solution_size": node.solution_size,
            "edges_remaining": node.edges_remaining, "lo": node.lo, "hi": node.hi,
            "inclusion": [int(v) for v in np.flatnonzero(node.inclusion)]}


def main():
    rng = random.Random(86421)
    cases = []
    for i in range(240):
        rule = ["degree_one", "degree_two_triangle", "high_degree", "fixpoint", "crown"][i % 5]
        if rule == "crown":  # crowns need sparse graphs with unmatched vertices
            n = rng.randint(4, 24)
            p = rng.choice([0.08, 0.12, 0.2])
        else:
            n = rng.randint(3, 40)
            p = rng.choice([0.05, 0.1, 0.2, 0.35, 0.6])
        g = make_graph(n, [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < p])
        budget = rng.randint(0, max(1, n // 2))
        width = rng.choice([8, 16, 32])
        node = SearchNode.for_graph(g, width, track_inclusion=True)
        case = {"n": n, "edges": [list(e) for e in g.edge_list()], "rule": rule,
                "budget": budget, "width": width, "root": {"lo": node.lo, "hi": node.hi}}
        if rule == "degree_one":
            oc = apply_degree_one(node, g)
        elif rule == "degree_two_triangle":
            oc = apply_degree_two_triangle(node, g)
        elif rule == "high_degree":
            oc = apply_high_degree(node, g, budget)
        elif rule == "crown":
            oc = crown_reduce(node, g)
        if rule == "fixpoint":
            out = np.full(n + 2, -1, dtype=np.int32)
            fo, pos = reduce_to_fixpoint(node, g, budget, out=out, pos=1)
            case["outcome"] = {"forced": fo.forced, "degree_one": fo.degree_one,
                               "degree_two_triangle": fo.degree_two_triangle,
                               "high_degree": fo.high_degree, "edges_removed": fo.edges_removed,
                               "pos": pos, "out": [int(x) for x in out[1:pos]]}
        elif rule == "crown":
            case["outcome"] = {"forced_vertices": oc.forced_vertices,
                               "independent_vertices": oc.independent_vertices,
                               "edges_removed": oc.edges_removed, "applied": oc.applied}
        else:
            case["outcome"] = {"applications": oc.applications, "forced": oc.forced,
                               "edges_removed": oc.edges_removed,
                               "forced_vertices": oc.forced_vertices}
        case["node"] = node_state(node)
        cases.append(case)
    # crowns with pendant fringes: leaves hung on a few hubs of a sparse core
    for i in range(60):
        core = rng.randint(4, 16)
        extra = rng.randint(2, 6)
        n = core + extra
        edges = [(u, v) for u in range(core) for v in range(u + 1, core) if rng.random() < 0.2]
        hubs = [rng.randrange(core) for _ in range(rng.randint(1, 3))]
        edges += [(core + j, rng.choice(hubs)) for j in range(extra)]
        g = make_graph(n, edges)
        width = rng.choice([8, 16, 32])
        node = SearchNode.for_graph(g, width, track_inclusion=True)
        case = {"n": n, "edges": [list(e) for e in g.edge_list()], "rule": "crown",
                "budget": 0, "width": width, "root": {"lo": node.lo, "hi": node.hi}}
        oc = crown_reduce(node, g)
        case["outcome"] = {"forced_vertices": oc.forced_vertices,
                           "independent_vertices": oc.independent_vertices,
                           "edges_removed": oc.edges_removed, "applied": oc.applied}
        case["node"] = node_state(node)
        cases.append(case)
    with open(os.path.join(HERE, "reductions.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))
    print(len(cases), "cases;", sum(bool(c["outcome"].get("applied")) for c in cases), "crowns")


if __name__ == "__main__":
    main()
