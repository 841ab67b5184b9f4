"""Generate the golden fixtures by running the REFERENCE itself.

Usage (in the build container, where /root/reference exists):

    python tests/golden/make_golden.py            # pure-Python reference
    REF_SRC=/tmp/refbuild/src python tests/golden/make_golden.py

``REF_SRC`` may point at a copy of /root/reference/pkg/src whose optional
Cython kernels were compiled in place (``python setup.py build_ext
--inplace`` on a /tmp copy); the reference's kernel parity tests hold the
compiled and pure backends bit-identical, so the fixtures are the same either
way -- only faster to produce for the 10^5-node workload entries.

The fixtures are small JSON files committed next to this script; nothing at
test time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.environ.get("REF_SRC", "/root/reference/pkg/src"))
sys.path.insert(0, ROOT)

from vcsolver import SolverConfig, brute_force_mvc, build_csr, root_reduce, solve  # noqa: E402
from vcsolver.graph import StaticGraph  # noqa: E402
from vcsolver.kernels import pure  # noqa: E402
from vcsolver.preprocess import greedy_bound  # noqa: E402
from vcsolver.reductions import crown_reduce  # noqa: E402
from vcsolver.graph import SearchNode  # noqa: E402

from paper_2512_18334_b200 import synth  # noqa: E402


def make_graph(n, edges):
    canon = sorted({(min(u, v), max(u, v)) for u, v in edges if u != v})
    return build_csr(canon, n)


def random_graph(rng, n, p):
    return make_graph(n, [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < p])


def edges_of(g):
    return [list(e) for e in g.edge_list()]


def stats_of(r):
    d = r.stats.as_dict()
    d.pop("phase_seconds")
    d.pop("degree_width")
    d["components_per_branch"] = {str(k): v for k, v in d["components_per_branch"].items()}
    return d


# -- kernel-level fixtures (pure.py) ----------------------------------------

def kernel_cases(count=150):
    rng = random.Random(20251)
    out = []
    for _ in range(count):
        n = rng.randint(1, 24)
        g = random_graph(rng, n, rng.choice([0.1, 0.3, 0.6]))
        deg = g.degree_array(32)
        # random partial state: drop a few vertices so dead entries appear
        for _ in range(rng.randint(0, 2)):
            pure.remove_vertex(deg, g.offsets, g.neighbors, rng.randrange(n))
        case = {"n": n, "edges": edges_of(g), "deg": deg.tolist()}
        off, nbr = g.offsets, g.neighbors
        budget = rng.randint(0, n)
        case["budget"] = budget
        res = {}
        for fn in ("degree_one_pass", "degree_two_triangle_pass"):
            d = deg.copy()
            o = np.zeros(2 * n + 2, dtype=np.int32)
            s = np.zeros(n + 1, dtype=np.int32)
            r = getattr(pure, fn)(d, off, nbr, 0, n - 1, o, 0, s)
            res[fn] = {"ret": list(r), "deg": d.tolist(), "out": o[: r[3]].tolist()}
        d = deg.copy()
        o = np.zeros(2 * n + 2, dtype=np.int32)
        s = np.zeros(n + 1, dtype=np.int32)
        r = pure.high_degree_pass(d, off, nbr, 0, n - 1, budget, o, 0, s)
        res["high_degree_pass"] = {"ret": list(r), "deg": d.tolist(), "out": o[: r[3]].tolist()}
        d = deg.copy()
        o = np.zeros(4 * n + 4, dtype=np.int32)
        r = pure.reduce_fixpoint(d, off, nbr, 0, n - 1, budget, o, 0, s)
        res["reduce_fixpoint"] = {"ret": list(r), "deg": d.tolist(), "out": o[: r[7]].tolist()}
        res["select_max_degree"] = pure.select_max_degree(deg, 0, n - 1)
        res["count_live"] = pure.count_live(deg, 0, n - 1)
        res["recompute_bounds"] = list(pure.recompute_bounds(deg, 0, n - 1))
        v = rng.randrange(n)
        case["v"] = v
        d = deg.copy()
        res["remove_vertex"] = {"ret": pure.remove_vertex(d, off, nbr, v), "deg": d.tolist()}
        d = deg.copy()
        o = np.zeros(n + 1, dtype=np.int32)
        r = pure.remove_neighbors(d, off, nbr, v, o, 0)
        res["remove_neighbors"] = {"ret": list(r), "deg": d.tolist(), "out": o[: r[2]].tolist()}
        live = [x for x in range(n) if deg[x] > 0]
        if live:
            src = rng.choice(live)
            case["src"] = src
            vis = np.zeros(n, dtype=np.int32)
            q = np.zeros(n, dtype=np.int32)
            r = pure.bfs_component(deg, off, nbr, vis, 1, q, src)
            res["bfs_component"] = {"ret": list(r), "members": sorted(q[: r[0]].tolist()),
                                    "queue": q[: r[0]].tolist(),
                                    "next": pure.next_live_unvisited(deg, vis, 1, 0, n - 1)}
        d = deg.copy()
        o = np.zeros(n + 1, dtype=np.int32)
        r = pure.greedy_cover(d, off, nbr, 0, n - 1, o, 0)
        res["greedy_cover"] = {"ret": list(r), "out": o[: r[1]].tolist()}
        case["expect"] = res
        out.append(case)
    return out


def crown_cases(count=200):
    rng = random.Random(5151)
    out = []
    for _ in range(count):
        n = rng.randint(4, 16)
        g = random_graph(rng, n, rng.choice([0.1, 0.2, 0.4]))
        node = SearchNode.for_graph(g, 32)
        oc = crown_reduce(node, g)
        out.append({"n": n, "edges": edges_of(g), "forced": oc.forced_vertices,
                    "independent": oc.independent_vertices, "edges_removed": oc.edges_removed})
    return out


def root_cases(count=200):
    rng = random.Random(4242)
    graphs = []
    for _ in range(count):
        n = rng.randint(1, 40)
        graphs.append(random_graph(rng, n, rng.choice([0.05, 0.1, 0.25, 0.5])))
    graphs.append(make_graph(1001, [(0, i) for i in range(1, 1001)]))
    graphs.append(make_graph(8, [(0, 1), (1, 2)] + [(3 + i, 3 + (i + 1) % 5) for i in range(5)]))
    graphs.append(make_graph(6, [(0, 1), (0, 2), (0, 3), (0, 4), (4, 5)]))
    out = []
    for g in graphs:
        for bound in (None, 2):
            pre = root_reduce(g, bound=bound)
            out.append({
                "n": g.num_vertices, "edges": edges_of(g), "bound": bound,
                "forced": pre.forced, "vertex_map": [int(x) for x in pre.vertex_map],
                "reduced_edges": edges_of(pre.graph), "rule_counts": pre.rule_counts,
                "greedy_original": pre.greedy_original, "greedy_reduced": pre.greedy_reduced,
                "width": pre.width,
            })
        out[-1]["greedy_members"] = greedy_bound(g, members=True)[1]
    return out


PETERSEN = [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (5, 7), (7, 9), (9, 6), (6, 8), (8, 5),
            (0, 5), (1, 6), (2, 7), (3, 8), (4, 9)]


def solve_cases():
    rng = random.Random(777)
    graphs = []
    densities = (0.1, 0.25, 0.5, 0.75)
    for i in range(240):
        r = random.Random(100_000 + i)
        graphs.append(("c01_%d" % i, random_graph(r, 1 + i % 18, densities[i % 4])))
    for seed in range(12):
        r = random.Random(9000 + seed)
        h = random_graph(r, 14, 0.5)
        e = h.edge_list()
        graphs.append(("twocopy_%d" % seed, make_graph(28, e + [(a + 14, b + 14) for a, b in e])))
    graphs.append(("petersen", make_graph(10, PETERSEN)))
    graphs.append(("petersen2", make_graph(20, PETERSEN + [(a + 10, b + 10) for a, b in PETERSEN])))
    c5 = [(i, (i + 1) % 5) for i in range(5)]
    graphs.append(("c5x3", make_graph(15, c5 + [(a + 5, b + 5) for a, b in c5]
                                      + [(a + 10, b + 10) for a, b in c5])))
    k4 = [(a, b) for a in range(4) for b in range(a + 1, 4)]
    graphs.append(("k4c5", make_graph(9, k4 + [(a + 4, b + 4) for a, b in c5])))
    for _ in range(30):
        n = rng.randint(20, 40)
        graphs.append(("mid_%d" % _, random_graph(rng, n, rng.choice([0.1, 0.15, 0.2]))))
    configs = {
        "det": dict(deterministic=True),
        "w1": dict(workers=1),
        "det_nocomp": dict(deterministic=True, use_components=False),
        "det_noroot": dict(deterministic=True, use_root_reduce=False),
        "det_nobounds": dict(deterministic=True, use_bounds=False),
        "det_nocrown": dict(deterministic=True, use_crown=False),
        "w1_nolb": dict(workers=1, load_balance=False),
    }
    out = []
    for name, g in graphs:
        case = {"name": name, "n": g.num_vertices, "edges": edges_of(g), "runs": {}}
        if g.num_vertices <= 26:
            case["brute"] = brute_force_mvc(g)[0]
        for cname, kw in configs.items():
            r = solve(g, SolverConfig(**kw))
            case["runs"][cname] = {"cover_size": r.cover_size, "found": r.found,
                                   "exact": r.exact, "stats": stats_of(r)}
        mvc = case["runs"]["det"]["cover_size"]
        pvc = {}
        for k in (mvc - 1, mvc, mvc + 1):
            if k < 0:
                continue
            r = solve(g, SolverConfig(mode="pvc", k=k, deterministic=True))
            pvc[str(k)] = {"found": r.found, "cover_size": r.cover_size, "stats": stats_of(r)}
        case["pvc"] = pvc
        out.append(case)
    return out


def workload_cases():
    out = {}
    for name in ("er200", "rgg2000"):
        n, off, nbr = synth.WORKLOADS[name]()
        g = StaticGraph(n, off, nbr)
        r = solve(g, SolverConfig(deterministic=True))
        mvc = r.cover_size
        entry = {"n": n, "m": int(off[-1] // 2), "mvc": mvc, "stats": stats_of(r), "pvc": {}}
        for k in (mvc - 1, mvc):
            rp = solve(g, SolverConfig(mode="pvc", k=k, deterministic=True))
            entry["pvc"][str(k)] = {"found": rp.found, "cover_size": rp.cover_size,
                                    "stats": stats_of(rp)}
        out[name] = entry
        print(name, mvc, flush=True)
    return out


# -- acceptance families (tests/test_acceptance.py:150-284) ------------------

def registry_dump(reg):
    """Every registry entry's fields (registry.py:24-88), in allocation order."""
    from vcsolver.registry import ParentEntry
    if reg is None:
        return None
    out = []
    for e in reg.entries:
        if isinstance(e, ParentEntry):
            out.append({"kind": "parent", "sum": e.sum, "sum_achieved": e.sum_achieved,
                        "live_comps": e.live_comps, "ancestor": e.ancestor,
                        "initial_sum": e.initial_sum, "folded_total": e.folded_total,
                        "children": list(e.children), "discovery_done": e.discovery_done})
        else:
            out.append({"kind": "child", "best": e.best, "achieved": e.achieved,
                        "live_nodes": e.live_nodes, "parent": e.parent})
    return out


def acceptance_cases():
    sys.path.insert(0, "/root/reference/pkg/tests")
    import test_acceptance as ta
    from helpers import PETERSEN_EDGES, clique_edges, cycle_edges, disjoint_union
    out = {"nested": [], "forests": [], "cliques": [], "cycles": [], "petersen_pair": None}

    def det_run(g):
        r = solve(g, SolverConfig(deterministic=True))
        return {"cover_size": r.cover_size, "stats": stats_of(r),
                "registry": registry_dump(r.registry),
                "nesting_depth": (ta.registry_nesting_depth(r.registry)
                                  if r.registry is not None else 0)}

    rng = random.Random(424)  # test_c06_nested_cascades
    for trial in range(50):
        g = ta.nested_chain(rng)
        size, wit = brute_force_mvc(g)
        out["nested"].append({"name": f"nested_{trial}", "n": g.num_vertices,
                              "edges": edges_of(g), "brute": [size, list(wit)],
                              "det": det_run(g)})
    for i in range(60):  # test_c07 forests
        rng = random.Random(500_000 + i)
        f = ta._random_forest(rng, rng.randint(1, 24))
        pre = root_reduce(f)
        size, wit = brute_force_mvc(f)
        out["forests"].append({"name": f"forest_{i}", "n": f.num_vertices, "edges": edges_of(f),
                               "forced": list(pre.forced), "rule_counts": dict(pre.rule_counts),
                               "brute": [size, list(wit)]})
    for n in range(2, 13):  # test_c08
        g = ta.make_graph(n, clique_edges(n))
        out["cliques"].append({"n": n, "edges": edges_of(g), "det": det_run(g),
                               "mvc": solve(g, SolverConfig()).cover_size})
    for n in range(3, 13):
        g = ta.make_graph(n, cycle_edges(n))
        out["cycles"].append({"n": n, "edges": edges_of(g), "det": det_run(g),
                              "mvc": solve(g, SolverConfig()).cover_size})
    pair = disjoint_union((10, PETERSEN_EDGES), (10, PETERSEN_EDGES))  # test_c05
    r = solve(pair, SolverConfig(deterministic=True, use_root_reduce=False))
    out["petersen_pair"] = {"n": pair.num_vertices, "edges": edges_of(pair),
                            "cover_size": r.cover_size, "stats": stats_of(r),
                            "registry": registry_dump(r.registry)}
    return out


def main():
    fixtures = {
        "kernels.json": kernel_cases,
        "crown.json": crown_cases,
        "root_reduce.json": root_cases,
        "solve.json": solve_cases,
        "workloads.json": workload_cases,
        "acceptance.json": acceptance_cases,
    }
    only = sys.argv[1:]
    for fname, fn in fixtures.items():
        if only and fname not in only:
            continue
        data = fn()
        with open(os.path.join(HERE, fname), "w") as f:
            json.dump(data, f, separators=(",", ":"))
        print("wrote", fname, len(data) if isinstance(data, list) else sorted(data))


if __name__ == "__main__":
    main()
