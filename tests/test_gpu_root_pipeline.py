"""Root pipeline parity on the device (preprocess.py:77 root_reduce, graph.py:99
induced_subgraph), for the paths the default sizes do not reach:

* the grid-wide cooperative fixpoint kernel (root_grid.cu), forced on every
  reference fixture with VCG_ROOT_GRID=1 -- same forced ids in the same
  order, same vertex map, rule counts and reduced graph as the reference;
* the frontier-driven kernel of the solve path (root_front.cu), forced with
  VCG_ROOT_GRID=2 -- same forced set, counts, map and reduced graph;
* the device compaction kernels (k_count_kept / k_gather_kept + scans),
  forced with VCG_DEVICE_COMPACT=1, and ``induced_subgraph`` on random keep
  sets against the oracle's restatement of graph.py:99;
* the full-size configurations (BASELINE configs[2], [3]) against
  tests/golden/scale.json (the pinned oracle's root pipeline and MVC)."""

from __future__ import annotations

import hashlib
import random

import numpy as np
import pytest

from helpers import csr, golden, stats_without_time

pytestmark = pytest.mark.gpu


def _sha(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=dtype)).tobytes()).hexdigest()


def _graph(case):
    import paper_2512_18334_b200 as vc

    n, off, nbr = csr(case["n"], case["edges"])
    return vc.StaticGraph(n, off, nbr)


@pytest.fixture
def grid_root(monkeypatch):
    monkeypatch.setenv("VCG_ROOT_GRID", "1")
    monkeypatch.setenv("VCG_DEVICE_COMPACT", "1")


def test_grid_root_reduce_bit_exact(grid_root):
    import paper_2512_18334_b200 as vc

    for case in golden("root_reduce.json"):
        g = _graph(case)
        pre = vc.root_reduce(g, bound=case["bound"])
        assert pre.forced == case["forced"], case.get("name")
        assert pre.vertex_map.tolist() == case["vertex_map"]
        assert pre.rule_counts == case["rule_counts"]
        assert pre.greedy_original == case["greedy_original"]
        assert pre.greedy_reduced == case["greedy_reduced"]
        assert pre.width == case["width"]
        rn = len(case["vertex_map"])
        _, roff, rnbr = csr(rn, case["reduced_edges"])
        assert pre.graph.offsets.tolist() == roff.tolist()
        assert pre.graph.neighbors.tolist() == rnbr.tolist()


def test_grid_root_solve_path_stats(grid_root):
    """The solve path (speculative MVC budget, PVC bounds) through the grid
    kernel and device compaction: deterministic statistics unchanged."""
    import paper_2512_18334_b200 as vc

    for case in golden("solve.json")[::3]:
        g = _graph(case)
        run = case["runs"]["det"]
        r = vc.solve(g, vc.SolverConfig(deterministic=True))
        assert r.cover_size == run["cover_size"], case["name"]
        assert stats_without_time(r.stats.as_dict()) == run["stats"], case["name"]
        for k, exp in case["pvc"].items():
            r = vc.solve(g, vc.SolverConfig(mode="pvc", k=int(k), deterministic=True))
            assert r.found == exp["found"], (case["name"], k)
            assert stats_without_time(r.stats.as_dict()) == exp["stats"], (case["name"], k)


@pytest.fixture
def front_root(monkeypatch):
    monkeypatch.setenv("VCG_ROOT_GRID", "2")
    monkeypatch.setenv("VCG_DEVICE_COMPACT", "1")


def test_front_root_reduce_same_sets(front_root):
    """The frontier kernel (root_front.cu, any-order callers) on every
    reference fixture: the same forced set, rule counts, vertex map and
    reduced graph as the reference (forced ids come back in index order)."""
    import paper_2512_18334_b200 as vc

    for case in golden("root_reduce.json"):
        g = _graph(case)
        pre = vc.root_reduce(g, bound=case["bound"], ordered=False)
        assert pre.kernel["kind"] == "frontier"
        assert pre.forced == sorted(case["forced"]), case.get("name")
        assert pre.vertex_map.tolist() == case["vertex_map"]
        assert pre.rule_counts == case["rule_counts"]
        assert pre.greedy_original == case["greedy_original"]
        assert pre.greedy_reduced == case["greedy_reduced"]
        rn = len(case["vertex_map"])
        _, roff, rnbr = csr(rn, case["reduced_edges"])
        assert pre.graph.offsets.tolist() == roff.tolist()
        assert pre.graph.neighbors.tolist() == rnbr.tolist()


def test_front_solve_path_stats(front_root):
    """Deterministic solves (greedy bound up front) and parallel MVC solves
    (speculative bound certified afterwards) through the frontier kernel."""
    import paper_2512_18334_b200 as vc

    for case in golden("solve.json")[::2]:
        g = _graph(case)
        run = case["runs"]["det"]
        r = vc.solve(g, vc.SolverConfig(deterministic=True))
        assert r.cover_size == run["cover_size"], case["name"]
        assert stats_without_time(r.stats.as_dict()) == run["stats"], case["name"]
        rp = vc.solve(g, vc.SolverConfig())
        assert rp.cover_size == run["cover_size"], case["name"]
        # the certified speculative root reduction is the reference's
        assert rp.stats.root_vertices_after == run["stats"]["root_vertices_after"], case["name"]
        for k, exp in case["pvc"].items():
            r = vc.solve(g, vc.SolverConfig(mode="pvc", k=int(k), deterministic=True))
            assert r.found == exp["found"], (case["name"], k)
            assert stats_without_time(r.stats.as_dict()) == exp["stats"], (case["name"], k)


def test_induced_subgraph_matches_oracle():
    import oracle
    import paper_2512_18334_b200 as vc

    rng = random.Random(7)
    for case in golden("solve.json")[::5]:
        n, off, nbr = csr(case["n"], case["edges"])
        g = vc.StaticGraph(n, off, nbr)
        for frac in (0.0, 0.3, 0.7, 1.0):
            keep = sorted(v for v in range(n) if rng.random() < frac)
            sub, vmap = vc.induced_subgraph(g, keep)
            assert vmap.tolist() == keep
            k = np.asarray(keep, dtype=np.int32)
            new_off = np.zeros(len(k) + 1, dtype=np.int64)
            new_nbr = np.zeros(max(len(nbr), 1), dtype=np.int32)
            L = oracle.lib()
            e = int(L.orc_induced_subgraph(oracle.I64(n), oracle._p(np.asarray(off, np.int64)),
                                           oracle._p(np.asarray(nbr, np.int32)), oracle._p(k),
                                           oracle.I64(len(k)), oracle._p(new_off),
                                           oracle._p(new_nbr)))
            assert sub.num_vertices == len(keep)
            assert sub.offsets.tolist() == new_off.tolist()
            assert sub.neighbors.tolist() == new_nbr[:e].tolist()


@pytest.mark.parametrize("name", ["ba100k", "planted1m"])
def test_scale_root_pipeline_matches_oracle(name):
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth

    exp = golden("scale.json")[name]
    n, off, nbr = synth.WORKLOADS[name]()
    assert (n, int(off[-1]) // 2) == (exp["n"], exp["m"])
    g = vc.StaticGraph(n, off, nbr)
    pre = vc.root_reduce(g)  # n > on-chip size: the grid-wide kernel, device compaction
    assert len(pre.forced) == exp["forced_count"]
    assert _sha(pre.forced, np.int32) == exp["forced_sha256"]
    assert _sha(pre.vertex_map, np.int64) == exp["vertex_map_sha256"]
    assert pre.rule_counts == exp["rule_counts"]
    assert pre.greedy_original == exp["greedy_original"]
    assert pre.greedy_reduced == exp["greedy_reduced"]
    assert _sha(np.concatenate([np.asarray(pre.graph.offsets, np.int64),
                                np.asarray(pre.graph.neighbors, np.int64)]),
                np.int64) == exp["reduced_sha256"]
    r = vc.solve(g, vc.SolverConfig(deterministic=True))
    assert r.cover_size == exp["mvc"]
    assert stats_without_time(r.stats.as_dict()) == {
        **exp["stats"],
        "components_per_branch": {str(k): v for k, v in exp["stats"]["components_per_branch"].items()},
    }
    # solve path (frontier kernel): the same set, in index order
    assert np.array_equal(r.forced_ids, np.sort(np.asarray(pre.forced_ids)))
    assert r.root_kernel["kind"] == "frontier"
    rp = vc.solve(g, vc.SolverConfig())
    assert rp.cover_size == exp["mvc"]
    assert rp.stats.rule_counts == r.stats.rule_counts


def _families():
    """Adversarial shapes for the frontier kernel's degree-one phase, which
    decides targets and tags them in one phase and decrements degrees
    speculatively: isolated candidate edges (every vertex degree 1), stars
    and double stars (many candidates on one target), long paths and
    caterpillars (one peel per sweep), pendant chains hanging off hubs that
    are themselves removed in the same sweep, triangles on paths (the
    triangle sweep after the degree-one cascade), plus random sparse graphs
    with many pendants."""
    rng = random.Random(7)
    out = []
    m = 400
    out.append(("matching", 2 * m, [(2 * i, 2 * i + 1) for i in range(m)]))
    out.append(("stars", 41 * 30, [(41 * s, 41 * s + j) for s in range(30) for j in range(1, 41)]))
    out.append(("double_stars", 62 * 20,
                [e for s in range(20) for e in [(62 * s, 62 * s + 1)] +
                 [(62 * s + (j & 1), 62 * s + 2 + j) for j in range(60)]]))
    out.append(("path", 3001, [(i, i + 1) for i in range(3000)]))
    out.append(("caterpillar", 3000, [(i, i + 1) for i in range(999)] +
                [(i % 1000, 1000 + i) for i in range(2000)]))
    hub_e = []
    for h in range(50):  # hub h (id 100 * h) with 40 pendant chains of length 1-3
        base = 100 * h
        nxt = base + 1
        for _ in range(30):
            ln = rng.randint(1, 3)
            prev = base
            for _ in range(ln):
                if nxt >= base + 100:
                    break
                hub_e.append((prev, nxt))
                prev, nxt = nxt, nxt + 1
        if h:
            hub_e.append((base, base - 100))  # hubs in a chain
    out.append(("hub_chains", 5000, hub_e))
    tri = [(i, i + 1) for i in range(1999)] + [(i, i + 2) for i in range(0, 1998, 3)]
    out.append(("triangles_on_path", 2000, tri))
    for s in range(4):
        n = 6000
        e = {(min(u, v), max(u, v)) for u, v in
             ((rng.randrange(n), rng.randrange(n)) for _ in range(4000 + 3000 * s)) if u != v}
        e |= {(rng.randrange(n // 4), v) for v in range(n // 4, n) if rng.random() < 0.6}
        out.append((f"random_pendants_{s}", n, sorted(e)))
    return out


def test_front_root_reduce_families(front_root):
    """The frontier kernel against the oracle's restatement of
    preprocess.py:77 on the adversarial families above: the same forced set,
    rule counts, vertex map and reduced graph."""
    import oracle
    import paper_2512_18334_b200 as vc

    for name, n, edges in _families():
        nn, off, nbr = csr(n, edges)
        want = oracle.root_reduce(nn, off, nbr)
        pre = vc.root_reduce(vc.StaticGraph(nn, off, nbr), ordered=False)
        assert pre.kernel["kind"] == "frontier", name
        assert pre.forced == sorted(want["forced"]), name
        assert pre.rule_counts == want["rule_counts"], name
        assert pre.vertex_map.tolist() == want["vertex_map"], name
        assert pre.graph.offsets.tolist() == want["offsets"].tolist(), name
        assert pre.graph.neighbors.tolist() == want["neighbors"].tolist(), name


def test_front_root_reduce_1024_thread_variant(front_root, monkeypatch):
    """The 1024-thread frontier kernel (graphs of >= 2^19 vertices; forced
    here with VCG_FRONT_BIGBLOCK) on every reference fixture and the
    adversarial families."""
    import oracle
    import paper_2512_18334_b200 as vc

    monkeypatch.setenv("VCG_FRONT_BIGBLOCK", "1")
    for case in golden("root_reduce.json"):
        g = _graph(case)
        pre = vc.root_reduce(g, bound=case["bound"], ordered=False)
        assert pre.forced == sorted(case["forced"]), case.get("name")
        assert pre.rule_counts == case["rule_counts"]
        assert pre.vertex_map.tolist() == case["vertex_map"]
    for name, n, edges in _families():
        nn, off, nbr = csr(n, edges)
        want = oracle.root_reduce(nn, off, nbr)
        pre = vc.root_reduce(vc.StaticGraph(nn, off, nbr), ordered=False)
        assert pre.forced == sorted(want["forced"]), name
        assert pre.rule_counts == want["rule_counts"], name
        assert pre.vertex_map.tolist() == want["vertex_map"], name
