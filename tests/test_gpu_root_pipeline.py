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
