"""Pin the C oracle to the reference's own outputs (tests/golden, made by
tests/golden/make_golden.py importing the reference).  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from helpers import csr, golden, stats_without_time


def _state(case):
    n, off, nbr = csr(case["n"], case["edges"])
    deg = np.asarray(case["deg"], dtype=np.uint32)
    return n, off, nbr, deg


def test_kernel_passes_match_reference():
    for case in golden("kernels.json"):
        n, off, nbr, deg = _state(case)
        exp = case["expect"]
        for fn in ("degree_one_pass", "degree_two_triangle_pass"):
            d = deg.copy()
            o = np.zeros(2 * n + 2, dtype=np.int32)
            s = np.zeros(n + 1, dtype=np.int32)
            r = getattr(oracle, fn)(d, off, nbr, 0, n - 1, o, 0, s)
            assert list(r) == exp[fn]["ret"], fn
            assert d.tolist() == exp[fn]["deg"], fn
            assert o[: r[3]].tolist() == exp[fn]["out"], fn
        d = deg.copy()
        o = np.zeros(2 * n + 2, dtype=np.int32)
        s = np.zeros(n + 1, dtype=np.int32)
        r = oracle.high_degree_pass(d, off, nbr, 0, n - 1, case["budget"], o, 0, s)
        assert list(r) == exp["high_degree_pass"]["ret"]
        assert d.tolist() == exp["high_degree_pass"]["deg"]
        d = deg.copy()
        o = np.zeros(4 * n + 4, dtype=np.int32)
        r = oracle.reduce_fixpoint(d, off, nbr, 0, n - 1, case["budget"], o, 0, s)
        assert list(r) == exp["reduce_fixpoint"]["ret"]
        assert d.tolist() == exp["reduce_fixpoint"]["deg"]
        assert o[: r[7]].tolist() == exp["reduce_fixpoint"]["out"]


def test_point_kernels_match_reference():
    for case in golden("kernels.json"):
        n, off, nbr, deg = _state(case)
        exp = case["expect"]
        assert oracle.select_max_degree(deg, 0, n - 1) == exp["select_max_degree"]
        assert oracle.count_live(deg, 0, n - 1) == exp["count_live"]
        assert list(oracle.recompute_bounds(deg, 0, n - 1)) == exp["recompute_bounds"]
        d = deg.copy()
        assert oracle.remove_vertex(d, off, nbr, case["v"]) == exp["remove_vertex"]["ret"]
        assert d.tolist() == exp["remove_vertex"]["deg"]
        d = deg.copy()
        o = np.zeros(n + 1, dtype=np.int32)
        r = oracle.remove_neighbors(d, off, nbr, case["v"], o, 0)
        assert list(r) == exp["remove_neighbors"]["ret"]
        assert o[: r[2]].tolist() == exp["remove_neighbors"]["out"]
        if "src" in case:
            vis = np.zeros(n, dtype=np.int32)
            q = np.zeros(n, dtype=np.int32)
            r = oracle.bfs_component(deg, off, nbr, vis, 1, q, case["src"])
            assert list(r) == exp["bfs_component"]["ret"]
            assert sorted(q[: r[0]].tolist()) == exp["bfs_component"]["members"]
            assert q[: r[0]].tolist() == exp["bfs_component"]["queue"]
            assert oracle.next_live_unvisited(deg, vis, 1, 0, n - 1) == exp["bfs_component"]["next"]
        d = deg.copy()
        o = np.zeros(n + 1, dtype=np.int32)
        r = oracle.greedy_cover(d, off, nbr, 0, n - 1, o, 0)
        assert list(r) == exp["greedy_cover"]["ret"]
        assert o[: r[1]].tolist() == exp["greedy_cover"]["out"]


def test_crown_matches_reference():
    fired = 0
    for case in golden("crown.json"):
        n, off, nbr = csr(case["n"], case["edges"])
        deg = np.diff(off).astype(np.uint32)
        live = np.nonzero(deg)[0]
        lo, hi = (int(live[0]), int(live[-1])) if len(live) else (max(n, 1), 0)
        forced, indep, er = oracle.crown_reduce(deg, off, nbr, lo, hi)
        assert forced == case["forced"]
        assert indep == case["independent"]
        assert er == case["edges_removed"]
        fired += bool(forced)
    assert fired >= 10


def test_root_reduce_matches_reference():
    for case in golden("root_reduce.json"):
        n, off, nbr = csr(case["n"], case["edges"])
        pre = oracle.root_reduce(n, off, nbr, bound=case["bound"])
        assert pre["forced"] == case["forced"]
        assert pre["vertex_map"] == case["vertex_map"]
        assert pre["rule_counts"] == case["rule_counts"]
        assert pre["greedy_original"] == case["greedy_original"]
        rn = len(case["vertex_map"])
        _, roff, rnbr = csr(rn, case["reduced_edges"])
        assert pre["offsets"].tolist() == roff.tolist()
        assert pre["neighbors"].tolist() == rnbr.tolist()
        assert oracle.greedy_bound(rn, roff, rnbr) == case["greedy_reduced"]
        if "greedy_members" in case:
            assert oracle.greedy_bound(n, off, nbr, members=True)[1] == case["greedy_members"]


_CFG = {
    "det": dict(deterministic=True),
    "w1": dict(workers=1),
    "det_nocomp": dict(deterministic=True, use_components=False),
    "det_noroot": dict(deterministic=True, use_root_reduce=False),
    "det_nobounds": dict(deterministic=True, use_bounds=False),
    "det_nocrown": dict(deterministic=True, use_crown=False),
    "w1_nolb": dict(workers=1, load_balance=False),
}


def test_solve_matches_reference_stats_exactly():
    for case in golden("solve.json"):
        n, off, nbr = csr(case["n"], case["edges"])
        for cname, run in case["runs"].items():
            r = oracle.solve(n, off, nbr, **_CFG[cname])
            assert r["cover_size"] == run["cover_size"], (case["name"], cname)
            assert stats_without_time(r["stats"]) == run["stats"], (case["name"], cname)
            assert r["registry_violations"] == 0
            if "brute" in case:
                assert r["cover_size"] == case["brute"]
        for k, exp in case["pvc"].items():
            r = oracle.solve(n, off, nbr, mode="pvc", k=int(k), deterministic=True)
            assert r["found"] == exp["found"], (case["name"], k)
            assert r["cover_size"] == exp["cover_size"]
            assert stats_without_time(r["stats"]) == exp["stats"]


def test_threaded_oracle_answers_are_schedule_independent():
    for case in golden("solve.json")[::7]:
        n, off, nbr = csr(case["n"], case["edges"])
        want = case["runs"]["det"]["cover_size"]
        for w in (2, 4):
            r = oracle.solve(n, off, nbr, workers=w)
            assert r["cover_size"] == want
            assert r["registry_violations"] == 0


@pytest.mark.parametrize("name", ["er200"])
def test_workload_er200_matches_reference(name):
    from paper_2512_18334_b200 import synth

    exp = golden("workloads.json")[name]
    n, off, nbr = synth.WORKLOADS[name]()
    r = oracle.solve(n, off, nbr, deterministic=True)
    assert r["cover_size"] == exp["mvc"]
    assert stats_without_time(r["stats"]) == exp["stats"]
