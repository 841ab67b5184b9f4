"""End-to-end parity of the GPU solver with the reference (tests/golden/
solve.json, root_reduce.json, workloads.json -- all produced by running
vcsolver itself, see tests/golden/make_golden.py).

* deterministic mode (one block) replays the reference's single-worker
  schedule: answers AND every statistic must be identical;
* parallel mode (every resident block): answers identical, registry
  quiescent and conserved.

The one-block parallel configurations ("w1") replay the reference's
single-worker statistics too, so they run with the warp tier off (the tier
changes the schedule, not the answers: tests/test_gpu_warp_tier.py)."""

from __future__ import annotations

import pytest

from helpers import assert_valid_cover, csr, golden, stats_without_time

pytestmark = pytest.mark.gpu

_CFG = {
    "det": dict(deterministic=True),
    "w1": dict(workers=1, warp_limit=0),
    "det_nocomp": dict(deterministic=True, use_components=False),
    "det_noroot": dict(deterministic=True, use_root_reduce=False),
    "det_nobounds": dict(deterministic=True, use_bounds=False),
    "det_nocrown": dict(deterministic=True, use_crown=False),
    "w1_nolb": dict(workers=1, load_balance=False, warp_limit=0),
}


def _graph(case):
    import paper_2512_18334_b200 as vc

    n, off, nbr = csr(case["n"], case["edges"])
    return vc.StaticGraph(n, off, nbr)


def test_root_reduce_bit_exact():
    import paper_2512_18334_b200 as vc

    for case in golden("root_reduce.json"):
        g = _graph(case)
        pre = vc.root_reduce(g, bound=case["bound"])
        assert pre.forced == case["forced"]
        assert pre.vertex_map.tolist() == case["vertex_map"]
        assert pre.rule_counts == case["rule_counts"]
        assert pre.greedy_original == case["greedy_original"]
        assert pre.greedy_reduced == case["greedy_reduced"]
        assert pre.width == case["width"]
        rn = len(case["vertex_map"])
        _, roff, rnbr = csr(rn, case["reduced_edges"])
        assert pre.graph.offsets.tolist() == roff.tolist()
        assert pre.graph.neighbors.tolist() == rnbr.tolist()
        if "greedy_members" in case:
            assert vc.greedy_bound(g, members=True)[1] == case["greedy_members"]


def test_deterministic_solve_matches_reference_stats():
    import paper_2512_18334_b200 as vc

    for case in golden("solve.json"):
        g = _graph(case)
        for cname, run in case["runs"].items():
            kw = dict(_CFG[cname])
            if "workers" in kw:  # reference workers=1 == one block
                kw["workers"] = 1
            r = vc.solve(g, vc.SolverConfig(check_registry=True, **kw))
            assert r.cover_size == run["cover_size"], (case["name"], cname)
            assert r.found == run["found"]
            assert stats_without_time(r.stats.as_dict()) == run["stats"], (case["name"], cname)
            if r.registry is not None:
                assert r.registry.quiescence_violations() == []
        for k, exp in case["pvc"].items():
            r = vc.solve(g, vc.SolverConfig(mode="pvc", k=int(k), deterministic=True))
            assert r.found == exp["found"], (case["name"], k)
            assert r.cover_size == exp["cover_size"]
            assert stats_without_time(r.stats.as_dict()) == exp["stats"], (case["name"], k)


def test_parallel_solve_answers_match_reference():
    import paper_2512_18334_b200 as vc

    for case in golden("solve.json"):
        g = _graph(case)
        want = case["runs"]["det"]["cover_size"]
        r = vc.solve(g, vc.SolverConfig(check_registry=True))
        assert r.cover_size == want, case["name"]
        assert r.exact
        if r.registry is not None:
            assert r.registry.quiescence_violations() == []
        for k, exp in case["pvc"].items():
            r = vc.solve(g, vc.SolverConfig(mode="pvc", k=int(k)))
            assert r.found == exp["found"], (case["name"], k)
            if exp["found"]:
                assert r.cover_size <= int(k)


@pytest.mark.parametrize("name", ["er200", "rgg2000"])
def test_workloads_match_reference(name):
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth

    exp = golden("workloads.json")[name]
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    r = vc.solve(g, vc.SolverConfig(deterministic=True))
    assert r.cover_size == exp["mvc"]
    assert stats_without_time(r.stats.as_dict()) == exp["stats"]
    r = vc.solve(g, vc.SolverConfig(check_registry=True))
    assert r.cover_size == exp["mvc"]
    assert r.registry.quiescence_violations() == []
    for k, e in exp["pvc"].items():
        r = vc.solve(g, vc.SolverConfig(mode="pvc", k=int(k)))
        assert r.found == e["found"], k


def test_record_cover_is_valid_and_minimum():
    """record_cover with components ON: the witness recorded during the
    search expands to a valid cover of exactly the reported size (the
    reference's witness pass turns components off, which is intractable on
    rgg2000)."""
    import paper_2512_18334_b200 as vc

    for case in golden("solve.json")[::3]:
        n, off, nbr = csr(case["n"], case["edges"])
        g = vc.StaticGraph(n, off, nbr)
        want = case["runs"]["det"]["cover_size"]
        for kw in (dict(), dict(deterministic=True)):
            r = vc.solve(g, vc.SolverConfig(record_cover=True, **kw))
            assert r.cover_size == want, case["name"]
            assert len(r.cover) == want
            assert_valid_cover(n, off, nbr, r.cover)
        r = vc.solve(g, vc.SolverConfig(mode="pvc", k=want, record_cover=True))
        assert r.found and len(r.cover) <= want
        assert_valid_cover(n, off, nbr, r.cover)


@pytest.mark.parametrize("name", ["er200", "rgg2000"])
def test_record_cover_on_workloads(name):
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth

    exp = golden("workloads.json")[name]
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    r = vc.solve(g, vc.SolverConfig(record_cover=True))
    assert r.cover_size == exp["mvc"] == len(r.cover)
    assert_valid_cover(n, off, nbr, r.cover)
    r = vc.solve(g, vc.SolverConfig(mode="pvc", k=exp["mvc"], record_cover=True))
    assert r.found and len(r.cover) <= exp["mvc"]
    assert_valid_cover(n, off, nbr, r.cover)


@pytest.mark.parametrize("threads", [128, 256, 512])
def test_hbm_workspace_split_heavy(monkeypatch, threads):
    """Workspaces in HBM (the launch plan for large reduced graphs, forced
    here with VCG_WS_GLOBAL) on the split-heavy rgg2000 workload with every
    resident block: answers identical, registry quiescent.  Regression test
    for the in-place label compression race (node_ops.cuh compress_labels),
    which lost degrees in component children and livelocked the degree-one
    sweep at >= 128-thread blocks."""
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth

    monkeypatch.setenv("VCG_WS_GLOBAL", "1")
    exp = golden("workloads.json")["rgg2000"]
    n, off, nbr = synth.WORKLOADS["rgg2000"]()
    g = vc.StaticGraph(n, off, nbr)
    for _ in range(3):
        r = vc.solve(g, vc.SolverConfig(threads=threads, check_registry=True))
        assert r.cover_size == exp["mvc"]
        assert r.registry.quiescence_violations() == []
    for k, e in exp["pvc"].items():
        r = vc.solve(g, vc.SolverConfig(mode="pvc", k=int(k), threads=threads))
        assert r.found == e["found"], k


def test_torus_time_budget_consistent():
    """torus60 (configs[4]) under a short time budget on the default launch
    plan (128-thread blocks, HBM workspaces): stops on time with a valid
    bound (the bipartite torus has a perfect matching: MVC = 1800)."""
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth

    n, off, nbr = synth.WORKLOADS["torus60"]()
    g = vc.StaticGraph(n, off, nbr)
    r = vc.solve(g, vc.SolverConfig(timeout=0.5))
    assert r.cover_size >= 1800
    assert not r.exact
    assert r.stats.tree_nodes_visited > 0


def test_deadline_far_in_future_is_exact():
    """A generous time limit arms the device deadline checks (block loop and
    warp-task poll) without ever firing them: answers stay exact.  Regression
    test for a narrowed deadline read in 32-bit warp tasks."""
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth

    for case in golden("solve.json")[::5]:
        g = _graph(case)
        r = vc.solve(g, vc.SolverConfig(timeout=120.0))
        assert r.exact and r.cover_size == case["runs"]["det"]["cover_size"], case["name"]
    exp = golden("workloads.json")["rgg2000"]
    n, off, nbr = synth.WORKLOADS["rgg2000"]()
    r = vc.solve(vc.StaticGraph(n, off, nbr), vc.SolverConfig(timeout=120.0))
    assert r.exact and r.cover_size == exp["mvc"]


def test_solve_batch_matches_sequential():
    """solve_batch (concurrent searches on per-thread streams, each with a
    share of the block slots) gives the sequential answers, repeatedly (the
    worker threads keep their pooled buffers across calls)."""
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth

    exp = golden("workloads.json")["rgg2000"]
    n, off, nbr = synth.WORKLOADS["rgg2000"]()
    g = vc.StaticGraph(n, off, nbr)
    opt = exp["mvc"]
    for _ in range(5):
        rs = vc.solve_batch(g, [vc.SolverConfig(mode="pvc", k=opt),
                                vc.SolverConfig(mode="pvc", k=opt - 1),
                                vc.SolverConfig()])
        assert rs[0].found and not rs[1].found and rs[2].cover_size == opt
    cases = golden("solve.json")[::7]
    graphs = [_graph(c) for c in cases]
    rs = vc.solve_batch(graphs, [vc.SolverConfig() for _ in cases])
    assert [r.cover_size for r in rs] == [c["runs"]["det"]["cover_size"] for c in cases]


def test_registry_reclamation_answers_and_reuse(monkeypatch):
    """Parallel solves recycle dead split groups (registry reclamation, off in
    the parity / audit modes; recycling from the first split here, from half
    the arena by default): answers unchanged, and a split-heavy search runs
    with fewer entries than it made splits."""
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth

    monkeypatch.setenv("VCG_RECLAIM_AT", "0")

    for case in golden("solve.json")[::3]:
        g = _graph(case)
        r = vc.solve(g, vc.SolverConfig())
        assert r.cover_size == case["runs"]["det"]["cover_size"], case["name"]
    exp = golden("workloads.json")["rgg2000"]
    n, off, nbr = synth.WORKLOADS["rgg2000"]()
    g = vc.StaticGraph(n, off, nbr)
    for _ in range(3):
        r = vc.solve(g, vc.SolverConfig())
        assert r.cover_size == exp["mvc"]
        assert len(r.registry) < r.stats.component_branches  # groups were reused
    # split-heavy and long (bounded): no arena / registry exhaustion
    n, off, nbr = synth.gnp(250, 0.06, 1)
    r = vc.solve(vc.StaticGraph(n, off, nbr), vc.SolverConfig(timeout=4.0))
    assert r.stats.component_branches > len(r.registry)
    assert r.cover_size is not None


def test_node_loads_with_and_without_tma(monkeypatch):
    """Node records enter the shared-memory workspace by a TMA bulk copy by
    default; the per-thread load path (VCG_NO_TMA=1) gives the same
    deterministic statistics, and both match the reference's."""
    import paper_2512_18334_b200 as vc

    cases = golden("solve.json")[::5]
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("VCG_NO_TMA", env)
        for case in cases:
            n, off, nbr = csr(case["n"], case["edges"])
            g = vc.StaticGraph(n, off, nbr)
            run = case["runs"]["det"]
            r = vc.solve(g, vc.SolverConfig(deterministic=True))
            assert r.cover_size == run["cover_size"], (case["name"], env)
            assert stats_without_time(r.stats.as_dict()) == run["stats"], (case["name"], env)
            p = vc.solve(g, vc.SolverConfig(check_registry=True))
            assert p.cover_size == run["cover_size"], (case["name"], env)
