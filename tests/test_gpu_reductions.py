"""The per-node reduction API (reductions.py mirror) on the device: the
reference's own reduction tests (tests/test_reductions.py), restated against
this package, plus every outcome field and the node's bookkeeping on 300
reference-generated cases (tests/golden/reductions.json).  Exact optima for
the safety checks come from the oracle."""

from __future__ import annotations

import random

import numpy as np
import pytest

import oracle
from helpers import golden

pytestmark = pytest.mark.gpu


def make_graph(n, edges):
    from paper_2512_18334_b200 import build_csr

    canon = sorted({(min(u, v), max(u, v)) for u, v in edges if u != v})
    return build_csr(canon, n)


def path_edges(n):
    return [(i, i + 1) for i in range(n - 1)]


def cycle_edges(n):
    return [(i, (i + 1) % n) for i in range(n)]


def clique_edges(n):
    return [(u, v) for u in range(n) for v in range(u + 1, n)]


def random_graph(rng, n, p):
    return make_graph(n, [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < p])


def exact(g):
    if g.num_edges == 0:
        return 0
    return oracle.solve(g.num_vertices, g.offsets, g.neighbors)["cover_size"]


def _node(g, track_inclusion=False, width=8):
    from paper_2512_18334_b200.graph import SearchNode

    return SearchNode.for_graph(g, width, track_inclusion=track_inclusion)


def _residual(g, node):
    deg = node.degrees
    return make_graph(g.num_vertices, [(u, v) for u, v in g.edge_list() if deg[u] and deg[v]])


def test_degree_one_on_path():
    from paper_2512_18334_b200.reductions import apply_degree_one

    g = make_graph(4, path_edges(4))
    node = _node(g, track_inclusion=True)
    oc = apply_degree_one(node, g)
    assert (oc.applications, oc.forced, oc.forced_vertices, oc.edges_removed) == (2, 2, [1, 2], 3)
    assert node.solution_size == 2 and node.edges_remaining == 0
    assert node.inclusion.tolist() == [False, True, True, False]
    assert node.lo > node.hi


def test_degree_two_triangle_rule():
    from paper_2512_18334_b200.reductions import apply_degree_two_triangle

    g = make_graph(3, cycle_edges(3))
    node = _node(g)
    oc = apply_degree_two_triangle(node, g)
    assert oc.applications == 1 and oc.forced_vertices == [1, 2]
    assert node.solution_size == 2 and node.edges_remaining == 0


def test_high_degree_budget_spans_passes():
    from paper_2512_18334_b200.reductions import apply_high_degree

    g = make_graph(9, [(0, 1), (0, 2), (0, 3), (0, 4), (5, 6), (5, 7), (5, 8)])
    node = _node(g)
    oc = apply_high_degree(node, g, 3)
    assert oc.applications == 2 and oc.forced_vertices == [0, 5]
    assert node.solution_size == 2 and node.edges_remaining == 0


def test_fixpoint_three_hub_tree_and_branch():
    from paper_2512_18334_b200.graph import remove_vertex
    from paper_2512_18334_b200.reductions import reduce_to_fixpoint

    edges = [(0, 1), (1, 2), (1, 4), (3, 4), (4, 5), (4, 7), (6, 7), (7, 8)]
    g = make_graph(9, edges)
    node = _node(g, track_inclusion=True)
    out = np.empty(9, dtype=np.int32)
    oc, pos = reduce_to_fixpoint(node, g, budget=100, out=out, pos=0)
    assert (oc.forced, oc.degree_one, oc.degree_two_triangle, oc.high_degree,
            oc.edges_removed) == (3, 3, 0, 0, 8)
    assert out[:pos].tolist() == [1, 4, 7]
    assert [int(v) for v in np.flatnonzero(node.inclusion)] == [1, 4, 7]
    node = _node(g)
    remove_vertex(node, g, 4, into_cover=True)
    oc, pos = reduce_to_fixpoint(node, g, budget=100, out=out, pos=0)
    assert oc.forced == 2 and sorted(out[:pos].tolist()) == [1, 7]
    assert node.solution_size == 3 and node.edges_remaining == 0


def test_fixpoint_threads_out_cursor_and_low_budget():
    from paper_2512_18334_b200.reductions import reduce_to_fixpoint

    g = make_graph(4, path_edges(4))
    node = _node(g)
    out = np.full(8, -1, dtype=np.int32)
    out[0] = 9
    _, pos = reduce_to_fixpoint(node, g, budget=100, out=out, pos=1)
    assert pos == 3 and out[:3].tolist() == [9, 1, 2]
    g = make_graph(4, clique_edges(4))
    node = _node(g)
    oc, _ = reduce_to_fixpoint(node, g, budget=1)
    assert oc.high_degree == 3 and node.solution_size == 3 and node.edges_remaining == 0


def test_rule_safety_random():
    from paper_2512_18334_b200.reductions import (apply_degree_one, apply_degree_two_triangle,
                                                  apply_high_degree, reduce_to_fixpoint)

    rng = random.Random(86420)
    for _ in range(120):
        n = rng.randint(3, 13)
        g = random_graph(rng, n, rng.choice([0.15, 0.3, 0.5, 0.8]))
        opt = exact(g)
        rule = rng.randrange(4)
        node = _node(g)
        if rule == 0:
            apply_degree_one(node, g)
        elif rule == 1:
            apply_degree_two_triangle(node, g)
        elif rule == 2:
            apply_high_degree(node, g, opt)
        else:
            reduce_to_fixpoint(node, g, budget=opt)
        assert node.solution_size + exact(_residual(g, node)) == opt


def test_special_component_values_match_oracle():
    from paper_2512_18334_b200.reductions import ComponentKind, solve_special_component

    for n in range(2, 9):
        assert solve_special_component(ComponentKind.CLIQUE, n) == exact(
            make_graph(n, clique_edges(n)))
    for n in range(4, 11):
        assert solve_special_component(ComponentKind.CHORDLESS_CYCLE, n) == exact(
            make_graph(n, cycle_edges(n)))


def test_crown_cases():
    from paper_2512_18334_b200.reductions import crown_reduce

    g = make_graph(6, [(0, 1), (0, 2), (0, 3), (0, 4), (4, 5)])
    node = _node(g)
    oc = crown_reduce(node, g)
    assert oc.applied and oc.forced_vertices == [0] and oc.independent_vertices == [2, 3]
    assert oc.edges_removed == 4 and node.solution_size == 1 and node.edges_remaining == 1
    g = make_graph(4, cycle_edges(4))
    node = _node(g)
    assert not crown_reduce(node, g).applied and node.edges_remaining == 4
    g = make_graph(3, [])
    assert not crown_reduce(_node(g), g).applied


def test_crown_iterates_with_rules():
    from paper_2512_18334_b200.reductions import crown_reduce, reduce_to_fixpoint

    rng = random.Random(11)
    for _ in range(20):
        g = random_graph(rng, 14, 0.25)
        opt = exact(g)
        node = _node(g)
        while True:
            before = node.solution_size
            reduce_to_fixpoint(node, g, budget=opt - node.solution_size)
            crown_reduce(node, g)
            if node.solution_size == before:
                break
        assert node.solution_size + exact(_residual(g, node)) == opt


def test_reductions_match_reference_golden():
    from paper_2512_18334_b200.graph import SearchNode
    from paper_2512_18334_b200.reductions import (apply_degree_one, apply_degree_two_triangle,
                                                  apply_high_degree, crown_reduce,
                                                  reduce_to_fixpoint)

    for case in golden("reductions.json"):
        g = make_graph(case["n"], case["edges"])
        node = SearchNode.for_graph(g, case["width"], track_inclusion=True)
        assert (node.lo, node.hi) == (case["root"]["lo"], case["root"]["hi"])
        rule, oc = case["rule"], case["outcome"]
        if rule == "fixpoint":
            out = np.full(case["n"] + 2, -1, dtype=np.int32)
            fo, pos = reduce_to_fixpoint(node, g, case["budget"], out=out, pos=1)
            got = {"forced": fo.forced, "degree_one": fo.degree_one,
                   "degree_two_triangle": fo.degree_two_triangle, "high_degree": fo.high_degree,
                   "edges_removed": fo.edges_removed, "pos": pos, "out": out[1:pos].tolist()}
        elif rule == "crown":
            co = crown_reduce(node, g)
            got = {"forced_vertices": co.forced_vertices,
                   "independent_vertices": co.independent_vertices,
                   "edges_removed": co.edges_removed, "applied": co.applied}
        else:
            fn = {"degree_one": apply_degree_one, "degree_two_triangle": apply_degree_two_triangle}
            ro = (apply_high_degree(node, g, case["budget"]) if rule == "high_degree"
                  else fn[rule](node, g))
            got = {"applications": ro.applications, "forced": ro.forced,
                   "edges_removed": ro.edges_removed, "forced_vertices": ro.forced_vertices}
        assert got == oc, (rule, case["n"])
        st = case["node"]
        assert node.degrees.tolist() == st["degrees"]
        assert (node.solution_size, node.edges_remaining, node.lo, node.hi) == (
            st["solution_size"], st["edges_remaining"], st["lo"], st["hi"])
        assert [int(v) for v in np.flatnonzero(node.inclusion)] == st["inclusion"]


def test_search_node_mirror():
    """test_graph.py:91-153, the SearchNode half, on the device node ops."""
    from paper_2512_18334_b200.graph import (SearchNode, recompute_node_bounds,
                                             remove_neighbors, remove_vertex)

    g = make_graph(4, path_edges(4))
    node = SearchNode.for_graph(g, 8)
    assert (node.solution_size, node.edges_remaining, node.lo, node.hi) == (0, 3, 0, 3)
    assert node.inclusion is None and node.live_count() == 4
    node = SearchNode.for_graph(g, 8, track_inclusion=True)
    clone = node.copy()
    assert remove_vertex(node, g, 1, into_cover=True) == 2
    assert (node.edges_remaining, node.solution_size) == (1, 1)
    assert node.degrees.tolist() == [0, 0, 1, 1]
    assert node.inclusion.tolist() == [False, True, False, False]
    assert remove_vertex(node, g, 0, into_cover=True) == 0 and node.solution_size == 2
    assert (clone.solution_size, clone.edges_remaining) == (0, 3)
    assert clone.degrees.tolist() == [1, 2, 2, 1] and not clone.inclusion.any()
    g = make_graph(5, clique_edges(5))
    node = SearchNode.for_graph(g, 8, track_inclusion=True)
    out = np.zeros(16, dtype=np.int32)
    removed, pos = remove_neighbors(node, g, 0, out, 0)
    assert removed == 4 and sorted(out[:pos].tolist()) == [1, 2, 3, 4]
    assert (node.solution_size, node.edges_remaining) == (4, 0)
    assert node.inclusion.tolist() == [False, True, True, True, True]
    g = make_graph(5, path_edges(5))
    node = SearchNode.for_graph(g, 8)
    remove_vertex(node, g, 0, into_cover=False)
    remove_vertex(node, g, 1, into_cover=True)
    recompute_node_bounds(node)
    assert (node.lo, node.hi) == (2, 4)
    for v in (2, 3, 4):
        remove_vertex(node, g, v, into_cover=False)
    recompute_node_bounds(node)
    assert node.lo > node.hi and node.live_count() == 0
