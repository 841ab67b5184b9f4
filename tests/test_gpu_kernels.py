"""Per-node device kernels vs the reference's own outputs (tests/golden/
kernels.json, generated from vcsolver.kernels.pure).  Each call runs one
thread block on the GPU through the C-ABI (vcg_node_op)."""

from __future__ import annotations

import numpy as np
import pytest

from helpers import csr, golden

pytestmark = pytest.mark.gpu


def _state(case, dtype):
    n, off, nbr = csr(case["n"], case["edges"])
    deg = np.asarray(case["deg"], dtype=dtype)
    return n, off, nbr, deg


@pytest.mark.parametrize("dtype", [np.uint32, np.uint8])
def test_rule_sweeps_bit_exact(dtype):
    from paper_2512_18334_b200 import kernels as K

    for case in golden("kernels.json"):
        n, off, nbr, deg = _state(case, dtype)
        exp = case["expect"]
        for fn in ("degree_one_pass", "degree_two_triangle_pass"):
            d = deg.copy()
            o = np.zeros(2 * n + 2, dtype=np.int32)
            r = getattr(K, fn)(d, off, nbr, 0, n - 1, o, 0, None)
            assert list(r) == exp[fn]["ret"], fn
            assert d.tolist() == exp[fn]["deg"], fn
            assert o[: r[3]].tolist() == exp[fn]["out"], fn
        d = deg.copy()
        o = np.zeros(2 * n + 2, dtype=np.int32)
        r = K.high_degree_pass(d, off, nbr, 0, n - 1, case["budget"], o, 0, None)
        assert list(r) == exp["high_degree_pass"]["ret"]
        assert d.tolist() == exp["high_degree_pass"]["deg"]
        assert o[: r[3]].tolist() == exp["high_degree_pass"]["out"]
        d = deg.copy()
        o = np.zeros(4 * n + 4, dtype=np.int32)
        r = K.reduce_fixpoint(d, off, nbr, 0, n - 1, case["budget"], o, 0, None)
        assert list(r) == exp["reduce_fixpoint"]["ret"]
        assert d.tolist() == exp["reduce_fixpoint"]["deg"]
        assert o[: r[7]].tolist() == exp["reduce_fixpoint"]["out"]


def test_point_kernels_bit_exact():
    from paper_2512_18334_b200 import kernels as K

    for case in golden("kernels.json"):
        n, off, nbr, deg = _state(case, np.uint32)
        exp = case["expect"]
        assert K.select_max_degree(deg, 0, n - 1) == exp["select_max_degree"]
        assert K.count_live(deg, 0, n - 1) == exp["count_live"]
        assert list(K.recompute_bounds(deg, 0, n - 1)) == exp["recompute_bounds"]
        d = deg.copy()
        assert K.remove_vertex(d, off, nbr, case["v"]) == exp["remove_vertex"]["ret"]
        assert d.tolist() == exp["remove_vertex"]["deg"]
        d = deg.copy()
        o = np.zeros(n + 1, dtype=np.int32)
        r = K.remove_neighbors(d, off, nbr, case["v"], o, 0)
        assert list(r) == exp["remove_neighbors"]["ret"]
        assert d.tolist() == exp["remove_neighbors"]["deg"]
        assert o[: r[2]].tolist() == exp["remove_neighbors"]["out"]
        if "src" in case:
            r, members = K.component(deg, off, nbr, case["src"])
            assert list(r) == exp["bfs_component"]["ret"]
            assert members == exp["bfs_component"]["members"]
            # kernels/__init__.py:42-43: BFS queue order, visited stamps
            vis = np.zeros(n, dtype=np.int32)
            q = np.zeros(n, dtype=np.int32)
            r = K.bfs_component(deg, off, nbr, vis, 1, q, case["src"])
            assert list(r) == exp["bfs_component"]["ret"]
            assert q[: r[0]].tolist() == exp["bfs_component"]["queue"]
            assert sorted(np.nonzero(vis == 1)[0].tolist()) == exp["bfs_component"]["members"]
            assert K.next_live_unvisited(deg, vis, 1, 0, n - 1) == exp["bfs_component"]["next"]
        d = deg.copy()
        o = np.zeros(n + 1, dtype=np.int32)
        r = K.greedy_cover(d, off, nbr, 0, n - 1, o, 0)
        assert list(r) == exp["greedy_cover"]["ret"]
        assert o[: r[1]].tolist() == exp["greedy_cover"]["out"]


def test_negative_budget_high_degree_closed_form():
    """budget < 0 makes every live vertex a candidate (stale nodes whose scope
    best dropped): the closed form must equal the in-order sweep."""
    import random

    import oracle
    from paper_2512_18334_b200 import kernels as K

    rng = random.Random(7)
    for _ in range(60):
        n = rng.randint(2, 40)
        edges = [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < 0.2]
        _, off, nbr = csr(n, edges)
        deg = np.diff(off).astype(np.uint32)
        for budget in (-3, -1, 0, 1, 2):
            d1, d2 = deg.copy(), deg.copy()
            o1 = np.zeros(2 * n + 2, np.int32)
            o2 = np.zeros(2 * n + 2, np.int32)
            s = np.zeros(n + 1, np.int32)
            r1 = oracle.high_degree_pass(d1, off, nbr, 0, n - 1, budget, o1, 0, s)
            r2 = K.high_degree_pass(d2, off, nbr, 0, n - 1, budget, o2, 0, None)
            assert tuple(r1) == tuple(r2)
            assert d1.tolist() == d2.tolist()
            assert o1[: r1[3]].tolist() == o2[: r2[3]].tolist()
