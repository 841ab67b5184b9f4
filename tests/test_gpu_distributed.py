"""The distributed solver's GPU backend on one GPU (world 1): device
expansion of the root's search tree + subtree searches seeded from it must
give the reference's answers."""

from __future__ import annotations

import pytest

from helpers import csr, golden

pytestmark = pytest.mark.gpu


def test_subtree_partition_answers():
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200.distributed import solve_distributed

    for case in golden("solve.json")[::4]:
        n, off, nbr = csr(case["n"], case["edges"])
        g = vc.StaticGraph(n, off, nbr)
        want = case["runs"]["det"]["cover_size"]
        for per in (1, 5):
            r = solve_distributed(g, vc.SolverConfig(), subtrees_per_rank=per)
            assert r.cover_size == want, (case["name"], per)
        for k, exp in case["pvc"].items():
            r = solve_distributed(g, vc.SolverConfig(mode="pvc", k=int(k)), subtrees_per_rank=5)
            assert r.found == exp["found"], (case["name"], k)


@pytest.mark.parametrize("name", ["er200", "rgg2000"])
def test_subtree_partition_workloads(name):
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth
    from paper_2512_18334_b200.distributed import solve_distributed

    exp = golden("workloads.json")[name]
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    for per in (4, 16):
        r = solve_distributed(g, vc.SolverConfig(), subtrees_per_rank=per)
        assert r.cover_size == exp["mvc"], per
    for k, e in exp["pvc"].items():
        r = solve_distributed(g, vc.SolverConfig(mode="pvc", k=int(k)), subtrees_per_rank=8)
        assert r.found == e["found"], k
