"""Full-size configurations (BASELINE.json configs[2], configs[3]) through
size-independent properties: the recorded cover is a valid vertex cover of
exactly the reported size, the PVC pair at k = opt / opt - 1 answers
yes / no (so the reported size is the minimum), and the deterministic
(reference-schedule) and parallel modes agree.  The optima are pinned to
the C oracle's (tests/golden/scale.json, make_scale_golden.py)."""

from __future__ import annotations

import pytest

from helpers import assert_valid_cover, golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["ba100k", "planted1m"])
def test_large_config_cover_and_pvc_pair(name):
    import numpy as np

    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth

    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    r = vc.solve(g, vc.SolverConfig(record_cover=True))
    assert r.exact
    assert len(r.cover) == r.cover_size == len(set(r.cover))
    assert_valid_cover(n, np.asarray(off), np.asarray(nbr), r.cover)
    opt = r.cover_size
    assert opt == golden("scale.json")[name]["mvc"]
    assert vc.solve(g, vc.SolverConfig(deterministic=True)).cover_size == opt
    assert vc.solve(g, vc.SolverConfig()).cover_size == opt
    yes = vc.solve(g, vc.SolverConfig(mode="pvc", k=opt))
    no = vc.solve(g, vc.SolverConfig(mode="pvc", k=opt - 1))
    assert yes.found and yes.cover_size <= opt
    assert not no.found


@pytest.mark.parametrize("name", ["gnp400", "torus60"])
def test_time_budget_configs_return_valid_covers(name):
    """configs[4] runs under a time budget (no exact answer in reach for
    either side).  As in the reference (engine.py:655), a timed-out solve
    reports its incumbent size but no cover; the incumbent is then
    witnessed by a PVC solve at k = incumbent, whose cover must be valid.
    The incumbent is no smaller than a maximal matching (torus60: a perfect
    matching, 1800)."""
    import numpy as np

    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth

    n, off, nbr = synth.WORKLOADS[name]()
    off, nbr = np.asarray(off), np.asarray(nbr)
    g = vc.StaticGraph(n, off, nbr)
    r = vc.solve(g, vc.SolverConfig(record_cover=True, timeout=1.0))
    assert not r.exact and r.cover is None
    best = r.cover_size
    w = vc.solve(g, vc.SolverConfig(mode="pvc", k=best, record_cover=True, timeout=30.0))
    assert w.found and w.cover is not None and len(w.cover) <= best
    assert_valid_cover(n, off, nbr, w.cover)
    matched = np.zeros(n, dtype=bool)
    lb = 0
    for v in range(n):
        if matched[v]:
            continue
        for x in nbr[off[v]:off[v + 1]]:
            if not matched[x] and x != v:
                matched[v] = matched[x] = True
                lb += 1
                break
    assert best >= lb
    if name == "torus60":
        assert best >= 1800
