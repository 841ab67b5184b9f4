"""The per-node reduction API's host pieces on CPU: closed-form component
classes (reductions.py:154-182, the reference's own cases) and the crown
entry point of the C-ABI (vcg_crown_reduce <- reductions.py:263) against
the reference's crowns (tests/golden/reductions.json, crown.json)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from helpers import csr, golden


def _crown(n, off, nbr, deg, lo, hi):
    from paper_2512_18334_b200 import _lib

    nbr = nbr if len(nbr) else np.zeros(1, dtype=np.int32)
    heads = np.empty(max(n, 1), dtype=np.int32)
    indep = np.empty(max(n, 1), dtype=np.int32)
    nh, ni, er = _lib.I64(), _lib.I64(), _lib.I64()
    _lib.check(_lib.lib.vcg_crown_reduce(n, off.ctypes.data, nbr.ctypes.data, deg.ctypes.data,
                                         lo, hi, heads.ctypes.data, C.byref(nh),
                                         indep.ctypes.data, C.byref(ni), C.byref(er)))
    return heads[:nh.value].tolist(), indep[:ni.value].tolist(), int(er.value)


def test_classify_special_components():
    from paper_2512_18334_b200.reductions import ComponentKind, classify_special_component

    assert classify_special_component(2, 1, 1) is ComponentKind.CLIQUE
    assert classify_special_component(3, 2, 2) is ComponentKind.CLIQUE
    assert classify_special_component(5, 4, 4) is ComponentKind.CLIQUE
    assert classify_special_component(4, 2, 2) is ComponentKind.CHORDLESS_CYCLE
    assert classify_special_component(9, 2, 2) is ComponentKind.CHORDLESS_CYCLE
    assert classify_special_component(4, 1, 2) is ComponentKind.GENERAL
    assert classify_special_component(6, 3, 4) is ComponentKind.GENERAL


def test_solve_special_components():
    from paper_2512_18334_b200.reductions import ComponentKind, solve_special_component

    assert solve_special_component(ComponentKind.CLIQUE, 2) == 1
    assert solve_special_component(ComponentKind.CLIQUE, 6) == 5
    assert solve_special_component(ComponentKind.CHORDLESS_CYCLE, 5) == 3
    assert solve_special_component(ComponentKind.CHORDLESS_CYCLE, 8) == 4
    with pytest.raises(ValueError):
        solve_special_component(ComponentKind.GENERAL, 4)


def test_crown_abi_matches_reference():
    fired = 0
    cases = [c for c in golden("reductions.json") if c["rule"] == "crown"]
    for case in cases:
        n, off, nbr = csr(case["n"], case["edges"])
        deg = np.diff(off).astype(np.uint32)
        heads, indep, er = _crown(n, off, nbr, deg, case["root"]["lo"], case["root"]["hi"])
        oc = case["outcome"]
        assert heads == oc["forced_vertices"]
        assert indep == oc["independent_vertices"]
        assert er == oc["edges_removed"]
        assert deg.tolist() == case["node"]["degrees"]
        fired += bool(heads)
    assert fired >= 40
    for case in golden("crown.json"):
        n, off, nbr = csr(case["n"], case["edges"])
        deg = np.diff(off).astype(np.uint32)
        live = np.nonzero(deg)[0]
        lo, hi = (int(live[0]), int(live[-1])) if len(live) else (max(n, 1), 0)
        heads, indep, er = _crown(n, off, nbr, deg, lo, hi)
        assert (heads, indep, er) == (case["forced"], case["independent"],
                                      case["edges_removed"])


def test_crown_abi_rejects_bad_arguments():
    from paper_2512_18334_b200 import _lib

    z = np.zeros(4, dtype=np.int64)
    rc = _lib.lib.vcg_crown_reduce(-1, z.ctypes.data, None, z.ctypes.data, 0, 0, None,
                                   None, None, None, None)
    assert rc == 1  # VCG_EINVAL
