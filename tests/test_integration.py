"""The reference-side binding of INTEGRATION.md (integration/vcsolver_gpu.py:
ctypes + numpy only, what a maintainer drops into vcsolver) against the
reference's answers and deterministic statistics."""

from __future__ import annotations

import importlib.util
import os
import types

import pytest

from helpers import csr, golden, stats_without_time

HERE = os.path.dirname(os.path.abspath(__file__))


def _binding():
    spec = importlib.util.spec_from_file_location(
        "vcsolver_gpu", os.path.join(os.path.dirname(HERE), "integration", "vcsolver_gpu.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_binding_loads_and_mirrors_the_abi():
    """CPU: the stub loads libvcgpu.so and its structs match the package's
    (which tests/test_capi_cpu.py checks against include/vcgpu.h)."""
    import ctypes as C

    from paper_2512_18334_b200 import _lib

    b = _binding()
    for mine, ref in ((b.Preprocessed, _lib.Preprocessed_t), (b.SearchConfig, _lib.SearchConfig_t),
                      (b.SearchResult, _lib.SearchResult_t)):
        assert [f[0] for f in mine._fields_] == [f[0] for f in ref._fields_]
        assert C.sizeof(mine) == C.sizeof(ref)


@pytest.mark.gpu
def test_binding_solves_like_the_reference():
    b = _binding()
    for case in golden("solve.json")[::6]:
        n, off, nbr = csr(case["n"], case["edges"])
        g = types.SimpleNamespace(num_vertices=n, offsets=off, neighbors=nbr)
        run = case["runs"]["det"]
        r = b.solve(g, types.SimpleNamespace(deterministic=True))
        assert r.cover_size == run["cover_size"], case["name"]
        assert stats_without_time(dict(r.stats, phase_seconds={}, degree_width=0)) == \
            run["stats"], case["name"]
        assert b.solve(g).cover_size == run["cover_size"]
        for k, exp in case["pvc"].items():
            r = b.solve(g, types.SimpleNamespace(mode="pvc", k=int(k)))
            assert r.found == exp["found"], (case["name"], k)
