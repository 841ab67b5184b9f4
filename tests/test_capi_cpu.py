"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/vcgpu.h declares, and fails loudly without a device."""

from __future__ import annotations

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "vcgpu.h")).read()
    return sorted(set(re.findall(r"\b(vcg_[a-z_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_2512_18334_b200 import _lib

    declared = _declared()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(_lib.lib, name), name
    assert set(_lib.EXPORTS) == set(declared)


def test_no_cpu_fallback_without_device():
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import _lib

    if _lib.device_count() > 0:
        pytest.skip("a device is present")
    g = vc.build_csr([(0, 1), (1, 2)], 3)
    with pytest.raises(_lib.GpuError):
        vc.solve(g)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2512_18334_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text, f


def test_warp_limit_validation():
    import paper_2512_18334_b200 as vc

    for ok in (-1, 0, 64, 128, 256):
        vc.SolverConfig(warp_limit=ok).validate()
    for bad in (-2, 257):
        with pytest.raises(ValueError):
            vc.SolverConfig(warp_limit=bad).validate()


def test_gpu_share_and_batch_validation():
    import paper_2512_18334_b200 as vc

    with pytest.raises(ValueError):
        vc.SolverConfig(gpu_share=0).validate()
    g = vc.StaticGraph(3, [0, 1, 2, 2], [1, 0])
    with pytest.raises(ValueError):
        vc.solve_batch([g, g], [vc.SolverConfig()])  # one graph per config
    assert vc.solve_batch(g, []) == []


def test_registry_object_needs_a_device():
    from paper_2512_18334_b200 import _lib
    from paper_2512_18334_b200.registry import Registry

    with pytest.raises(_lib.GpuError):
        Registry()
