"""Host-side C++ of the root pipeline (csrc/host_algos.cpp: the greedy bound
and the crown rule) against the oracle on CPU.  The file is compiled here
with g++ into a scratch library -- it is plain C++, the same source the
CUDA library links -- and called through a two-function C shim."""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import oracle
from helpers import csr, golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = r'''
#include "host_algos.h"
extern "C" int64_t t_greedy(int64_t n, const int64_t* off, const int32_t* nbr, int32_t* members) {
  return vcg::greedy_cover_host(n, off, nbr, members);
}
'''


@pytest.fixture(scope="module")
def hostlib(tmp_path_factory):
    d = tmp_path_factory.mktemp("hostalgos")
    shim = d / "shim.cpp"
    shim.write_text(SHIM)
    src = os.path.join(ROOT, "paper_2512_18334_b200", "csrc")
    so = d / "libhost.so"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I", src, str(shim),
                           os.path.join(src, "host_algos.cpp"), "-o", str(so)])
    lib = C.CDLL(str(so))
    lib.t_greedy.restype = C.c_int64
    lib.t_greedy.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    return lib


def _greedy(lib, n, off, nbr):
    off = np.ascontiguousarray(off, dtype=np.int64)
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    out = np.zeros(max(n, 1), dtype=np.int32)
    size = lib.t_greedy(n, off.ctypes.data, nbr.ctypes.data, out.ctypes.data)
    return size, out[:size].tolist()


def test_greedy_matches_oracle_on_golden_graphs(hostlib):
    for case in golden("solve.json"):
        n, off, nbr = csr(case["n"], case["edges"])
        assert _greedy(hostlib, n, off, nbr) == oracle.greedy_bound(n, off, nbr, members=True), \
            case["name"]


@pytest.mark.parametrize("seed", range(6))
def test_greedy_matches_oracle_random(hostlib, seed):
    from paper_2512_18334_b200 import synth

    rng = np.random.default_rng(seed)
    n = int(rng.integers(50, 3000))
    kind = seed % 3
    if kind == 0:
        n, off, nbr = synth.er(n, float(rng.uniform(1, 12)), seed)
    elif kind == 1:
        n, off, nbr = synth.ba(n, int(rng.integers(1, 5)), seed)
    else:
        n, off, nbr = synth.rgg(n, float(rng.uniform(0.02, 0.06)), seed)
    assert _greedy(hostlib, n, off, nbr) == oracle.greedy_bound(n, off, nbr, members=True)
