"""Small independent references of the reference API (oracle.py:28-97):
``brute_force_mvc`` (every vertex subset checked on the device,
``vcg_brute_force_mvc``) and the greedy cover (the device greedy kernel,
kernels.greedy_cover).  Deliberately different algorithms from the search,
so the two cross-validate, as in the reference."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, kernels
from .graph import StaticGraph

MAX_ORACLE_VERTICES = 26


def brute_force_mvc(g: StaticGraph) -> tuple[int, tuple[int, ...]]:
    """oracle.py:28 -- exact minimum vertex cover size and the
    lexicographically smallest minimum cover (n <= 26)."""
    n = g.num_vertices
    if n > MAX_ORACLE_VERTICES:
        raise ValueError(f"oracle limited to {MAX_ORACLE_VERTICES} vertices, got {n}")
    off = np.ascontiguousarray(g.offsets, dtype=np.int64)
    nbr = np.ascontiguousarray(g.neighbors, dtype=np.int32)
    if len(nbr) == 0:
        nbr = np.zeros(1, dtype=np.int32)
    size = C.c_int64()
    wit = np.zeros(max(n, 1), dtype=np.int32)
    _lib.check(_lib.lib.vcg_brute_force_mvc(n, off.ctypes.data, nbr.ctypes.data, C.byref(size),
                                            wit.ctypes.data))
    return int(size.value), tuple(int(x) for x in wit[: size.value])


def greedy_cover_members(g: StaticGraph) -> list[int]:
    """oracle.py:87 -- the greedy cover in pick order (ties to the lowest index)."""
    n = g.num_vertices
    if n == 0 or g.num_edges == 0:
        return []
    deg = np.diff(np.asarray(g.offsets, dtype=np.int64)).astype(np.uint32)
    out = np.empty(n, dtype=np.int32)
    size, _ = kernels.greedy_cover(deg, g.offsets, g.neighbors, 0, n - 1, out, 0)
    return [int(x) for x in out[:size]]


def greedy_cover(g: StaticGraph) -> int:
    """oracle.py:82 -- size of the greedy cover."""
    return len(greedy_cover_members(g))


__all__ = ["MAX_ORACLE_VERTICES", "brute_force_mvc", "greedy_cover", "greedy_cover_members"]
