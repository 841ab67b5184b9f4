"""Per-node kernel API of ``vcsolver.kernels`` (kernels/__init__.py:38-49),
each call executed by ONE thread block on the device (``vcg_node_op``).

This is the parity surface: the same functions, arguments and return tuples
as the reference's ``pure``/``_native`` backends, so the reference's kernel
tests read the same against this module.  (The search kernel runs the same
device functions; per-call launches here are for parity, not speed.)
``deg`` arrays are updated in place, like the reference.
"""

from __future__ import annotations

import numpy as np

from . import _lib

BACKEND = "cuda-sm_100a"
_OPS = {
    "degree_one_pass": 0, "degree_two_triangle_pass": 1, "high_degree_pass": 2,
    "reduce_fixpoint": 3, "recompute_bounds": 4, "select_max_degree": 5, "count_live": 6,
    "remove_vertex": 7, "remove_neighbors": 8, "component": 9, "bfs_component": 10,
    "next_live_unvisited": 11, "greedy_cover": 12,
}
_WIDTH = {1: 8, 2: 16, 4: 32, 8: 32}


def _call(op, deg, off, nbr, lo=0, hi=-1, budget=0, v=0, out=None, pos=0, _buf=None):
    n = len(deg)
    if n == 0:
        raise ValueError("empty degree array")
    off = np.ascontiguousarray(off, dtype=np.int64)
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    if len(nbr) == 0:
        nbr = np.zeros(1, dtype=np.int32)
    width = _WIDTH[np.dtype(deg.dtype).itemsize]
    d32 = np.ascontiguousarray(deg, dtype=np.uint32)
    buf = np.zeros(4 * n + 4, dtype=np.int32) if _buf is None else _buf
    if out is not None:
        k = min(len(out), len(buf))
        buf[:k] = out[:k]
    ret = np.zeros(8, dtype=np.int64)
    _lib.check(_lib.lib.vcg_node_op(_OPS[op], width, n, off.ctypes.data, nbr.ctypes.data,
                                    d32.ctypes.data, int(lo), int(hi), int(budget), int(v),
                                    buf.ctypes.data, int(pos), ret.ctypes.data))
    deg[:] = d32.astype(deg.dtype)
    if out is not None:
        k = min(len(out), len(buf))
        out[:k] = buf[:k]
    return ret, buf


def remove_vertex(deg, off, nbr, v):
    ret, _ = _call("remove_vertex", deg, off, nbr, v=v)
    return int(ret[0])


def remove_neighbors(deg, off, nbr, v, out, pos):
    ret, _ = _call("remove_neighbors", deg, off, nbr, v=v, out=out, pos=pos)
    return int(ret[0]), int(ret[1]), int(ret[2])


def degree_one_pass(deg, off, nbr, lo, hi, out, pos, scratch):
    ret, _ = _call("degree_one_pass", deg, off, nbr, lo, hi, out=out, pos=pos)
    return tuple(int(x) for x in ret[:4])


def degree_two_triangle_pass(deg, off, nbr, lo, hi, out, pos, scratch):
    ret, _ = _call("degree_two_triangle_pass", deg, off, nbr, lo, hi, out=out, pos=pos)
    return tuple(int(x) for x in ret[:4])


def high_degree_pass(deg, off, nbr, lo, hi, budget, out, pos, scratch):
    ret, _ = _call("high_degree_pass", deg, off, nbr, lo, hi, budget, out=out, pos=pos)
    return tuple(int(x) for x in ret[:4])


def reduce_fixpoint(deg, off, nbr, lo, hi, budget, out, pos, scratch):
    ret, _ = _call("reduce_fixpoint", deg, off, nbr, lo, hi, budget, out=out, pos=pos)
    return tuple(int(x) for x in ret[:8])


def recompute_bounds(deg, lo, hi):
    off = np.zeros(len(deg) + 1, dtype=np.int64)
    ret, _ = _call("recompute_bounds", deg.copy(), off, np.zeros(1, np.int32), lo, hi)
    return int(ret[0]), int(ret[1])


def select_max_degree(deg, lo, hi):
    off = np.zeros(len(deg) + 1, dtype=np.int64)
    ret, _ = _call("select_max_degree", deg.copy(), off, np.zeros(1, np.int32), lo, hi)
    return int(ret[0])


def count_live(deg, lo, hi):
    off = np.zeros(len(deg) + 1, dtype=np.int64)
    ret, _ = _call("count_live", deg.copy(), off, np.zeros(1, np.int32), lo, hi)
    return int(ret[0])


def component(deg, off, nbr, source, lo=0, hi=None):
    """Component of a live ``source`` (the set bfs_component visits, pure.py:258):
    returns ((size, degree_sum, min_degree, max_degree, min_vertex, max_vertex),
    sorted members)."""
    if deg[source] == 0:
        raise ValueError("bfs_component: source vertex is not live")
    hi = len(deg) - 1 if hi is None else hi
    ret, buf = _call("component", deg.copy(), off, nbr, lo, hi, v=source)
    size = int(ret[0])
    return tuple(int(x) for x in ret[:6]), buf[:size].tolist()


def bfs_component(deg, off, nbr, visited, stamp, queue, source):
    """pure.py:258 -- the component of a live ``source`` in BFS queue order:
    members get ``stamp`` in ``visited`` and fill ``queue[0:size]``.  Returns
    (size, degree_sum, min_degree, max_degree, min_vertex, max_vertex)."""
    if deg[source] == 0:
        raise ValueError("bfs_component: source vertex is not live")
    n = len(deg)
    buf = np.zeros(4 * n + 4, dtype=np.int32)
    buf[:n] = visited[:n]
    ret, buf = _call("bfs_component", deg.copy(), off, nbr, budget=stamp, v=source, out=None,
                     pos=0, _buf=buf)
    size = int(ret[0])
    visited[:n] = buf[:n]
    queue[:size] = buf[n:n + size]
    return tuple(int(x) for x in ret[:6])


def next_live_unvisited(deg, visited, stamp, start, hi):
    """pure.py:297 -- first live vertex of [start, hi] not carrying ``stamp``, or -1."""
    n = len(deg)
    if start > hi:
        return -1
    buf = np.zeros(4 * n + 4, dtype=np.int32)
    buf[:n] = visited[:n]
    off = np.zeros(n + 1, dtype=np.int64)
    ret, _ = _call("next_live_unvisited", deg.copy(), off, np.zeros(1, np.int32), start, hi,
                   budget=stamp, _buf=buf)
    return int(ret[0])


def greedy_cover(deg, off, nbr, lo, hi, out, pos):
    """pure.py:306 -- max-degree greedy cover (lowest index on ties) on the
    device; destroys ``deg`` like the reference, members to ``out[pos..]``.
    Returns (size, new_pos)."""
    ret, _ = _call("greedy_cover", deg, off, nbr, lo, hi, out=out, pos=pos)
    return int(ret[0]), int(ret[1])
