"""Per-node reduction API of ``vcsolver.reductions`` (reductions.py:1-320).

The same names, outcome records and side effects on a host ``SearchNode``
as the reference, so a caller of the reference's single-rule API (its
tests, or a custom driver) finds the same surface.  The rules execute on the
device, one thread block per call (``kernels`` -> ``vcg_node_op``, the same
device functions the search kernel runs at every node); the crown is the
library's host C++ matching (``vcg_crown_reduce``, the routine the root
pipeline runs between its device fixpoint passes).  The solve path never
calls this module: the search kernel applies the rules inside its own loop.
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib, kernels
from .graph import SearchNode, StaticGraph


@dataclass
class ReductionOutcome:
    """reductions.py:27: what one rule did to a node."""

    applications: int = 0
    forced: int = 0
    edges_removed: int = 0
    forced_vertices: list[int] = field(default_factory=list)


@dataclass
class FixpointOutcome:
    """reductions.py:37: per-rule application counts of one fixpoint run."""

    forced: int = 0
    degree_one: int = 0
    degree_two_triangle: int = 0
    high_degree: int = 0
    edges_removed: int = 0


def _record(node: SearchNode, out: np.ndarray, start: int, stop: int) -> list[int]:
    forced = [int(x) for x in out[start:stop]]
    node.solution_size += stop - start
    if node.inclusion is not None:
        for v in forced:
            node.inclusion[v] = 1
    return forced


def _run_rule(node: SearchNode, g: StaticGraph, pass_fn, *extra) -> ReductionOutcome:
    # reductions.py:60: sweep until a pass applies nothing; the high-degree
    # budget shrinks by the vertices each pass forced
    out = np.empty(len(node.degrees), dtype=np.int32)
    outcome = ReductionOutcome()
    pos = 0
    while True:
        applied, forced, edges, pos = pass_fn(node.degrees, g.offsets, g.neighbors, node.lo,
                                              node.hi, *extra, out, pos, None)
        outcome.applications += applied
        outcome.edges_removed += edges
        node.edges_remaining -= edges
        if applied == 0:
            break
        if extra:
            extra = (extra[0] - forced,)
    outcome.forced_vertices = _record(node, out, 0, pos)
    outcome.forced = pos
    recompute_node_bounds_inplace(node)
    return outcome


def recompute_node_bounds_inplace(node: SearchNode) -> None:
    """reductions.py:91."""
    node.lo, node.hi = kernels.recompute_bounds(node.degrees, node.lo, node.hi)


def apply_degree_one(node: SearchNode, g: StaticGraph) -> ReductionOutcome:
    """reductions.py:95: force the neighbour of every degree-one vertex, to
    exhaustion."""
    return _run_rule(node, g, kernels.degree_one_pass)


def apply_degree_two_triangle(node: SearchNode, g: StaticGraph) -> ReductionOutcome:
    """reductions.py:100: force both neighbours of every degree-2 vertex whose
    neighbours are adjacent."""
    return _run_rule(node, g, kernels.degree_two_triangle_pass)


def apply_high_degree(node: SearchNode, g: StaticGraph, budget: int) -> ReductionOutcome:
    """reductions.py:105: force every live vertex of degree above the
    remaining budget."""
    return _run_rule(node, g, kernels.high_degree_pass, budget)


def reduce_to_fixpoint(node: SearchNode, g: StaticGraph, budget: int, out=None, pos: int = 0,
                       scratch=None) -> tuple[FixpointOutcome, int]:
    """reductions.py:110: all rules to a joint fixpoint (one device block);
    forced ids land in ``out[pos:]``.  Returns (outcome, new_pos)."""
    if out is None:
        out = np.empty(len(node.degrees), dtype=np.int32)
    start = pos
    forced, d1, d2t, hd, edges, lo, hi, pos = kernels.reduce_fixpoint(
        node.degrees, g.offsets, g.neighbors, node.lo, node.hi, budget, out, pos, scratch)
    node.lo = lo
    node.hi = hi
    node.edges_remaining -= edges
    _record(node, out, start, pos)
    return FixpointOutcome(forced=forced, degree_one=d1, degree_two_triangle=d2t,
                           high_degree=hd, edges_removed=edges), pos


class ComponentKind(enum.Enum):
    """reductions.py:154."""

    CLIQUE = "clique"
    CHORDLESS_CYCLE = "chordless_cycle"
    GENERAL = "general"


def classify_special_component(size: int, min_degree: int, max_degree: int) -> ComponentKind:
    """reductions.py:160: closed-form classes from the degree summary (the
    search kernel's ``try_split`` applies the same test on the device).  K3
    counts as a clique."""
    if min_degree == max_degree:
        if min_degree == size - 1:
            return ComponentKind.CLIQUE
        if min_degree == 2 and size >= 3:
            return ComponentKind.CHORDLESS_CYCLE
    return ComponentKind.GENERAL


def solve_special_component(kind: ComponentKind, size: int) -> int:
    """reductions.py:175: exact cover size of a special component."""
    if kind is ComponentKind.CLIQUE:
        return size - 1
    if kind is ComponentKind.CHORDLESS_CYCLE:
        return (size + 1) // 2
    raise ValueError("general components have no closed-form cover size")


@dataclass
class CrownOutcome:
    """reductions.py:185."""

    forced_vertices: list[int] = field(default_factory=list)
    independent_vertices: list[int] = field(default_factory=list)
    edges_removed: int = 0

    @property
    def applied(self) -> bool:
        return bool(self.forced_vertices)


def crown_reduce(node: SearchNode, g: StaticGraph) -> CrownOutcome:
    """reductions.py:263: find one crown (greedy maximal matching, maximum
    bipartite matching of its unmatched side, alternating closure from the
    unmatched candidates) and force its heads into the cover."""
    outcome = CrownOutcome()
    if node.lo > node.hi:
        return outcome
    n = len(node.degrees)
    deg = np.ascontiguousarray(node.degrees, dtype=np.uint32)
    off = np.ascontiguousarray(g.offsets, dtype=np.int64)
    nbr = np.ascontiguousarray(g.neighbors, dtype=np.int32)
    if len(nbr) == 0:
        nbr = np.zeros(1, dtype=np.int32)
    heads = np.empty(max(n, 1), dtype=np.int32)
    indep = np.empty(max(n, 1), dtype=np.int32)
    nh, ni, er = _lib.I64(), _lib.I64(), _lib.I64()
    _lib.check(_lib.lib.vcg_crown_reduce(n, off.ctypes.data, nbr.ctypes.data, deg.ctypes.data,
                                         int(node.lo), int(node.hi), heads.ctypes.data,
                                         C.byref(nh), indep.ctypes.data, C.byref(ni),
                                         C.byref(er)))
    if nh.value == 0:
        return outcome
    node.degrees[:] = deg.astype(node.degrees.dtype)
    outcome.forced_vertices = [int(h) for h in heads[:nh.value]]
    outcome.independent_vertices = [int(v) for v in indep[:ni.value]]
    outcome.edges_removed = int(er.value)
    if node.inclusion is not None:
        for h in outcome.forced_vertices:
            node.inclusion[h] = 1
    node.solution_size += len(outcome.forced_vertices)
    node.edges_remaining -= outcome.edges_removed
    recompute_node_bounds_inplace(node)
    return outcome
