"""Root reduction + compaction (mirror of vcsolver.preprocess, preprocess.py:28-148).

The lightweight rules run to a fixpoint on the device, the crown rule's
matching runs natively on the host, survivors are compacted into a fresh CSR
on the device (``vcg_root_reduce``), and the degree width is the smallest of
8/16/32 bits that holds the reduced maximum degree (§4.4).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import SUPPORTED_WIDTHS, DeviceGraph, StaticGraph, width_capacity

ROOT_RULE_KEYS = ("degree_one", "degree_two_triangle", "high_degree", "crown")


def greedy_bound(g: StaticGraph, members: bool = False):
    """preprocess.py:28 -- max-degree greedy cover size (optionally the picks)."""
    if g.num_vertices == 0 or g.num_edges == 0:
        return (0, []) if members else 0
    out = np.zeros(g.num_vertices, dtype=np.int32) if members else None
    size = C.c_int64()
    _lib.check(_lib.lib.vcg_greedy_bound(g.device().handle,
                                         out.ctypes.data if members else None, C.byref(size)))
    if members:
        return int(size.value), out[: size.value].tolist()
    return int(size.value)


def select_width(max_degree: int, override: int | None = None) -> int:
    """preprocess.py:42 -- smallest supported width whose capacity fits."""
    if override is not None:
        if override not in SUPPORTED_WIDTHS:
            raise ValueError(
                f"unsupported degree width {override}; choose one of {SUPPORTED_WIDTHS}")
        if max_degree > width_capacity(override):
            raise ValueError(f"max degree {max_degree} does not fit degree width {override}")
        return override
    for width in SUPPORTED_WIDTHS:
        if max_degree <= width_capacity(width):
            return width
    raise ValueError(f"max degree {max_degree} exceeds every supported width")


class LazyForced:
    """The root reduction's forced ids, left on the device with the reduced
    graph (vcg_graph_forced) and downloaded on first use: the solve path
    only needs their count.  Behaves like the int32 array it stands for."""

    def __init__(self, graph: StaticGraph, count: int):
        self._graph = graph
        self._count = count
        self._arr = None

    def _get(self) -> np.ndarray:
        if self._arr is None:
            out = np.empty(max(self._count, 1), dtype=np.int32)
            cnt = C.c_int64()
            _lib.check(_lib.lib.vcg_graph_forced(self._graph.device().handle, out.ctypes.data,
                                                 C.byref(cnt)))
            self._arr = out[: cnt.value]
        return self._arr

    def __len__(self) -> int:
        return self._count

    def __array__(self, dtype=None, copy=None):
        a = self._get()
        return a if dtype is None else a.astype(dtype)

    def __getitem__(self, i):
        return self._get()[i]

    def __iter__(self):
        return iter(self._get())

    def tolist(self) -> list:
        return self._get().tolist()

    @property
    def dtype(self):
        return np.dtype(np.int32)

    @property
    def shape(self):
        return (self._count,)

    def __repr__(self) -> str:
        return f"LazyForced({self._count} ids on the device)"


@dataclass
class Preprocessed:
    """preprocess.py:61 -- result of the root reduction pass."""

    graph: StaticGraph
    vertex_map: np.ndarray  # reduced id -> original id
    forced_ids: np.ndarray  # int32, original ids forced into the cover (or LazyForced)
    greedy_original: int
    greedy_reduced: int
    width: int
    rule_counts: dict[str, int] = field(default_factory=dict)
    seconds: dict[str, float] = field(default_factory=dict)
    kernel: dict = field(default_factory=dict)  # rule kernels: device ms, launches, scans, kind
    # lazy_greedy: the smallest greedy_original under which the speculative
    # reduction equals the reference's (-1: no speculation); see solve()
    spec_need: int = -1

    @property
    def forced(self) -> list[int]:
        """The reference's ``forced`` list (built on first access: a 1M-vertex
        root reduction forces ~10^5 vertices, and the solve path only needs
        their count)."""
        cached = self.__dict__.get("_forced_list")
        if cached is None:
            cached = self.forced_ids.tolist()
            self.__dict__["_forced_list"] = cached
        return cached

    @property
    def forced_count(self) -> int:
        return len(self.forced_ids)


def root_reduce(g: StaticGraph, enabled: bool = True, crown: bool = True,
                bound: int | None = None, width_override: int | None = None,
                need_greedy_original: bool = True, ordered: bool = True,
                lazy_greedy: bool = False, speculate: bool = True,
                lazy_forced: bool = False) -> Preprocessed:
    """preprocess.py:77 root_reduce on the device.

    ``need_greedy_original=False`` (used by PVC solves, where the bound is k)
    skips the greedy cover of the input graph; ``greedy_original`` is then -1.
    ``ordered=False`` (the solve path) returns ``forced`` in index order
    instead of the reference's forcing order -- same set, same rule counts --
    so the device can run the fused order-free sweeps on chip.
    ``lazy_greedy=True`` (the MVC solve path) skips the greedy cover of the
    input: ``greedy_original`` is then -1, the search starts from
    ``greedy_reduced`` (achieved) and ``spec_need`` says which greedy value
    the speculative reduction assumed (solve() certifies it against the
    optimum).  ``speculate=False`` runs the rules with the real bound.
    ``lazy_forced=True`` (the solve path) leaves the forced ids on the device
    until first use (``forced_ids`` is then a LazyForced)."""
    n = g.num_vertices
    info = _lib.Preprocessed_t()
    forced = None if lazy_forced else np.empty(max(n, 1), dtype=np.int32)  # written by the library
    vmap = np.empty(max(n, 1), dtype=np.int64)
    h = C.c_void_p()
    _lib.check(_lib.lib.vcg_root_reduce(
        g.device().handle,
        (1 if enabled else 0) | (0 if ordered else 2) | (4 if lazy_greedy else 0)
        | (0 if speculate else 8), int(crown),
        0 if bound is None else (2 if need_greedy_original else 1),
        int(bound) if bound is not None else 0, C.byref(info),
        None if forced is None else forced.ctypes.data, vmap.ctypes.data, C.byref(h)))
    reduced = StaticGraph.from_device(DeviceGraph(h.value))
    forced_ids = (LazyForced(reduced, int(info.forced_count)) if forced is None
                  else forced[: info.forced_count])
    md = int(info.max_degree_reduced)
    return Preprocessed(
        graph=reduced,
        vertex_map=vmap[: info.n_reduced].copy(),
        forced_ids=forced_ids,
        greedy_original=int(info.greedy_original),
        greedy_reduced=int(info.greedy_reduced),
        width=select_width(md, width_override),
        rule_counts=dict(zip(ROOT_RULE_KEYS, (int(x) for x in info.rule_counts))),
        seconds={"device_reduce": info.seconds[0], "crown": info.seconds[1],
                 "compaction": info.seconds[2]},
        kernel={"ms": info.kernel_ms, "launches": int(info.kernel_launches),
                "scans": int(info.kernel_scans), "sweeps": int(info.kernel_sweeps),
                "walked": int(info.kernel_walked), "barriers": int(info.kernel_barriers),
                "kind": ("none", "block_smem", "block_hbm", "grid",
                         "frontier")[int(info.kernel_kind)]},
        spec_need=int(info.spec_need) if lazy_greedy else -1,
    )
