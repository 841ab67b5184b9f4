"""``vcsolver.registry`` (registry.py:1-224): the completion registry.

``Registry()`` is the reference's protocol object, backed by the search
kernel's own device registry (``vcg_registry_*``): the same HBM arena and
atomic encodings the search uses (child best as ``best * 2 + !achieved``
under atomicMin, live counters, parent sums), one protocol operation per
call -- and ``concurrent`` runs thousands of device threads through the same
operations at once, which is how the search actually exercises them.
``Registry.snapshot`` is the read-only view a solve returns
(``SolveResult.registry``).  Both give ``entry(idx)`` as the reference's
``ChildEntry`` / ``ParentEntry`` records and the reference's per-entry
quiescence / conservation diagnostics.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib

NEW_CHILD, NEW_PARENT, ATOMIC_MIN_BEST, BEST_SNAPSHOT = 0, 1, 2, 3
INC_LIVE_NODES, DEC_LIVE_NODES, ADD_TO_SUM = 4, 5, 6
INC_LIVE_COMPS, DEC_LIVE_COMPS, MARK_DISCOVERY_DONE = 7, 8, 9
FIELDS = 12  # int32 fields per entry row (include/vcgpu.h registry_out)


class RegistryProtocolError(RuntimeError):
    """registry.py:20: a live counter went negative or an entry was used
    after completion."""


@dataclass
class ChildEntry:
    """registry.py:24 ChildEntry, as read back from the device."""

    best: int
    achieved: bool
    live_nodes: int
    parent: int | None


@dataclass
class ParentEntry:
    """registry.py:44 ParentEntry, as read back from the device."""

    sum: int
    sum_achieved: bool
    live_comps: int
    ancestor: int
    initial_sum: int
    folded_total: int
    children: list[int]
    discovery_done: bool


def _decode(f, children: list[int]) -> ChildEntry | ParentEntry:
    key, live, link, kind = int(f[0]), int(f[1]), int(f[2]), int(f[3])
    if kind == 0:
        return ChildEntry(best=key >> 1, achieved=not (key & 1), live_nodes=live,
                          parent=None if link < 0 else link)
    return ParentEntry(sum=int(f[4]), sum_achieved=bool(f[5]), live_comps=live, ancestor=link,
                       initial_sum=int(f[6]), folded_total=int(f[7]), children=children,
                       discovery_done=bool(f[10]))


_PROTOCOL_TEXT = {
    INC_LIVE_NODES: "live-node increment on a completed entry",
    DEC_LIVE_NODES: "live-node count went negative",
    INC_LIVE_COMPS: "component increment on a finalized entry",
    DEC_LIVE_COMPS: "component count went negative",
}


class Registry:
    """registry.py:79 Registry on the device (capacity: arena entries)."""

    def __init__(self, capacity: int = 1 << 16):
        h = C.c_void_p()
        _lib.check(_lib.lib.vcg_registry_create(int(capacity), C.byref(h)))
        self._h = h.value
        self._rows = None
        self._count = None
        self._cache = None
        self._finalizer = weakref.finalize(self, _lib.lib.vcg_registry_destroy, self._h)

    @classmethod
    def snapshot(cls, count: int, raw: np.ndarray | None = None) -> "Registry":
        """A solve's registry as copied back from HBM (search layout:
        children of a parent are the contiguous [first_child, +nchild)); the
        entries are only known when the solve read them back
        (``check_registry=True`` or ``deterministic=True``)."""
        self = cls.__new__(cls)
        self._h = None
        self._count = count
        self._rows = None if raw is None else np.asarray(raw).reshape(-1, FIELDS)[:count]
        self._cache = None
        return self

    # -- reading ------------------------------------------------------------

    def _table(self) -> np.ndarray:
        if self._h is None:
            if self._rows is None:
                raise RuntimeError("solve with check_registry=True (or deterministic=True) to "
                                   "read the registry entries back from the device")
            return self._rows
        n = _lib.I64()
        _lib.check(_lib.lib.vcg_registry_download(self._h, None, 0, C.byref(n)))
        rows = np.zeros((max(n.value, 1), FIELDS), dtype=np.int32)
        _lib.check(_lib.lib.vcg_registry_download(self._h, rows.ctypes.data, n.value,
                                                  C.byref(n)))
        return rows[:n.value]

    def _children(self, rows: np.ndarray, i: int) -> list[int]:
        if self._h is None:  # search layout
            return list(range(int(rows[i, 8]), int(rows[i, 8]) + int(rows[i, 9])))
        # protocol object: children in registration order = index order
        return [int(c) for c in np.flatnonzero((rows[:, 3] == 0) & (rows[:, 2] == i))]

    @property
    def entries(self) -> list:
        if self._cache is not None:
            return self._cache
        rows = self._table()
        out = [_decode(rows[i], self._children(rows, i) if rows[i, 3] else [])
               for i in range(len(rows))]
        if self._h is None:
            self._cache = out  # a snapshot never changes
        return out

    def __len__(self) -> int:
        if self._h is None:
            return self._count
        return int(_lib.lib.vcg_registry_size(self._h))

    @property
    def count(self) -> int:
        return len(self)

    def entry(self, idx: int):
        rows = self._table()
        if not 0 <= idx < len(rows):
            raise IndexError(idx)
        return _decode(rows[idx], self._children(rows, idx) if rows[idx, 3] else [])

    # -- protocol (registry.py:94-177) ----------------------------------------

    def _op(self, op: int, idx: int = -1, a: int = 0, b: int = 0, c: int = 0):
        if self._h is None:
            raise RuntimeError("a solve's registry snapshot is read-only")
        ret = (_lib.I64 * 2)()
        rc = _lib.lib.vcg_registry_op(self._h, op, int(idx), int(a), int(b), int(c), ret)
        if rc == 5:  # VCG_EPROTOCOL
            _lib.lib.vcg_last_error()
            raise RegistryProtocolError(f"entry {idx}: {_PROTOCOL_TEXT[op]}")
        if rc == 1 and op in (NEW_CHILD, NEW_PARENT):
            raise ValueError(_lib.lib.vcg_last_error().decode())
        if rc == 1:
            raise IndexError(_lib.lib.vcg_last_error().decode())
        _lib.check(rc)
        return int(ret[0]), int(ret[1])

    def new_child_entry(self, best_init: int, parent: int | None = None,
                        achieved: bool = True) -> int:
        return self._op(NEW_CHILD, -1, best_init, -1 if parent is None else parent,
                        int(bool(achieved)))[0]

    def new_parent_entry(self, initial_sum: int, ancestor: int) -> int:
        return self._op(NEW_PARENT, -1, initial_sum, ancestor)[0]

    def atomic_min_best(self, idx: int, candidate: int, achieved: bool) -> int:
        """registry.py:123: lower best to candidate if smaller (an equal
        achieved candidate upgrades the flag); returns the prior best."""
        return self._op(ATOMIC_MIN_BEST, idx, candidate, int(bool(achieved)))[0]

    def best_snapshot(self, idx: int) -> tuple[int, bool]:
        best, ach = self._op(BEST_SNAPSHOT, idx)
        return best, bool(ach)

    def inc_live_nodes(self, idx: int) -> int:
        return self._op(INC_LIVE_NODES, idx)[0]

    def dec_live_nodes(self, idx: int) -> int:
        return self._op(DEC_LIVE_NODES, idx)[0]

    def add_to_sum(self, idx: int, delta: int, achieved: bool, folded: bool = False) -> int:
        return self._op(ADD_TO_SUM, idx, delta, int(bool(achieved)), int(bool(folded)))[0]

    def inc_live_comps(self, idx: int) -> int:
        return self._op(INC_LIVE_COMPS, idx)[0]

    def dec_live_comps(self, idx: int) -> int:
        return self._op(DEC_LIVE_COMPS, idx)[0]

    def mark_discovery_done(self, idx: int) -> None:
        self._op(MARK_DISCOVERY_DONE, idx)

    def concurrent(self, ops, idx, a=None, b=None, rounds: int = 1) -> np.ndarray:
        """All len(idx) device threads at once: thread i runs ``rounds``
        passes of the operation sequence ``ops`` on entry idx[i] with
        arguments (a[i], b[i]); returns each thread's last result.  Raises
        RegistryProtocolError if any thread violated the protocol."""
        if self._h is None:
            raise RuntimeError("a solve's registry snapshot is read-only")
        ops = np.ascontiguousarray(np.atleast_1d(ops), dtype=np.int32)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        a = None if a is None else np.ascontiguousarray(a, dtype=np.int64)
        b = None if b is None else np.ascontiguousarray(b, dtype=np.int64)
        ret = np.zeros(max(len(idx), 1), dtype=np.int64)
        err = C.c_int(0)
        _lib.check(_lib.lib.vcg_registry_concurrent(
            self._h, ops.ctypes.data, len(ops), int(rounds), idx.ctypes.data,
            None if a is None else a.ctypes.data, None if b is None else b.ctypes.data,
            len(idx), ret.ctypes.data, C.byref(err)))
        if err.value:
            raise RegistryProtocolError(f"protocol violation {err.value} under contention")
        return ret[:len(idx)]

    # -- diagnostics (registry.py:198-224) ---------------------------------

    def quiescence_violations(self) -> list[str]:
        """registry.py:198 -- entries still holding live counts."""
        out = []
        for i, e in enumerate(self.entries):
            if isinstance(e, ChildEntry):
                if e.live_nodes != 0:
                    out.append(f"child entry {i}: live_nodes == {e.live_nodes}")
            elif e.live_comps != 0:
                out.append(f"parent entry {i}: live_comps == {e.live_comps}")
        return out

    def conservation_violations(self) -> list[str]:
        """registry.py:211 -- parents whose sum disagrees with initial +
        folded + children bests."""
        entries = self.entries
        out = []
        for i, e in enumerate(entries):
            if isinstance(e, ParentEntry):
                kids = [entries[c].best for c in e.children]
                expected = e.initial_sum + e.folded_total + sum(kids)
                if e.sum != expected:
                    out.append(f"parent entry {i}: sum {e.sum} != {expected} "
                               f"(initial {e.initial_sum} + folded {e.folded_total} "
                               f"+ children {kids})")
        return out
