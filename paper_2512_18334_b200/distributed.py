"""Multi-GPU solve of ONE instance: root subtrees self-scheduled across ranks,
with the best bound and termination exchanged while the searches run.

One process per GPU (torch.distributed; NCCL or gloo for the final
reductions).  Every rank runs the same deterministic root pipeline
(``root_reduce``) and the same breadth-first expansion of the root's search
tree (``vcg_expand``, one device block, the reference's node semantics),
which yields open subtrees that partition the remaining search:

    MVC = min(best, min_i(S_i + MVC(subtree_i)))

Load balance (engine.py:245-273 take/steal, :413 offload -- here across
processes): subtrees are not dealt statically; an idle rank takes the next
one from a shared ticket counter (an atomic ``add`` on the process group's
c10d store), largest residual first (LPT), so a rank stuck in a deep subtree
never holds up the others and the ranks finish within one short subtree of
each other.

Bound and termination propagation (engine.py:453-495 across processes),
default ``exchange="peer"``: the global best cover size and the PVC stop
flag are two device words on rank 0's GPU, mapped into every rank by CUDA
IPC (NVLink peer memory across GPUs).  Every running search kernel polls
them (block loop and warp-tier loop), lowers its subtree's root bound to
global best - S_i, and publishes its own covers (+ S_i) and a PVC answer with
system-scope atomics -- no host in the loop.  Fallback ``exchange="store"``
(a rank that cannot map the words): the best is a compare-and-set minimum
in the c10d store, relayed to each running kernel by a host thread through
a ``vcg_exchange`` (device words read and written by DMA on the copy
engines).  Either way a PVC answer stops the ticket loop everywhere.

A subtree whose residual graph is disconnected is solved by the
component-aware search itself.  Reference behaviour replaced: engine.py:200
``_Engine.run`` (threads over one shared worklist); the answer and the
result format are those of ``engine.solve`` (engine.py:561).
"""

from __future__ import annotations

import ctypes as C
import itertools
import threading
import time
from dataclasses import dataclass

import numpy as np

from .engine import RULE_KEYS, SolveResult, SolverConfig, Stats


@dataclass
class Subtrees:
    S: np.ndarray        # cover size so far of each open subtree
    deg: np.ndarray      # [count, n] residual degrees (int32)
    best: int            # best cover found by the expansion's own leaves
    nodes: int           # tree nodes the expansion processed


@dataclass
class SubtreeResult:
    best: int | None     # subtree cover size below the bound, if one was found
    nodes: int
    found: bool          # PVC: the subtree reached its budget
    hist: dict
    timed_out: bool


# ------------------------------------------------------------ coordination --

_CALLS = itertools.count()


class Coordinator:
    """Global best, PVC stop and the subtree ticket counter of one distributed
    solve: the process group's c10d store when there is one (atomic ``add``,
    ``compare_set``), else process-local state."""

    def __init__(self, store=None, prefix: str = "vcg/"):
        self.store = store
        self.p = prefix
        # one store request at a time per process: the ticket loop and the
        # exchanger thread share the client connection
        self._lock = threading.Lock()
        self._best = None
        self._ticket = 0
        self._found = False

    def ticket(self) -> int:
        with self._lock:
            if self.store is not None:
                return int(self.store.add(self.p + "ticket", 1)) - 1
            t = self._ticket
            self._ticket += 1
            return t

    def offer(self, v: int) -> None:
        """best = min(best, v)."""
        v = int(v)
        with self._lock:
            if self._best is not None and v >= self._best:
                return  # this process already knows a cover at least as small
            if self.store is None:
                self._best = v
                return
            key, want = self.p + "best", str(v).encode()
            cur = self.store.compare_set(key, "", want)  # sets an absent key
            while cur != want and int(cur) > v:
                cur = self.store.compare_set(key, cur, want)
            self._best = min(v, int(cur))

    def best(self) -> int:
        with self._lock:
            if self.store is None:
                return self._best
            b = int(self.store.get(self.p + "best"))
            self._best = b if self._best is None else min(self._best, b)
            return b

    def set_found(self) -> None:
        with self._lock:
            if self.store is None:
                self._found = True
            else:
                self.store.set(self.p + "found", "1")
                self._found = True

    def found(self) -> bool:
        with self._lock:
            if self.store is None or self._found:
                return self._found
            self._found = self.store.check([self.p + "found"])
            return self._found


def _dist():
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return None
    return dist if dist.is_available() and dist.is_initialized() else None


def _allreduce(values, op, group=None):
    """All-reduce a small int64 vector (MIN, MAX or SUM) across the group."""
    dist = _dist()
    if dist is None:
        return list(values)
    import torch

    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    t = torch.tensor(list(values), dtype=torch.int64, device=device)
    ops = {"min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM}
    dist.all_reduce(t, op=ops[op], group=group)
    return [int(x) for x in t.cpu().tolist()]


class PeerCoordinator(Coordinator):
    """The global best and PVC stop as device words (vcg_peer): allocated on
    rank 0's GPU, mapped into every other rank by CUDA IPC -- NVLink peer
    memory across GPUs -- so the running search kernels read the global bound
    and publish their covers / the PVC stop themselves with system-scope
    atomics (no host thread relaying).  Tickets stay on the store."""

    def __init__(self, store, prefix, peer):
        super().__init__(store, prefix)
        self.peer = peer  # vcg_peer* (c_void_p)

    def offer(self, v: int) -> None:
        from . import _lib

        v = int(v)
        with self._lock:
            if self._best is not None and v >= self._best:
                return
            _lib.check(_lib.lib.vcg_peer_offer(self.peer, v, 0))
            self._best = v

    def _read(self):
        from . import _lib

        b, st = C.c_int64(), C.c_int()
        _lib.check(_lib.lib.vcg_peer_read(self.peer, C.byref(b), C.byref(st)))
        return int(b.value), bool(st.value)

    def best(self) -> int:
        with self._lock:
            b = self._read()[0]
            self._best = b if self._best is None else min(self._best, b)
            return b

    def set_found(self) -> None:
        from . import _lib

        with self._lock:
            _lib.check(_lib.lib.vcg_peer_offer(self.peer, -1, 1))
            self._found = True

    def found(self) -> bool:
        with self._lock:
            if not self._found:
                self._found = self._read()[1]
            return self._found


def _open_peer(dist, group, rank):
    """Rank 0 creates the peer words, every rank maps them; None unless every
    rank succeeded (the store exchange is the fallback)."""
    from . import _lib

    h = C.c_void_p()
    blob = [None]
    ok = 1
    if rank == 0:
        handle = (C.c_char * 64)()
        ok = int(_lib.lib.vcg_peer_create(C.byref(h)) == 0 and
                 _lib.lib.vcg_peer_handle(h, handle) == 0)
        blob[0] = bytes(handle) if ok else None
    dist.broadcast_object_list(blob, src=dist.get_global_rank(group, 0) if group else 0,
                               group=group)
    if rank != 0:
        ok = int(blob[0] is not None and
                 _lib.lib.vcg_peer_open(C.create_string_buffer(blob[0], 64), C.byref(h)) == 0)
    if _allreduce([ok], "min", group)[0]:
        return h
    if h.value:
        _lib.lib.vcg_peer_destroy(h)
    return None


def _close_peer(coord, dist, group, rank):
    from . import _lib

    if not isinstance(coord, PeerCoordinator):
        return
    if rank != 0:  # mappings are closed before the owner frees the words
        _lib.lib.vcg_peer_destroy(coord.peer)
    dist.barrier(group=group)
    if rank == 0:
        _lib.lib.vcg_peer_destroy(coord.peer)


def _coordinator(group, exchange="store"):
    dist = _dist()
    call = next(_CALLS)  # every rank makes the same sequence of calls
    if dist is None or dist.get_world_size(group) == 1:
        return Coordinator()
    from torch.distributed import distributed_c10d as c10d

    store, prefix = c10d._get_default_store(), f"vcg/solve{call}/"
    if exchange == "peer":
        peer = _open_peer(dist, group, dist.get_rank(group))
        if peer is not None:
            return PeerCoordinator(store, prefix, peer)
    return Coordinator(store, prefix)


# ----------------------------------------------------------------- backend --

class GpuBackend:
    """The product path: root pipeline, expansion and subtree search on the GPU."""

    def __init__(self):
        self._xch = {}

    def root_reduce(self, g, cfg):
        from .preprocess import root_reduce

        bound = cfg.k if cfg.mode == "pvc" else None
        return root_reduce(g, enabled=cfg.use_root_reduce, crown=cfg.use_crown, bound=bound,
                           width_override=cfg.width, need_greedy_original=bound is None,
                           ordered=False)

    def expand(self, rg, cfg, best_init, target) -> Subtrees:
        from . import _lib

        n = rg.num_vertices
        cap = 2 * target + 8
        sub_S = np.zeros(cap, dtype=np.int32)
        sub_deg = np.zeros((cap, n), dtype=np.int32)
        ec = _lib.ExpandConfig_t(target, best_init, int(cfg.use_components), int(cfg.use_bounds))
        er = _lib.ExpandResult_t()
        _lib.check(_lib.lib.vcg_expand(rg.device().handle, C.byref(ec), C.byref(er),
                                       sub_S.ctypes.data, sub_deg.ctypes.data, cap))
        k = int(er.count)
        return Subtrees(sub_S[:k].copy(), sub_deg[:k].copy(), int(er.best), int(er.nodes))

    def _exchange(self):
        from . import _lib

        dev = _lib.get_device()
        x = self._xch.get(dev)
        if x is None:
            h = C.c_void_p()
            _lib.check(_lib.lib.vcg_exchange_create(C.byref(h)))
            x = self._xch[dev] = h
        return x

    def search_subtree(self, rg, cfg, width, root_deg, bound, k_red, coord, S_i,
                       timeout=None) -> SubtreeResult:
        """Search one subtree for a cover < bound, exchanging bounds with the
        other ranks through ``coord`` while the kernel runs."""
        from dataclasses import replace

        from . import _lib
        from .engine import run_search

        deg = np.ascontiguousarray(root_deg, dtype=np.int32)
        sub_cfg = replace(cfg, timeout=timeout)
        if isinstance(coord, PeerCoordinator):
            # the kernel itself reads / updates the global words
            def peer_hook(sc):
                sc.root_deg = deg.ctypes.data
                sc.peer = coord.peer
                sc.peer_offset = S_i

            res, hist, _ = run_search(rg, sub_cfg, width, bound, False, k_red,
                                      config_hook=peer_hook)
            improved = int(res.best) < bound and bool(res.best_achieved)
            return SubtreeResult(int(res.best) if improved else None,
                                 int(res.tree_nodes_visited), bool(res.found), hist,
                                 bool(res.timed_out))
        x = self._exchange()
        _lib.check(_lib.lib.vcg_exchange_reset(x))
        _lib.check(_lib.lib.vcg_exchange_post(x, int(bound), int(coord.found())))
        dev = _lib.get_device()
        done = threading.Event()

        def exchanger():  # the host side of the in-flight exchange
            _lib.set_device(dev)
            lb = C.c_int64()
            posted = (int(bound), 0)
            while not done.wait(0.001):
                _lib.check(_lib.lib.vcg_exchange_peek(x, C.byref(lb)))
                if lb.value < (1 << 31) - 1:
                    coord.offer(S_i + lb.value)
                now = (coord.best() - S_i, int(coord.found()))
                if now != posted:  # post only news (a DMA and a stream sync)
                    _lib.check(_lib.lib.vcg_exchange_post(x, now[0], now[1]))
                    posted = now

        def hook(sc):
            sc.root_deg = deg.ctypes.data
            sc.exchange = x

        t = threading.Thread(target=exchanger, daemon=True)
        t.start()
        try:
            res, hist, _ = run_search(rg, sub_cfg, width, bound, False, k_red, config_hook=hook)
        finally:
            done.set()
            t.join()
        improved = int(res.best) < bound and bool(res.best_achieved)
        return SubtreeResult(int(res.best) if improved else None, int(res.tree_nodes_visited),
                             bool(res.found), hist, bool(res.timed_out))


# ------------------------------------------------------------------- solve --

def solve_distributed(g, config: SolverConfig | None = None, group=None,
                      subtrees_per_rank: int = 8, backend=None,
                      exchange: str = "auto") -> SolveResult:
    """engine.py:561 solve, one instance across every rank of ``group``.

    ``exchange``: "peer" -- the global best / stop as device words every
    rank's kernels update directly (CUDA IPC / NVLink peer memory);
    "store" -- the c10d store, relayed to each running kernel by a host
    thread through a vcg_exchange; "auto" -- peer for the GPU backend,
    falling back to the store when a rank cannot map the words."""
    cfg = config if config is not None else SolverConfig()
    cfg.validate()
    if cfg.record_cover:
        raise ValueError("record_cover is not supported by solve_distributed; use solve()")
    be = backend if backend is not None else GpuBackend()
    dist = _dist()
    rank = dist.get_rank(group) if dist else 0
    world = dist.get_world_size(group) if dist else 1
    if exchange not in ("auto", "peer", "store"):
        raise ValueError(f"unknown exchange {exchange!r}")
    use_peer = exchange == "peer" or (exchange == "auto" and isinstance(be, GpuBackend))
    t_start = time.perf_counter()
    deadline = None if cfg.timeout is None else t_start + cfg.timeout

    stats = Stats()
    stats.rule_counts = dict.fromkeys(RULE_KEYS, 0)
    stats.root_vertices_before = g.num_vertices
    stats.phase_seconds = {"root_reduce": 0.0, "search": 0.0, "reconstruct": 0.0}
    pre = be.root_reduce(g, cfg)
    stats.phase_seconds["root_reduce"] = time.perf_counter() - t_start
    for key, val in pre.rule_counts.items():
        stats.rule_counts[key] = stats.rule_counts.get(key, 0) + val
    stats.root_vertices_after = pre.graph.num_vertices
    stats.degree_width = pre.width
    rg = pre.graph
    result = SolveResult(cover_size=None, found=False, exact=True, cover=None, stats=stats,
                         mode=cfg.mode, k=cfg.k, forced_ids=pre.forced_ids)
    if cfg.mode == "pvc" and pre.forced_count > cfg.k:
        return result
    if rg.num_edges == 0:
        result.found = True
        result.cover_size = pre.forced_count
        return result
    k_red = cfg.k - pre.forced_count if cfg.mode == "pvc" else None
    if cfg.mode == "pvc":
        if pre.greedy_reduced <= k_red:
            result.found = True
            result.cover_size = pre.forced_count + pre.greedy_reduced
            return result
        best_init = min(pre.greedy_reduced, k_red + 1)
    else:
        best_init = max(1, min(pre.greedy_reduced, pre.greedy_original - pre.forced_count))

    coord = _coordinator(group, "peer" if use_peer else "store")
    t1 = time.perf_counter()
    sub = be.expand(rg, cfg, best_init, max(1, subtrees_per_rank * world))
    best0 = min(best_init, sub.best)
    # a subtree without edges is a leaf cover of S_i vertices, not a search
    edge_free = sub.deg.sum(axis=1) == 0 if len(sub.S) else np.zeros(0, dtype=bool)
    if edge_free.any():
        best0 = min(best0, int(sub.S[edge_free].min()))
    coord.offer(best0)
    if k_red is not None and best0 <= k_red:
        coord.set_found()
    # tickets in longest-processing-time order: the subtrees with the most
    # residual edges first (the same order on every rank), so the last
    # tickets are the short ones and the ranks finish together
    cand = np.nonzero(~edge_free)[0]
    order = cand[np.argsort(-sub.deg[cand].sum(axis=1), kind="stable")] if len(cand) else cand
    nodes = sub.nodes if rank == 0 else 0
    hist: dict[int, int] = {}
    timed_out = False
    while not coord.found():
        t = coord.ticket()
        if t >= len(order):
            break
        remaining = None
        if deadline is not None:
            remaining = deadline - time.perf_counter()
            if remaining <= 0:
                timed_out = True
                break
        i = int(order[t])
        S_i = int(sub.S[i])
        bound = coord.best() - S_i
        if bound < 1:  # a subtree with edges needs >= 1 more vertex: pruned
            continue
        kr = None if k_red is None else k_red - S_i
        r = be.search_subtree(rg, cfg, pre.width, sub.deg[i], bound, kr, coord, S_i,
                              timeout=remaining)
        nodes += r.nodes
        for key, c in r.hist.items():
            hist[key] = hist.get(key, 0) + c
        if r.best is not None:
            coord.offer(S_i + r.best)
        if r.found or (k_red is not None and coord.best() <= k_red):
            coord.set_found()
        timed_out = timed_out or r.timed_out
    stats.phase_seconds["search"] = time.perf_counter() - t1
    if dist is not None:
        dist.barrier(group=group)
    best = coord.best()
    nodes, = _allreduce([nodes], "sum", group)
    timed_out = bool(_allreduce([int(timed_out)], "max", group)[0])
    found = coord.found() or (k_red is not None and best <= k_red)
    if dist is not None and world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, hist, group=group)
        hist = {}
        for h in parts:
            for key, c in h.items():
                hist[key] = hist.get(key, 0) + c
        _close_peer(coord, dist, group, rank)
    stats.tree_nodes_visited = nodes
    stats.components_per_branch = hist
    if cfg.mode == "mvc":
        result.found = True
        result.cover_size = pre.forced_count + best
        result.exact = not timed_out
    else:
        result.found = found
        result.exact = found or not timed_out
        result.cover_size = pre.forced_count + best if found else None
    return result


__all__ = ["solve_distributed", "GpuBackend", "Subtrees", "SubtreeResult", "Coordinator",
           "PeerCoordinator"]
