"""Multi-GPU solve of ONE instance: root-subtree partitioning across ranks.

One process per GPU (torch.distributed, NCCL over NVLink on a GPU node).
Every rank runs the deterministic root pipeline (``root_reduce``) and the
same breadth-first expansion of the root's search tree (``vcg_expand``, one
device block, the reference's node semantics), which yields open subtrees
that partition the remaining search:

    MVC = min(best, min_i(S_i + MVC(subtree_i)))

Subtrees are dealt round-robin (subtree i -> rank i mod world).  Each rank
solves its subtree of the round with the persistent search kernel, bounded
by the current global best minus S_i, then the ranks all-reduce (MIN) the
best bound -- the bound exchange that lets every rank prune with the best
cover found anywhere -- and, for PVC, stop as soon as any rank reached k
(termination propagation).  A subtree whose residual graph is disconnected
is solved by the component-aware search itself.

Reference behaviour replaced: engine.py:200 ``_Engine.run`` (threads over one
shared worklist); the answer and the result format are those of
``engine.solve`` (engine.py:561).
"""

from __future__ import annotations

import ctypes as C
import math
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


class GpuBackend:
    """The product path: root pipeline, expansion and subtree search on the GPU."""

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

    def search_subtree(self, rg, cfg, width, root_deg, bound, k_red):
        """Search one subtree for a cover < bound: (best or None, nodes, found, hist)."""
        from .engine import run_search

        deg = np.ascontiguousarray(root_deg, dtype=np.int32)

        def seed_root(sc):
            sc.root_deg = deg.ctypes.data

        res, hist, _ = run_search(rg, cfg, width, bound, False, k_red, config_hook=seed_root)
        improved = int(res.best) < bound
        return (int(res.best) if improved else None), int(res.tree_nodes_visited), \
            bool(res.found), hist


def _dist():
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return None
    return dist if dist.is_available() and dist.is_initialized() else None


def _allreduce(values, op, group=None):
    """All-reduce a small int64 vector (MIN or SUM) across the group."""
    dist = _dist()
    if dist is None:
        return list(values)
    import torch

    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    t = torch.tensor(list(values), dtype=torch.int64, device=device)
    dist.all_reduce(t, op={"min": dist.ReduceOp.MIN, "sum": dist.ReduceOp.SUM}[op], group=group)
    return [int(x) for x in t.cpu().tolist()]


def solve_distributed(g, config: SolverConfig | None = None, group=None,
                      subtrees_per_rank: int = 8, backend=None) -> SolveResult:
    """engine.py:561 solve, one instance across every rank of ``group``."""
    cfg = config if config is not None else SolverConfig()
    cfg.validate()
    be = backend if backend is not None else GpuBackend()
    dist = _dist()
    rank = dist.get_rank(group) if dist else 0
    world = dist.get_world_size(group) if dist else 1

    stats = Stats()
    stats.rule_counts = dict.fromkeys(RULE_KEYS, 0)
    stats.root_vertices_before = g.num_vertices
    stats.phase_seconds = {"root_reduce": 0.0, "search": 0.0, "reconstruct": 0.0}
    t0 = time.perf_counter()
    pre = be.root_reduce(g, cfg)
    stats.phase_seconds["root_reduce"] = time.perf_counter() - t0
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

    t1 = time.perf_counter()
    sub = be.expand(rg, cfg, best_init, max(1, subtrees_per_rank * world))
    best = min(best_init, sub.best)
    nodes = sub.nodes if rank == 0 else 0
    found = k_red is not None and best <= k_red
    count = len(sub.S)
    hist: dict[int, int] = {}
    for r in range(math.ceil(count / world) if not found else 0):
        i = r * world + rank
        local = best
        lfound = 0
        if i < count:
            bound = best - int(sub.S[i])
            if bound >= 1:
                kr = None if k_red is None else k_red - int(sub.S[i])
                got, nd, f, h = be.search_subtree(rg, cfg, pre.width, sub.deg[i], bound, kr)
                nodes += nd
                for key, c in h.items():
                    hist[key] = hist.get(key, 0) + c
                if got is not None:
                    local = min(local, int(sub.S[i]) + got)
                lfound = int(f)
        best, = _allreduce([local], "min", group)
        if k_red is not None:
            anyf, = _allreduce([lfound], "sum", group)
            if anyf or best <= k_red:
                found = True
                break
    stats.phase_seconds["search"] = time.perf_counter() - t1
    nodes, = _allreduce([nodes], "sum", group)
    stats.tree_nodes_visited = nodes
    stats.components_per_branch = hist
    if cfg.mode == "mvc":
        result.found = True
        result.cover_size = pre.forced_count + best
    else:
        result.found = found or best <= k_red
        result.cover_size = pre.forced_count + best if result.found else None
    return result


__all__ = ["solve_distributed", "GpuBackend", "Subtrees"]
