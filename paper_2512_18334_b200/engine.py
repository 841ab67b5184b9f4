"""solve(): the reference's solve pipeline driving the B200 search kernel.

Mirrors ``vcsolver.engine`` (engine.py:45-659): same ``SolverConfig`` fields,
same ``SolveResult`` / ``Stats`` shapes and the same phase logic (root
reduction, PVC early exits, root bound initialisation, search, result
assembly).  The search itself is ``vcg_search`` -- one persistent CUDA kernel
in which every resident thread block is one worker of the reference engine.

Differences from the reference, by design:
* ``workers`` counts thread blocks; 0 (the default) fills every resident
  block slot of the GPU.  ``deterministic=True`` runs one block and replays
  the reference's single-worker schedule exactly (same statistics).
* The registry lives in HBM; ``SolveResult.registry`` is a view of it
  (``Registry``: entries, ``entry(idx)``, the reference's per-entry
  quiescence / conservation diagnostics), copied back in the parity modes.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import StaticGraph
from .preprocess import Preprocessed, greedy_bound, root_reduce
from .registry import ChildEntry, ParentEntry, Registry  # noqa: F401  (re-exported)

RULE_KEYS = (
    "degree_one",
    "degree_two_triangle",
    "high_degree",
    "crown",
    "clique_component",
    "cycle_component",
)


@dataclass
class SolverConfig:
    """engine.py:45 SolverConfig (``workers`` = GPU thread blocks, 0 = all)."""

    mode: str = "mvc"
    k: int | None = None
    workers: int = 0
    use_components: bool = True
    use_root_reduce: bool = True
    use_bounds: bool = True
    use_crown: bool = True
    load_balance: bool = True
    deterministic: bool = False
    width: int | None = None
    record_cover: bool = False
    timeout: float | None = None
    worklist_threshold: int | None = None
    threads: int = 0  # block size; 0 = chosen from the reduced graph size
    check_registry: bool = False
    # warp tier: subproblems with <= warp_limit live vertices (max 256) are
    # solved by one warp each as bitmask tasks; 0 = off, -1 = auto (128 on
    # small dense reduced graphs, else 64).  Parallel mode only
    # (deterministic / record_cover runs keep the reference's node schedule).
    warp_limit: int = -1
    # concurrent searches sharing the GPU (solve_batch sets it): each takes
    # 1/gpu_share of the resident block slots
    gpu_share: int = 1
    _disable_pruning: bool = False

    def validate(self) -> None:
        if self.mode not in ("mvc", "pvc"):
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.mode == "pvc":
            if self.k is None or self.k < 0:
                raise ValueError("pvc mode needs a non-negative k")
        if self.workers < 0:
            raise ValueError("workers must be >= 0")
        if self.timeout is not None and self.timeout <= 0:
            raise ValueError("timeout must be positive")
        if self.worklist_threshold is not None and self.worklist_threshold < 1:
            raise ValueError("worklist threshold must be >= 1")
        if not -1 <= self.warp_limit <= 256:
            raise ValueError("warp_limit must be in [-1, 256]")
        if self.gpu_share < 1:
            raise ValueError("gpu_share must be >= 1")


@dataclass
class Stats:
    """engine.py:79 Stats (Table III/IV counters)."""

    tree_nodes_visited: int = 0
    component_branches: int = 0
    components_per_branch: dict[int, int] = field(default_factory=dict)
    rule_counts: dict[str, int] = field(default_factory=dict)
    root_vertices_before: int = 0
    root_vertices_after: int = 0
    degree_width: int = 0
    max_stack_depth: int = 0
    worklist_pushes: int = 0
    worklist_pops: int = 0
    phase_seconds: dict[str, float] = field(default_factory=dict)

    def as_dict(self) -> dict:
        return {
            "tree_nodes_visited": self.tree_nodes_visited,
            "component_branches": self.component_branches,
            "components_per_branch": dict(sorted(self.components_per_branch.items())),
            "rule_counts": dict(self.rule_counts),
            "root_vertices_before": self.root_vertices_before,
            "root_vertices_after": self.root_vertices_after,
            "degree_width": self.degree_width,
            "max_stack_depth": self.max_stack_depth,
            "worklist_pushes": self.worklist_pushes,
            "worklist_pops": self.worklist_pops,
            "phase_seconds": dict(self.phase_seconds),
        }


RegistrySummary = Registry  # round-1 name


@dataclass
class SolveResult:
    """engine.py:109 SolveResult."""

    cover_size: int | None
    found: bool
    exact: bool
    cover: list[int] | None
    stats: Stats
    mode: str
    k: int | None = None
    registry: Registry | None = None
    root_index: int | None = None
    forced_ids: np.ndarray | None = None  # int32 root-forced ids (``forced`` as a list)
    warp_tasks: int = 0     # warp-tier tasks solved
    warp_nodes: int = 0     # tree nodes processed by the warp tier
    search_ms: float = 0.0  # device time of the search kernel
    blocks: int = 0         # search-kernel launch: resident blocks (workers)
    threads: int = 0        # and threads per block
    phase_cycles: dict = field(default_factory=dict)  # block time by phase (SM cycles)
    root_kernel: dict = field(default_factory=dict)   # root rule kernels (Preprocessed.kernel)
    kernel_interval_ns: tuple = (0, 0)  # device %globaltimer: search kernel start, drain end

    @property
    def forced(self) -> list[int]:
        """engine.py:120 ``forced``: original ids the root reduction forced
        (built from ``forced_ids`` on first access)."""
        cached = self.__dict__.get("_forced_list")
        if cached is None:
            cached = [] if self.forced_ids is None else self.forced_ids.tolist()
            self.__dict__["_forced_list"] = cached
        return cached


def run_search(rg: StaticGraph, cfg: SolverConfig, width: int, best_init: int,
               achieved_init: bool, k_red: int | None, record: bool = False,
               config_hook=None):
    """One vcg_search call; returns (SearchResult_t, histogram dict, cover or None).

    With ``record`` the nodes carry scoped cover bitsets and the kernel
    records witnesses, so a cover of the root's best comes back with the
    search itself (components stay on, unlike the reference's witness pass)."""
    sc = _lib.SearchConfig_t()
    sc.width = width
    sc.pvc = int(k_red is not None)
    sc.k_red = int(k_red) if k_red is not None else -1
    sc.best_init = int(best_init)
    sc.best_init_achieved = int(achieved_init)
    sc.use_components = int(cfg.use_components)
    sc.use_bounds = int(cfg.use_bounds)
    sc.disable_pruning = int(cfg._disable_pruning)
    sc.deterministic = int(cfg.deterministic)
    sc.load_balance = int(cfg.load_balance)
    sc.workers = int(cfg.workers)
    sc.threads = int(cfg.threads)
    sc.worklist_threshold = int(cfg.worklist_threshold or 0)
    sc.timeout = float(cfg.timeout or 0.0)
    sc.check_registry = int(cfg.check_registry)
    sc.warp_limit = int(cfg.warp_limit)
    sc.gpu_share = int(cfg.gpu_share)
    cover = None
    if record:
        cover = np.zeros(max(rg.num_vertices, 1), dtype=np.int32)
        sc.record_cover = 1
        sc.cover_out = cover.ctypes.data
    if config_hook is not None:
        config_hook(sc)  # e.g. seed the search with a subtree root (distributed.py)
    reg_raw = None
    if cfg.check_registry or cfg.deterministic:
        # the registry view (registry.py) is read back for the parity modes
        cap = 1 << 20 if cfg.check_registry else 1 << 16  # calloc'd: untouched pages are free
        reg_raw = np.zeros((cap, 12), dtype=np.int32)
        sc.registry_out = reg_raw.ctypes.data
        sc.registry_cap = cap
    res = _lib.SearchResult_t()
    hist = np.zeros(rg.num_vertices + 2, dtype=np.int64)
    _lib.check(_lib.lib.vcg_search(rg.device().handle, C.byref(sc), C.byref(res),
                                   hist.ctypes.data))
    if res.error:
        raise _lib.GpuError(f"search kernel reported device error {res.error}")
    h = {int(i): int(c) for i, c in enumerate(hist) if c}
    local = cover[: res.cover_size].tolist() if record and res.cover_size >= 0 else None
    count = int(res.registry_entries)
    res.registry_view = Registry.snapshot(
        count, reg_raw if reg_raw is not None and count <= len(reg_raw) else None)
    return res, h, local


def witness_cover(rg: StaticGraph, cfg: SolverConfig, width: int, target: int,
                  recorded: list[int] | None) -> list[int]:
    """engine.py:514 _witness_cover: a concrete cover of size <= target.

    Normally the search's own recorded witness; when the root's best is an
    initial bound no leaf attained (the greedy cover, or the all-forced cap),
    the greedy members or a recording PVC pass at k = target supply it."""
    if recorded is not None and len(recorded) <= target:
        return recorded
    greedy, members = greedy_bound(rg, members=True)
    if greedy <= target:
        return members
    sub = SolverConfig(mode="pvc", k=target, workers=cfg.workers, threads=cfg.threads,
                       use_components=cfg.use_components, use_bounds=cfg.use_bounds)
    res, _, local = run_search(rg, sub, width, target + 1, False, target, record=True)
    if local is None or len(local) > target:
        raise RuntimeError("cover reconstruction failed to reach the target size")
    return local


def _assemble_cover(g: StaticGraph, pre: Preprocessed, local: list[int]) -> list[int]:
    """engine.py:550 -- map a reduced-graph cover to original ids and verify it."""
    forced = np.asarray(pre.forced_ids, dtype=np.int64)
    local_orig = np.asarray(pre.vertex_map, dtype=np.int64)[np.asarray(local, dtype=np.int64)]
    cover_arr = np.union1d(forced, local_orig)
    cover = cover_arr.tolist()
    covered = np.zeros(g.num_vertices, dtype=bool)
    covered[cover_arr] = True
    heads = np.repeat(np.arange(g.num_vertices), np.diff(g.offsets))
    if not np.all(covered[heads] | covered[g.neighbors]):
        raise RuntimeError("reconstructed cover misses an edge")
    return cover


def solve(g: StaticGraph, config: SolverConfig | None = None) -> SolveResult:
    """engine.py:561 solve: MVC, or PVC's decision form with budget k.

    Parallel MVC solves skip the greedy cover of the input (the reference's
    root bound, preprocess.py:28): the root rules run with a speculative
    budget and report the smallest greedy value they assumed
    (``spec_need``).  Every cover -- the greedy one included -- has at least
    the optimum's size, so an optimum >= spec_need certifies the reduction;
    otherwise the greedy is computed, and if it is below spec_need too the
    solve reruns with the real bound.  Deterministic solves compute the
    greedy up front (the reference's search order needs its exact value)."""
    cfg = config if config is not None else SolverConfig()
    cfg.validate()
    lazy = cfg.mode == "mvc" and not cfg.deterministic and cfg.use_root_reduce
    result, pre = _solve(g, cfg, lazy)
    if lazy and pre.spec_need >= 0:
        if not (result.exact and result.cover_size >= pre.spec_need):
            if greedy_bound(g) < pre.spec_need:  # the real bound would have fired
                result, _ = _solve(g, cfg, False)
    return result


def _solve(g: StaticGraph, cfg: SolverConfig, lazy: bool):
    stats = Stats()
    stats.rule_counts = dict.fromkeys(RULE_KEYS, 0)
    stats.root_vertices_before = g.num_vertices
    stats.phase_seconds = {"root_reduce": 0.0, "search": 0.0, "reconstruct": 0.0}

    t0 = time.perf_counter()
    bound = cfg.k if cfg.mode == "pvc" else None
    pre = root_reduce(g, enabled=cfg.use_root_reduce, crown=cfg.use_crown, bound=bound,
                      width_override=cfg.width, need_greedy_original=bound is None,
                      ordered=False, lazy_greedy=lazy, lazy_forced=True)
    stats.phase_seconds["root_reduce"] = time.perf_counter() - t0
    for key, val in pre.rule_counts.items():
        stats.rule_counts[key] = stats.rule_counts.get(key, 0) + val
    stats.root_vertices_after = pre.graph.num_vertices
    stats.degree_width = pre.width
    rg = pre.graph

    result = SolveResult(cover_size=None, found=False, exact=True, cover=None, stats=stats,
                         mode=cfg.mode, k=cfg.k, forced_ids=pre.forced_ids,
                         root_kernel=dict(pre.kernel))

    if cfg.mode == "pvc" and pre.forced_count > cfg.k:
        return result, pre

    if rg.num_edges == 0:
        result.found = True
        result.cover_size = pre.forced_count
        if cfg.record_cover:
            result.cover = _assemble_cover(g, pre, [])
            result.cover_size = len(result.cover)
        return result, pre

    k_red = cfg.k - pre.forced_count if cfg.mode == "pvc" else None
    greedy_reduced = pre.greedy_reduced
    if cfg.mode == "pvc":
        if greedy_reduced <= k_red:
            result.found = True
            result.cover_size = pre.forced_count + greedy_reduced
            if cfg.record_cover:
                _, members = greedy_bound(rg, members=True)
                result.cover = _assemble_cover(g, pre, members)
                result.cover_size = len(result.cover)
            return result, pre
        best_init = min(greedy_reduced, k_red + 1)
        achieved_init = greedy_reduced <= k_red + 1
    else:
        # greedy_original == -1: skipped by the library because a matching
        # lower bound proved greedy_reduced <= greedy_original - forced
        cap = (pre.greedy_original - pre.forced_count if pre.greedy_original >= 0
               else greedy_reduced)
        best_init = max(1, min(greedy_reduced, cap))
        achieved_init = greedy_reduced <= cap

    t1 = time.perf_counter()
    res, hist, recorded = run_search(rg, cfg, pre.width, best_init, achieved_init, k_red,
                                     record=cfg.record_cover)
    stats.phase_seconds["search"] = time.perf_counter() - t1
    result.search_ms = float(res.kernel_ms)
    result.kernel_interval_ns = (int(res.kernel_t0_ns), int(res.kernel_t1_ns))
    result.blocks = int(res.workers)
    result.threads = int(res.threads)
    result.phase_cycles = dict(zip(_lib.PHASES, (int(x) for x in res.phase_cycles)))
    result.phase_cycles["warp_task_cycles"] = int(res.warp_cycles)
    result.phase_cycles["warp_epoch_cycles"] = int(res.warp_epoch_cycles)
    result.phase_cycles["warp_task_max_cycles"] = int(res.warp_task_max_cycles)
    for i, nm in enumerate(("t_node_last_ns", "t_task_first_ns", "t_task_last_ns",
                            "warp_task_max_nodes", "warp_task_max_n", "warp_fix_cycles",
                            "warp_comp_cycles", "warp_split_cycles")):
        result.phase_cycles[nm] = int(res.trace[i])
    result.warp_tasks = int(res.warp_tasks)
    result.warp_nodes = int(res.warp_nodes)
    for i, nm in enumerate(("scan", "degree_one", "triangle", "high_degree")):
        result.phase_cycles[f"fix_{nm}_cycles"] = int(res.fix_cycles[i])
        result.phase_cycles[f"fix_{nm}_count"] = int(res.fix_count[i])
    stats.tree_nodes_visited = int(res.tree_nodes_visited)
    stats.component_branches = int(res.component_branches)
    stats.components_per_branch = hist
    for i, key in enumerate(RULE_KEYS):
        if key == "crown":
            continue
        stats.rule_counts[key] = stats.rule_counts.get(key, 0) + int(res.rule_counts[i])
    stats.max_stack_depth = int(res.max_stack_depth)
    stats.worklist_pushes = int(res.worklist_pushes)
    stats.worklist_pops = int(res.worklist_pops)
    result.registry = res.registry_view
    result.root_index = 0

    best = int(res.best)
    timed_out = bool(res.timed_out)
    if cfg.mode == "mvc":
        result.found = True
        result.cover_size = pre.forced_count + best
        result.exact = not timed_out
        have_target = True
    else:
        found = bool(res.found) or best <= k_red
        result.found = found
        result.exact = found or not timed_out
        result.cover_size = pre.forced_count + best if found else None
        have_target = found

    if cfg.record_cover and have_target and result.exact:
        t2 = time.perf_counter()
        local = witness_cover(rg, cfg, pre.width, best, recorded)
        result.cover = _assemble_cover(g, pre, local)
        result.cover_size = len(result.cover)
        stats.phase_seconds["reconstruct"] = time.perf_counter() - t2
    return result, pre


def solve_batch(graphs, configs) -> list[SolveResult]:
    """Several independent solves at once on one GPU (e.g. the PVC pair
    k = opt / opt - 1): each runs on its own host thread, stream and pooled
    buffers with 1/len(configs) of the resident block slots
    (``gpu_share``), so the latency-bound searches overlap on the device.
    ``graphs`` is one StaticGraph for all configs or one per config.
    Results are those of ``solve`` (same answers; schedules differ)."""
    from concurrent.futures import ThreadPoolExecutor
    from dataclasses import replace

    configs = list(configs)
    if not isinstance(graphs, (list, tuple)):
        graphs = [graphs] * len(configs)
    if len(graphs) != len(configs):
        raise ValueError("one graph per config (or a single graph)")
    k = len(configs)
    if k <= 1:
        return [solve(graphs[0], configs[0])] if k else []
    shared = [replace(c, gpu_share=max(c.gpu_share, k)) if not c.deterministic else c
              for c in configs]
    for g in graphs:  # upload once, before the threads share the handle
        g.device()
    global _BATCH_POOL
    if _BATCH_POOL is None or _BATCH_POOL._max_workers < k:
        # long-lived workers: each keeps its stream and pooled device buffers
        # (a replaced pool's threads exit; their buffers go back to the
        # library's per-device context pool)
        if _BATCH_POOL is not None:
            _BATCH_POOL.shutdown(wait=True)
        _BATCH_POOL = ThreadPoolExecutor(max_workers=k, thread_name_prefix="vcg-batch")
    dev = _lib.get_device()  # worker threads start on device 0: adopt the caller's

    def on_device(g, c):
        _lib.set_device(dev)
        return solve(g, c)

    futs = [_BATCH_POOL.submit(on_device, g, c) for g, c in zip(graphs, shared)]
    return [f.result() for f in futs]


_BATCH_POOL = None


def _shutdown_pool() -> None:
    global _BATCH_POOL
    if _BATCH_POOL is not None:
        _BATCH_POOL.shutdown(wait=True)
        _BATCH_POOL = None


_lib.at_shutdown(_shutdown_pool)
