"""vcsolver/gpu.py -- the binding a maintainer adds to the reference package
(`vcsolver`) to run its `solve` path on a B200 through `libvcgpu.so`.

Self-contained: ctypes + numpy only (no import of paper_2512_18334_b200), so
it can be dropped into the reference tree as is.  ``solve(g, config)`` takes
the reference's ``StaticGraph`` (num_vertices / offsets / neighbors) and
``SolverConfig`` (any object with its fields) and keeps engine.py:561's phase
logic: root reduction (preprocess.py:77) -> PVC early exits -> root bound ->
search (engine.py:200) -> result, with the reference's result fields.  The
struct layouts mirror include/vcgpu.h field for field.
"""

from __future__ import annotations

import ctypes as C
import os
from types import SimpleNamespace

import numpy as np

I64, P = C.c_int64, C.c_void_p
LIB_PATH = os.environ.get("VCG_LIB", os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
    "paper_2512_18334_b200", "_build", "libvcgpu.so"))


class Preprocessed(C.Structure):  # vcg_preprocessed
    _fields_ = [
        ("n_reduced", I64), ("m_reduced", I64), ("forced_count", I64),
        ("greedy_original", I64), ("greedy_reduced", I64), ("max_degree_reduced", I64),
        ("rule_counts", I64 * 4), ("seconds", C.c_double * 3), ("kernel_ms", C.c_double),
        ("kernel_launches", I64), ("kernel_scans", I64), ("kernel_kind", I64),
        ("kernel_sweeps", I64), ("kernel_walked", I64), ("kernel_barriers", I64),
        ("spec_need", I64),
    ]


class SearchConfig(C.Structure):  # vcg_search_config
    _fields_ = [
        ("width", C.c_int), ("pvc", C.c_int), ("k_red", I64), ("best_init", I64),
        ("best_init_achieved", C.c_int), ("use_components", C.c_int), ("use_bounds", C.c_int),
        ("disable_pruning", C.c_int), ("deterministic", C.c_int), ("load_balance", C.c_int),
        ("workers", C.c_int), ("threads", C.c_int), ("worklist_threshold", I64),
        ("timeout", C.c_double), ("check_registry", C.c_int), ("record_cover", C.c_int),
        ("cover_out", P), ("root_deg", P), ("warp_limit", C.c_int), ("gpu_share", C.c_int),
        ("registry_out", P), ("registry_cap", I64), ("exchange", P), ("peer", P),
        ("peer_offset", I64),
    ]


class SearchResult(C.Structure):  # vcg_search_result
    _fields_ = [
        ("best", I64), ("best_achieved", C.c_int), ("found", C.c_int), ("timed_out", C.c_int),
        ("error", C.c_int), ("tree_nodes_visited", I64), ("component_branches", I64),
        ("worklist_pushes", I64), ("worklist_pops", I64), ("max_stack_depth", I64),
        ("rule_counts", I64 * 6), ("registry_entries", I64), ("registry_violations", I64),
        ("kernel_ms", C.c_double), ("workers", C.c_int), ("threads", C.c_int),
        ("records_loaded", I64), ("records_stored", I64), ("slot_bytes", I64),
        ("phase_cycles", I64 * 10), ("cover_size", I64), ("fix_cycles", I64 * 4),
        ("fix_count", I64 * 4), ("warp_tasks", I64), ("warp_nodes", I64), ("warp_cycles", I64),
        ("warp_limit", C.c_int), ("warp_epoch_cycles", I64), ("warp_task_max_cycles", I64),
        ("trace", I64 * 8), ("kernel_t0_ns", I64), ("kernel_t1_ns", I64),
    ]


RULES = ("degree_one", "degree_two_triangle", "high_degree", "crown", "clique_component",
         "cycle_component")

_lib = C.CDLL(LIB_PATH)
_lib.vcg_last_error.restype = C.c_char_p
_lib.vcg_graph_create.argtypes = [I64, P, P, C.POINTER(P)]
_lib.vcg_graph_destroy.argtypes = [P]
_lib.vcg_graph_num_vertices.argtypes = [P]
_lib.vcg_graph_num_vertices.restype = I64
_lib.vcg_graph_num_edges.argtypes = [P]
_lib.vcg_graph_num_edges.restype = I64
_lib.vcg_root_reduce.argtypes = [P, C.c_int, C.c_int, C.c_int, I64, C.POINTER(Preprocessed),
                                 P, P, C.POINTER(P)]
_lib.vcg_search.argtypes = [P, C.POINTER(SearchConfig), C.POINTER(SearchResult), P]


def _check(rc):
    if rc:
        raise RuntimeError(f"libvcgpu error {rc}: {_lib.vcg_last_error().decode()}")


class _Graph:
    def __init__(self, n, offsets, neighbors):
        self.off = np.ascontiguousarray(offsets, dtype=np.int64)
        self.nbr = np.ascontiguousarray(neighbors, dtype=np.int32)
        if len(self.nbr) == 0:
            self.nbr = np.zeros(1, dtype=np.int32)
        self.h = P()
        _check(_lib.vcg_graph_create(n, self.off.ctypes.data, self.nbr.ctypes.data,
                                     C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            _lib.vcg_graph_destroy(self.h)


def _width(max_degree):  # preprocess.py:42 select_width
    for w in (8, 16, 32):
        if max_degree <= (1 << w) - 2:
            return w
    raise ValueError("max degree exceeds every supported width")


def solve(g, config=None):
    """engine.py:561 solve on the GPU; the reference's result fields."""
    cfg = config if config is not None else SimpleNamespace()
    get = lambda k, d: getattr(cfg, k, d)  # noqa: E731
    mode, k = get("mode", "mvc"), get("k", None)
    n = g.num_vertices
    stats = {"tree_nodes_visited": 0, "component_branches": 0, "components_per_branch": {},
             "rule_counts": dict.fromkeys(RULES, 0), "root_vertices_before": n,
             "root_vertices_after": 0, "max_stack_depth": 0, "worklist_pushes": 0,
             "worklist_pops": 0}
    out = SimpleNamespace(cover_size=None, found=False, exact=True, stats=stats, mode=mode,
                          k=k, forced=[])
    G = _Graph(n, g.offsets, g.neighbors)
    info = Preprocessed()
    forced = np.zeros(max(n, 1), dtype=np.int32)
    vmap = np.zeros(max(n, 1), dtype=np.int64)
    red = P()
    _check(_lib.vcg_root_reduce(G.h, 1 if get("use_root_reduce", True) else 0,
                                int(get("use_crown", True)), 1 if mode == "pvc" else 0,
                                int(k or 0), C.byref(info), forced.ctypes.data,
                                vmap.ctypes.data, C.byref(red)))
    R = SimpleNamespace(h=red)
    try:
        fc = int(info.forced_count)
        out.forced = forced[:fc].tolist()
        for i, key in enumerate(RULES[:4]):
            stats["rule_counts"][key] += int(info.rule_counts[i])
        stats["root_vertices_after"] = int(info.n_reduced)
        if mode == "pvc" and fc > k:
            return out
        if info.m_reduced == 0:
            out.found, out.cover_size = True, fc
            return out
        gr = int(info.greedy_reduced)
        if mode == "pvc":
            k_red = k - fc
            if gr <= k_red:
                out.found, out.cover_size = True, fc + gr
                return out
            best_init, ach = min(gr, k_red + 1), gr <= k_red + 1
        else:
            k_red = None
            cap = int(info.greedy_original) - fc
            best_init, ach = max(1, min(gr, cap)), gr <= cap
        sc = SearchConfig(width=_width(int(info.max_degree_reduced)), pvc=int(mode == "pvc"),
                          k_red=-1 if k_red is None else k_red, best_init=best_init,
                          best_init_achieved=int(ach),
                          use_components=int(get("use_components", True)),
                          use_bounds=int(get("use_bounds", True)),
                          deterministic=int(get("deterministic", False)),
                          load_balance=int(get("load_balance", True)),
                          workers=int(get("workers", 0) if not get("deterministic", False)
                                      else 1),
                          timeout=float(get("timeout", None) or 0.0), warp_limit=-1,
                          gpu_share=1)
        res = SearchResult()
        hist = np.zeros(int(info.n_reduced) + 2, dtype=np.int64)
        _check(_lib.vcg_search(red, C.byref(sc), C.byref(res), hist.ctypes.data))
        if res.error:
            raise RuntimeError(f"search kernel reported device error {res.error}")
        stats["tree_nodes_visited"] = int(res.tree_nodes_visited)
        stats["component_branches"] = int(res.component_branches)
        stats["components_per_branch"] = {int(i): int(c) for i, c in enumerate(hist) if c}
        for i, key in enumerate(RULES):
            if key != "crown":
                stats["rule_counts"][key] += int(res.rule_counts[i])
        stats["max_stack_depth"] = int(res.max_stack_depth)
        stats["worklist_pushes"] = int(res.worklist_pushes)
        stats["worklist_pops"] = int(res.worklist_pops)
        best = int(res.best)
        if mode == "mvc":
            out.found, out.cover_size, out.exact = True, fc + best, not res.timed_out
        else:
            out.found = bool(res.found) or best <= k_red
            out.exact = out.found or not res.timed_out
            out.cover_size = fc + best if out.found else None
        return out
    finally:
        _lib.vcg_graph_destroy(R.h)
