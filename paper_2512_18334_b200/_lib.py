"""ctypes binding of the in-tree CUDA library (``_build/libvcgpu.so``).

The C-ABI is declared in ``include/vcgpu.h``.  There is no fallback: if the
library is missing the import fails loudly, and every compute call fails
with ``VCG_ENODEV`` when no CUDA device is present.
"""

from __future__ import annotations

import atexit
import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VCG_LIB") or os.path.join(_HERE, "_build", "libvcgpu.so")
CSRC = os.path.join(_HERE, "csrc")

I64 = C.c_int64
P = C.c_void_p


class GpuError(RuntimeError):
    """A C-ABI call failed (bad input, no device, CUDA error, resource)."""


class Preprocessed_t(C.Structure):
    _fields_ = [
        ("n_reduced", I64), ("m_reduced", I64), ("forced_count", I64),
        ("greedy_original", I64), ("greedy_reduced", I64), ("max_degree_reduced", I64),
        ("rule_counts", I64 * 4), ("seconds", C.c_double * 3),
        ("kernel_ms", C.c_double), ("kernel_launches", I64), ("kernel_scans", I64),
        ("kernel_kind", I64), ("kernel_sweeps", I64), ("kernel_walked", I64), ("kernel_barriers", I64),
        ("spec_need", I64),
    ]


class SearchConfig_t(C.Structure):
    _fields_ = [
        ("width", C.c_int), ("pvc", C.c_int), ("k_red", I64), ("best_init", I64),
        ("best_init_achieved", C.c_int), ("use_components", C.c_int), ("use_bounds", C.c_int),
        ("disable_pruning", C.c_int), ("deterministic", C.c_int), ("load_balance", C.c_int),
        ("workers", C.c_int), ("threads", C.c_int), ("worklist_threshold", I64),
        ("timeout", C.c_double), ("check_registry", C.c_int), ("record_cover", C.c_int),
        ("cover_out", C.c_void_p), ("root_deg", C.c_void_p), ("warp_limit", C.c_int),
        ("gpu_share", C.c_int), ("registry_out", C.c_void_p), ("registry_cap", I64),
        ("exchange", C.c_void_p), ("peer", C.c_void_p), ("peer_offset", I64),
    ]


class ExpandConfig_t(C.Structure):
    _fields_ = [("target", I64), ("best_init", I64), ("use_components", C.c_int),
                ("use_bounds", C.c_int)]


class ExpandResult_t(C.Structure):
    _fields_ = [("count", I64), ("best", I64), ("nodes", I64)]


class SearchResult_t(C.Structure):
    _fields_ = [
        ("best", I64), ("best_achieved", C.c_int), ("found", C.c_int), ("timed_out", C.c_int),
        ("error", C.c_int), ("tree_nodes_visited", I64), ("component_branches", I64),
        ("worklist_pushes", I64), ("worklist_pops", I64), ("max_stack_depth", I64),
        ("rule_counts", I64 * 6), ("registry_entries", I64), ("registry_violations", I64),
        ("kernel_ms", C.c_double), ("workers", C.c_int), ("threads", C.c_int),
        ("records_loaded", I64), ("records_stored", I64), ("slot_bytes", I64),
        ("phase_cycles", I64 * 10), ("cover_size", I64),
        ("fix_cycles", I64 * 4), ("fix_count", I64 * 4),
        ("warp_tasks", I64), ("warp_nodes", I64), ("warp_cycles", I64), ("warp_limit", C.c_int),
        ("warp_epoch_cycles", I64), ("warp_task_max_cycles", I64), ("trace", I64 * 8),
        ("kernel_t0_ns", I64), ("kernel_t1_ns", I64),
    ]


PHASES = ("idle", "load", "reduce", "label", "split", "select", "exclude", "include",
          "registry", "other")


EXPORTS = (
    "vcg_graph_create", "vcg_graph_create_borrowed", "vcg_graph_destroy", "vcg_graph_num_vertices", "vcg_graph_num_edges",
    "vcg_graph_download", "vcg_induced_subgraph", "vcg_greedy_bound", "vcg_root_reduce",
    "vcg_search", "vcg_node_op", "vcg_last_error", "vcg_device_count", "vcg_launch_count",
    "vcg_set_device", "vcg_get_device", "vcg_expand", "vcg_shutdown", "vcg_brute_force_mvc",
    "vcg_exchange_create", "vcg_exchange_destroy", "vcg_exchange_reset", "vcg_exchange_post",
    "vcg_exchange_peek", "vcg_peer_create", "vcg_peer_handle", "vcg_peer_open",
    "vcg_peer_destroy", "vcg_peer_offer", "vcg_peer_read", "vcg_graph_forced",
    "vcg_crown_reduce", "vcg_registry_create", "vcg_registry_destroy", "vcg_registry_size",
    "vcg_registry_op", "vcg_registry_concurrent", "vcg_registry_download",
)


def build(force: bool = False) -> str:
    """Compile the library for sm_100a with nvcc (make in csrc/)."""
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    srcs.append(os.path.join(os.path.dirname(_HERE), "include", "vcgpu.h"))
    stale = force or not os.path.exists(LIB_PATH) or any(
        os.path.getmtime(s) > os.path.getmtime(LIB_PATH) for s in srcs)
    if stale:
        subprocess.check_call(["make", "-s", "-C", CSRC])
    return LIB_PATH


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build() or make -C {CSRC})")
    lib = C.CDLL(LIB_PATH)
    lib.vcg_last_error.restype = C.c_char_p
    lib.vcg_graph_num_vertices.restype = I64
    lib.vcg_graph_num_edges.restype = I64
    lib.vcg_launch_count.restype = I64
    lib.vcg_graph_create.argtypes = [I64, P, P, C.POINTER(P)]
    lib.vcg_graph_create_borrowed.argtypes = [I64, P, P, C.POINTER(P)]
    lib.vcg_graph_destroy.argtypes = [P]
    lib.vcg_graph_num_vertices.argtypes = [P]
    lib.vcg_graph_num_edges.argtypes = [P]
    lib.vcg_graph_download.argtypes = [P, P, P]
    lib.vcg_induced_subgraph.argtypes = [P, P, I64, C.POINTER(P)]
    lib.vcg_greedy_bound.argtypes = [P, P, C.POINTER(I64)]
    lib.vcg_root_reduce.argtypes = [P, C.c_int, C.c_int, C.c_int, I64,
                                    C.POINTER(Preprocessed_t), P, P, C.POINTER(P)]
    lib.vcg_search.argtypes = [P, C.POINTER(SearchConfig_t), C.POINTER(SearchResult_t), P]
    lib.vcg_expand.argtypes = [P, C.POINTER(ExpandConfig_t), C.POINTER(ExpandResult_t), P, P, I64]
    lib.vcg_node_op.argtypes = [C.c_int, C.c_int, I64, P, P, P, I64, I64, I64, I64, P, I64, P]
    lib.vcg_brute_force_mvc.argtypes = [I64, P, P, C.POINTER(I64), P]
    lib.vcg_registry_create.argtypes = [I64, C.POINTER(P)]
    lib.vcg_registry_destroy.argtypes = [P]
    lib.vcg_registry_size.argtypes = [P]
    lib.vcg_registry_size.restype = I64
    lib.vcg_registry_op.argtypes = [P, C.c_int, I64, I64, I64, I64, P]
    lib.vcg_registry_concurrent.argtypes = [P, P, C.c_int, C.c_int, P, P, P, I64, P, P]
    lib.vcg_registry_download.argtypes = [P, P, I64, C.POINTER(I64)]
    lib.vcg_crown_reduce.argtypes = [I64, P, P, P, I64, I64, P, C.POINTER(I64), P,
                                     C.POINTER(I64), C.POINTER(I64)]
    lib.vcg_exchange_create.argtypes = [C.POINTER(P)]
    lib.vcg_exchange_destroy.argtypes = [P]
    lib.vcg_exchange_reset.argtypes = [P]
    lib.vcg_exchange_post.argtypes = [P, I64, C.c_int]
    lib.vcg_exchange_peek.argtypes = [P, C.POINTER(I64)]
    lib.vcg_peer_create.argtypes = [C.POINTER(P)]
    lib.vcg_peer_handle.argtypes = [P, P]
    lib.vcg_peer_open.argtypes = [P, C.POINTER(P)]
    lib.vcg_peer_destroy.argtypes = [P]
    lib.vcg_peer_offer.argtypes = [P, I64, C.c_int]
    lib.vcg_peer_read.argtypes = [P, C.POINTER(I64), C.POINTER(C.c_int)]
    lib.vcg_graph_forced.argtypes = [P, P, C.POINTER(I64)]
    lib.vcg_shutdown.restype = None
    return lib


lib = _load()

_exit_hooks = []


def at_shutdown(fn) -> None:
    """Run ``fn`` at interpreter exit before the library stops releasing
    device memory (the solve_batch pool registers its shutdown here)."""
    _exit_hooks.append(fn)


@atexit.register
def _shutdown() -> None:
    # join the library's worker threads first, then make every later device
    # release a no-op: objects finalised after this point (and thread-local
    # contexts) leave their memory to the process exit, so no CUDA call runs
    # while the CUDA runtimes tear down
    for fn in reversed(_exit_hooks):
        try:
            fn()
        except Exception:  # noqa: BLE001 -- best effort at exit
            pass
    lib.vcg_shutdown()


def check(rc: int) -> None:
    if rc != 0:
        msg = lib.vcg_last_error().decode(errors="replace")
        raise GpuError(f"vcgpu error {rc}: {msg}")


def device_count() -> int:
    return int(lib.vcg_device_count())


def launch_count() -> int:
    """Kernels launched by the library so far in this process."""
    return int(lib.vcg_launch_count())


def set_device(device: int) -> None:
    check(lib.vcg_set_device(int(device)))


def get_device() -> int:
    """The calling thread's current CUDA device."""
    return int(lib.vcg_get_device())
