"""B200-native component-aware branch-and-reduce vertex cover (MVC / PVC).

Drop-in for the solve path of the reference package ``vcsolver``
(arxiv/paper_2512_18334): same entry points and result format, with the
root reduction, compaction and the whole search running as hand-written
sm_100a CUDA kernels behind the C-ABI in ``include/vcgpu.h``.
"""

from .engine import SolveResult, SolverConfig, Stats, solve, solve_batch
from .exhaustive import brute_force_mvc
from .graph import StaticGraph, build_csr, induced_subgraph
from .preprocess import Preprocessed, greedy_bound, root_reduce, select_width

BACKEND = "cuda-sm_100a"
__version__ = "0.1.0"

__all__ = [
    "BACKEND",
    "Preprocessed",
    "SolveResult",
    "SolverConfig",
    "StaticGraph",
    "Stats",
    "brute_force_mvc",
    "build_csr",
    "greedy_bound",
    "induced_subgraph",
    "root_reduce",
    "select_width",
    "solve",
    "solve_batch",
    "__version__",
]
