"""Two ranks on one GPU solve the strong instance with each exchange mode
(torchrun --nproc-per-node 2): answer and time per mode."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

dist.init_process_group("gloo")
torch.cuda.set_device(0)
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402
from paper_2512_18334_b200.distributed import solve_distributed  # noqa: E402

n, off, nbr = synth.gnp(180, 0.08, 1)
g = vc.StaticGraph(n, off, nbr)
for mode in ("peer", "store", "peer"):
    dist.barrier()
    t = time.perf_counter()
    r = solve_distributed(g, vc.SolverConfig(), subtrees_per_rank=32, exchange=mode)
    dt = time.perf_counter() - t
    yes = solve_distributed(g, vc.SolverConfig(mode="pvc", k=136), subtrees_per_rank=32,
                            exchange=mode)
    no = solve_distributed(g, vc.SolverConfig(mode="pvc", k=135), subtrees_per_rank=32,
                           exchange=mode)
    if dist.get_rank() == 0:
        print(f"{mode}: mvc={r.cover_size} exact={r.exact} nodes={r.stats.tree_nodes_visited} "
              f"{dt:.3f} s; pvc 136 {yes.found}, 135 {no.found}", flush=True)
dist.destroy_process_group()
