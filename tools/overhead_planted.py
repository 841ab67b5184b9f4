"""Where planted1m's time-to-solution goes: the whole solve() vs the bare
vcg_root_reduce call vs the root kernel (CUDA events / perf_counter)."""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import _lib, synth  # noqa: E402

n, off, nbr = synth.WORKLOADS["planted1m"]()
g = vc.StaticGraph(n, off, nbr)
g.device()
for _ in range(3):
    vc.solve(g)
forced = np.empty(n, dtype=np.int32)
vmap = np.empty(n, dtype=np.int64)


def ev(fn, reps=20):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        out.append((e0.elapsed_time(e1), (time.perf_counter() - t) * 1e3, r))
    return statistics.median(x[0] for x in out), statistics.median(x[1] for x in out), out[-1][2]


def bare():
    info = _lib.Preprocessed_t()
    h = C.c_void_p()
    _lib.check(_lib.lib.vcg_root_reduce(g.device().handle, 1 | 2 | 4, 1, 0, 0, C.byref(info),
                                        forced.ctypes.data, vmap.ctypes.data, C.byref(h)))
    _lib.lib.vcg_graph_destroy(h)
    return info.kernel_ms


a = ev(lambda: vc.solve(g))
b = ev(bare)
print(f"solve(): {a[0]:.3f} ms events, {a[1]:.3f} ms host; kernel {a[2].root_kernel['ms']:.3f} ms")
print(f"vcg_root_reduce bare: {b[0]:.3f} ms events, {b[1]:.3f} ms host; kernel {b[2]:.3f} ms")
