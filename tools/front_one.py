"""One lazy root_reduce (frontier kernel) of a large config, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ba100k"
n, off, nbr = synth.WORKLOADS[name]()
g = vc.StaticGraph(n, off, nbr)
for _ in range(3):
    pre = vc.root_reduce(g, ordered=False, lazy_greedy=True)
print(name, pre.kernel)
