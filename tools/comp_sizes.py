"""Component structure of a workload's reduced graph (root reduction output)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
import scipy.sparse.csgraph as cg  # noqa: E402

import paper_2512_18334_b200 as vc  # noqa: E402
from paper_2512_18334_b200 import synth  # noqa: E402

n, off, nbr = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "rgg2000"]()
pre = vc.root_reduce(vc.StaticGraph(n, off, nbr))
rg = pre.graph
rn = rg.num_vertices
A = sp.csr_matrix((np.ones(len(rg.neighbors)), rg.neighbors, rg.offsets), shape=(rn, rn))
k, lab = cg.connected_components(A, directed=False)
sizes = np.sort(np.bincount(lab))[::-1]
print(f"reduced n={rn} m={rg.num_edges} components={k} largest={sizes[:12].tolist()} "
      f">64: {int((sizes > 64).sum())} >128: {int((sizes > 128).sum())}")
