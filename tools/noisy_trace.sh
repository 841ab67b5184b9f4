#!/bin/bash
# Root pipeline phases of planted1m with 3x noise (the configs[3] variant
# whose rules leave a residual: crown round, device compaction, search)
VCG_TRACE=1 python -c "
import sys; sys.path.insert(0, '.')
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.planted(1_000_000, 50_000, 1, oo=1.0)
g = vc.StaticGraph(n, off, nbr)
for _ in range(3):
    r = vc.solve(g)
print(r.cover_size, r.stats.phase_seconds)
" 2>&1 | grep -E "rules round|crown round|compaction|phase|431" | tail -5
