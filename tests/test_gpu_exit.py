"""Process lifecycle: a user process that imports the package (with or
without torch), solves (solve and solve_batch) and exits must exit with
status 0 -- no crash in library or CUDA-runtime teardown.

Regression test for the round-1 driver record (pytest rc 139 at interpreter
exit after every test had passed)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROG = r"""
import sys
sys.path.insert(0, {root!r})
if {torch}:
    import torch
    torch.zeros(1, device="cuda")
import paper_2512_18334_b200 as vc
from paper_2512_18334_b200 import synth
n, off, nbr = synth.er(200, 4.0, 1)
g = vc.StaticGraph(n, off, nbr)
opt = vc.solve(g).cover_size
if {batch}:
    rs = vc.solve_batch(g, [vc.SolverConfig(mode="pvc", k=opt),
                            vc.SolverConfig(mode="pvc", k=opt - 1)])
    assert rs[0].found and not rs[1].found
if {thread}:
    import threading
    t = threading.Thread(target=lambda: vc.solve(g))
    t.start(); t.join()
print("ok", opt)
"""


@pytest.mark.gpu
@pytest.mark.parametrize("torch_first", [False, True])
@pytest.mark.parametrize("batch", [False, True])
@pytest.mark.parametrize("thread", [False, True])
def test_clean_exit(torch_first, batch, thread):
    src = PROG.format(root=ROOT, torch=torch_first, batch=batch, thread=thread)
    p = subprocess.run([sys.executable, "-X", "faulthandler", "-c", src],
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, (p.returncode, p.stdout[-2000:], p.stderr[-4000:])
    assert p.stdout.startswith("ok")
