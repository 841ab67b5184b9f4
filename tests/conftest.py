import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    # the product package loads its in-tree CUDA library at import: make sure
    # it is built (nvcc cross-compiles for sm_100a without a GPU)
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_2512_18334_b200", "csrc")])
