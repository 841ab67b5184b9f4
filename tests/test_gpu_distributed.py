"""The distributed solver's GPU backend on one GPU: world 1 (device expansion
of the root's search tree + subtree searches seeded from it), the in-flight
vcg_exchange of one search, and world 2 (two processes sharing cuda:0) --
the reference's answers throughout."""

from __future__ import annotations

import pytest

from helpers import csr, golden

pytestmark = pytest.mark.gpu


def test_subtree_partition_answers():
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200.distributed import solve_distributed

    for case in golden("solve.json")[::4]:
        n, off, nbr = csr(case["n"], case["edges"])
        g = vc.StaticGraph(n, off, nbr)
        want = case["runs"]["det"]["cover_size"]
        for per in (1, 5):
            r = solve_distributed(g, vc.SolverConfig(), subtrees_per_rank=per)
            assert r.cover_size == want, (case["name"], per)
        for k, exp in case["pvc"].items():
            r = solve_distributed(g, vc.SolverConfig(mode="pvc", k=int(k)), subtrees_per_rank=5)
            assert r.found == exp["found"], (case["name"], k)


@pytest.mark.parametrize("name", ["er200", "rgg2000"])
def test_subtree_partition_workloads(name):
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import synth
    from paper_2512_18334_b200.distributed import solve_distributed

    exp = golden("workloads.json")[name]
    n, off, nbr = synth.WORKLOADS[name]()
    g = vc.StaticGraph(n, off, nbr)
    for per in (4, 16):
        r = solve_distributed(g, vc.SolverConfig(), subtrees_per_rank=per)
        assert r.cover_size == exp["mvc"], per
    for k, e in exp["pvc"].items():
        r = solve_distributed(g, vc.SolverConfig(mode="pvc", k=int(k)), subtrees_per_rank=8)
        assert r.found == e["found"], k


def test_exchange_bound_stop_and_publish():
    """vcg_exchange on one search: the kernel publishes its best achieved root
    cover; an external bound at the optimum leaves nothing better to find; an
    external stop ends the search."""
    import ctypes as C

    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import _lib, synth
    from paper_2512_18334_b200.engine import run_search

    exp = golden("workloads.json")["rgg2000"]
    n, off, nbr = synth.WORKLOADS["rgg2000"]()
    g = vc.StaticGraph(n, off, nbr)
    pre = vc.root_reduce(g, ordered=False)
    rg, opt_red = pre.graph, exp["mvc"] - pre.forced_count
    x = C.c_void_p()
    _lib.check(_lib.lib.vcg_exchange_create(C.byref(x)))
    lb = C.c_int64()
    try:
        def hook(sc):
            sc.exchange = x

        cfg = vc.SolverConfig()
        _lib.check(_lib.lib.vcg_exchange_reset(x))
        res, _, _ = run_search(rg, cfg, pre.width, pre.greedy_reduced, True, None,
                               config_hook=hook)
        _lib.check(_lib.lib.vcg_exchange_peek(x, C.byref(lb)))
        assert int(res.best) == opt_red and lb.value == opt_red
        full_nodes = int(res.tree_nodes_visited)
        # a cover of opt size exists elsewhere: nothing better here
        _lib.check(_lib.lib.vcg_exchange_reset(x))
        _lib.check(_lib.lib.vcg_exchange_post(x, opt_red, 0))
        res, _, _ = run_search(rg, cfg, pre.width, pre.greedy_reduced, True, None,
                               config_hook=hook)
        assert int(res.best) == opt_red
        assert int(res.tree_nodes_visited) <= 1.1 * full_nodes  # schedule noise only
        # external stop: the kernel ends without an answer
        _lib.check(_lib.lib.vcg_exchange_reset(x))
        _lib.check(_lib.lib.vcg_exchange_post(x, -1, 1))
        res, _, _ = run_search(rg, cfg, pre.width, pre.greedy_reduced, True, None,
                               config_hook=hook)
        assert int(res.tree_nodes_visited) < full_nodes
    finally:
        _lib.lib.vcg_exchange_destroy(x)


def _gpu_worker(rank, world, port, cases, q, exchange="auto"):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), VCG_WATCHDOG_S="120")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200.distributed import solve_distributed

    out = []
    for name, n, edges, opt, pvc in cases:
        n, off, nbr = csr(n, edges)
        g = vc.StaticGraph(n, off, nbr)
        r = solve_distributed(g, vc.SolverConfig(), subtrees_per_rank=3, exchange=exchange)
        ks = {int(k): solve_distributed(g, vc.SolverConfig(mode="pvc", k=int(k)),
                                        subtrees_per_rank=3, exchange=exchange).found
              for k in pvc}
        out.append((name, r.cover_size, r.exact, ks))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["peer", "store"])
def test_two_ranks_share_one_gpu(exchange):
    """The GPU backend at world size 2 (two processes on cuda:0 over gloo):
    subtrees from the store's ticket counter; bounds and PVC stops through the
    peer words (CUDA IPC, updated by the kernels themselves) or through the
    store and each rank's vcg_exchange -- the reference's answers on every
    rank."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cases = [(c["name"], c["n"], c["edges"], c["runs"]["det"]["cover_size"],
              {k: e["found"] for k, e in c["pvc"].items()})
             for c in golden("solve.json")[::9] if c["n"] > 0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, cases, q, exchange))
             for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0] == res[1]
    for (name, _, _, opt, pvc), (name2, mvc, exact, ks) in zip(cases, res[0]):
        assert name == name2 and mvc == opt and exact, name
        assert ks == {int(k): f for k, f in pvc.items()}, name


def _peer_worker(rank, port, q):
    """Both ranks map rank 0's peer words; covers offered by each are seen by
    both, a stop set by one is seen by the other."""
    import ctypes as C
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2512_18334_b200 import distributed as D

    coord = D._coordinator(None, "peer")
    kind = type(coord).__name__
    coord.offer(100 - rank)
    dist.barrier()
    b1 = coord.best()
    if rank == 1:
        coord.set_found()
    dist.barrier()
    f = coord.found()
    D._close_peer(coord, dist, None, rank)
    q.put((rank, kind, b1, f))
    dist.destroy_process_group()


def test_peer_words_two_processes():
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (k, b, f)) for r, k, b, f in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert res[r] == ("PeerCoordinator", 99, True), res
