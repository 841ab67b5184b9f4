"""N>1 path of the distributed solver on CPU: world_size 2 over gloo.

The GPU pieces (root pipeline, expansion, subtree search) are replaced by an
oracle-backed backend with the same contract, so what is tested here is the
partitioning itself: identical expansion on every rank, subtrees taken from
the c10d store's ticket counter, the global best kept as a compare-and-set
minimum in the store, PVC termination through the store's stop flag, and the
combination MVC = min(best, min_i S_i + MVC(subtree_i))."""

from __future__ import annotations

import os
import socket
import types

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from helpers import csr, golden


class OracleBackend:
    def root_reduce(self, g, cfg):
        bound = cfg.k if cfg.mode == "pvc" else None
        pre = oracle.root_reduce(g.num_vertices, g.offsets, g.neighbors, bound=bound)
        rn = len(pre["vertex_map"])
        rg = types.SimpleNamespace(num_vertices=rn, num_edges=len(pre["neighbors"]) // 2,
                                   offsets=pre["offsets"], neighbors=pre["neighbors"])
        greedy_red = oracle.greedy_bound(rn, pre["offsets"], pre["neighbors"])
        return types.SimpleNamespace(graph=rg, rule_counts=pre["rule_counts"],
                                     forced=pre["forced"], forced_count=len(pre["forced"]),
                                     forced_ids=np.asarray(pre["forced"], dtype=np.int32),
                                     greedy_original=pre["greedy_original"],
                                     greedy_reduced=greedy_red, width=32)

    def expand(self, rg, cfg, best_init, target):
        """Host restatement of k_expand (capi.cu): BFS, reference node semantics."""
        from paper_2512_18334_b200.distributed import Subtrees

        n, off, nbr = rg.num_vertices, rg.offsets, rg.neighbors
        deg0 = np.diff(off).astype(np.uint32)
        live = np.nonzero(deg0)[0]
        root = (0, int(deg0.sum() // 2), int(live[0]), int(live[-1]), deg0, False)
        fifo = [root]
        best, nodes, head = best_init, 0, 0
        out = np.zeros(4 * n + 4, dtype=np.int32)
        scratch = np.zeros(n + 1, dtype=np.int32)
        while head < len(fifo) and len(fifo) - head < target:
            S0, E0, lo0, hi0, deg, split = fifo[head]
            if split:
                if all(f[5] for f in fifo[head:]):
                    break
                fifo.append(fifo[head])
                head += 1
                continue
            head += 1
            nodes += 1
            deg = deg.copy()
            r = oracle.reduce_fixpoint(deg, off, nbr, lo0, hi0, best - S0 - 1, out, 0, scratch)
            S, E, lo, hi = S0 + r[0], E0 - r[4], r[5], r[6]
            rem = best - S - 1
            if S >= best or E > rem * rem:
                continue
            if E == 0:
                best = S
                continue
            if cfg.use_components:
                vis = np.zeros(n, dtype=np.int32)
                q = np.zeros(n, dtype=np.int32)
                src = oracle.next_live_unvisited(deg, vis, 1, lo, hi)
                size = oracle.bfs_component(deg, off, nbr, vis, 1, q, src)[0]
                if size < oracle.count_live(deg, lo, hi):
                    fifo.append((S, E, lo, hi, deg, True))
                    continue
            v = oracle.select_max_degree(deg, lo, hi)
            ex = deg.copy()
            rm, ed, _ = oracle.remove_neighbors(ex, off, nbr, v, out, 0)
            fifo.append((S + rm, E - ed, lo, hi, ex, False))
            inc = deg.copy()
            e2 = oracle.remove_vertex(inc, off, nbr, v)
            fifo.append((S + 1, E - e2, lo, hi, inc, False))
        opened = fifo[head:]
        return Subtrees(np.array([f[0] for f in opened], dtype=np.int32),
                        np.array([f[4] for f in opened], dtype=np.int32).reshape(len(opened), n),
                        int(best), nodes)

    def search_subtree(self, rg, cfg, width, root_deg, bound, k_red, coord, S_i, timeout=None):
        from paper_2512_18334_b200.distributed import SubtreeResult

        off, nbr = rg.offsets, rg.neighbors
        alive = np.asarray(root_deg) > 0
        heads = np.repeat(np.arange(rg.num_vertices), np.diff(off))
        keep = alive[heads] & alive[nbr] & (heads < nbr)
        n2, o2, b2 = csr(rg.num_vertices, np.stack([heads[keep], nbr[keep]], 1))
        mvc = oracle.solve(n2, o2, b2, deterministic=True)["cover_size"]
        found = k_red is not None and mvc <= k_red
        return SubtreeResult(mvc if mvc < bound else None, 1, found, {}, False)


def _graph(case):
    n, off, nbr = csr(case["n"], case["edges"])
    return types.SimpleNamespace(num_vertices=n, offsets=off, neighbors=nbr)


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_18334_b200 import SolverConfig
    from paper_2512_18334_b200.distributed import solve_distributed

    out = []
    for case in cases:
        g = _graph(case)
        opt = case["runs"]["det"]["cover_size"]
        r = solve_distributed(g, SolverConfig(), subtrees_per_rank=3, backend=OracleBackend())
        yes = solve_distributed(g, SolverConfig(mode="pvc", k=opt), subtrees_per_rank=3,
                                backend=OracleBackend())
        no = solve_distributed(g, SolverConfig(mode="pvc", k=opt - 1), subtrees_per_rank=3,
                               backend=OracleBackend()) if opt > 0 else None
        out.append((case["name"], opt, r.cover_size, yes.found, None if no is None else no.found))
    q.put((rank, out))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_partition_matches_reference():
    cases = [c for c in golden("solve.json") if c["name"].startswith(("mid_", "twocopy_", "petersen"))]
    cases = cases[:14]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0] == results[1]  # every rank reports the same answer
    for name, opt, mvc, yes, no in results[0]:
        assert mvc == opt, name
        assert yes is True, name
        assert no in (False, None), name


def test_single_process_partition_matches_reference():
    from paper_2512_18334_b200 import SolverConfig
    from paper_2512_18334_b200.distributed import solve_distributed

    for case in golden("solve.json")[::11]:
        g = _graph(case)
        want = case["runs"]["det"]["cover_size"]
        r = solve_distributed(g, SolverConfig(), subtrees_per_rank=4, backend=OracleBackend())
        assert r.cover_size == want, case["name"]


def _ticket_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_18334_b200.distributed import _coordinator

    coord = _coordinator(None)
    coord.offer(1000 + rank)
    mine = []
    while True:
        t = coord.ticket()
        if t >= 200:
            break
        mine.append(t)
        coord.offer(900 - t)
    dist.barrier()
    q.put((rank, mine, coord.best(), coord.found()))
    dist.destroy_process_group()


def test_store_coordinator_two_ranks():
    """Tickets are handed out exactly once across ranks; the store's best is
    the minimum every rank offered."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ticket_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (m, b, f)) for r, m, b, f in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    taken = res[0][0] + res[1][0]
    assert sorted(taken) == list(range(200))
    assert res[0][1] == res[1][1] == 900 - 199
    assert res[0][2] is False
