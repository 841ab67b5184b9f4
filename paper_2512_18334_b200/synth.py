"""Seeded synthetic graphs of the shapes named in BASELINE.json's configs.

Host-side data plumbing only (numpy): every generator returns a canonical
``(num_vertices, offsets, neighbors)`` CSR triple -- sorted neighbour slices,
both directions, no self-loops or duplicates -- which is exactly the
``StaticGraph`` layout of the reference (vcsolver/graph.py:33-123).

The five workloads (BASELINE.json ``configs``):

0. ``er``       Erdos-Renyi G(n=200, avg degree 4)
1. ``rgg``      2,000-vertex random geometric graph in the unit square; the
                radius 0.027 sits just past the point where it splits into
                many components and the reference needs ~10^5 tree nodes
2. ``ba``       Barabasi-Albert preferential attachment, m=3 (2 % single-edge
                arrivals: the root reduction shatters it)
3. ``planted``  planted small cover plus noise (1M vertices; the root
                reduction solves it outright)
4. ``gnp`` / ``torus``  dense-ish G(400, 0.1) and the 60x60 torus: beyond
                exact branch-and-reduce within any budget here -- measured as
                search-tree nodes/s over a fixed time budget
"""

from __future__ import annotations

import numpy as np


def csr_from_pairs(pairs, n: int):
    """Canonicalise an (E, 2) int array into CSR (offsets int64, neighbors int32)."""
    e = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if len(e):
        if int(e.min()) < 0 or int(e.max()) >= n:
            raise ValueError("edge endpoint out of range")
        e = e[e[:, 0] != e[:, 1]]
        e = np.sort(e, axis=1)
        key = np.unique(e[:, 0] * np.int64(n) + e[:, 1])
        u = key // n
        v = key % n
        both_src = np.concatenate([u, v])
        both_dst = np.concatenate([v, u])
        order = np.lexsort((both_dst, both_src))
        src = both_src[order]
        nbr = both_dst[order].astype(np.int32)
        counts = np.bincount(src, minlength=n)
    else:
        nbr = np.zeros(0, dtype=np.int32)
        counts = np.zeros(n, dtype=np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return n, off, nbr


def er(n: int = 200, avg_degree: float = 4.0, seed: int = 1):
    rng = np.random.default_rng(seed)
    p = avg_degree / (n - 1)
    iu, ju = np.triu_indices(n, 1)
    m = rng.random(len(iu)) < p
    return csr_from_pairs(np.stack([iu[m], ju[m]], 1), n)


def gnp(n: int = 400, p: float = 0.1, seed: int = 1):
    return er(n, p * (n - 1), seed)


def rgg(n: int = 2000, radius: float = 0.027, seed: int = 1):
    """Random geometric graph: points uniform in [0,1)^2, edge iff dist < radius."""
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    # cell grid keeps this O(n) in memory for large n
    cells = max(1, int(1.0 / radius))
    cx = np.minimum((pts[:, 0] * cells).astype(np.int64), cells - 1)
    cy = np.minimum((pts[:, 1] * cells).astype(np.int64), cells - 1)
    cell = cx * cells + cy
    order = np.argsort(cell, kind="stable")
    starts = np.searchsorted(cell[order], np.arange(cells * cells + 1))
    pairs = []
    r2 = radius * radius
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            nx, ny = cx + dx, cy + dy
            ok = (nx >= 0) & (nx < cells) & (ny >= 0) & (ny < cells)
            idx = np.nonzero(ok)[0]
            nc = nx[idx] * cells + ny[idx]
            lo, hi = starts[nc], starts[nc + 1]
            cnt = hi - lo
            src = np.repeat(idx, cnt)
            off = np.repeat(lo - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
            dst = order[np.arange(cnt.sum()) + off]
            keep = src < dst
            src, dst = src[keep], dst[keep]
            d = ((pts[src] - pts[dst]) ** 2).sum(1)
            m = d < r2
            pairs.append(np.stack([src[m], dst[m]], 1))
    return csr_from_pairs(np.concatenate(pairs) if pairs else np.zeros((0, 2)), n)


def ba(n: int = 100_000, m: int = 3, seed: int = 1, pendant: float = 0.02):
    """Barabasi-Albert preferential attachment with m = 3 edges per new vertex
    ("dual BA": with probability ``pendant`` a new vertex attaches a single
    edge instead).  Pure m = 3 BA has minimum degree 3 and nothing for the
    reduction rules to start from; 2 % pendant arrivals are enough for the
    degree-one / high-degree cascade to shatter the whole graph at the root,
    which is the "heavy reduction then compaction" regime of configs[2]."""
    rng = np.random.default_rng(seed)
    src = np.empty(n * m, dtype=np.int64)
    dst = np.empty(n * m, dtype=np.int64)
    repeated = np.empty(2 * n * m + m, dtype=np.int64)
    repeated[:m] = np.arange(m)
    nrep = m
    k = 0
    ks = np.where(rng.random(n) < pendant, 1, m)
    for v in range(m, n):
        mv = int(ks[v])
        chosen = set()
        while len(chosen) < mv:
            chosen.add(int(repeated[rng.integers(nrep)]))
        for t in chosen:
            src[k] = v
            dst[k] = t
            k += 1
        c = np.fromiter(chosen, dtype=np.int64, count=mv)
        repeated[nrep:nrep + mv] = c
        repeated[nrep + mv:nrep + 2 * mv] = v
        nrep += 2 * mv
    return csr_from_pairs(np.stack([src[:k], dst[:k]], 1), n)


def planted(n: int = 1_000_000, cover: int = 50_000, seed: int = 1, cc: float = 1.0,
            oo: float = 0.3):
    """Planted cover C (|C| = cover) plus noise.

    Every vertex outside C attaches to 2 or 3 random members of C; ``cc*|C|``
    random C-C edges and ``oo*n`` random outside-outside noise edges are added,
    so the optimum exceeds |C| only through the noise.
    """
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    C, O = perm[:cover], perm[cover:]
    k = rng.choice([2, 3], size=len(O))
    src = np.repeat(O, k)
    dst = C[rng.integers(0, cover, size=len(src))]
    ne = int(cc * cover)
    a, b = C[rng.integers(0, cover, ne)], C[rng.integers(0, cover, ne)]
    no = int(oo * n)
    x, y = O[rng.integers(0, len(O), no)], O[rng.integers(0, len(O), no)]
    pairs = np.concatenate([np.stack([src, dst], 1), np.stack([a, b], 1), np.stack([x, y], 1)])
    return csr_from_pairs(pairs, n)


def torus(a: int = 60, b: int = 60):
    i, j = np.meshgrid(np.arange(a), np.arange(b), indexing="ij")
    v = (i * b + j).ravel()
    right = (i * b + (j + 1) % b).ravel()
    down = (((i + 1) % a) * b + j).ravel()
    return csr_from_pairs(np.concatenate([np.stack([v, right], 1), np.stack([v, down], 1)]), a * b)


WORKLOADS = {
    "er200": lambda: er(200, 4.0, 1),
    "rgg2000": lambda: rgg(2000, 0.027, 1),
    "ba100k": lambda: ba(100_000, 3, 1),
    "planted1m": lambda: planted(1_000_000, 50_000, 1),
    "gnp400": lambda: gnp(400, 0.1, 1),
    "torus60": lambda: torus(60, 60),
}
