"""Shared fixture loading and graph builders for the test suite."""

from __future__ import annotations

import functools
import json
import os
import random

import numpy as np

from paper_2512_18334_b200.synth import csr_from_pairs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def csr(n, edges):
    """(n, offsets, neighbors) from an edge list (dedup, no self-loops)."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    return csr_from_pairs(e, n)


def random_edges(rng: random.Random, n: int, p: float):
    return [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < p]


def stats_without_time(stats: dict) -> dict:
    d = dict(stats)
    d.pop("phase_seconds", None)
    d.pop("degree_width", None)
    d["components_per_branch"] = {str(k): v for k, v in d["components_per_branch"].items()}
    return d


def assert_valid_cover(n, off, nbr, cover):
    covered = np.zeros(n, dtype=bool)
    covered[np.asarray(cover, dtype=np.int64)] = True
    heads = np.repeat(np.arange(n), np.diff(off))
    assert np.all(covered[heads] | covered[nbr]), "cover misses an edge"
