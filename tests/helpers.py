"""Test helpers: replicas of the reference test fixtures
(/root/reference/proj/tests/support/test_helpers.hpp) driven by the same
mt19937_64 stream, and graph plumbing between the oracle and the device."""
from __future__ import annotations

import math

import numpy as np

from oracle import pyoracle as po


class Stream:
    """std::mt19937_64 + uniform_unit (rng.hpp:11-13), drawn through the oracle."""

    def __init__(self, orc, seed, chunk=1 << 16):
        self.orc, self.seed, self.chunk = orc, seed, chunk
        self.buf = np.zeros(0)
        self.pos = 0
        self.total = 0

    def unit(self) -> float:
        if self.pos >= self.buf.size:
            self.total += self.chunk
            _, u = po.mt_draws(self.orc, self.seed, self.total)
            self.buf = u[self.total - self.chunk:]
            self.pos = 0
        x = float(self.buf[self.pos])
        self.pos += 1
        return x


def random_graph(rng: Stream, n, max_card=3, extra_edge_prob=0.2):
    """bptest::random_graph (test_helpers.hpp:90-132)."""
    cards = [2 + int(rng.unit() * (max_card - 1)) for _ in range(n)]
    positive = lambda: math.exp(2.0 * rng.unit() - 1.0)  # noqa: E731
    unaries = [[positive() for _ in range(c)] for c in cards]
    edges = []

    def add(i, j):
        edges.append((i, j, [positive() for _ in range(cards[i] * cards[j])]))

    for v in range(1, n):
        add(int(rng.unit() * v), v)
    for i in range(n - 1):
        for j in range(i + 1, n):
            if rng.unit() < extra_edge_prob:
                add(i, j)
    seen, uniq = set(), []
    for e in edges:
        if (e[0], e[1]) not in seen:
            seen.add((e[0], e[1]))
            uniq.append(e)
    return cards, unaries, uniq


def random_tree(rng: Stream, n, c):
    """bptest::random_tree (test_helpers.hpp:136-155)."""
    cards = [2] * n
    unaries = []
    for _ in range(n):
        u = [rng.unit(), rng.unit()]
        for k in range(2):
            while u[k] == 0.0:
                u[k] = rng.unit()
        unaries.append(u)
    edges = []
    for v in range(1, n):
        parent = int(rng.unit() * v)
        lam = rng.unit() - 0.5
        a, d = math.exp(lam * c), math.exp(-lam * c)
        edges.append((parent, v, [a, d, d, a]))
    return cards, unaries, edges


def flatten(cards, unaries, edges):
    un = np.concatenate([np.asarray(u, np.float64) for u in unaries]) if unaries else np.zeros(0)
    ep = np.asarray([[e[0], e[1]] for e in edges], np.uint32).reshape(-1, 2)
    tb = np.concatenate([np.asarray(e[2], np.float64) for e in edges]) if edges else np.zeros(0)
    return np.asarray(cards, np.uint32), un, ep, tb


def both(bp, lib, cards, unaries, edges):
    """The same model on the device and in an oracle library."""
    c, u, ep, tb = flatten(cards, unaries, edges)
    return bp.PairwiseMRF.from_arrays(c, u, ep, tb), po.Graph.from_arrays(lib, c, u, ep, tb), ep


def path_graph(n):
    """path_graph (test_schedulers.cpp:19-27)."""
    return [2] * n, [[0.6, 0.4]] * n, [(v, v + 1, [2.0, 0.5, 0.5, 2.0]) for v in range(n - 1)]


def oracle_config(cfg):
    """bp.SchedulerConfig -> oracle config."""
    return po.make_config(int(cfg.kind), epsilon=cfg.epsilon, p=cfg.p, splash_depth=cfg.splash_depth,
                          low_p=cfg.low_p, high_p=cfg.high_p, edge_ratio_threshold=cfg.edge_ratio_threshold,
                          max_iterations=cfg.max_iterations, time_limit=cfg.time_limit, seed=cfg.seed)


def lattice_arrays(orc, rows, cols, seed, c=2.0):
    """rows x cols Ising lattice in generate_ising's edge order (per vertex the
    right edge, then the down edge, generators.cpp:37-43) as build_graph input:
    unaries (u, u') per vertex, then one lambda = u - 0.5 per edge, table
    {e^{lambda c}, e^{-lambda c}, e^{-lambda c}, e^{lambda c}}; a zero draw in a
    unary becomes 0.5.  Vectorised: any shape, including C > 512 strips."""
    V = rows * cols
    v = np.arange(V, dtype=np.int64)
    col = v % cols
    right = np.stack([v, v + 1], 1)
    down = np.stack([v, v + cols], 1)
    pairs = np.stack([right, down], 1).reshape(-1, 2)
    mask = np.stack([col + 1 < cols, v + cols < V], 1).reshape(-1)
    ep = pairs[mask].astype(np.uint32)
    E = ep.shape[0]
    _, u = po.mt_draws(orc, seed, 2 * V + E)
    unary = u[: 2 * V].copy()
    unary[unary == 0.0] = 0.5
    lam = u[2 * V:] - 0.5
    a, d = np.exp(lam * c), np.exp(-lam * c)
    tb = np.stack([a, d, d, a], 1).reshape(-1)
    return np.full(V, 2, np.uint32), unary, ep, tb
