"""GPU parity of Residual Splash (rs_frontier, schedulers.cpp:169-192;
build_splash :136-167; apply_splash_frontier :253-291).

Three layers, mirroring the reference's test_schedulers.cpp splash cases:
  * the device's parallel greedy claiming equals the sequential walk of
    rs_frontier run on the device's own (fp32) vertex residuals -- exact;
  * the same splashes applied by both engines keep the messages within 1e-5;
  * full runs converge like the reference with marginals within 1e-4.
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.helpers import Stream, both, oracle_config, path_graph, random_graph

pytestmark = pytest.mark.gpu

MSG_TOL = 1e-5
BELIEF_TOL = 1e-4


def _sequential_rs(off, adj, src, vres, p, h):
    """rs_frontier + build_splash (schedulers.cpp:136-192), pure Python."""
    V = len(vres)
    k = max(1, int(np.floor(p * V + 0.5)))
    order = sorted(range(V), key=lambda v: (-vres[v], v))
    claimed = [None] * V
    roots, eoff, edges = [], [0], []
    for r in order:
        if len(roots) >= k:
            break
        if claimed[r] is not None:
            continue
        claimed[r] = r
        queue, visited = [(r, 0)], []
        while queue:
            v, dep = queue.pop(0)
            visited.append(v)
            if dep < h:
                for a in range(off[v], off[v + 1]):
                    w = src[adj[a]]
                    if claimed[w] is None:
                        claimed[w] = r
                        queue.append((w, dep + 1))
        for v in visited:
            edges += [int(adj[a]) ^ 1 for a in range(off[v], off[v + 1])]
        roots.append(r)
        eoff.append(len(edges))
    return roots, eoff, edges


def _topology(og):
    off, adj = og.incoming()
    a = og.arrays()
    src = np.empty(2 * a.endpoints.shape[0], np.int64)
    src[0::2] = a.endpoints[:, 0]
    src[1::2] = a.endpoints[:, 1]
    return off, adj, src


def _vertex_residuals(off, adj, r):
    V = len(off) - 1
    return [max([r[adj[a]] for a in range(off[v], off[v + 1])], default=0.0) for v in range(V)]


def _check_rs_exact(de, og, p, h):
    off, adj, src = _topology(og)
    res = de.residuals()
    vres = _vertex_residuals(off, adj, res)
    roots, eoff, edges = de.rs_frontier(p, h)
    want_roots, want_eoff, want_edges = _sequential_rs(off, adj, src, vres, p, h)
    assert list(roots) == want_roots
    assert list(eoff) == want_eoff
    assert list(edges) == want_edges
    return roots, eoff, edges


@pytest.mark.parametrize("n,c,seed,p,h", [(12, 2.5, 1, 1 / 16, 2), (16, 2.5, 7, 1 / 128, 2), (10, 3.0, 3, 0.3, 1),
                                          (9, 2.0, 5, 1.0, 0), (14, 2.5, 2, 1 / 8, 3),
                                          # deep splashes: the distance-propagation ready test (h > 8)
                                          (20, 2.5, 4, 1 / 64, 9), (24, 2.5, 6, 1 / 128, 12),
                                          (16, 2.0, 8, 1 / 32, 25)])
def test_rs_frontier_equals_sequential_walk_ising(bp, orc, n, c, seed, p, h):
    og = po.Graph.ising(orc, n, c, seed)
    a = og.arrays()
    dg = bp.PairwiseMRF.from_arrays(a.cardinalities, a.unary, a.endpoints, a.tables)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rs, p=p, splash_depth=h)
    de = bp.EngineState(dg, cfg)
    for step in range(6):
        roots, eoff, edges = _check_rs_exact(de, og, p, h)
        de.apply_splashes(roots, eoff, edges)


def test_rs_frontier_equals_sequential_walk_random_graphs(bp, orc):
    rng = Stream(orc, 77)
    for rep in range(5):
        cards, un, ed = random_graph(rng, 12 + 3 * rep, 4, 0.3)
        dg, og, ep = both(bp, orc, cards, un, ed)
        de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rs))
        de.set_endpoints(ep)
        for p, h in ((0.25, 2), (0.1, 1), (0.5, 2)):
            _check_rs_exact(de, og, p, h)


def test_deep_rs_frontier_random_graphs(bp, orc):
    rng = Stream(orc, 91)
    for rep in range(3):
        cards, un, ed = random_graph(rng, 40 + 10 * rep, 4, 0.1)
        dg, og, ep = both(bp, orc, cards, un, ed)
        de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rs))
        de.set_endpoints(ep)
        for p, h in ((0.05, 9), (0.1, 14)):
            roots, eoff, edges = _check_rs_exact(de, og, p, h)
            de.apply_splashes(roots, eoff, edges)


def test_rs_frontier_matches_reference_when_order_is_unambiguous(bp, orc):
    """Device splashes == the reference's own rs_frontier on the same state
    (holds whenever fp32 vertex residuals order like the fp64 ones)."""
    og = po.Graph.ising(orc, 12, 2.5, 4)
    a = og.arrays()
    dg = bp.PairwiseMRF.from_arrays(a.cardinalities, a.unary, a.endpoints, a.tables)
    de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rs))
    oe = po.Engine(og, po.make_config("rs"))
    roots, eoff, edges = de.rs_frontier(1 / 16, 2)
    oroots, oeoff, oedges = oe.rs_frontier(1 / 16, 2)
    assert list(roots) == list(oroots)
    assert list(eoff) == list(oeoff)
    assert list(edges) == list(oedges)


def test_splash_apply_lockstep_with_reference_splashes(bp, orc):
    """The reference's splashes applied by both engines (overlay Gauss-Seidel)."""
    for n, c, seed, p, h in ((12, 2.5, 11, 1 / 16, 2), (10, 2.0, 3, 0.2, 1)):
        og = po.Graph.ising(orc, n, c, seed)
        a = og.arrays()
        dg = bp.PairwiseMRF.from_arrays(a.cardinalities, a.unary, a.endpoints, a.tables)
        de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rs))
        oe = po.Engine(og, po.make_config("rs"))
        for t in range(15):
            roots, eoff, edges = oe.rs_frontier(p, h)
            de.apply_splashes(roots, eoff, edges)
            oe.apply_splashes(roots, eoff, edges)
            assert np.max(np.abs(de.messages() - oe.messages())) <= MSG_TOL, t
            assert np.max(np.abs(de.residuals() - oe.residuals())) <= MSG_TOL, t
            if oe.unconverged == 0:
                break


def test_splash_apply_generic_cardinalities(bp, orc):
    rng = Stream(orc, 5)
    cards, un, ed = random_graph(rng, 14, 4, 0.25)
    dg, og, ep = both(bp, orc, cards, un, ed)
    de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rs))
    de.set_endpoints(ep)
    oe = po.Engine(og, po.make_config("rs"))
    for t in range(10):
        roots, eoff, edges = oe.rs_frontier(0.2, 2)
        de.apply_splashes(roots, eoff, edges)
        oe.apply_splashes(roots, eoff, edges)
        assert np.max(np.abs(de.messages() - oe.messages())) <= MSG_TOL, t


def test_overlapping_splashes_rejected(bp, orc):
    cards, un, ed = path_graph(6)
    dg, og, ep = both(bp, orc, cards, un, ed)
    de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rs))
    with pytest.raises(bp.ModelError):
        de.apply_splashes([0, 1], [0, 2, 3], [1, 3, 1])


def test_splash_depth_zero_equals_apply_frontier(bp, orc):
    """h = 0 splash == apply_frontier of its edges (test_schedulers.cpp:336-351)."""
    og = po.Graph.ising(orc, 8, 2.5, 9)
    a = og.arrays()
    dg = bp.PairwiseMRF.from_arrays(a.cardinalities, a.unary, a.endpoints, a.tables)
    d1 = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rs))
    d2 = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rs))
    roots, eoff, edges = d1.rs_frontier(1 / 16, 0)
    d1.apply_splashes(roots, eoff, edges)
    d2.apply_frontier(np.sort(edges))
    assert np.max(np.abs(d1.messages() - d2.messages())) <= 1e-6


@pytest.mark.parametrize("n,c,seed,p,h", [(10, 2.0, 1, 1 / 16, 2), (20, 2.0, 2, 1 / 32, 2), (16, 2.5, 3, 1 / 8, 1),
                                          (16, 2.0, 5, 1 / 64, 10)])
def test_rs_run_matches_reference(bp, orc, n, c, seed, p, h):
    g = bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed))
    og = po.Graph.ising(orc, n, c, seed)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rs, p=p, splash_depth=h, max_iterations=200000)
    r = bp.run(g, cfg)
    o = po.run(og, oracle_config(cfg))
    assert o.converged and r.converged  # instances chosen to converge
    assert np.max(np.abs(r.beliefs.values - o.beliefs)) <= BELIEF_TOL
    # frontier_size = splash edges; messages_updated_total = its sum (schedulers.cpp:335,343)
    assert sum(t.frontier_size for t in r.trace) == r.messages_updated_total
    assert len(r.trace) == r.iterations


def test_rs_run_tree_exact(bp, orc):
    from tests.helpers import random_tree
    from tests.test_gpu_parity import _enumerate
    rng = Stream(orc, 14)
    cards, un, ed = random_tree(rng, 12, 2.0)
    dg, og, ep = both(bp, orc, cards, un, ed)
    exact = _enumerate(cards, un, ed)
    r = bp.run(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rs, epsilon=1e-8, p=0.25, max_iterations=100000))
    assert r.converged
    assert np.max(np.abs(r.beliefs.values - exact)) <= 1e-6


def test_rs_run_er_graph(bp, orc):
    """Erdos-Renyi instance (config 3 shape, small): converged marginals vs the oracle."""
    g = bp.generate_er(2000, 4000, 2.0, 3)
    og = po.Graph.er(orc, 2000, 4000, 2.0, 3)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rs, p=1 / 128, splash_depth=2, max_iterations=100000)
    r = bp.run(g, cfg)
    o = po.run(og, oracle_config(cfg))
    assert o.converged and r.converged
    assert np.max(np.abs(r.beliefs.values - o.beliefs)) <= BELIEF_TOL
