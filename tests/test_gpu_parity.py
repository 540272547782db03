"""GPU parity tests: the CUDA engine (through the C ABI) against the fp64
oracle (oracle/bp_oracle.c, pinned bitwise to the reference in
tests/test_oracle.py).

Tolerances (north_star): LBP per-iteration messages within 1e-5 abs (fp32
device vs fp64 reference); converged marginals within 1e-4."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.helpers import Stream, both, oracle_config, path_graph, random_graph, random_tree

pytestmark = pytest.mark.gpu

MSG_TOL = 1e-5
BELIEF_TOL = 1e-4


def _lockstep_lbp(bp, orc, dg, og, ep, iters, eps=1e-5):
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, epsilon=eps)
    de = bp.EngineState(dg, cfg)
    de.set_endpoints(ep)
    oe = po.Engine(og, oracle_config(cfg))
    worst = 0.0
    for t in range(iters):
        dm, om = de.messages(), oe.messages()
        worst = max(worst, float(np.max(np.abs(dm - om))) if dm.size else 0.0)
        assert worst <= MSG_TOL, (t, worst)
        # candidates and residuals of the one-step lookahead cache
        dr, orr = de.residuals(), oe.residuals()
        assert np.max(np.abs(dr - orr), initial=0.0) <= MSG_TOL
        # unconverged count: equal up to residuals within fp32 noise of eps
        near = int(np.sum(np.abs(orr - eps) < 2e-6))
        assert abs(de.unconverged_count() - oe.unconverged) <= near, (t, de.unconverged_count(), oe.unconverged)
        if oe.unconverged == 0:
            break
        de.step()
        oe.apply_frontier(oe.frontier_lbp())
    return worst


def test_lbp_lockstep_ising_binary(bp, orc):
    og = po.Graph.ising(orc, 10, 2.5, 11)
    a = og.arrays()
    dg = bp.PairwiseMRF.from_arrays(a.cardinalities, a.unary, a.endpoints, a.tables)
    _lockstep_lbp(bp, orc, dg, og, a.endpoints, 40)


def test_lbp_lockstep_random_generic(bp, orc):
    rng = Stream(orc, 202)
    for rep in range(6):
        cards, un, ed = random_graph(rng, 3 + rep % 6, 4)
        dg, og, ep = both(bp, orc, cards, un, ed)
        _lockstep_lbp(bp, orc, dg, og, ep, 25)


def test_generated_ising_equals_reference_instance(bp, orc):
    """bp_graph_generate_ising builds the same instance as generate_ising."""
    dg = bp.generate_ising(bp.IsingParams(n=9, c=2.5, seed=4))
    og = po.Graph.ising(orc, 9, 2.5, 4)
    _lockstep_lbp(bp, orc, dg, og, og.arrays().endpoints, 20)


def test_generated_chain_and_potts(bp, orc):
    dg = bp.generate_chain(bp.ChainParams(length=40, c=2.0, seed=40))
    og = po.Graph.chain(orc, 40, 2.0, 40)
    _lockstep_lbp(bp, orc, dg, og, og.arrays().endpoints, 45)
    dp = bp.generate_potts(6, 3, 2.5, 7)
    op = po.Graph.potts(orc, 6, 3, 2.5, 7)
    _lockstep_lbp(bp, orc, dp, op, op.arrays().endpoints, 20)


@pytest.mark.parametrize("n,c,seed", [(10, 1.5, 1), (20, 2.0, 3), (30, 1.0, 5)])
def test_lbp_run_matches_oracle(bp, orc, n, c, seed):
    g = bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed))
    og = po.Graph.ising(orc, n, c, seed)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=3000)
    r = bp.run(g, cfg)
    o = po.run(og, oracle_config(cfg))
    assert o.converged and r.converged  # instances chosen to converge
    assert abs(r.iterations - o.iterations) <= 1
    assert len(r.trace) == r.iterations
    assert np.max(np.abs(r.beliefs.values - o.beliefs)) <= BELIEF_TOL
    assert r.messages_updated_total == r.iterations * 2 * g.num_edges()


def test_tree_exactness_all_device_schedulers(bp, orc):
    """every scheduler solves a tree exactly (test_schedulers.cpp:418-434)."""
    rng = Stream(orc, 14)
    cards, un, ed = random_tree(rng, 12, 2.0)
    dg, og, ep = both(bp, orc, cards, un, ed)
    # exact marginals by enumeration
    exact = _enumerate(cards, un, ed)
    for kind in (bp.SchedulerKind.lbp, bp.SchedulerKind.rbp, bp.SchedulerKind.rnbp):
        cfg = bp.SchedulerConfig(kind=kind, epsilon=1e-8, p=0.25, max_iterations=1000000)
        r = bp.run(dg, cfg)
        assert r.converged, kind
        assert np.max(np.abs(r.beliefs.values - exact)) <= 1e-6, kind


def _enumerate(cards, un, ed):
    import itertools
    n = len(cards)
    marg = [np.zeros(c) for c in cards]
    for a in itertools.product(*[range(c) for c in cards]):
        w = 1.0
        for v in range(n):
            w *= un[v][a[v]]
        for i, j, t in ed:
            w *= t[a[i] * cards[j] + a[j]]
        for v in range(n):
            marg[v][a[v]] += w
    return np.concatenate([m / m.sum() for m in marg])


def test_rnbp_injected_frontier_lockstep(bp, orc):
    """Device Philox frontier applied to both engines: states stay in lockstep."""
    og = po.Graph.ising(orc, 12, 2.5, 2)
    a = og.arrays()
    dg = bp.PairwiseMRF.from_arrays(a.cardinalities, a.unary, a.endpoints, a.tables)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, seed=99)
    de = bp.EngineState(dg, cfg)
    oe = po.Engine(og, oracle_config(cfg))
    for t in range(30):
        f = de.rnbp_frontier(0.5)
        res = oe.residuals()
        # every selected edge is unconverged (filter 1), ascending order
        assert np.all(np.diff(f.astype(np.int64)) > 0)
        assert np.all(res[f] >= cfg.epsilon - 2e-6)
        de.apply_frontier(f)
        oe.apply_frontier(f)
        assert np.max(np.abs(de.messages() - oe.messages())) <= MSG_TOL
        if oe.unconverged == 0:
            break


def test_rnbp_p1_is_unconverged_set(bp, orc):
    """rnbp_frontier with p=1 is exactly the unconverged set (test_schedulers.cpp:228-239)."""
    rng = Stream(orc, 3)
    cards, un, ed = random_graph(rng, 10)
    dg, og, ep = both(bp, orc, cards, un, ed)
    de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp))
    f = de.rnbp_frontier(1.0)
    r = de.residuals()
    eps = np.float32(1e-5)
    if eps < 1e-5:  # the device compares against the smallest float >= epsilon
        eps = np.nextafter(eps, np.float32(np.inf))
    assert np.array_equal(f, np.nonzero(r >= eps)[0])


def test_rnbp_fallback_picks_one_survivor(bp, orc):
    cards, un, ed = path_graph(4)
    dg, og, ep = both(bp, orc, cards, un, ed)
    de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, seed=123))
    f = de.rnbp_frontier(1e-300)
    assert f.size == 1
    assert de.residuals()[f[0]] >= 1e-5


def test_rbp_topk_exact_against_select_top_k(bp, orc):
    """Device radix select == select_top_k (schedulers.cpp:105-116) on the device residuals."""
    og = po.Graph.ising(orc, 16, 2.5, 6)
    a = og.arrays()
    dg = bp.PairwiseMRF.from_arrays(a.cardinalities, a.unary, a.endpoints, a.tables)
    de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rbp))
    D = dg.num_directed_edges()
    for step in range(12):
        r = de.residuals().astype(np.float32).astype(np.float64)
        for p in (1.0 / 256, 1.0 / 16, 0.3, 0.999):
            k = max(1, int(np.floor(p * D + 0.5)))
            want = np.sort(po.select_top_k(orc, r, k))
            got = de.rbp_frontier(p)
            assert np.array_equal(got, want), (step, p)
        de.apply_frontier(de.rbp_frontier(0.3))


def test_rbp_topk_ties_across_chunks(bp, orc):
    """select_top_k's id order among equal keys across tie chunks and list
    blocks: a 100^2 grid (5 chunks of 8192 edges) whose residuals go to
    exactly 0 as edges commit (K* = 0 with partial ties), and a coupling-free
    grid whose residuals are all 0 (the k lowest ids)."""
    og = po.Graph.ising(orc, 100, 2.5, 8)
    a = og.arrays()
    dg = bp.PairwiseMRF.from_arrays(a.cardinalities, a.unary, a.endpoints, a.tables)
    de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rbp))
    D = dg.num_directed_edges()
    for step in range(4):
        r = de.residuals().astype(np.float32).astype(np.float64)
        for p in (1.0 / 64, 0.5, 0.9):
            k = max(1, int(np.floor(p * D + 0.5)))
            want = np.sort(po.select_top_k(orc, r, k))
            assert np.array_equal(de.rbp_frontier(p), want), (step, p)
        de.apply_frontier(de.rbp_frontier(0.6))
    flat = bp.generate_ising(bp.IsingParams(n=60, c=0.0, seed=3))
    fe = bp.EngineState(flat, bp.SchedulerConfig(kind=bp.SchedulerKind.rbp))
    assert not np.any(fe.residuals())
    k = int(np.floor(0.3 * flat.num_directed_edges() + 0.5))
    assert np.array_equal(fe.rbp_frontier(0.3), np.arange(k))


def test_rbp_frontier_size_rounding(bp, orc):
    """k = max(1, llround(p * 2|E|)): round(12.5) = 13 (test_schedulers.cpp:76-84)."""
    cards, un, ed = path_graph(101)
    dg, og, ep = both(bp, orc, cards, un, ed)
    de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rbp))
    assert de.rbp_frontier(1.0 / 16.0).size == 13
    assert de.rbp_frontier(1e-9).size == 1
    assert de.rbp_frontier(1.0).size == 200


@pytest.mark.parametrize("kind", ["rnbp", "rbp"])
def test_converged_marginals_match_reference(bp, orc, kind):
    """Converged marginals under every scheduler within 1e-4 of the reference's."""
    for n, c, seed in [(10, 2.0, 1), (20, 2.0, 2)]:
        g = bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed))
        og = po.Graph.ising(orc, n, c, seed)
        cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(kind), low_p=0.5, p=1 / 16,
                                 max_iterations=200000, seed=seed)
        r = bp.run(g, cfg)
        o = po.run(og, oracle_config(cfg))
        assert r.converged and o.converged
        assert np.max(np.abs(r.beliefs.values - o.beliefs)) <= BELIEF_TOL


def test_caps_are_not_errors(bp, orc):
    g = bp.generate_ising(bp.IsingParams(n=6, c=3.0, seed=1))
    r = bp.run(g, bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=1))
    assert not r.converged and r.iterations == 1 and len(r.trace) == 1


def test_zero_edge_graph(bp, orc):
    g = bp.build_graph([2, 3], [[0.2, 0.6], [1, 1, 2]], [])
    for kind in (bp.SchedulerKind.lbp, bp.SchedulerKind.rbp, bp.SchedulerKind.rnbp):
        r = bp.run(g, bp.SchedulerConfig(kind=kind))
        assert r.converged and r.iterations == 0
        assert abs(r.beliefs.at(0)[0] - 0.25) < 1e-6
        assert abs(r.beliefs.at(1)[2] - 0.5) < 1e-6


@pytest.mark.parametrize("n,c,seed,p", [(100, 2.5, 500, 0.5), (60, 3.0, 7, 0.5), (20, 2.0, 3, 0.05)])
def test_rnbp_persistent_tail_matches_graph_loop(bp, orc, n, c, seed, p):
    """The persistent list-mode kernel runs the same iterations as the
    per-kernel graph loop: identical traces (frontier sizes, counts).  p = 0.05
    on short lists makes empty attempt-0 draws common, so the in-kernel retry
    (attempt 1) and the single-survivor fallback run too (50 single-edge
    frontiers in the 20x20 run)."""
    g = bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed))
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=p, high_p=p if p < 0.5 else 1.0,
                             max_iterations=3000, seed=seed)
    a = bp.run(g, cfg)
    b = bp.run_ex(g, cfg, flags=bp.RUN_NO_PERSIST)
    assert a.trace_signature() == b.trace_signature()
    assert np.max(np.abs(a.beliefs.values - b.beliefs.values)) <= 1e-6
    assert a.gpu_launches <= b.gpu_launches + 2  # + the persistent launch chained behind each graph chunk


def _lattice_arrays(orc, rows, cols, seed, c=2.0):
    """rows x cols Ising lattice in generate_ising's edge order, as build_graph input."""
    rng = Stream(orc, seed)
    V = rows * cols
    unary = []
    for _ in range(V):
        a, b = rng.unit(), rng.unit()
        unary += [a or 0.5, b or 0.5]
    ep, tb = [], []
    for r in range(rows):
        for col in range(cols):
            v = r * cols + col
            for w in ([v + 1] if col + 1 < cols else []) + ([v + cols] if r + 1 < rows else []):
                lam = rng.unit() - 0.5
                a, d = np.exp(lam * c), np.exp(-lam * c)
                ep.append((v, w))
                tb += [a, d, d, a]
    return (np.full(V, 2, np.uint32), np.asarray(unary), np.asarray(ep, np.uint32).reshape(-1, 2),
            np.asarray(tb))


@pytest.mark.parametrize("rows,cols", [(7, 11), (13, 4), (1, 9), (9, 1)])
def test_nonsquare_lattice_detected_and_exact(bp, orc, rows, cols):
    """Descriptor lattices (any rows x cols) take the arithmetic-neighbour path;
    LBP stays in lockstep with the oracle and converged runs agree."""
    cards, un, ep, tb = _lattice_arrays(orc, rows, cols, 17 + rows)
    dg = bp.PairwiseMRF.from_arrays(cards, un, ep, tb)
    og = po.Graph.from_arrays(orc, cards, un, ep, tb)
    _lockstep_lbp(bp, orc, dg, og, ep, 30)
    for kind in ("lbp", "rnbp", "rbp", "rs"):
        cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(kind), low_p=0.5, p=0.25, max_iterations=20000)
        r = bp.run(dg, cfg)
        o = po.run(og, oracle_config(cfg))
        assert o.converged and r.converged, kind
        assert np.max(np.abs(r.beliefs.values - o.beliefs)) <= BELIEF_TOL, kind


@pytest.mark.parametrize("name", ["er", "potts4", "potts8"])
def test_rnbp_persistent_tail_generic_graphs(bp, name):
    """The persistent tail on CSR (non-lattice) binary graphs and on generic
    q-state graphs (atomic target dedupe, generic vertex update) runs the same
    iterations as the per-kernel graph loop."""
    g = {"er": lambda: bp.generate_er(20000, 40000, 2.5, 1),
         "potts4": lambda: bp.generate_potts(64, 4, 1.5, 2),
         "potts8": lambda: bp.generate_potts(48, 8, 1.0, 5)}[name]()
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=3000, seed=3)
    a = bp.run(g, cfg)
    b = bp.run_ex(g, cfg, flags=bp.RUN_NO_PERSIST)
    assert a.trace_signature() == b.trace_signature()
    assert np.max(np.abs(a.beliefs.values - b.beliefs.values)) == 0.0
    assert a.gpu_launches < b.gpu_launches  # the persistent kernel took over


@pytest.mark.timeout(300)
def test_rnbp_persistent_tail_potts_multipass(bp):
    """Potts 1024^2, q = 8: the candidate list at the handover (~10^5 entries)
    takes several passes of the persistent grid per phase; the run must match
    the graph loop iteration for iteration."""
    g = bp.generate_potts(1024, 8, 2.5, 0)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=200, seed=1)
    a = bp.run(g, cfg)
    b = bp.run_ex(g, cfg, flags=bp.RUN_NO_PERSIST)
    assert a.trace_signature() == b.trace_signature()
    assert np.max(np.abs(a.beliefs.values - b.beliefs.values)) == 0.0


@pytest.mark.timeout(180)
def test_rnbp_persistent_tail_potts_4096(bp):
    """Potts 4096^2, q = 8, first 20 RnBP iterations (the persistent grid on a
    list of ~10^6 entries): identical to the graph loop.  Guards the set-up
    race fixed this round (legacy-stream memsets of recycled device blocks were
    not ordered before the engine's non-blocking stream)."""
    g = bp.generate_potts(4096, 8, 2.5, 0)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=20, time_limit=60)
    a = bp.run_ex(g, cfg, beliefs=False)
    b = bp.run_ex(g, cfg, beliefs=False, flags=bp.RUN_NO_PERSIST)
    assert a.trace_signature() == b.trace_signature()


@pytest.mark.parametrize("maxq", [20, 40, 64, 100])
def test_large_cardinalities(bp, orc, maxq):
    """q up to 128 (message strides 64, 128): LBP lockstep and converged marginals
    under RnBP / RBP / RS against the oracle."""
    rng = Stream(orc, 300 + maxq)
    cards, un, ed = random_graph(rng, 8, maxq, 0.3)
    cards[0] = maxq  # at least one vertex at the maximum
    un[0] = [rng.unit() + 0.5 for _ in range(maxq)]
    ed = [(i, j, t if i != 0 else [rng.unit() + 0.5 for _ in range(cards[i] * cards[j])]) for i, j, t in ed]
    dg, og, ep = both(bp, orc, cards, un, ed)
    _lockstep_lbp(bp, orc, dg, og, ep, 12)
    for kind in ("rnbp", "rbp", "rs"):
        cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(kind), low_p=0.5, p=0.3, max_iterations=5000)
        r = bp.run(dg, cfg)
        o = po.run(og, oracle_config(cfg))
        assert r.converged and o.converged, kind
        assert float(np.max(np.abs(r.beliefs.values - o.beliefs))) <= BELIEF_TOL, kind


@pytest.mark.parametrize("n,q,c,seed,low_p", [(16, 3, 1.0, 1, 0.5), (20, 8, 1.0, 2, 0.5), (24, 4, 1.5, 5, 0.7),
                                              (40, 8, 1.0, 3, 0.3)])
def test_potts_rnbp_run_matches_oracle(bp, orc, n, q, c, seed, low_p):
    """RnBP on Potts lattices with q-vectors of 4 / 8 floats (the select's
    quad commits, the lanes-over-states touched refresh): converges like the
    reference, converged marginals within 1e-4 (north_star), and the
    per-kernel graph loop gives the same run as the default path."""
    g = bp.generate_potts(n, q, c, seed)
    og = po.Graph.potts(orc, n, q, c, seed)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=low_p, max_iterations=5000, seed=seed)
    r = bp.run(g, cfg)
    o = po.run(og, oracle_config(cfg))
    assert o.converged, "instance chosen to converge"
    assert r.converged
    assert np.max(np.abs(r.beliefs.values - o.beliefs)) <= BELIEF_TOL
    b = bp.run_ex(g, cfg, flags=bp.RUN_NO_PERSIST)
    assert r.trace_signature() == b.trace_signature()
