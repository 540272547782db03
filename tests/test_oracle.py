"""CPU tests of the oracle (test infrastructure): the C restatement
(oracle/bp_oracle.c) is pinned against (a) the reference itself compiled in
process (oracle/_ref), bit for bit, and (b) the committed golden fixtures and
the known-answer tests of the reference's own suites."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from tests.helpers import Stream, flatten, path_graph, random_graph, random_tree

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


@pytest.fixture(scope="module")
def small():
    with open(os.path.join(GOLDEN, "reference_small.json")) as f:
        return json.load(f)


# ---------------------------------------------------------------- golden vectors

def test_mt19937_64_golden(orc, small):
    for seed, vals in small["mt19937_64"].items():
        raw, unit = po.mt_draws(orc, int(seed), 8)
        assert [int(x) for x in raw] == vals
        assert np.array_equal(unit, (raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)
    raw, _ = po.mt_draws(orc, 5489, 10000)
    assert int(raw[-1]) == small["mt19937_64_5489_10000th"] == 9981545732273789042


def test_generated_instances_match_reference(orc, small):
    for inst in small["instances"]:
        a = po.Graph.ising(orc, inst["n"], inst["c"], inst["seed"]).arrays()
        assert _sha(a.unary) == inst["unary_sha"]
        assert _sha(a.endpoints.astype(np.uint32)) == inst["endpoints_sha"]
        assert _sha(a.tables) == inst["tables_sha"]


def test_runs_match_reference_fixtures(orc, small):
    for case in small["runs"]:
        gk = case["graph"]
        g = (po.Graph.ising(orc, gk["n"], gk["c"], gk["seed"]) if gk["kind"] == "ising"
             else po.Graph.chain(orc, gk["n"], gk["c"], gk["seed"]))
        ck = dict(case["config"])
        kind = ck.pop("kind")
        r = po.run(g, po.make_config(kind, **ck))
        assert r.converged == case["converged"], case["config"]
        assert r.iterations == case["iterations"]
        assert r.messages_updated_total == case["messages_updated_total"]
        assert hashlib.sha256(r.signature().encode()).hexdigest()[:32] == case["trace_signature_sha"]
        assert _sha(r.beliefs) == case["beliefs_sha"]


# ---------------------------------------------------------------- bitwise vs the reference

@pytest.mark.parametrize("kind", ["lbp", "rbp", "rs", "rnbp", "srbp"])
def test_oracle_bitwise_equals_reference(orc, ref, kind):
    rng = Stream(orc, 91)
    graphs = [("ising", 7, 2.5, 3), ("ising", 12, 3.0, 9)]
    for n, c, seed in [(g[1], g[2], g[3]) for g in graphs]:
        go, gr = po.Graph.ising(orc, n, c, seed), po.Graph.ising(ref, n, c, seed)
        cfg = po.make_config(kind, p=0.2, max_iterations=2000 if kind == "srbp" else 200, seed=5, low_p=0.5)
        a, b = po.run(go, cfg), po.run(gr, cfg)
        assert a.signature() == b.signature()
        assert np.array_equal(a.beliefs, b.beliefs)
    for rep in range(4):  # mixed cardinalities
        cards, un, ed = random_graph(rng, 5 + rep, 4)
        c, u, ep, tb = flatten(cards, un, ed)
        go, gr = po.Graph.from_arrays(orc, c, u, ep, tb), po.Graph.from_arrays(ref, c, u, ep, tb)
        cfg = po.make_config(kind, p=0.3, max_iterations=500, seed=rep)
        a, b = po.run(go, cfg), po.run(gr, cfg)
        assert a.signature() == b.signature()
        assert np.array_equal(a.beliefs, b.beliefs)


def test_lockstep_phases_bitwise_equal_reference(orc, ref):
    go, gr = po.Graph.ising(orc, 9, 2.5, 4), po.Graph.ising(ref, 9, 2.5, 4)
    cfg = po.make_config("rnbp", seed=3)
    eo, er = po.Engine(go, cfg), po.Engine(gr, cfg)
    for t in range(15):
        assert np.array_equal(eo.residuals(), er.residuals())
        assert np.array_equal(eo.candidates(), er.candidates())
        fo, fr = eo.rnbp_frontier(0.5), er.rnbp_frontier(0.5)
        assert np.array_equal(fo, fr)
        assert np.array_equal(np.sort(eo.rbp_frontier(0.1)), np.sort(er.rbp_frontier(0.1)))
        ro, oo, so = eo.rs_frontier(0.05, 2)
        rr, orr, sr = er.rs_frontier(0.05, 2)
        assert np.array_equal(ro, rr) and np.array_equal(oo, orr) and np.array_equal(so, sr)
        eo.apply_frontier(fo)
        er.apply_frontier(fr)
        assert np.array_equal(eo.messages(), er.messages())
        assert eo.unconverged == er.unconverged
    ro, oo, so = eo.rs_frontier(0.1, 2)
    eo.apply_splashes(ro, oo, so)
    er.apply_splashes(ro, oo, so)
    assert np.array_equal(eo.messages(), er.messages())


# ---------------------------------------------------------------- known-answer tests
# (test_mrf_core.cpp / test_schedulers.cpp / test_generators.cpp of the reference)

def _graph(orc, cards, unaries, edges):
    c, u, ep, tb = flatten(cards, unaries, edges)
    return po.Graph.from_arrays(orc, c, u, ep, tb)


def test_hand_derived_update(orc):
    """unnormalized (1.7, 0.8) -> (0.68, 0.32)  (test_mrf_core.cpp:123-130)"""
    g = _graph(orc, [2, 2], [[0.8, 0.2], [0.5, 0.5]], [(0, 1, [2.0, 0.5, 0.5, 2.0])])
    e = po.Engine(g, po.make_config("lbp"))
    m = e.update_message(0)
    assert abs(m[0] - 0.68) <= 1e-12 and abs(m[1] - 0.32) <= 1e-12


def test_directed_ids_and_incoming_csr(orc):
    """ids 2e / 2e+1, CSR of incoming edges in edge-id order (test_mrf_core.cpp:24-51)"""
    g = _graph(orc, [2, 2], [[0.8, 0.2], [0.5, 0.5]], [(0, 1, [2.0, 0.5, 0.5, 2.0])])
    off, adj = g.incoming()
    assert off.tolist() == [0, 1, 2] and adj.tolist() == [1, 0]
    rng = Stream(orc, 11)
    for rep in range(10):
        cards, un, ed = random_graph(rng, 2 + rep % 8)
        gg = _graph(orc, cards, un, ed)
        off, adj = gg.incoming()
        assert sorted(adj.tolist()) == list(range(2 * len(ed)))
        for v in range(len(cards)):
            seg = adj[off[v]:off[v + 1]]
            assert np.all(np.diff(seg.astype(np.int64)) > 0)
            for d in seg:
                e = d >> 1
                tgt = ed[e][1] if d % 2 == 0 else ed[e][0]
                assert tgt == v


@pytest.mark.parametrize("bad", [
    ([2, 2, 2, 2], [[1, 1]] * 4, [(3, 3, [1, 1, 1, 1])]),           # self-loop
    ([2, 2], [[1, 1], [1, 1]], [(0, 1, [1, 0.0, 1, 1])]),              # zero pairwise entry
    ([2, 2], [[1, 0.0], [1, 1]], []),                                  # zero unary entry
    ([2, 2], [[1, 1], [1, 1]], [(0, 1, [1] * 4), (0, 1, [1] * 4)]),    # duplicate edge
    ([2, 2], [[1, 1], [1, 1]], [(1, 0, [1, 1, 1, 1])]),               # endpoints must be ordered
    ([2, 2], [[1, 1], [1, 1]], [(0, 1, [1, float("inf"), 1, 1])]),     # non-finite
])
def test_build_graph_rejects(orc, bad):
    """test_mrf_core.cpp:53-68"""
    with pytest.raises(po.OracleError) as ei:
        _graph(orc, *bad)
    assert ei.value.code == 2  # model_error


def test_select_top_k_and_rounding(orc):
    """test_schedulers.cpp:51-84"""
    assert sorted(po.select_top_k(orc, [0.5, 0.3, 0.9, 0.1], 2).tolist()) == [0, 2]
    assert po.select_top_k(orc, [0.4, 0.4, 0.1], 1).tolist() == [0]
    assert po.select_top_k(orc, [0.5, 0.3, 0.9, 0.1], 99).size == 4
    assert po.select_top_k(orc, [0.5, 0.3, 0.9, 0.1], 0).size == 0
    g = _graph(orc, *path_graph(101))
    e = po.Engine(g, po.make_config("rbp"))
    assert e.rbp_frontier(1.0 / 16.0).size == 13  # llround(12.5) = 13
    assert e.rbp_frontier(1e-9).size == 1
    assert np.array_equal(np.sort(e.rbp_frontier(1.0)), e.frontier_lbp())


@pytest.mark.parametrize("lib", ["orc", "ref"])
def test_splash_bfs_order_and_claims(lib):
    """build_splash golden vectors (test_schedulers.cpp:117-157)"""
    L = po.load(lib) if lib == "orc" or os.path.exists(po.PATHS["ref"]) else pytest.skip("no ref")
    g = _graph(L, *path_graph(5))
    e = po.Engine(g, po.make_config("rs"))
    U = np.uint32(0xFFFFFFFF)
    claimed = np.full(5, U, np.uint32)
    assert e.build_splash(2, 0, claimed).tolist() == [3, 4]  # h=0: (2->1), (2->3)
    assert claimed.tolist().count(int(U)) == 4 and claimed[2] == 2
    claimed = np.full(5, U, np.uint32)
    assert e.build_splash(2, 2, claimed).tolist() == [3, 4, 1, 2, 5, 6, 0, 7]
    assert claimed.tolist() == [2] * 5
    g6 = _graph(L, *path_graph(6))
    e6 = po.Engine(g6, po.make_config("rs"))
    claimed = np.full(6, U, np.uint32)
    e6.build_splash(1, 1, claimed)
    e6.build_splash(4, 1, claimed)
    assert claimed.tolist() == [1, 1, 1, 4, 4, 4]
    with pytest.raises(po.OracleError):
        e6.build_splash(4, 1, claimed)


def test_edge_ratio_rule(orc):
    """test_schedulers.cpp:294-313"""
    cfg = po.make_config("rnbp", low_p=0.7, high_p=1.0)
    sp = lambda a, b: po.select_parallelism(orc, a, b, cfg)  # noqa: E731
    assert sp(100, 95) == 0.7 and sp(100, 50) == 1.0 and sp(0, 50) == 1.0
    assert sp(1000, 900) == 1.0 and sp(1000, 901) == 0.7


def test_rnbp_p1_and_fallback(orc):
    """test_schedulers.cpp:228-269"""
    rng = Stream(orc, 3)
    cards, un, ed = random_graph(rng, 10)
    e = po.Engine(_graph(orc, cards, un, ed), po.make_config("rnbp"))
    assert np.array_equal(e.rnbp_frontier(1.0), np.nonzero(e.residuals() >= 1e-5)[0])
    e2 = po.Engine(_graph(orc, *path_graph(4)), po.make_config("rnbp", seed=123))
    f = e2.rnbp_frontier(1e-300)
    assert f.size == 1 and e2.residuals()[f[0]] >= 1e-5


def test_chain_converges_within_length_and_caps(orc):
    """test_schedulers.cpp:436-456"""
    for length in (10, 33, 80):
        r = po.run(po.Graph.chain(orc, length, 2.0, length), po.make_config("lbp", max_iterations=length + 5))
        assert r.converged and r.iterations <= length and len(r.trace) == r.iterations
    r = po.run(po.Graph.ising(orc, 6, 3.0, 1), po.make_config("lbp", max_iterations=1))
    assert not r.converged and r.iterations == 1 and len(r.trace) == 1


def test_ising_table_and_c0(orc):
    """test_generators.cpp:13-19, 77-87"""
    a = po.Graph.ising(orc, 3, 1.0, 0).arrays()
    lam = math.log(a.tables[0])  # = lambda * c
    assert abs(a.tables[1] - math.exp(-lam)) < 1e-15 and a.tables[0] == a.tables[3]
    r = po.run(po.Graph.ising(orc, 5, 0.0, 3), po.make_config("lbp"))
    assert r.converged and r.iterations <= 2


def test_tree_exactness_all_schedulers(orc):
    """test_schedulers.cpp:418-434"""
    rng = Stream(orc, 14)
    cards, un, ed = random_tree(rng, 9, 2.0)
    g = _graph(orc, cards, un, ed)
    import itertools
    n = len(cards)
    marg = [np.zeros(2) for _ in range(n)]
    for a in itertools.product(*[range(2)] * n):
        w = 1.0
        for v in range(n):
            w *= un[v][a[v]]
        for i, j, t in ed:
            w *= t[a[i] * 2 + a[j]]
        for v in range(n):
            marg[v][a[v]] += w
    exact = np.concatenate([m / m.sum() for m in marg])
    for kind in ("lbp", "srbp", "rbp", "rs", "rnbp"):
        r = po.run(g, po.make_config(kind, epsilon=1e-8, p=0.25, max_iterations=1000000))
        assert r.converged, kind
        assert np.max(np.abs(r.beliefs - exact)) <= 1e-6, kind


def test_new_generators_are_deterministic(orc):
    """Potts / Erdos-Renyi instance definitions."""
    a = po.Graph.potts(orc, 5, 4, 2.5, 1).arrays()
    b = po.Graph.potts(orc, 5, 4, 2.5, 1).arrays()
    assert np.array_equal(a.tables, b.tables) and a.cardinalities.tolist() == [4] * 25
    t = a.tables[:16].reshape(4, 4)
    assert np.allclose(t, t.T) and len(set(np.round(t.ravel(), 12))) == 2
    e = po.Graph.er(orc, 200, 400, 2.5, 3).arrays()
    ep = e.endpoints.astype(np.int64)
    assert e.num_edges == 400 and np.all(ep[:, 0] < ep[:, 1])
    keys = ep[:, 0] * 1000 + ep[:, 1]
    assert np.all(np.diff(keys) > 0)  # sorted, unique


def test_oracle_reproduces_reference_suite_fixtures(orc):
    """The C restatement reproduces the reference's suite fixtures bitwise
    (tests/golden/reference_suites.json, generated from oracle/_ref)."""
    import json
    import os
    from tests.golden.make_golden import h
    with open(os.path.join(os.path.dirname(__file__), "golden", "reference_suites.json")) as f:
        suites = json.load(f)["suites"]
    for suite, seed, name in (("ising100", 513, "lbp"), ("hard30", 700, "rnbp_low0.1"), ("hard30", 709, "lbp")):
        sp = suites[suite]
        row = next(r for r in sp["rows"] if r["seed"] == seed)[name]
        g = po.Graph.ising(orc, sp["n"], sp["c"], seed)
        kw = dict(low_p=float(name.split("low")[1]), high_p=1.0, edge_ratio_threshold=0.9,
                  seed=seed - sp["seeds"][0]) if name != "lbp" else {}
        r = po.run(g, po.make_config("lbp" if name == "lbp" else "rnbp", max_iterations=sp["max_iterations"],
                                     time_limit=1e9, **kw), trace_cap=1)
        assert (r.converged, r.iterations, r.messages_updated_total) == \
            (row["converged"], row["iterations"], row["messages_updated_total"])
        assert h(r.beliefs) == row["beliefs_sha"]
