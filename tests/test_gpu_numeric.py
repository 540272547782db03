"""numeric_error parity (normalize_in_place, messages.cpp:41-49): the reference
throws when a message's (or a belief's) unnormalised total mass falls below
1e-300.  graph.cu bounds that mass for every model at build time; models that
can reach it are built with log-domain tables and the device computes the
reference's mass exactly (generic_logmatvec), so bp.run raises NumericError
exactly where the reference's run throws numeric_error -- and models that are
merely flagged run the log-domain path to the same results."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.helpers import flatten, oracle_config

pytestmark = pytest.mark.gpu

KINDS = ("lbp", "rbp", "rnbp", "rs")


def _both(bp, orc, cards, unaries, edges):
    c, u, ep, tb = flatten(cards, unaries, edges)
    return bp.PairwiseMRF.from_arrays(c, u, ep, tb), po.Graph.from_arrays(orc, c, u, ep, tb)


def _cfg(bp, kind):
    return bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(kind), low_p=0.5, p=0.25, max_iterations=2000)


def _oracle_raises_numeric(og, cfg):
    with pytest.raises(po.OracleError) as ei:
        po.run(og, oracle_config(cfg))
    assert ei.value.code == 3  # ORC_NUMERIC = numeric_error
    return ei.value


@pytest.mark.parametrize("kind", KINDS)
def test_collapse_at_the_first_refresh(bp, orc, kind):
    """Tiny potentials: the EngineState ctor's first refresh underflows
    (mass 2e-320), in the reference and on the device."""
    dg, og = _both(bp, orc, [2, 2], [[1e-160, 1e-160], [1.0, 1.0]], [(0, 1, [1e-160] * 4)])
    cfg = _cfg(bp, kind)
    _oracle_raises_numeric(og, cfg)
    with pytest.raises(bp.NumericError):
        bp.run(dg, cfg)


@pytest.mark.parametrize("kind", ("lbp", "rnbp"))
def test_collapse_during_the_run(bp, orc, kind):
    """Star: four confident leaves pull the centre two ways (messages ~1e-200
    after the first commit), so the centre's next outgoing messages have mass
    ~4e-400: the reference throws in iteration 0's refresh, so does the device."""
    strong = [1.0, 1e-200]
    unaries = [[1.0, 1.0], strong, strong[::-1], strong, strong[::-1], [1.0, 1.0]]
    table = [1.0, 1e-200, 1e-200, 1.0]
    dg, og = _both(bp, orc, [2] * 6, unaries, [(0, v, table) for v in range(1, 6)])
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(kind), low_p=1.0, max_iterations=100)
    _oracle_raises_numeric(og, cfg)
    with pytest.raises(bp.NumericError):
        bp.run(dg, cfg)


@pytest.mark.parametrize("kind", KINDS)
def test_flagged_model_without_collapse_matches_reference(bp, orc, kind):
    """A chain with near-deterministic couplings (1e-200 off the diagonal) is
    flagged by the build-time bound (two such incoming messages could carry
    mass 1e-400) but never collapses: the log-domain path runs and converges
    to the reference's marginals."""
    n = 12
    unaries = [[0.7, 0.3]] + [[1.0, 1.0]] * (n - 2) + [[0.7, 0.3]]
    edges = [(v, v + 1, [1.0, 1e-200, 1e-200, 1.0]) for v in range(n - 1)]
    dg, og = _both(bp, orc, [2] * n, unaries, edges)
    assert not dg.binary  # built with the log-domain (q-state) layout
    cfg = _cfg(bp, kind)
    o = po.run(og, oracle_config(cfg))
    r = bp.run(dg, cfg)
    assert o.converged and r.converged
    assert np.max(np.abs(r.beliefs.values - o.beliefs)) <= 1e-4


def test_ordinary_models_keep_the_fast_layout(bp, orc):
    """Generated and ordinary descriptor models pass the bound: binary log-odds layout."""
    og = po.Graph.ising(orc, 8, 2.5, 1)
    a = og.arrays()
    assert bp.PairwiseMRF.from_arrays(a.cardinalities, a.unary, a.endpoints, a.tables).binary
