"""Edge-case configurations against the oracle (tools/edge_config_check.py as a
test): extreme p / low_p / high_p / thresholds, splash depth 0 / 1, iteration
caps 0 / 1 / 2, large epsilon, on an Ising lattice, a Potts lattice and a
random mixed-cardinality graph.  LBP / RBP / RS are deterministic: verdict,
iteration count and update total equal the reference's; every run agrees
on marginals (1e-4 converged, 1e-5 under a cap)."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.helpers import Stream, flatten, oracle_config, random_graph

pytestmark = pytest.mark.gpu

CONFIGS = [("rbp", dict(p=1.0)), ("rbp", dict(p=1e-6, max_iterations=400)), ("rs", dict(p=1.0, splash_depth=2)),
           ("rs", dict(p=1e-6, splash_depth=2)), ("rs", dict(p=0.2, splash_depth=0, max_iterations=50)),
           ("rs", dict(p=0.2, splash_depth=1)), ("rnbp", dict(low_p=1.0)), ("rnbp", dict(low_p=0.5, high_p=0.5)),
           ("rnbp", dict(low_p=0.5, edge_ratio_threshold=1.0)), ("lbp", dict(max_iterations=0)),
           ("lbp", dict(max_iterations=1)), ("rbp", dict(p=0.3, max_iterations=2)), ("rnbp", dict(max_iterations=1)),
           ("rs", dict(p=0.3, max_iterations=0)), ("lbp", dict(epsilon=0.5)), ("rnbp", dict(epsilon=0.5)),
           ("rbp", dict(p=0.2, epsilon=1e-3))]


def _models(bp, orc):
    cards, un, edges = random_graph(Stream(orc, 3), 40, 3, 0.08)
    a = flatten(cards, un, edges)
    return [(bp.generate_ising(bp.IsingParams(n=20, c=1.5, seed=4)), po.Graph.ising(orc, 20, 1.5, 4)),
            (bp.generate_potts(12, 3, 1.0, 2), po.Graph.potts(orc, 12, 3, 1.0, 2)),
            (bp.PairwiseMRF.from_arrays(*a), po.Graph.from_arrays(orc, *a))]


@pytest.mark.parametrize("kind,kw", CONFIGS, ids=[f"{k}-{'-'.join(f'{a}={b}' for a, b in kw.items())}" for k, kw in CONFIGS])
def test_edge_config_matches_oracle(bp, orc, kind, kw):
    for dg, og in _models(bp, orc):
        kw2 = dict(kw)
        kw2.setdefault("max_iterations", 3000)
        cfg = bp.SchedulerConfig(kind=getattr(bp.SchedulerKind, kind), seed=7, **kw2)
        r = bp.run(dg, cfg)
        o = po.run(og, oracle_config(cfg))
        assert r.converged == o.converged
        diff = float(np.max(np.abs(r.beliefs.values - o.beliefs)))
        if kind != "rnbp":
            assert r.iterations == o.iterations
            assert r.messages_updated_total == o.messages_updated_total
            assert diff <= (1e-4 if r.converged else 1e-5)
        elif r.converged:
            assert diff <= 1e-4
        else:  # capped after the same deterministic first iteration(s)
            assert r.iterations == o.iterations


def test_edge_ratio_threshold_zero_is_rejected_like_the_reference(bp, orc):
    dg, og = _models(bp, orc)[0]
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, edge_ratio_threshold=0.0)
    with pytest.raises(ValueError):
        bp.run(dg, cfg)
    with pytest.raises(po.OracleError):
        po.run(og, oracle_config(cfg))
