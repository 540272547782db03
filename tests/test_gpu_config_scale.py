"""Parity at the BASELINE configs' own scale (BASELINE.json configs 2-4),
against the fp64 oracle (pinned bitwise to the reference, test_oracle.py):

* config 3's graph (Erdos-Renyi G(1e6, 2e6)): LBP fused sweeps (the CSR
  vertex kernel) per iteration <= 1e-5; Residual Splash with the reference's
  own splashes (rs_frontier) applied by both engines, messages and residuals
  <= 1e-5 per iteration;
* config 2 (Ising 1000^2, C = 2.5): RnBP with the device's Philox frontiers
  injected into the reference engine (apply_frontier), messages <= 1e-5 per
  iteration through the dense phase -- the frontier semantics (filter r >=
  eps, ascending ids) checked on every iteration;
* config 4's family (Potts q = 8, 1024^2): LBP sweeps with four states per
  lane per iteration <= 1e-5, and the touched refresh (RnBP frontiers
  injected) <= 1e-5.

The oracle is single-threaded fp64, so each case runs a few iterations."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.helpers import oracle_config
from tests.test_gpu_lbp_sweeps import fused_lockstep

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

MSG_TOL = 1e-5


def test_er1m_lbp_sweeps(bp, orc):
    dg = bp.generate_er(1_000_000, 2_000_000, 2.5, 0)
    og = po.Graph.er(orc, 1_000_000, 2_000_000, 2.5, 0)
    fused_lockstep(bp, dg, og, og.arrays().endpoints, 3, kernel="auto")


def test_er1m_rs_reference_splashes(bp, orc):
    og = po.Graph.er(orc, 1_000_000, 2_000_000, 2.5, 0)
    a = og.arrays()
    dg = bp.PairwiseMRF.from_arrays(a.cardinalities, a.unary, a.endpoints, a.tables)
    de = bp.EngineState(dg, bp.SchedulerConfig(kind=bp.SchedulerKind.rs))
    oe = po.Engine(og, po.make_config("rs"))
    for t in range(3):
        roots, eoff, edges = oe.rs_frontier(1 / 128, 2)
        assert len(roots) == int(1_000_000 / 128 + 0.5)  # llround (schedulers.cpp:172-173)
        de.apply_splashes(roots, eoff, edges)
        oe.apply_splashes(roots, eoff, edges)
        assert np.max(np.abs(de.messages() - oe.messages())) <= MSG_TOL, t
        assert np.max(np.abs(de.residuals() - oe.residuals())) <= MSG_TOL, t


def test_ising1000_rnbp_injected_frontiers(bp, orc):
    og = po.Graph.ising(orc, 1000, 2.5, 0)
    dg = bp.generate_ising(bp.IsingParams(n=1000, c=2.5, seed=0))
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, seed=0)
    de = bp.EngineState(dg, cfg)
    oe = po.Engine(og, oracle_config(cfg))
    for t in range(4):
        f = de.rnbp_frontier(0.5)
        res = oe.residuals()
        assert np.all(np.diff(f.astype(np.int64)) > 0)
        assert np.all(res[f] >= cfg.epsilon - 2e-6)
        # about half of the unconverged edges (Bernoulli(0.5))
        assert abs(len(f) - oe.unconverged / 2) < 6 * np.sqrt(oe.unconverged / 4) + 0.01 * oe.unconverged
        de.apply_frontier(f)
        oe.apply_frontier(f)
        de.advance_iteration()
        oe.advance()
        assert np.max(np.abs(de.messages() - oe.messages())) <= MSG_TOL, t


def test_potts1024_q8_sweeps_and_refresh(bp, orc):
    n, q = 1024, 8
    dg = bp.generate_potts(n, q, 2.5, 0)
    og = po.Graph.potts(orc, n, q, 2.5, 0)
    ep = og.arrays().endpoints
    fused_lockstep(bp, dg, og, ep, 3, kernel="auto", expect="qlanes")
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, seed=3)
    de = bp.EngineState(dg, cfg)
    de.set_endpoints(ep)
    oe = po.Engine(og, oracle_config(cfg))
    for t in range(3):
        f = de.rnbp_frontier(0.5)
        de.apply_frontier(f)
        oe.apply_frontier(f)
        de.advance_iteration()
        oe.advance()
        assert np.max(np.abs(de.messages() - oe.messages())) <= MSG_TOL, t
        assert np.max(np.abs(de.residuals() - oe.residuals())) <= MSG_TOL, t
