"""Parity of the PRODUCTION LBP sweeps against the fp64 oracle.

bp.run executes LBP as one fused sweep per iteration (kernels_lbp.cuh
k_lbp_lattice for binary Ising lattices of >= 2^21 vertices, the register-tiled
lattice sweep below that, k_lattice_qsweep -- lanes over states -- for q-state
lattices with q <= 8, the vertex-centric k_vertex_update for CSR graphs and
larger q).  EngineState.lbp_sweep runs exactly that kernel once, so the
reference's per-iteration state can be compared after every sweep:
messages() = m_t, candidates() = f(m_t), unconverged = #{r(m_t) >= eps}
(the reference's EngineState after t apply_frontier(frontier_lbp()) calls,
schedulers.cpp:99-103, 226-251).

Tolerances (north_star): LBP per-iteration messages within 1e-5 abs (fp32
device vs fp64 reference); converged marginals within 1e-4."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.helpers import lattice_arrays, oracle_config

pytestmark = pytest.mark.gpu

MSG_TOL = 1e-5
BELIEF_TOL = 1e-4


def fused_lockstep(bp, dg, og, ep, iters, kernel="auto", expect=None, eps=1e-5):
    """Per iteration: device fused sweep vs reference apply_frontier(frontier_lbp())."""
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, epsilon=eps)
    de = bp.EngineState(dg, cfg)
    de.set_endpoints(ep)
    oe = po.Engine(og, oracle_config(cfg))
    worst = 0.0
    for t in range(iters):
        ran = de.lbp_sweep(kernel)
        if expect is not None:
            assert ran == expect, (ran, expect)
        assert de.iteration() == t
        dm, om = de.messages(), oe.messages()
        dc, oc = de.candidates(), oe.candidates()
        worst = max(worst, float(np.max(np.abs(dm - om), initial=0.0)), float(np.max(np.abs(dc - oc), initial=0.0)))
        assert worst <= MSG_TOL, (t, worst)
        orr = oe.residuals()
        near = int(np.sum(np.abs(orr - eps) < 2e-6))
        assert abs(de.unconverged_count() - oe.unconverged) <= near, (t, de.unconverged_count(), oe.unconverged)
        if oe.unconverged == 0:
            break
        oe.apply_frontier(oe.frontier_lbp())
    return worst


def _descriptor_lattice(bp, orc, rows, cols, seed, c=2.5):
    cards, un, ep, tb = lattice_arrays(orc, rows, cols, seed, c)
    return bp.PairwiseMRF.from_arrays(cards, un, ep, tb), po.Graph.from_arrays(orc, cards, un, ep, tb), ep


# Shapes that reach every branch of the TMA sweep: 2 rows (first == last - 1),
# one partial 512-column strip, exactly one strip, strips + a ragged end, a
# one-column tail strip, tall-narrow, and a grid big enough for several tiles
# per block.
TMA_SHAPES = [(2, 5), (3, 513), (7, 1030), (33, 1024), (5, 1537), (64, 3), (300, 700), (257, 2049)]


@pytest.mark.parametrize("rows,cols", TMA_SHAPES)
def test_tma_sweep_lockstep_descriptor_lattices(bp, orc, rows, cols):
    """k_lbp_lattice forced on descriptor lattices of any shape: <= 1e-5 per iteration."""
    dg, og, ep = _descriptor_lattice(bp, orc, rows, cols, 40 + rows)
    fused_lockstep(bp, dg, og, ep, 12, kernel="tma", expect="tma")


@pytest.mark.parametrize("rows,cols", TMA_SHAPES[:6])
def test_tiles_sweep_lockstep_descriptor_lattices(bp, orc, rows, cols):
    """The register-tiled lattice sweep on the same shapes."""
    dg, og, ep = _descriptor_lattice(bp, orc, rows, cols, 40 + rows)
    fused_lockstep(bp, dg, og, ep, 12, kernel="tiles", expect="tiles")


def test_tma_sweep_on_a_single_row_falls_back(bp, orc):
    """A 1-row lattice has no vertical edges: the TMA sweep is not eligible and
    the tiles sweep runs (and stays exact)."""
    dg, og, ep = _descriptor_lattice(bp, orc, 1, 700, 3)
    fused_lockstep(bp, dg, og, ep, 8, kernel="tma", expect="tiles")


@pytest.mark.timeout(900)
def test_production_sweep_2048_tma(bp, orc):
    """2048^2 Ising (>= 2^21 vertices): bp.run's automatic choice is the TMA
    sweep; 10 fused iterations against the reference, <= 1e-5 each."""
    n = 2048
    dg = bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=1))
    og = po.Graph.ising(orc, n, 2.5, 1)
    fused_lockstep(bp, dg, og, og.arrays().endpoints, 10, kernel="auto", expect="tma")


@pytest.mark.timeout(600)
def test_production_sweep_1000_tiles(bp, orc):
    """BASELINE config 2 (1000^2, C = 2.5): the automatic choice is the tiles
    sweep; 10 fused iterations, <= 1e-5 each."""
    dg = bp.generate_ising(bp.IsingParams(n=1000, c=2.5, seed=0))
    og = po.Graph.ising(orc, 1000, 2.5, 0)
    fused_lockstep(bp, dg, og, og.arrays().endpoints, 10, kernel="auto", expect="tiles")


@pytest.mark.parametrize("n,q,c,seed", [(9, 3, 2.5, 1), (16, 8, 2.5, 2), (40, 4, 1.5, 3), (12, 5, 2.0, 4),
                                        (33, 16, 1.5, 6)])
@pytest.mark.parametrize("kernel", ["auto", "vertex"])
def test_potts_lattice_sweep_lockstep(bp, orc, n, q, c, seed, kernel):
    """q-state lattices: lanes over states (k_lattice_qsweep, q <= 8, the
    production kernel) and the thread-per-vertex path (forced, and q > 8):
    fused sweeps <= 1e-5 per iteration."""
    dg = bp.generate_potts(n, q, c, seed)
    og = po.Graph.potts(orc, n, q, c, seed)
    expect = "qlanes" if kernel == "auto" and q <= 8 else "vertex"
    fused_lockstep(bp, dg, og, og.arrays().endpoints, 25, kernel=kernel, expect=expect)


@pytest.mark.parametrize("rows,cols,q", [(7, 9, 3), (5, 33, 8)])
def test_dense_table_lattice_sweep_lockstep(bp, orc, rows, cols, q):
    """Non-Potts q-state lattice tables (dense, asymmetric): lanes over states
    with the shuffled dense contraction, both edge directions."""
    from tests.helpers import Stream
    rng = Stream(orc, 100 + q)
    V = rows * cols
    unary = [rng.unit() + 0.05 for _ in range(V * q)]
    ep, tb = [], []
    for r in range(rows):
        for col in range(cols):
            v = r * cols + col
            for w in ([v + 1] if col + 1 < cols else []) + ([v + cols] if r + 1 < rows else []):
                ep.append((v, w))
                tb += [np.exp(2.0 * (rng.unit() - 0.5)) for _ in range(q * q)]
    cards = np.full(V, q, np.uint32)
    ep = np.asarray(ep, np.uint32)
    dg = bp.PairwiseMRF.from_arrays(cards, np.asarray(unary), ep, np.asarray(tb))
    og = po.Graph.from_arrays(orc, cards, np.asarray(unary), ep, np.asarray(tb))
    fused_lockstep(bp, dg, og, ep, 20, expect="qlanes")


def test_er_sweep_lockstep(bp, orc):
    """CSR (non-lattice) binary graph: the vertex-centric sweep."""
    dg = bp.generate_er(3000, 6000, 2.5, 4)
    og = po.Graph.er(orc, 3000, 6000, 2.5, 4)
    fused_lockstep(bp, dg, og, og.arrays().endpoints, 25, expect="vertex")


@pytest.mark.parametrize("kernel", ["tma", "tiles"])
@pytest.mark.parametrize("n,c,seed", [(24, 1.5, 1), (40, 2.0, 3)])
def test_lbp_run_forced_kernel_matches_oracle(bp, orc, kernel, n, c, seed):
    """Whole runs through bp.run with the sweep kernel forced (BP_RUN_LBP_*):
    same verdict, iterations within 1 (fp32 vs fp64 at the eps boundary),
    converged marginals within 1e-4."""
    g = bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed))
    og = po.Graph.ising(orc, n, c, seed)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=5000)
    flags = bp.RUN_LBP_TMA if kernel == "tma" else bp.RUN_LBP_TILES
    r = bp.run_ex(g, cfg, flags=flags)
    o = po.run(og, oracle_config(cfg))
    assert o.converged, "instance chosen to converge"
    assert r.converged
    assert abs(r.iterations - o.iterations) <= 1
    assert np.max(np.abs(r.beliefs.values - o.beliefs)) <= BELIEF_TOL
    assert r.messages_updated_total == r.iterations * 2 * g.num_edges()


@pytest.mark.parametrize("n,q,c,seed", [(12, 3, 1.0, 1), (20, 8, 1.0, 2), (16, 4, 1.5, 5)])
def test_potts_lbp_run_matches_oracle(bp, orc, n, q, c, seed):
    """LBP runs on Potts lattices (the q <= 8 lattice sweep) against the oracle."""
    g = bp.generate_potts(n, q, c, seed)
    og = po.Graph.potts(orc, n, q, c, seed)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=5000)
    r = bp.run(g, cfg)
    o = po.run(og, oracle_config(cfg))
    assert o.converged, "instance chosen to converge"
    assert r.converged
    assert abs(r.iterations - o.iterations) <= 1
    assert np.max(np.abs(r.beliefs.values - o.beliefs)) <= BELIEF_TOL


@pytest.mark.parametrize("rows,cols", [(3, 513), (9, 1100)])
def test_tma_run_descriptor_lattice_converges_like_oracle(bp, orc, rows, cols):
    """Multi-strip descriptor lattices run to convergence with the TMA sweep."""
    cards, un, ep, tb = lattice_arrays(orc, rows, cols, 5, 1.0)
    dg = bp.PairwiseMRF.from_arrays(cards, un, ep, tb)
    og = po.Graph.from_arrays(orc, cards, un, ep, tb)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=5000)
    r = bp.run_ex(dg, cfg, flags=bp.RUN_LBP_TMA)
    o = po.run(og, oracle_config(cfg))
    assert o.converged and r.converged
    assert abs(r.iterations - o.iterations) <= 1
    assert np.max(np.abs(r.beliefs.values - o.beliefs)) <= BELIEF_TOL
