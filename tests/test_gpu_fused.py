"""The fused dense RnBP sweep (csrc/kernels_fused.cuh) against the two-launch
select + refresh loop it replaces (k_rnbp_select + k_vertex_update<Delta>,
rnbp_frontier + apply_frontier, schedulers.cpp:194-251): same Philox draws,
same commits, same refresh arithmetic, so the runs must agree BIT FOR BIT --
trace (frontier sizes, unconverged counts), iterations, update totals, final
messages and beliefs -- and both against the fp64 oracle's converged
marginals (1e-4)."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.helpers import lattice_arrays

pytestmark = pytest.mark.gpu


def _cfg(bp, seed=0, low_p=0.5, high_p=1.0, iters=10000, thr=0.9):
    return bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=low_p, high_p=high_p, edge_ratio_threshold=thr,
                              max_iterations=iters, time_limit=1e9, seed=seed)


def _pair(bp, g, cfg, flags=0):
    a = bp.run_ex(g, cfg, flags=flags, messages=True, kernel_timing=bool(flags & bp.RUN_KERNEL_TIMING))
    b = bp.run_ex(g, cfg, flags=flags | bp.RUN_NO_FUSED, messages=True)
    return a, b


def _assert_same(a, b):
    assert a.iterations == b.iterations and a.converged == b.converged
    assert a.messages_updated_total == b.messages_updated_total
    assert a.message_evaluations == b.message_evaluations and a.vertex_visits == b.vertex_visits
    for col in ("iteration", "frontier_size", "unconverged"):
        assert np.array_equal(a.trace.column(col), b.trace.column(col)), col
    assert np.array_equal(a.messages, b.messages)
    assert np.array_equal(a.beliefs.values, b.beliefs.values)


# (lattices up to 16K vertices run the dense phase in one 16-CTA cluster
# launch, up to 48K in one cooperative-grid launch: k_rnbp_fused_persist)
@pytest.mark.parametrize("n,c,seed,low_p", [(30, 2.5, 1, 0.5), (64, 2.5, 7, 0.3), (100, 2.5, 500, 0.5),
                                            (100, 1.0, 3, 0.7), (150, 2.5, 9, 0.5), (200, 2.5, 11, 0.3),
                                            (260, 2.5, 2, 0.5)])
def test_fused_run_equals_two_launch_loop(bp, n, c, seed, low_p):
    g = bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed))
    a, b = _pair(bp, g, _cfg(bp, seed=seed, low_p=low_p))
    _assert_same(a, b)
    assert a.kernel_stats is None


@pytest.mark.parametrize("iters", [1, 2, 3, 20, 21])
def test_fused_window_parity_fixup(bp, iters):
    """capped windows of odd and even length: the state returns to the
    canonical buffers whichever set the last sweep wrote"""
    g = bp.generate_ising(bp.IsingParams(n=1000, c=2.5, seed=0))
    a, b = _pair(bp, g, _cfg(bp, seed=0, iters=iters))
    _assert_same(a, b)
    assert a.iterations == iters and a.messages_updated_total > 0


@pytest.mark.parametrize("n", [100, 180])
@pytest.mark.parametrize("iters", [1, 2, 3, 21])
def test_fused_persistent_windows(bp, n, iters):
    """capped windows inside the persistent dense launch (cluster at 100^2,
    grid at 180^2): odd and even sweep counts leave the canonical state"""
    g = bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=4))
    a, b = _pair(bp, g, _cfg(bp, seed=4, iters=iters))
    _assert_same(a, b)
    assert a.iterations == iters


def test_fused_nonsquare_and_descriptor_lattices(bp, orc):
    """lattices from host arrays (detected numbering), several shapes"""
    for rows, cols, seed in ((7, 300, 1), (300, 7, 2), (1, 50, 3), (2, 513, 4)):
        cards, un, ep, tb = lattice_arrays(orc, rows, cols, seed, 2.0)
        g = bp.PairwiseMRF.from_arrays(cards, un, ep, tb)
        a, b = _pair(bp, g, _cfg(bp, seed=seed))
        _assert_same(a, b)


def test_fused_kernel_timing_path(bp):
    """the non-graph host loop (per-launch CUDA events) runs the same sweeps"""
    g = bp.generate_ising(bp.IsingParams(n=200, c=2.5, seed=9))
    a, b = _pair(bp, g, _cfg(bp, seed=9, iters=300), flags=bp.RUN_KERNEL_TIMING)
    _assert_same(a, b)
    assert a.kernel_stats["fused"]["launches"] > 0 and a.kernel_stats["select"]["launches"] > 0


@pytest.mark.parametrize("seed", range(6))
def test_fused_empty_frontier_hands_the_iteration_back(bp, seed):
    """tiny lattices at p = 0.02: attempt 0 often selects nothing; the fused
    phase then aborts and the retry / fallback of the per-kernel loop redoes
    the iteration -- still identical to the two-launch loop"""
    g = bp.generate_ising(bp.IsingParams(n=3, c=2.5, seed=seed))
    a, b = _pair(bp, g, _cfg(bp, seed=seed, low_p=0.02, high_p=0.02))
    _assert_same(a, b)


def test_fused_high_p_only(bp):
    """p = 1 everywhere (no Philox draws): every survivor commits"""
    g = bp.generate_ising(bp.IsingParams(n=80, c=1.5, seed=4))
    a, b = _pair(bp, g, _cfg(bp, seed=4, low_p=1.0, high_p=1.0))
    _assert_same(a, b)


@pytest.mark.parametrize("n,c,seed", [(40, 2.5, 5), (100, 1.5, 501)])
def test_fused_converged_marginals_match_oracle(bp, orc, n, c, seed):
    g = bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed))
    r = bp.run(g, _cfg(bp, seed=seed))
    o = po.run(po.Graph.ising(orc, n, c, seed), po.make_config("rnbp", low_p=0.5, high_p=1.0, max_iterations=10000,
                                                               seed=seed))
    assert r.converged and o.converged
    assert float(np.max(np.abs(r.beliefs.values - o.beliefs))) <= 1e-4


# ---- the SMEM-staged fused sweep (kernels_fused_tma.cuh): bulk-copied rows,
# strip boundaries, ragged strips, blocks starting mid-strip -- bit for bit
@pytest.mark.parametrize("rows,cols", [(2, 5), (3, 257), (7, 600), (33, 256), (40, 513), (1, 300), (300, 7),
                                       (64, 1000), (129, 255)])
def test_fused_tma_equals_two_launch_loop(bp, orc, rows, cols):
    cards, un, ep, tb = lattice_arrays(orc, rows, cols, rows + cols, 2.0)
    g = bp.PairwiseMRF.from_arrays(cards, un, ep, tb)
    for iters, lp in ((7, 0.5), (60, 0.3)):
        cfg = _cfg(bp, seed=rows, low_p=lp, iters=iters)
        a = bp.run_ex(g, cfg, flags=bp.RUN_FUSED_TMA, messages=True)
        b = bp.run_ex(g, cfg, flags=bp.RUN_NO_FUSED, messages=True)
        _assert_same(a, b)
        assert a.fused_iterations > 0


@pytest.mark.parametrize("n,iters", [(1000, 20), (2048, 9)])
def test_fused_tma_windows(bp, n, iters):
    """the staged sweep forced at 1000^2 and 2048^2"""
    g = bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=1))
    cfg = _cfg(bp, seed=1, iters=iters)
    a = bp.run_ex(g, cfg, flags=bp.RUN_FUSED_TMA, messages=True)
    b = bp.run_ex(g, cfg, flags=bp.RUN_NO_FUSED, messages=True)
    _assert_same(a, b)
