"""Row-band partition on one GPU: P bands in one process,
halos moved by LocalExchange (the data movement NcclExchange does between
GPUs).  Owned messages must be bitwise identical to the unpartitioned run for
every P -- the GPU-count independence contract (thread_pool.hpp:13-16)."""
import numpy as np
import pytest

from paper_1909_11469_b200 import parallel as par

pytestmark = pytest.mark.gpu


def _lockstep(bp, n, c, seed, nparts, iters, eps=1e-5):
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=iters, epsilon=eps)
    bands = [par.BandLBP(n, c, seed, p, nparts, cfg, 0) for p in range(nparts)]
    ex = par.LocalExchange(bands)
    for _ in range(iters + 1):
        for b in bands:
            b.sweep()
        ex.exchange_all()
        for b in bands:
            b.finish()
    return bands, [b.status() for b in bands]


@pytest.mark.parametrize("nparts", [2, 3, 5])
def test_band_lbp_bitwise_equals_unpartitioned(bp, nparts):
    n, c, seed, iters = 23, 2.5, 3, 17
    full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed)),
                  bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=iters))
    want = full.beliefs.values.reshape(n, n, 2)
    bands, st = _lockstep(bp, n, c, seed, nparts, iters)
    for b, s in zip(bands, st):
        assert s.stopped and s.iterations == full.iterations == iters and s.converged == full.converged
        got = b.owned_beliefs()
        assert np.array_equal(got, want[b.info.row0:b.info.row1]), b.info
    # every directed edge is owned (and counted) by exactly one band
    assert sum(s.messages_updated_total for s in st) == full.messages_updated_total


def test_band_lbp_converges_like_unpartitioned(bp):
    n, c, seed = 30, 1.0, 8
    full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed)),
                  bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=500))
    assert full.converged
    bands, st = _lockstep(bp, n, c, seed, 4, full.iterations + 5)
    for b, s in zip(bands, st):
        assert s.converged and s.iterations == full.iterations
        assert np.array_equal(b.owned_beliefs(), full.beliefs.values.reshape(n, n, 2)[b.info.row0:b.info.row1])


def test_band_rows_cover_grid():
    for n in (7, 16, 1000):
        for p in (1, 2, 3, 7):
            rows = [par.band_rows(n, k, p) for k in range(p)]
            assert rows[0][0] == 0 and rows[-1][1] == n
            assert all(rows[k][1] == rows[k + 1][0] for k in range(p - 1))
            total = sum(par.owned_directed_edges(n, r0, r1) for r0, r1, _, _ in rows)
            assert total == 4 * n * (n - 1)


@pytest.mark.parametrize("nparts", [1, 2, 3])
def test_band_rnbp_equals_unpartitioned(bp, nparts):
    """RnBP over bands: same iterations, updates and beliefs as the one-GPU
    run (Philox keyed by global edge ids; retry/fallback across bands)."""
    n, c, seed = 20, 2.0, 4
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=400, seed=seed)
    full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed)), cfg)
    bands = [par.BandRnBP(n, c, seed, p, nparts, cfg, 0) for p in range(nparts)]
    st = par.run_band_rnbp(bands, par.LocalComm(), cfg.max_iterations)
    assert st.converged == full.converged and st.iterations == full.iterations
    assert st.messages_updated_total == full.messages_updated_total
    want = full.beliefs.values.reshape(n, n, 2)
    for b in bands:
        assert np.array_equal(b.owned_beliefs(), want[b.info.row0:b.info.row1])


def test_band_rbp_single_band_equals_unpartitioned(bp):
    """One band = the whole grid: local top-k == global select_top_k, same run."""
    n, c, seed = 16, 2.0, 6
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rbp, p=1 / 16, max_iterations=3000)
    full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed)), cfg)
    (b,) = bands = [par.BandRBP(n, c, seed, 0, 1, cfg, 0)]
    st = par.run_band_rnbp(bands, par.LocalComm(), cfg.max_iterations)
    assert st.converged == full.converged and st.iterations == full.iterations
    assert st.messages_updated_total == full.messages_updated_total
    assert np.array_equal(b.owned_beliefs(), full.beliefs.values.reshape(n, n, 2))


@pytest.mark.parametrize("nparts", [2, 3])
def test_band_rbp_local_frontiers_converge_to_the_fixed_point(bp, orc, nparts):
    """P bands with per-partition local top-k: a different schedule, the same
    converged marginals (within 1e-4 of the reference's)."""
    from oracle import pyoracle as po
    from tests.helpers import oracle_config
    n, c, seed = 18, 1.5, 2
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rbp, p=1 / 8, max_iterations=20000)
    o = po.run(po.Graph.ising(orc, n, c, seed), oracle_config(cfg))
    bands = [par.BandRBP(n, c, seed, p, nparts, cfg, 0) for p in range(nparts)]
    st = par.run_band_rnbp(bands, par.LocalComm(), cfg.max_iterations)
    assert st.converged and o.converged
    want = np.asarray(o.beliefs).reshape(n, n, 2)
    for b in bands:
        assert np.max(np.abs(b.owned_beliefs() - want[b.info.row0:b.info.row1])) <= 1e-4


def test_band_rs_single_band_equals_unpartitioned(bp):
    n, c, seed = 14, 2.0, 3
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rs, p=1 / 16, splash_depth=2, max_iterations=3000)
    full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed)), cfg)
    (b,) = bands = [par.BandRS(n, c, seed, 0, 1, cfg, 0)]
    st = par.run_band_rnbp(bands, par.LocalComm(), cfg.max_iterations)
    assert st.converged == full.converged and st.iterations == full.iterations
    assert st.messages_updated_total == full.messages_updated_total
    assert np.array_equal(b.owned_beliefs(), full.beliefs.values.reshape(n, n, 2))


@pytest.mark.parametrize("nparts", [2, 4])
def test_band_rs_local_splashes_converge_to_the_fixed_point(bp, orc, nparts):
    from oracle import pyoracle as po
    from tests.helpers import oracle_config
    n, c, seed = 16, 1.5, 5
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rs, p=1 / 16, splash_depth=2, max_iterations=20000)
    o = po.run(po.Graph.ising(orc, n, c, seed), oracle_config(cfg))
    bands = [par.BandRS(n, c, seed, p, nparts, cfg, 0) for p in range(nparts)]
    st = par.run_band_rnbp(bands, par.LocalComm(), cfg.max_iterations)
    assert st.converged and o.converged
    want = np.asarray(o.beliefs).reshape(n, n, 2)
    for b in bands:
        assert np.max(np.abs(b.owned_beliefs() - want[b.info.row0:b.info.row1])) <= 1e-4


def test_band_loops_through_nccl_torchrun():
    """The NCCL transport path (NcclExchange / NcclComm on the band's external
    stream) under torchrun; world size = the GPUs present (1 here)."""
    import os
    import subprocess
    import sys

    import torch
    ngpu = torch.cuda.device_count()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ngpu}",
           "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(root, "tools", "band_nccl_check.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]
    assert "OK" in p.stdout, p.stdout + p.stderr[-2000:]


# ---- the C++ driver (csrc/partition.cu, bp_band_run): the same contract
@pytest.mark.parametrize("nparts", [1, 2, 3, 5])
def test_cpp_driver_lbp_bitwise_equals_unpartitioned(bp, nparts):
    n, c, seed, iters = 23, 2.5, 3, 17
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=iters)
    full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed)), cfg)
    bands = [par.Band(cfg, p, nparts, 0, n=n, c=c, seed=seed) for p in range(nparts)]
    st = par.run_bands(bands, par.BandComm.local())
    assert st.stopped and st.iterations == full.iterations == iters and st.converged == full.converged
    want = full.beliefs.values.reshape(n, n, 2)
    for b in bands:
        assert np.array_equal(b.owned_beliefs(), want[b.info.row0:b.info.row1]), b.info
    assert sum(b.status().messages_updated_total for b in bands) == full.messages_updated_total


@pytest.mark.parametrize("nparts", [1, 2, 3])
def test_cpp_driver_rnbp_equals_unpartitioned(bp, nparts):
    n, c, seed = 20, 2.0, 4
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=400, seed=seed)
    full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed)), cfg)
    bands = [par.Band(cfg, p, nparts, 0, n=n, c=c, seed=seed) for p in range(nparts)]
    st = par.run_bands(bands, par.BandComm.local())
    assert st.converged == full.converged and st.iterations == full.iterations
    assert st.messages_updated_total == full.messages_updated_total
    want = full.beliefs.values.reshape(n, n, 2)
    for b in bands:
        assert np.array_equal(b.owned_beliefs(), want[b.info.row0:b.info.row1])


def test_cpp_driver_rnbp_fallback_across_bands(bp):
    """Tiny low_p: empty attempt-0 draws, retries and single-survivor
    fallbacks picked across bands (ascending global ids) -- same run."""
    n, c, seed = 12, 2.0, 3
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.02, high_p=0.02, max_iterations=300, seed=seed)
    full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed)), cfg)
    bands = [par.Band(cfg, p, 3, 0, n=n, c=c, seed=seed) for p in range(3)]
    st = par.run_bands(bands, par.BandComm.local())
    assert st.iterations == full.iterations and st.messages_updated_total == full.messages_updated_total
    want = full.beliefs.values.reshape(n, n, 2)
    for b in bands:
        assert np.array_equal(b.owned_beliefs(), want[b.info.row0:b.info.row1])


@pytest.mark.parametrize("kind", ["lbp", "rnbp"])
def test_cpp_driver_any_lattice_descriptor(bp, orc, kind):
    """Bands of a caller's own lattice (build_graph arrays, non-square): the
    same run as the whole graph on one device."""
    from tests.helpers import lattice_arrays
    rows, cols = 17, 40
    arrays = lattice_arrays(orc, rows, cols, 9, 2.0)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(kind), low_p=0.5, max_iterations=60, seed=2)
    full = bp.run(bp.PairwiseMRF.from_arrays(*arrays), cfg)
    bands = [par.Band(cfg, p, 3, 0, arrays=arrays) for p in range(3)]
    st = par.run_bands(bands, par.BandComm.local())
    assert st.iterations == full.iterations and st.converged == full.converged
    want = full.beliefs.values.reshape(rows, cols, 2)
    for b in bands:
        assert np.array_equal(b.owned_beliefs(), want[b.info.row0:b.info.row1])


def test_cpp_driver_nccl_single_rank(bp):
    """The NCCL transport of the C++ driver (libnccl loaded at first use) with
    one rank: communicator set-up, the all-reduce on the band stream."""
    n, c, seed = 16, 2.0, 1
    comm = par.BandComm.nccl(par.nccl_unique_id(), 0, 1, 0)
    for kind in ("lbp", "rnbp"):
        cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(kind), low_p=0.5, max_iterations=50, seed=seed)
        full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed)), cfg)
        band = par.Band(cfg, 0, 1, 0, n=n, c=c, seed=seed)
        st = par.run_bands([band], comm)
        assert st.iterations == full.iterations
        assert np.array_equal(band.owned_beliefs(), full.beliefs.values.reshape(n, n, 2))


# ---- vertex-range partition of ANY binary model (bp_graph_create_part):
# random graphs, cut messages exchanged with every peer part
def _er(orc, n, m, c, seed):
    from oracle import pyoracle as po
    a = po.Graph.er(orc, n, m, c, seed).arrays()
    return a.cardinalities, a.unary, a.endpoints, a.tables


def _owned(parts):
    return np.concatenate([p.owned_beliefs() for p in parts]).reshape(-1)


@pytest.mark.parametrize("nparts", [1, 2, 3, 5])
def test_parts_lbp_random_graph_bitwise_equals_unpartitioned(bp, orc, nparts):
    arrays = _er(orc, 3000, 6000, 2.5, 1)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=25)
    full = bp.run(bp.PairwiseMRF.from_arrays(*arrays), cfg)
    parts = [par.Part(cfg, p, nparts, arrays) for p in range(nparts)]
    infos = [p.info for p in parts]
    assert sum(i.v1 - i.v0 for i in infos) == 3000
    assert sum(i.send_messages for i in infos) == sum(i.recv_messages for i in infos)
    assert sum(i.owned_directed for i in infos) == 2 * 6000
    st = par.run_bands(parts, par.BandComm.local())
    assert st.iterations == full.iterations == 25 and st.converged == full.converged
    assert np.array_equal(_owned(parts), full.beliefs.values)
    assert sum(p.status().messages_updated_total for p in parts) == full.messages_updated_total


def test_parts_lbp_converges_like_unpartitioned(bp, orc):
    arrays = _er(orc, 2000, 3000, 1.0, 2)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=2000)
    full = bp.run(bp.PairwiseMRF.from_arrays(*arrays), cfg)
    parts = [par.Part(cfg, p, 4, arrays) for p in range(4)]
    st = par.run_bands(parts, par.BandComm.local())
    assert full.converged and st.converged and st.iterations == full.iterations
    assert np.array_equal(_owned(parts), full.beliefs.values)


@pytest.mark.parametrize("nparts", [1, 2, 3])
def test_parts_rnbp_random_graph_equals_unpartitioned(bp, orc, nparts):
    """RnBP draws are keyed by GLOBAL edge ids, so the partitioned run commits
    exactly the unpartitioned frontiers"""
    arrays = _er(orc, 2000, 4000, 2.0, 3)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=400, seed=7)
    full = bp.run(bp.PairwiseMRF.from_arrays(*arrays), cfg)
    parts = [par.Part(cfg, p, nparts, arrays) for p in range(nparts)]
    st = par.run_bands(parts, par.BandComm.local())
    assert st.converged == full.converged and st.iterations == full.iterations
    assert st.messages_updated_total == full.messages_updated_total
    assert np.array_equal(_owned(parts), full.beliefs.values)


def test_parts_rnbp_fallback_across_parts(bp, orc):
    """low_p: empty attempt-0 draws, retries and single-survivor fallbacks
    picked across parts (ascending global directed ids)"""
    arrays = _er(orc, 60, 90, 2.0, 4)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.02, high_p=0.02, max_iterations=300, seed=3)
    full = bp.run(bp.PairwiseMRF.from_arrays(*arrays), cfg)
    parts = [par.Part(cfg, p, 3, arrays) for p in range(3)]
    st = par.run_bands(parts, par.BandComm.local())
    assert st.iterations == full.iterations and st.messages_updated_total == full.messages_updated_total
    assert np.array_equal(_owned(parts), full.beliefs.values)


def test_parts_generic_binary_tables_and_lattices(bp, orc):
    """non-Ising binary tables (bptest::random_graph, test_helpers.hpp:90-132)
    and a lattice given as arrays: vertex ranges partition any binary model"""
    from tests.helpers import Stream, lattice_arrays, random_graph
    cards, un, ed = random_graph(Stream(orc, 77), 300, 2, 0.02)
    rg = (np.asarray(cards, np.uint32), np.concatenate([np.asarray(u, float) for u in un]),
          np.asarray([(i, j) for i, j, _ in ed], np.uint32), np.concatenate([np.asarray(t, float) for _, _, t in ed]))
    for arrays in (rg, lattice_arrays(orc, 13, 29, 5, 2.0)):
        for kind in ("lbp", "rnbp"):
            cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(kind), low_p=0.5, max_iterations=80, seed=1)
            full = bp.run(bp.PairwiseMRF.from_arrays(*arrays), cfg)
            parts = [par.Part(cfg, p, 3, arrays) for p in range(3)]
            st = par.run_bands(parts, par.BandComm.local())
            assert st.iterations == full.iterations and st.converged == full.converged
            assert np.array_equal(_owned(parts), full.beliefs.values)


def test_parts_reject_what_they_do_not_partition(bp, orc):
    arrays = _er(orc, 100, 150, 2.0, 5)
    with pytest.raises(Exception, match="LBP and RnBP"):
        par.Part(bp.SchedulerConfig(kind=bp.SchedulerKind.rbp), 0, 2, arrays)
    with pytest.raises(Exception):
        par.Part(bp.SchedulerConfig(kind=bp.SchedulerKind.lbp), 2, 2, arrays)
