"""CPU tests of the product boundary (no GPU needed, no device compute):
libbp_b200.so loads, exports every symbol declared in include/bp_cuda.h, and
its host-side logic (config validation, EdgeRatio rule, graph validation,
host instance arrays) behaves like the reference."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bp_cuda.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^BP_API\s+[\w\s\*]+?\b(bp_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol(bp):
    lib = ctypes.CDLL(bp.library_path())
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.bp_abi_version() == 1


def test_sm100a_cubin_embedded(bp):
    """the library carries sm_100a SASS (built with -gencode arch=compute_100a,code=sm_100a)"""
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", bp.library_path()], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_config_validation_matches_reference(bp, orc):
    """SchedulerConfig::validate (schedulers.cpp:78-90) -> ValueError"""
    bad = [dict(p=0.0), dict(p=1.5), dict(epsilon=0.0), dict(low_p=0.9, high_p=0.5),
           dict(edge_ratio_threshold=0.0), dict(time_limit=0.0), dict(epsilon=float("nan"))]
    for kw in bad:
        with pytest.raises(ValueError):
            bp.SchedulerConfig(**kw).validate()
        assert orc.validate_config(ctypes.byref(po.make_config("lbp", **kw))) == 1
    bp.SchedulerConfig().validate()


def test_select_parallelism_matches_oracle(bp, orc):
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.7, high_p=1.0)
    ocfg = po.make_config("rnbp", low_p=0.7, high_p=1.0)
    assert bp.select_parallelism(1000, 900, cfg) == 1.0
    assert bp.select_parallelism(1000, 901, cfg) == 0.7
    assert bp.select_parallelism(0, 123, cfg) == 1.0
    rng = np.random.default_rng(8)
    for _ in range(300):
        prev, now = int(rng.integers(0, 1000)), int(rng.integers(0, 1100))
        assert bp.select_parallelism(prev, now, cfg) == po.select_parallelism(orc, prev, now, ocfg)


def test_scheduler_kind_strings(bp):
    """to_string / scheduler_from_string (schedulers.cpp:58-76)"""
    K = bp.SchedulerKind
    assert [str(k) for k in K] == ["lbp", "srbp", "rbp", "rs", "rnbp"]
    assert K.from_string("serial_rbp") == K.serial_rbp and K.from_string("nope") is None


@pytest.mark.parametrize("bad,msg", [
    (([2, 2, 2, 2], [[1, 1]] * 4, [(3, 3, [1, 1, 1, 1])]), "self-loop"),
    (([2, 2], [[1, 1], [1, 1]], [(0, 1, [1, 0.0, 1, 1])]), "strictly positive"),
    (([2, 2], [[1, 0.0], [1, 1]], []), "strictly positive"),
    (([2, 2], [[1, 1], [1, 1]], [(0, 1, [1] * 4), (0, 1, [1] * 4)]), "duplicate"),
    (([2, 2], [[1, 1], [1, 1]], [(0, 1, [1, 1, 1])]), "entries"),
    (([2, 2], [[1, 1, 1], [1, 1]], []), "entries"),
    (([2, 2], [[1, 1], [1, 1]], [(1, 0, [1, 1, 1, 1])]), "i < j"),
    (([0, 2], [[], [1, 1]], []), "cardinality 0"),
    # several violations: the reference's first one (vertex order, then edge
    # order with range / self-loop / order / duplicate / entries per edge)
    (([2, 2, 2], [[1, 1]] * 3, [(0, 1, [1, 0.0, 1, 1]), (2, 2, [1] * 4)]), r"pairwise\(0,1\)"),
    (([2, 2, 2], [[1, 1]] * 3, [(0, 1, [1] * 4), (0, 1, [1] * 4), (1, 2, [1, -1, 1, 1])]), "duplicate edge \\(0, 1\\)"),
    (([2, 2, 2], [[1, 1], [1, float("inf")], [1, 1]], [(2, 2, [1] * 4)]), r"unary\(1\)"),
    (([2, 3, 2], [[1, 1], [1, 1, 1], [1, 1]], [(0, 1, [1] * 6), (1, 2, [1] * 5 + [float("nan")])]), r"pairwise\(1,2\)"),
])
def test_build_graph_validation_is_host_side(bp, bad, msg):
    """model_error cases of build_graph (mrf.cpp:28-91) are raised before any
    device work, so they are checked here without a GPU."""
    with pytest.raises(bp.ModelError, match=msg):
        bp.build_graph(*bad)


def test_host_instance_arrays_equal_reference_generator(bp, orc):
    """bp_generate_ising_arrays reproduces generate_ising bit for bit."""
    for n, c, seed in ((1, 2.5, 0), (2, 1.0, 3), (17, 2.5, 500)):
        cards, un, ep, tb = bp.generate_ising_arrays(bp.IsingParams(n=n, c=c, seed=seed))
        a = po.Graph.ising(orc, n, c, seed).arrays()
        assert np.array_equal(cards, a.cardinalities)
        assert np.array_equal(un, a.unary) and np.array_equal(tb, a.tables)
        assert np.array_equal(ep, a.endpoints)


def test_import_fails_loudly_without_extension(tmp_path):
    """no CPU fallback: the package refuses to import when the .so is missing"""
    import shutil
    import subprocess
    import sys
    pkg = tmp_path / "paper_1909_11469_b200"
    shutil.copytree(os.path.join(ROOT, "paper_1909_11469_b200"), pkg,
                    ignore=shutil.ignore_patterns("*.so", "csrc", "__pycache__"))
    r = subprocess.run([sys.executable, "-c", "import paper_1909_11469_b200"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "build the CUDA extension" in r.stderr


def test_host_philox_known_answer(bp):
    """The host restatement of the device draw (bp_philox_u53, used by the
    band fallback) on Random123's first philox4x32-10 known-answer vector
    (counter 0, key 0 -> 6627e8d5 e169c58d bc57ac4c 9b00dbd8): edge pair 0,
    iteration 0, attempt 0, seed 0; d = 0 takes words 0-1, d = 1 words 2-3."""
    assert bp.philox_u53(0, 0, 0, 0) == ((0x6627E8D5 << 32) | 0xE169C58D) >> 11
    assert bp.philox_u53(0, 0, 0, 1) == ((0xBC57AC4C << 32) | 0x9B00DBD8) >> 11


def test_host_er_arrays_equal_reference_style_generator(bp, orc):
    """bp_generate_er_arrays: the ER instance the oracle builds."""
    for n, m, c, seed in ((10, 12, 2.5, 0), (500, 900, 2.0, 3)):
        cards, un, ep, tb = bp.generate_er_arrays(n, m, c, seed)
        a = po.Graph.er(orc, n, m, c, seed).arrays()
        assert np.array_equal(cards, a.cardinalities) and np.array_equal(ep.reshape(-1), a.endpoints.reshape(-1))
        assert np.array_equal(un, a.unary) and np.array_equal(tb, a.tables)
