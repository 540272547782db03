"""Bulk .pgm ingest (csrc/pgm.cpp) against the reference's
own parse_model / serialize_model (model_io.cpp:98-181, compiled in
oracle/_ref): parsed arrays bit for bit, and the reference's first
parse_error -- message and line -- on malformed text.  Host only, except the
last test (the parsed model run on the device)."""
import numpy as np
import pytest

from oracle import pyoracle as po


def _ref_arrays(ref, text):
    a = po.Graph.parse(ref, text).arrays()
    return a.cardinalities, a.unary, a.endpoints, a.tables


def _same(bp, ref, text):
    mine = bp.parse_model_arrays(text)
    theirs = _ref_arrays(ref, text)
    for m, t in zip(mine, theirs):
        assert np.array_equal(np.asarray(m).reshape(-1), np.asarray(t).reshape(-1))


def test_serialized_generated_models_parse_bit_for_bit(bp, ref):
    for g in (po.Graph.ising(ref, 40, 2.5, 3), po.Graph.chain(ref, 30, 1.5, 1), po.Graph.ising(ref, 1, 1.0, 0)):
        _same(bp, ref, g.serialize())


def test_large_model_takes_the_parallel_path(bp, ref):
    """a 300x300 grid (~8 MB of text, several line-aligned chunks)"""
    text = po.Graph.ising(ref, 300, 2.5, 7).serialize()
    assert len(text) > 4 << 20
    _same(bp, ref, text)


@pytest.mark.parametrize("text", [
    "pgm 3\n2 0\n2 2 2\n0.5 1.5\n1 1 # comment\n2 1\n0 1 1 2 2 1\n1 2 1 0.5 0.5 1\n",
    "# header comment\npgm\t2 1 0\r\n2 3\r\n1e0 2.5E-1\n1 1 1\n0 1 1 2 3 4 5 6\n",  # mixed cardinalities
    "pgm 2 0 0 2 2 1 1 1 1",
    "pgm 0 0 0\n",
])
def test_hand_written_models(bp, ref, text):
    _same(bp, ref, text)


def test_model_errors_come_after_a_clean_parse(bp, ref):
    text = "pgm 2 1 0 2 2 1 1 1 1 1 0 1 1 1 1"  # i > j: build_graph's model_error
    with pytest.raises(po.OracleError, match="i < j"):
        po.Graph.parse(ref, text)
    arrays = bp.parse_model_arrays(text)
    with pytest.raises(bp.ModelError, match="i < j"):
        bp.PairwiseMRF.from_arrays(*arrays)


@pytest.mark.parametrize("text", [
    "",
    "pgx 1 0 0 2 1 1",
    "pgm 1 0 1 2 1 1",                       # unsupported version
    "pgm 2 0 0\n2 0\n1 1\n",                 # cardinality out of range
    "pgm 2 0 0\n2 2\n1 1\n1 x\n",            # bad unary entry
    "pgm 2 0 0\n2 2\n1 1\n1 inf\n",          # non-finite
    "pgm 2 1 0\n2 2\n1 1\n1 1\n0 5 1 1 1 1\n",  # endpoint out of range
    "pgm 2 1 0\n2 2\n1 1\n1 1\n\n0 1 1 1 1\n",  # missing entry: end of input
    "pgm 2 0 0\n2 2\n1 1\n1 1\n7\n",         # trailing token
    "pgm 2 1 0\n2 2\n1 1\n1 1\n0 -1 1 1 1 1\n",
    "pgm 2.5 0 0",
    "pgm 3 1 0\n2 2 3\n1 1\n1 1\n1 1 1\n0 2 1 1 1 1 1 nan\n",  # mixed cards, sequential path
])
def test_parse_errors_match_the_reference(bp, ref, text):
    with pytest.raises(po.OracleError) as theirs:
        po.Graph.parse(ref, text)
    assert theirs.value.code == 8
    with pytest.raises(bp.ParseError) as mine:
        bp.parse_model_arrays(text)
    assert str(mine.value) in str(theirs.value)


def test_parse_error_in_a_large_model_reports_the_first_line(bp, ref):
    lines = po.Graph.ising(ref, 200, 2.5, 2).serialize().splitlines(keepends=True)
    k = len(lines) // 2
    lines[k] = lines[k].replace(" ", " 1e999 ", 1)  # a non-finite entry in the middle
    lines[k + 10] = lines[k + 10].replace(" ", " zz ", 1)
    text = "".join(lines)
    with pytest.raises(po.OracleError) as theirs:
        po.Graph.parse(ref, text)
    with pytest.raises(bp.ParseError) as mine:
        bp.parse_model_arrays(text)
    assert str(mine.value) in str(theirs.value)
    assert mine.value.line == k + 1


@pytest.mark.gpu
def test_parsed_model_runs_like_the_arrays(bp, ref):
    text = po.Graph.ising(ref, 60, 2.5, 11).serialize()
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=3000, seed=2)
    a = bp.run(bp.parse_model(text), cfg)
    b = bp.run(bp.PairwiseMRF.from_arrays(*_ref_arrays(ref, text)), cfg)
    assert a.iterations == b.iterations and np.array_equal(a.beliefs.values, b.beliefs.values)
