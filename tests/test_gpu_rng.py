"""The device random stream of RnBP (rnbp_frontier, schedulers.cpp:194-216).

The reference draws uniform_unit(mt19937_64) per survivor in id order
(rng.hpp:11-13, schedulers.cpp:207-209); the device draws Philox4x32-10 keyed
by (seed, iteration, attempt, edge) so frontiers do not depend on launch
shape or GPU count.  Pinned here:
* the device Philox4x32-10 against the published Random123 known-answer
  vectors (kat_vectors, philox4x32 R=10);
* the host restatement used by the band fallback equals the device draw;
* the Bernoulli(p) selection concentrates like the reference's
  (test_schedulers.cpp:271-292);
* the device EdgeRatio rule (schedulers.cpp:218-224, 326-327) from run traces:
  on iterations where the rule picks high_p = 1 the frontier is exactly the
  start-of-iteration unconverged set."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# Random123 kat_vectors: philox4x32 10 <ctr0..3> <key0..1> -> <out0..3>
KAT = [
    ((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
     (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff, 0xffffffff, 0xffffffff, 0xffffffff), (0xffffffff, 0xffffffff),
     (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
]


def test_device_philox_known_answers(bp):
    ctr = np.array([k[0] for k in KAT], np.uint32)
    key = np.array([k[1] for k in KAT], np.uint32)
    out = bp.philox4x32_10_device(ctr, key)
    assert out.tolist() == [list(k[2]) for k in KAT]


def test_host_draw_equals_device_draw(bp):
    rng = np.random.default_rng(5)
    for seed, it, att in [(0, 0, 0), (17, 3, 1), (2**40 + 7, 2**33 + 5, 2), (123, 9999, 0)]:
        d = rng.integers(0, 2**40, size=2000, dtype=np.uint64)
        dev = bp.philox_u53_device(seed, it, att, d)
        host = np.array([bp.philox_u53(seed, it, att, int(x)) for x in d], np.uint64)
        assert np.array_equal(dev, host)


def test_draws_are_uniform(bp):
    d = np.arange(1 << 20, dtype=np.uint64)
    u = bp.philox_u53_device(3, 1, 0, d).astype(np.float64) * 2.0 ** -53
    assert u.min() >= 0.0 and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 5 * np.sqrt(1 / 12 / u.size)
    hist = np.bincount((u * 64).astype(np.int64), minlength=64)
    exp = u.size / 64
    chi2 = float(np.sum((hist - exp) ** 2 / exp))
    assert chi2 < 120  # 63 dof: p ~ 3e-5


def test_frontier_sizes_concentrate_around_p_survivors(bp):
    """test_schedulers.cpp:271-292 on the device: chain(501), p = 0.4, 100
    seeds; >= 97 sizes within 3 standard deviations of p * survivors."""
    g = bp.generate_chain(bp.ChainParams(length=501, c=2.0, seed=42))
    p = 0.4
    in_range = 0
    for seed in range(100):
        e = bp.EngineState(g, bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, seed=seed))
        survivors = int(np.sum(e.residuals() >= 1e-5))
        assert survivors > 900
        f = e.rnbp_frontier(p)
        assert np.all(e.residuals()[f] >= 1e-5)  # never a converged message
        mean, sigma = survivors * p, np.sqrt(survivors * p * (1 - p))
        in_range += abs(f.size - mean) <= 3 * sigma
    assert in_range >= 97


@pytest.mark.parametrize("p", [0.05, 0.3, 0.7])
def test_frontier_rate_on_a_large_grid(bp, p):
    """One draw over ~4M survivors: within 5 sigma of p * survivors."""
    g = bp.generate_ising(bp.IsingParams(n=1000, c=2.5, seed=0))
    e = bp.EngineState(g, bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, seed=9))
    survivors = e.unconverged_count()
    f = e.rnbp_frontier(p)
    assert abs(f.size - p * survivors) <= 5 * np.sqrt(survivors * p * (1 - p))


def _edge_ratio_check(trace, low_p, thr=0.9):
    """Replays select_parallelism over a run trace (high_p = 1): returns the
    number of high and low iterations checked."""
    fs = [t.frontier_size for t in trace]
    un = [t.unconverged for t in trace]
    start = [fs[0]] + un[:-1]  # unconverged at the start of iteration t (iteration 0: all survivors selected)
    high = low = 0
    for t in range(len(trace)):
        if t == 0:
            pick_high = True  # prev_unconverged unset (schedulers.cpp:219)
        else:
            pick_high = not (start[t] / start[t - 1] > thr) if start[t - 1] else True
        if pick_high:
            assert fs[t] == start[t], (t, fs[t], start[t])
            high += 1
        else:
            assert fs[t] <= start[t]
            if start[t] >= 2000:  # binomial concentration (retry / fallback only bite on tiny sets)
                assert abs(fs[t] - low_p * start[t]) <= 6 * np.sqrt(start[t] * low_p * (1 - low_p)) + 1, t
            low += 1
    return high, low


@pytest.mark.parametrize("n,c,seed,low_p", [(100, 2.5, 500, 0.5), (300, 2.5, 1, 0.3), (1000, 2.5, 0, 0.5)])
def test_device_edge_ratio_rule_from_traces(bp, n, c, seed, low_p):
    """Both device copies of the rule (the graph loop's select and the
    persistent tail) follow select_parallelism exactly: high_p = 1 iterations
    select precisely the start-of-iteration unconverged set."""
    g = bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed))
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=low_p, high_p=1.0, max_iterations=3000, seed=seed)
    for flags in (0, bp.RUN_NO_PERSIST):
        r = bp.run_ex(g, cfg, flags=flags)
        high, low = _edge_ratio_check(r.trace, low_p)
        assert high >= 1 and low >= 1


def test_advance_iteration_rekeys_the_draws(bp):
    """EngineState::advance_iteration (schedulers.hpp:75): each lockstep
    iteration draws with its own Philox keys, so the frontier stays a
    Bernoulli(p) sample of the survivors (without advancing, the edges left
    out once would be left out again)."""
    g = bp.generate_ising(bp.IsingParams(n=300, c=2.5, seed=4))
    de = bp.EngineState(g, bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, seed=5))
    for t in range(4):
        s = de.unconverged_count()
        f = de.rnbp_frontier(0.5)
        assert abs(len(f) - s / 2) < 6 * np.sqrt(s / 4), (t, len(f), s)
        assert de.iteration() == t
        de.apply_frontier(f)
        de.advance_iteration()
