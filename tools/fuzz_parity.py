"""Randomised parity fuzz against the oracle: random model families / sizes /
schedulers / parameters.  Every run must match the reference's verdict and
marginals (1e-4; RnBP 2e-4, the reference's own seed-to-seed spread being
~1e-4); deterministic schedulers also its iteration count within 2% (+-1):
RBP / RS pick top-k by fp32 residuals, so near-ties in the fp64 order can
select other edges and long runs drift by a few iterations.
usage: python tools/fuzz_parity.py [CASES] [SEED]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from tests.helpers import Stream, flatten, lattice_arrays, oracle_config, random_graph  # noqa: E402

orc = po.load()
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
K = bp.SchedulerKind
bad = 0
t0 = time.time()
worst = {"lbp": [0.0, 0.0], "rbp": [0.0, 0.0], "rs": [0.0, 0.0], "rnbp": [0.0, 0.0]}  # max diff, max iteration drift
for i in range(cases):
    fam = rng.choice(["ising", "lattice", "potts", "random", "er"])
    s = int(rng.integers(1, 10**6))
    if fam == "ising":
        n = int(rng.integers(2, 50)); c = float(rng.uniform(0.5, 2.5))
        dg, og, desc = bp.generate_ising(bp.IsingParams(n=n, c=c, seed=s)), po.Graph.ising(orc, n, c, s), f"ising n={n} c={c:.2f}"
    elif fam == "lattice":
        r, cc = int(rng.integers(1, 40)), int(rng.integers(2, 70)); c = float(rng.uniform(0.5, 2.0))
        a = lattice_arrays(orc, r, cc, s, c)
        dg, og, desc = bp.PairwiseMRF.from_arrays(*a), po.Graph.from_arrays(orc, *a), f"lattice {r}x{cc} c={c:.2f}"
    elif fam == "potts":
        n, q = int(rng.integers(3, 30)), int(rng.integers(2, 10)); c = float(rng.uniform(0.3, 1.5))
        dg, og, desc = bp.generate_potts(n, q, c, s), po.Graph.potts(orc, n, q, c, s), f"potts n={n} q={q} c={c:.2f}"
    elif fam == "random":
        n, mq = int(rng.integers(5, 150)), int(rng.integers(2, 6))
        cards, un, edges = random_graph(Stream(orc, s), n, mq, float(rng.uniform(0.0, 0.1)))
        a = flatten(cards, un, edges)
        dg, og, desc = bp.PairwiseMRF.from_arrays(*a), po.Graph.from_arrays(orc, *a), f"random n={n} maxq={mq}"
    else:
        n = int(rng.integers(50, 5000)); m = int(n * rng.uniform(1.0, 2.5)); c = float(rng.uniform(0.5, 2.5))
        dg, og, desc = bp.generate_er(n, m, c, s), po.Graph.er(orc, n, m, c, s), f"er n={n} m={m} c={c:.2f}"
    kind = rng.choice(["lbp", "rbp", "rs", "rnbp"])
    kw = {}
    if kind == "rbp":
        kw["p"] = float(10 ** rng.uniform(-3, 0))
    elif kind == "rs":
        kw["p"] = float(10 ** rng.uniform(-2.5, 0)); kw["splash_depth"] = int(rng.integers(1, 4))
    elif kind == "rnbp":
        kw["low_p"] = float(rng.uniform(0.1, 1.0))
    cfg = bp.SchedulerConfig(kind=getattr(K, kind), max_iterations=2000, seed=int(rng.integers(0, 1000)), **kw)
    r = bp.run(dg, cfg)
    o = po.run(og, oracle_config(cfg))
    both = r.converged and o.converged
    diff = float(np.max(np.abs(r.beliefs.values - o.beliefs), initial=0.0))
    drift = abs(r.iterations - o.iterations) / max(o.iterations, 1)
    if both:
        worst[kind][0] = max(worst[kind][0], diff)
    worst[kind][1] = max(worst[kind][1], drift)
    if kind == "rnbp":
        flag = r.converged != o.converged or (both and diff > 2e-4)
    else:
        flag = (r.converged != o.converged or (abs(r.iterations - o.iterations) > 1 and drift > 0.02) or
                (both and diff > 1e-4))
    bad += flag
    if flag or i % 25 == 0:
        print(f"{i:4d} {desc:34s} {kind:4s} {kw} device {r.converged} {r.iterations} | oracle {o.converged} "
              f"{o.iterations} | diff {diff:.1e} {'<-- MISMATCH' if flag else ''}", flush=True)
print(f"cases {cases} mismatches {bad} in {time.time() - t0:.0f} s")
print("per scheduler: max converged-marginal diff, max relative iteration drift:",
      {k: (f"{v[0]:.1e}", f"{v[1]:.3f}") for k, v in worst.items()})
