"""Scheduler x graph-family matrix against the oracle: every scheduler's run()
on lattices (Ising, Potts q = 3..16, dense q-state tables), random mixed-
cardinality graphs and ER graphs; prints one line per case and flags a case
where the verdicts differ or converged marginals are more than 1e-4 apart."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from tests.helpers import Stream, flatten, lattice_arrays, oracle_config, random_graph  # noqa: E402

orc = po.load()


def dense_q_lattice(rows, cols, q, seed):
    _, _, ep, _ = lattice_arrays(orc, rows, cols, seed, 1.0)
    rng = np.random.default_rng(seed)
    V, E = rows * cols, ep.shape[0]
    un = np.exp(rng.uniform(-1, 1, V * q))
    tb = np.exp(rng.uniform(-1, 1, E * q * q))
    return np.full(V, q, np.uint32), un, ep, tb


cases = []
for q in (3, 5, 8, 16):
    cases.append((f"potts16_q{q}", lambda q=q: (bp.generate_potts(16, q, 1.0, q), po.Graph.potts(orc, 16, q, 1.0, q))))
for q in (3, 8):
    def mk(q=q):
        a = dense_q_lattice(12, 19, q, 7 + q)
        return bp.PairwiseMRF.from_arrays(*a), po.Graph.from_arrays(orc, *a)
    cases.append((f"dense12x19_q{q}", mk))
def rg():
    cards, un, edges = random_graph(Stream(orc, 11), 60, 4, 0.05)
    a = flatten(cards, un, edges)
    return bp.PairwiseMRF.from_arrays(*a), po.Graph.from_arrays(orc, *a)
cases.append(("random60", rg))
cases.append(("er3000", lambda: (bp.generate_er(3000, 6000, 2.0, 4), po.Graph.er(orc, 3000, 6000, 2.0, 4))))
def lat():
    a = lattice_arrays(orc, 17, 41, 3, 1.5)
    return bp.PairwiseMRF.from_arrays(*a), po.Graph.from_arrays(orc, *a)
cases.append(("ising17x41", lat))
cases.append(("ising30", lambda: (bp.generate_ising(bp.IsingParams(n=30, c=2.0, seed=2)), po.Graph.ising(orc, 30, 2.0, 2))))

if "--big" in sys.argv:  # list mode / persistent tails on q-state and CSR graphs, caps, other thresholds
    cases = [("potts100_q4", lambda: (bp.generate_potts(100, 4, 1.0, 1), po.Graph.potts(orc, 100, 4, 1.0, 1))),
             ("potts90_q8", lambda: (bp.generate_potts(90, 8, 1.5, 2), po.Graph.potts(orc, 90, 8, 1.5, 2))),
             ("er30000", lambda: (bp.generate_er(30000, 60000, 2.0, 5), po.Graph.er(orc, 30000, 60000, 2.0, 5))),
             ("ising100_c2.5", lambda: (bp.generate_ising(bp.IsingParams(n=100, c=2.5, seed=501)),
                                        po.Graph.ising(orc, 100, 2.5, 501)))]
    EXTRA = [("rnbp_eps1e-3", {"low_p": 0.5, "epsilon": 1e-3}), ("lbp_eps1e-8", {"epsilon": 1e-8}),
             ("rbp_p1/64", {"p": 1 / 64}), ("rnbp_eps1e-8", {"low_p": 0.5, "epsilon": 1e-8})]
else:
    EXTRA = []
scheds = [("lbp", {}), ("rbp", {"p": 0.25}), ("rs", {"p": 0.25, "splash_depth": 2}), ("rs_h4", {"p": 0.1, "splash_depth": 4}),
          ("rnbp", {"low_p": 0.5}), ("rnbp_p07", {"low_p": 0.7})] + EXTRA
bad = 0
for name, mk in cases:
    dg, og = mk()
    for sname, kw in scheds:
        kind = sname.split("_")[0]
        cap = 2000 if "--big" in sys.argv else 3000
        cfg = bp.SchedulerConfig(kind=getattr(bp.SchedulerKind, kind), max_iterations=cap, seed=5, **kw)
        try:
            r = bp.run(dg, cfg)
        except Exception as e:  # noqa: BLE001
            print(f"{name:16s} {sname:9s} DEVICE ERROR {e}")
            bad += 1
            continue
        o = po.run(og, oracle_config(cfg))
        diff = float(np.max(np.abs(r.beliefs.values - o.beliefs))) if r.converged and o.converged else float("nan")
        tol = 1e-4 if cfg.epsilon >= 1e-5 else 1e-6
        flag = (r.converged != o.converged) or (r.converged and o.converged and diff > tol)
        flag = flag or (not r.converged and not o.converged and r.iterations != o.iterations)
        bad += flag
        print(f"{name:16s} {sname:9s} device {r.converged!s:5s} {r.iterations:5d} | oracle {o.converged!s:5s} "
              f"{o.iterations:5d} | belief diff {diff:.2e} {'<-- MISMATCH' if flag else ''}")
print("mismatches", bad)
