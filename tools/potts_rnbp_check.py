"""RnBP on a small Potts lattice against the oracle: converged / iterations /
updates and the trace around the stall (debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from tests.helpers import oracle_config  # noqa: E402

n, q, c, seed, lp = 16, 3, 1.0, 1, 0.5
if len(sys.argv) > 1:
    n, q, c, seed, lp = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5])
orc = po.load()
g = bp.generate_potts(n, q, c, seed)
og = po.Graph.potts(orc, n, q, c, seed)
for kind in ("rnbp", "lbp", "rbp"):
    cfg = bp.SchedulerConfig(kind=getattr(bp.SchedulerKind, kind), low_p=lp, p=0.25, max_iterations=300, seed=seed)
    r = bp.run(g, cfg)
    o = po.run(og, oracle_config(cfg))
    print(kind, "device converged", r.converged, "its", r.iterations, "| oracle", o.converged, o.iterations,
          "| max belief diff", float(np.max(np.abs(r.beliefs.values - o.beliefs))))
    if kind == "rnbp":
        print([(x.iteration, x.frontier_size, x.unconverged) for x in r.trace[8:40]])
        de = bp.EngineState(g, cfg)
        oe = po.Engine(og, oracle_config(cfg))
        print("t0 unconverged device", de.unconverged_count(), "oracle", oe.unconverged)
        dr, orr = de.residuals(), oe.residuals()
        print("residual max diff at t0", float(np.max(np.abs(dr - orr))))
