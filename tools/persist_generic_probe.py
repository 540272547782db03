import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1909_11469_b200 as bp
K = bp.SchedulerKind
cases = [("er", bp.generate_er(20000, 40000, 2.5, 1)), ("potts", bp.generate_potts(64, 4, 1.5, 2)), ("potts8", bp.generate_potts(48, 8, 1.0, 5))]
for name, g in cases:
    if g is None:
        print(name, "skipped"); continue
    cfg = bp.SchedulerConfig(kind=K.rnbp, low_p=0.5, max_iterations=3000, seed=3)
    a = bp.run(g, cfg); b = bp.run_ex(g, cfg, flags=bp.RUN_NO_PERSIST)
    print(name, a.iterations, a.converged, "same", a.trace_signature() == b.trace_signature(),
          "maxdiff", float(np.max(np.abs(a.beliefs.values - b.beliefs.values))), "launches", a.gpu_launches, b.gpu_launches)
