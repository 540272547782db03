"""First trace mismatch between the persistent tail and the graph loop (Potts 4096^2 q=8 RnBP)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = bp.generate_potts(n, 8, 2.5, 0)
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=20, time_limit=60)
b = bp.run_ex(g, cfg, beliefs=False, flags=bp.RUN_NO_PERSIST)
a = bp.run_ex(g, cfg, beliefs=False)
ta = np.stack([a.trace.column(c) for c in ("frontier_size", "unconverged")], 1)
tb = np.stack([b.trace.column(c) for c in ("frontier_size", "unconverged")], 1)
print("iterations", a.iterations, b.iterations, "launches", a.gpu_launches, b.gpu_launches)
m = min(len(ta), len(tb))
bad = np.nonzero(np.any(ta[:m] != tb[:m], axis=1))[0]
print("first mismatch", bad[:5], [(ta[i].tolist(), tb[i].tolist()) for i in bad[:3]])
print("unconverged persist", ta[:, 1].tolist())
print("unconverged graph  ", tb[:, 1].tolist())
