"""racecheck repro: RBP on the flagged chain of test_gpu_numeric, with and without CUDA graphs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

n = 12
un = np.array([0.7, 0.3] + [1.0, 1.0] * (n - 2) + [0.7, 0.3])
ep = np.array([(v, v + 1) for v in range(n - 1)], np.uint32)
tb = np.array([1.0, 1e-200, 1e-200, 1.0] * (n - 1))
g = bp.PairwiseMRF.from_arrays(np.full(n, 2, np.uint32), un, ep, tb)
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rbp, p=0.25, max_iterations=2000)
flags = bp.RUN_NO_GRAPHS if sys.argv[1:] == ["nographs"] else 0
r = bp.run_ex(g, cfg, flags=flags)
print("converged", r.converged, r.iterations)
