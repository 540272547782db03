"""ms per LBP iteration (device time of a 2000-iteration run) on n x n Ising grids."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

for n, it in ((1000, 2000), (2048, 1000), (4096, 300), (8192, 100)):
    g = bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=0))
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=it, time_limit=1e9)
    bp.run_ex(g, cfg, beliefs=False)
    r = bp.run_ex(g, cfg, beliefs=False)
    print(f"n={n}: {1e3 * r.device_ms / max(1, r.iterations):.2f} us/iter")
    del g
