"""ms per LBP sweep on the 16384^2 Ising grid (kernel-timed update launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

g = bp.generate_ising(bp.IsingParams(n=16384, c=2.5, seed=0))
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=30, time_limit=1e9)
bp.run_ex(g, cfg, beliefs=False)
for _ in range(2):
    r = bp.run_ex(g, cfg, beliefs=False, kernel_timing=True)
    k = r.kernel_stats["update"]
    print(f"16K LBP {k['ms'] / (r.iterations + 1):.4f} ms/sweep ({k['launches']} launches)")
