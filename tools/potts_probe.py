"""ms per LBP sweep and per RnBP iteration on the Potts 4096^2 q=8 grid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

g = bp.generate_potts(4096, 8, 2.5, 0)
for kind, it in ((bp.SchedulerKind.lbp, 20), (bp.SchedulerKind.rnbp, 20)):
    cfg = bp.SchedulerConfig(kind=kind, low_p=0.5, max_iterations=it, time_limit=1e9)
    bp.run_ex(g, cfg, beliefs=False)
    r = bp.run_ex(g, cfg, beliefs=False)
    print(f"potts 4096^2 q=8 {kind}: {r.device_ms / max(1, r.iterations):.3f} ms/iter")
