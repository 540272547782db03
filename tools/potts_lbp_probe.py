"""Potts 4096^2 q=8 LBP: lanes-over-states sweep vs the vertex kernel, ms per sweep."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = bp.generate_potts(n, 8, 2.5, 0)
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=10, time_limit=1e9)
for name, fl in (("auto (lanes)", 0), ("vertex", bp.RUN_LBP_VERTEX)):
    bp.run_ex(g, cfg, flags=fl, beliefs=False)
    r = bp.run_ex(g, cfg, flags=fl, beliefs=False, kernel_timing=True)
    k = r.kernel_stats["update"]
    print(f"{name}: {k['ms'] / k['launches']:.3f} ms per sweep over {k['launches']} sweeps")
for name, fl in (("auto (lanes)", 0), ("vertex", bp.RUN_LBP_VERTEX)):
    for it in (10, 40):
        c2 = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=it, time_limit=1e9)
        r = bp.run_ex(g, c2, flags=fl, beliefs=False)
        r = bp.run_ex(g, c2, flags=fl, beliefs=False)
        print(f"graph mode {name} {it} its: {r.device_ms / (r.iterations + 1):.3f} ms per sweep")
