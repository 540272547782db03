"""Regression check of the main device numbers (one JSON line): headline
window (RnBP 1000^2, 20 iterations), LBP us/iteration at 1000^2, LBP ms/sweep
at 16384^2 (TMA) and Potts 4096^2 q=8."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_11469_b200 as bp  # noqa: E402

out = {}
bel = torch.empty(2 * 16384 * 16384 // 8, dtype=torch.float64, device="cuda")
g = bp.generate_ising(bp.IsingParams(n=1000, c=2.5, seed=0))
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=20, time_limit=1e9)
for _ in range(3):
    r = bp.run_ex(g, cfg, beliefs_device_ptr=bel.data_ptr())
out["window20_ms"] = min(bp.run_ex(g, cfg, beliefs_device_ptr=bel.data_ptr()).device_ms for _ in range(5))
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=2000, time_limit=1e9)
bp.run_ex(g, cfg, beliefs=False)
r = bp.run_ex(g, cfg, beliefs=False)
out["lbp1000_us_per_it"] = r.device_ms / (r.iterations + 1) * 1e3
del g
if "--big" in sys.argv:
    g = bp.generate_ising(bp.IsingParams(n=16384, c=2.5, seed=0))
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=30, time_limit=1e9)
    bp.run_ex(g, cfg, beliefs=False)
    r = bp.run_ex(g, cfg, beliefs=False)
    out["lbp16k_ms_per_sweep"] = r.device_ms / (r.iterations + 1)
    del g
    g = bp.generate_potts(4096, 8, 2.5, 0)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=10, time_limit=1e9)
    bp.run_ex(g, cfg, beliefs=False)
    r = bp.run_ex(g, cfg, beliefs=False)
    out["potts4096_ms_per_sweep"] = r.device_ms / (r.iterations + 1)
print(json.dumps({k: round(v, 4) for k, v in out.items()}))
