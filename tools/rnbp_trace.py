"""Per-iteration timing of one RnBP run from the device trace (globaltimer)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g = bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=seed))
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=10000, time_limit=1e9, seed=seed)
bp.run(g, cfg)
r = bp.run(g, cfg)
t = np.array([x.elapsed_seconds for x in r.trace])
f = np.array([x.frontier_size for x in r.trace])
u = np.array([x.unconverged for x in r.trace])
dt = np.diff(np.concatenate([[0.0], t])) * 1e6
print(f"n={n} iterations={r.iterations} device_ms={r.device_ms:.1f} launches={r.gpu_launches}")
for a, b in ((0, 10), (10, 100), (100, 1000), (1000, 5000), (5000, 10000)):
    if a >= len(dt):
        break
    s = slice(a, min(b, len(dt)))
    print(f"iters {a:5d}-{b:5d}: us/iter median {np.median(dt[s]):7.2f} mean {dt[s].mean():7.2f}  "
          f"frontier median {np.median(f[s]):9.0f}  unconverged median {np.median(u[s]):9.0f}")
rk = bp.run_ex(g, cfg, kernel_timing=True)
print({k: (round(v["ms"], 2), v["launches"]) for k, v in rk.kernel_stats.items() if v["launches"]})
