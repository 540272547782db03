import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1909_11469_b200 as bp
g = bp.generate_ising(bp.IsingParams(n=1000, c=2.5, seed=2))
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=10000, time_limit=1e9, seed=2)
for rep in range(6):
    r = bp.run_ex(g, cfg, beliefs=(rep % 2 == 0))
    t = r.trace.column("elapsed_seconds"); dt = np.diff(np.concatenate([[0.0], t])) * 1e6
    w = [(0, 100), (100, 1000), (1000, 5000), (5000, 10000)]
    print(f"device {r.device_ms:7.1f} ms last-iter-at {t[-1]*1e3:7.1f} ms first {t[0]*1e6:7.1f} us", " ".join(f"[{a}-{b}] sum {dt[a:b].sum()/1e3:6.1f} ms max {dt[a:b].max():8.1f}us" for a, b in w))
