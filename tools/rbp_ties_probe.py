"""Residual distribution at the RBP top-k threshold (1000^2, p = 1/256): how
many edges share the k-th key, how many residuals are exactly zero."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

g = bp.generate_ising(bp.IsingParams(n=1000, c=2.5, seed=0))
de = bp.EngineState(g, bp.SchedulerConfig(kind=bp.SchedulerKind.rbp, p=1 / 256, max_iterations=1000))
done = 0
for t in (0, 1, 10, 100, 300):
    while done < t:
        de.step()
        done += 1
    r = de.residuals()
    k = int(round(r.size / 256))
    kth = np.partition(r, r.size - k)[r.size - k]
    print(f"it {t}: k {k} kth {kth:.3e} ties {(r == kth).sum()} above {(r > kth).sum()} zeros {(r == 0).sum()} "
          f"nonzero {(r > 0).sum()}", flush=True)
