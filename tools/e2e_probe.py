"""Stage times of the end-to-end call (graph from host arrays, run, beliefs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

cards, un, ep, tb = bp.generate_ising_arrays(bp.IsingParams(n=1000, c=2.5, seed=0))
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=10000, time_limit=1e9)
for rep in range(3):
    t0 = time.perf_counter()
    g = bp.PairwiseMRF.from_arrays(cards, un, ep, tb)
    t1 = time.perf_counter()
    r = bp.run(g, cfg)
    t2 = time.perf_counter()
    s = r.beliefs.values.sum()
    t3 = time.perf_counter()
    del g
    print(f"graph {1e3 * (t1 - t0):.1f} ms  run {1e3 * (t2 - t1):.1f} ms (device {r.device_ms:.1f})  "
          f"beliefs {1e3 * (t3 - t2):.1f} ms")
