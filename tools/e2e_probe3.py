"""e2e steps exactly as bench.py times them (L2 flush, graph from host arrays, run, beliefs), 8 seeds."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
arrs = {s: bp.generate_ising_arrays(bp.IsingParams(n=1000, c=2.5, seed=s)) for s in range(8)}
cfg = lambda s, it=10000: bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=it,
                                              time_limit=1e9, seed=s)
bp.run(bp.PairwiseMRF.from_arrays(*arrs[0]), cfg(0, 10))
for s in range(8):
    flush.zero_(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = bp.PairwiseMRF.from_arrays(*arrs[s])
    t1 = time.perf_counter()
    r = bp.run(g, cfg(s))
    t2 = time.perf_counter()
    _ = r.beliefs.values.sum()
    t3 = time.perf_counter()
    del g
    t4 = time.perf_counter()
    print(f"seed {s}: graph {1e3*(t1-t0):6.1f} run {1e3*(t2-t1):6.1f} (device {r.device_ms:6.1f}) "
          f"sum {1e3*(t3-t2):4.1f} del {1e3*(t4-t3):5.1f} ms", flush=True)
