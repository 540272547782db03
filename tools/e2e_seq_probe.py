"""The bench's e2e sequence with per-phase timing (find the slow step)."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
kw = lambda s, it=20: dict(low_p=0.5, high_p=1.0, edge_ratio_threshold=0.9, epsilon=1e-5, max_iterations=it,  # noqa
                           time_limit=1e9, seed=s)
K = bp.SchedulerKind.rnbp
graphs = {s: bp.generate_ising(bp.IsingParams(n=1000, c=2.5, seed=s)) for s in range(5)}
bel = torch.empty(2 * 10 ** 6, dtype=torch.float64, device="cuda")
for s in range(3):
    bp.run_ex(graphs[s], bp.SchedulerConfig(kind=K, **kw(s)), beliefs_device_ptr=bel.data_ptr())
for s in range(5):
    flush.zero_()
    bp.run_ex(graphs[s], bp.SchedulerConfig(kind=K, **kw(s)), beliefs_device_ptr=bel.data_ptr())
torch.cuda.synchronize()
host = {s: bp.generate_ising_arrays(bp.IsingParams(n=1000, c=2.5, seed=s)) for s in range(5)}
for s in range(3):
    a = bp.generate_ising_arrays(bp.IsingParams(n=1000, c=2.5, seed=s))
    g = bp.PairwiseMRF.from_arrays(*a)
    r = bp.run(g, bp.SchedulerConfig(kind=K, **kw(s)))
    del g, r
gc.disable()
for s in range(5):
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = bp.PairwiseMRF.from_arrays(*host[s])
    t1 = time.perf_counter()
    r = bp.run(g, bp.SchedulerConfig(kind=K, **kw(s)))
    t2 = time.perf_counter()
    _ = float(r.beliefs.values[-1])
    del g
    t3 = time.perf_counter()
    print(f"step {s}: graph {1e3*(t1-t0):6.2f} run {1e3*(t2-t1):6.2f} (device {r.device_ms:5.2f}) del {1e3*(t3-t2):5.2f}",
          file=sys.stderr, flush=True)
gc.enable()
