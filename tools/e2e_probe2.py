import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1909_11469_b200 as bp
arrs = [bp.generate_ising_arrays(bp.IsingParams(n=1000, c=2.5, seed=s)) for s in range(4)]
cfg = lambda s: bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=10000, time_limit=1e9, seed=s)
for s in range(4):
    cards, un, ep, tb = arrs[s]
    t0 = time.perf_counter(); g = bp.PairwiseMRF.from_arrays(cards, un, ep, tb); t1 = time.perf_counter()
    r = bp.run(g, cfg(s)); t2 = time.perf_counter(); del g; t3 = time.perf_counter()
    print(f"seed {s}: graph {1e3*(t1-t0):.1f} run {1e3*(t2-t1):.1f} (device {r.device_ms:.1f}) del {1e3*(t3-t2):.1f} ms", flush=True)
