import sys, time, numpy as np
sys.path.insert(0,'.')
import paper_1909_11469_b200 as bp
for n in (100, 1000):
    g = bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=0))
    for kind, kw in (("lbp", {}), ("rnbp", dict(low_p=0.5)), ("rbp", dict(p=1/256))):
        cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(kind), max_iterations=1000 if n==1000 else 10000, **kw)
        bp.run(g, cfg)
        t=time.time(); r = bp.run(g, cfg); t=time.time()-t
        print(n, kind, r.converged, r.iterations, f"wall {r.wall_time:.4f} dev {r.device_ms:.2f}ms upd/s {r.messages_updated_total/r.wall_time:.3e} evals {r.message_evaluations}", flush=True)
        rk = bp.run_ex(g, cfg, kernel_timing=True)
        print("   timing", {k:(round(v['ms'],3), v['launches']) for k,v in rk.kernel_stats.items() if v['launches']}, flush=True)
