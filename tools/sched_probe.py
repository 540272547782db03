"""Kernel-class breakdown of one scheduler run on the 1000^2 Ising grid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "rbp"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
g = bp.generate_ising(bp.IsingParams(n=1000, c=2.5, seed=0))
K = bp.SchedulerKind
cfg = {"rbp": bp.SchedulerConfig(kind=K.rbp, p=1 / 256, max_iterations=iters, time_limit=1e9),
       "rs": bp.SchedulerConfig(kind=K.rs, p=1 / 256, splash_depth=2, max_iterations=iters, time_limit=1e9),
       "lbp": bp.SchedulerConfig(kind=K.lbp, max_iterations=iters, time_limit=1e9)}[kind]
bp.run_ex(g, cfg, beliefs=False)
r = bp.run_ex(g, cfg, beliefs=False)
print(f"{kind}: iterations {r.iterations} device {r.device_ms:.2f} ms = {1e3 * r.device_ms / max(1, r.iterations):.1f} us/iter")
rk = bp.run_ex(g, cfg, beliefs=False, kernel_timing=True)
print({k: (round(v["ms"], 2), v["launches"]) for k, v in rk.kernel_stats.items() if v["launches"]})
