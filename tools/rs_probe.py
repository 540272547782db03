"""One Residual-Splash run on ER(1M, 2M) for profiling."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5
g = bp.generate_er(1_000_000, 2_000_000, 2.5, 0)
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rs, p=1 / 128, splash_depth=2, max_iterations=iters, time_limit=1e9)
fl = bp.RUN_NO_GRAPHS if "--nograph" in sys.argv else 0
bp.run_ex(g, cfg, beliefs=False, flags=fl)
r = bp.run_ex(g, cfg, beliefs=False, flags=fl)
print(f"rs er1M iterations={r.iterations} device_ms={r.device_ms:.2f} ms/iter={r.device_ms / max(1, r.iterations):.3f} "
      f"splashes={r.splashes} rounds={r.splash_rounds} updates={r.messages_updated_total}")
