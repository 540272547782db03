"""Potts 4096^2 q=8 RnBP dense window: kernel classes per iteration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

g = bp.generate_potts(4096, 8, 2.5, 0)
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, high_p=1.0, max_iterations=20, time_limit=1e9, seed=1)
bp.run_ex(g, cfg, beliefs=False)
r = bp.run_ex(g, cfg, beliefs=False)
print(f"graph mode: {r.device_ms / r.iterations:.3f} ms per iteration, visits {r.vertex_visits}, evals {r.message_evaluations}")
k = bp.run_ex(g, cfg, beliefs=False, kernel_timing=True).kernel_stats
print({a: (round(b["ms"] / 20, 3), b["launches"]) for a, b in k.items() if b["launches"]})
r = bp.run_ex(g, bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, high_p=1.0, max_iterations=3, time_limit=1e9,
                                    seed=1), beliefs=False, kernel_timing=True)
print("3 its:", [(x.iteration, x.frontier_size, x.unconverged) for x in r.trace],
      {a: (round(b["ms"], 3), b["launches"]) for a, b in r.kernel_stats.items() if b["launches"]})
