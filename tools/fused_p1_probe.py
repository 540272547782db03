"""Fused sweep cost with and without Philox draws (p = 1: every survivor commits, no draw)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
g = bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=0))
bel = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
for lp, hp in ((0.5, 0.5), (1.0, 1.0)):
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=lp, high_p=hp, max_iterations=20, time_limit=1e9, seed=0)
    for _ in range(3):
        r = bp.run_ex(g, cfg, beliefs_device_ptr=bel.data_ptr())
    k = bp.run_ex(g, cfg, kernel_timing=True, beliefs_device_ptr=bel.data_ptr()).kernel_stats["fused"]
    print(f"p={lp}: run {r.device_ms:.3f} ms, fused {k['ms'] / 20 * 1e3:.1f} us per sweep")
