"""Fused sweep: SMEM-staged vs register version, us per sweep."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
it = 20 if n <= 4096 else 10
g = bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=0))
bel = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=it, time_limit=1e9, seed=0)
for name, fl in (("tma", bp.RUN_FUSED_TMA), ("regs", bp.RUN_FUSED_REGS)):
    for _ in range(3):
        r = bp.run_ex(g, cfg, flags=fl, beliefs_device_ptr=bel.data_ptr())
    k = bp.run_ex(g, cfg, flags=fl, kernel_timing=True, beliefs_device_ptr=bel.data_ptr())
    ks = k.kernel_stats["fused"]
    print(f"n={n} {name}: run {r.device_ms:.3f} ms, fused {ks['ms'] / k.fused_iterations * 1e3:.1f} us per sweep "
          f"({ks['bytes'] / (ks['ms'] / 1e3) / 1e9:.0f} GB/s incl. skipped launches)")
