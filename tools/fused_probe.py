"""RnBP 1000^2 window: fused vs two-launch, device ms per run and kernel shares."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=0))
bel = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=iters, time_limit=1e9, seed=0)
for name, fl in (("fused", 0), ("two-launch", bp.RUN_NO_FUSED)):
    for rep in range(4):
        r = bp.run_ex(g, cfg, flags=fl, beliefs_device_ptr=bel.data_ptr())
    print(f"{name}: device {r.device_ms:.3f} ms for {r.iterations} its ({r.device_ms / r.iterations * 1e3:.1f} us/it), "
          f"launches {r.gpu_launches}, updates {r.messages_updated_total}")
    k = bp.run_ex(g, cfg, flags=fl, kernel_timing=True, beliefs_device_ptr=bel.data_ptr()).kernel_stats
    print("   ", {a: (round(b["ms"], 3), b["launches"]) for a, b in k.items() if b["launches"]})
