"""Device ms per iteration and kernel shares of one scheduler on an Ising grid:
python tools/sched_probe.py KIND N ITERS [P] [FLAGS]  (KIND: lbp rbp rs rnbp)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

torch.cuda.set_device(0)
kind = sys.argv[1] if len(sys.argv) > 1 else "rbp"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
p = float(sys.argv[4]) if len(sys.argv) > 4 else 1 / 256
fl = int(sys.argv[5]) if len(sys.argv) > 5 else 0
g = bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=0))
bel = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
cfg = bp.SchedulerConfig(kind=getattr(bp.SchedulerKind, kind), p=p, low_p=0.5, max_iterations=iters, time_limit=1e9,
                         seed=0)
for rep in range(3):
    r = bp.run_ex(g, cfg, flags=fl, beliefs_device_ptr=bel.data_ptr())
print(f"{kind} {n}^2: device {r.device_ms:.3f} ms for {r.iterations} its ({r.device_ms / r.iterations * 1e3:.2f} us/it), "
      f"launches {r.gpu_launches}, updates {r.messages_updated_total}")
k = bp.run_ex(g, cfg, flags=fl, kernel_timing=True, beliefs_device_ptr=bel.data_ptr()).kernel_stats
print("   ", {a: (round(b["ms"], 3), b["launches"]) for a, b in k.items() if b["launches"]})
