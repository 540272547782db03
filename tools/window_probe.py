"""RnBP window on an Ising grid: best device ms per iteration over repeats, plus a
checksum of the run (updates, beliefs) so two builds can be compared bit for bit.

usage: [BPB_LIB=path/to/libbp_b200.so] python tools/window_probe.py N ITERS [REPEATS]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 7
g = bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=0))
bel = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=iters, time_limit=1e9, seed=0)
ms = []
for rep in range(reps):
    r = bp.run_ex(g, cfg, beliefs_device_ptr=bel.data_ptr())
    ms.append(r.device_ms)
k = bp.run_ex(g, cfg, kernel_timing=True, beliefs_device_ptr=bel.data_ptr()).kernel_stats
print(json.dumps({"lib": os.environ.get("BPB_LIB", "in-tree"), "n": n, "iterations": r.iterations,
                  "us_per_it_best": min(ms) / r.iterations * 1e3, "us_per_it_median": sorted(ms)[len(ms) // 2] / r.iterations * 1e3,
                  "fused_ms": round(k.get("fused", {}).get("ms", 0.0), 4),
                  "updates": r.messages_updated_total, "belief_sum": float(bel.sum().item()),
                  "belief_l1": float(bel.abs().sum().item())}))
