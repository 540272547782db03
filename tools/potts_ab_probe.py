"""Potts 4096^2 q=8 RnBP 20-iteration window: device ms per iteration, select /
refresh ms per iteration, and a checksum of the run (updates, frontier trace,
beliefs) so two builds (BPB_LIB) can be compared bit for bit."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
q = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = bp.generate_potts(n, q, 2.5, 0)
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, high_p=1.0, max_iterations=20, time_limit=1e9, seed=1)
bel = torch.empty(q * n * n, dtype=torch.float64, device="cuda")
ms = []
for _ in range(5):
    r = bp.run_ex(g, cfg, beliefs_device_ptr=bel.data_ptr())
    ms.append(r.device_ms)
k = bp.run_ex(g, cfg, beliefs=False, kernel_timing=True).kernel_stats
print(json.dumps({"lib": os.environ.get("BPB_LIB", "in-tree"), "n": n, "q": q,
                  "ms_per_it": min(ms) / r.iterations, "classes_ms_per_it": {a: round(b["ms"] / r.iterations, 4)
                                                                      for a, b in k.items() if b["launches"]},
                  "updates": r.messages_updated_total, "trace": sum((i + 1) * x.frontier_size for i, x in enumerate(r.trace)),
                  "belief_sum": float((bel * torch.arange(bel.numel(), device="cuda", dtype=torch.float64).remainder(97)).sum().item())}))
