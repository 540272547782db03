"""Headline-window timing probe: RnBP 1000^2 C=2.5 run() capped at N iterations,
persistent loop kernels vs the per-kernel graph loop; LBP us/iteration.
BPB_DEBUG_PHASES=1 prints the loop kernels' phase clocks."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_11469_b200 as bp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
gs = [bp.generate_ising(bp.IsingParams(n=n, c=2.5, seed=s)) for s in range(4)]
bel = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
for iters in (20, 100, 10000):
    for flags, name in ((0, "loops"), (bp.RUN_NO_PERSIST, "graph")):
        out = []
        for rep in range(2):
            for s, g in enumerate(gs):
                cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=iters, time_limit=1e9, seed=s)
                t = time.perf_counter()
                r = bp.run_ex(g, cfg, flags=flags, beliefs_device_ptr=bel.data_ptr())
                w = time.perf_counter() - t
                out.append(f"{r.device_ms:.3f}/{w*1e3:.2f}")
        print(f"rnbp iters={iters} {name}: device_ms/wall_ms {' '.join(out)}  its={r.iterations} upd={r.messages_updated_total} launches={r.gpu_launches}", flush=True)
for flags, name in ((0, "loops"), (bp.RUN_NO_PERSIST, "graph")):
    r = bp.run_ex(gs[0], bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=20, time_limit=1e9),
                  kernel_timing=True, flags=flags, beliefs_device_ptr=bel.data_ptr())
    print(f"rnbp20 {name} kernel stats", {k: (round(v["ms"], 3), v["launches"]) for k, v in r.kernel_stats.items() if v["launches"]}, flush=True)
for flags, name in ((0, "loops"), (bp.RUN_NO_PERSIST, "graph")):
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=2000, time_limit=1e9)
    bp.run_ex(gs[0], cfg, flags=flags, beliefs_device_ptr=bel.data_ptr())
    r = bp.run_ex(gs[0], cfg, flags=flags, beliefs_device_ptr=bel.data_ptr())
    print(f"lbp {name}: {r.device_ms / (r.iterations + 1) * 1e3:.2f} us/iteration, its {r.iterations}", flush=True)
    r = bp.run_ex(gs[0], bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=200, time_limit=1e9),
                  kernel_timing=True, flags=flags, beliefs_device_ptr=bel.data_ptr())
    print(f"lbp200 {name} kernel stats", {k: (round(v["ms"], 3), v["launches"]) for k, v in r.kernel_stats.items() if v["launches"]}, flush=True)
