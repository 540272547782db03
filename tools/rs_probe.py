"""Residual Splash device ms per iteration (ER-1M config 3 at p = 1/128 and
1/256, the 1000^2 grid, ER-30000 at h = 3) with a run checksum, to A/B builds
(BPB_LIB)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

out = {"lib": os.environ.get("BPB_LIB", "in-tree")}
er = bp.generate_er(1000000, 2000000, 2.5, 0)
cases = (("er1m_p128", er, 1 / 128, 2, 20), ("er1m_p256", er, 1 / 256, 2, 20),
         ("ising1000_p256", bp.generate_ising(bp.IsingParams(n=1000, c=2.5, seed=0)), 1 / 256, 2, 50),
         ("er30k_h3", bp.generate_er(30000, 60000, 2.0, 5), 0.1, 3, 3))
for name, g, p, h, its in cases:
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rs, p=p, splash_depth=h, max_iterations=its, time_limit=1e9, seed=0)
    ms = []
    for _ in range(3):
        r = bp.run(g, cfg)
        ms.append(r.device_ms)
    out[name] = {"ms_per_it": round(min(ms) / r.iterations, 4), "updates": r.messages_updated_total,
                 "rounds": r.splash_rounds, "bel": float(r.beliefs.values.sum())}
print(json.dumps(out))
