"""Two consecutive runs on one graph: both must run the same iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

for kind_name, maker in (("potts2048", lambda: bp.generate_potts(2048, 8, 2.5, 0)),
                         ("potts4096", lambda: bp.generate_potts(4096, 8, 2.5, 0)),
                         ("ising4096", lambda: bp.generate_ising(bp.IsingParams(n=4096, c=2.5, seed=0)))):
    g = maker()
    for kind in (bp.SchedulerKind.lbp, bp.SchedulerKind.rnbp):
        cfg = bp.SchedulerConfig(kind=kind, low_p=0.5, max_iterations=20, time_limit=60)
        out = []
        for _ in range(2):
            r = bp.run_ex(g, cfg, beliefs=False)
            out.append((r.iterations, r.converged, r.messages_updated_total, round(r.device_ms, 1)))
        print(kind_name, kind, out, flush=True)
    del g
