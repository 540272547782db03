"""One short run of the engine for ncu: kernels launched directly (no CUDA
graph) so every launch is visible to the profiler."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1000)
ap.add_argument("--kind", default="rnbp")
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--potts", type=int, default=0, help="q > 0: Potts grid with q states")
ap.add_argument("--graphs", action="store_true")
ap.add_argument("--er", action="store_true", help="Erdos-Renyi G(n, 2n) instead of a grid")
a = ap.parse_args()
g = (bp.generate_er(a.n, 2 * a.n, 2.5, 0) if a.er else bp.generate_potts(a.n, a.potts, 2.5, 0) if a.potts else
     bp.generate_ising(bp.IsingParams(n=a.n, c=2.5, seed=0)))
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(a.kind), low_p=0.5, p=1 / 256, max_iterations=a.iters)
r = bp.run_ex(g, cfg, flags=0 if a.graphs else bp.RUN_NO_GRAPHS, batch=a.iters)
print(f"{a.kind} n={a.n} iterations={r.iterations} updates={r.messages_updated_total} device_ms={r.device_ms:.3f}")
