import paper_1909_11469_b200 as bp, numpy as np
for n, c, p in [(12, 1.0, 0.1), (16, 1.5, 0.1), (20, 2.0, 0.05), (30, 2.0, 0.05), (24, 1.0, 0.03)]:
    g = bp.generate_ising(bp.IsingParams(n=n, c=c, seed=3))
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=p, high_p=p, max_iterations=3000, seed=3)
    r = bp.run(g, cfg); b = bp.run_ex(g, cfg, flags=bp.RUN_NO_PERSIST)
    f = np.array([x.frontier_size for x in r.trace]); u = np.array([x.unconverged for x in r.trace])
    print(n, c, p, r.iterations, r.converged, "f==1:", int((f == 1).sum()), "u<=3:", int((u <= 3).sum()),
          "launches", r.gpu_launches, b.gpu_launches, "same", r.trace_signature() == b.trace_signature())
