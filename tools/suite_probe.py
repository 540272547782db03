import json, sys, numpy as np
sys.path.insert(0, '.')
import paper_1909_11469_b200 as bp
g = json.load(open('tests/golden/reference_suites.json'))['suites']
for suite, name, low in (("ising100", "rnbp_low0.5", 0.5), ("ising100", "rnbp_low0.7", 0.7), ("hard30", "rnbp_low0.1", 0.1)):
    sp = g[suite]
    ref = [r[name]["iterations"] if r[name]["converged"] else -1 for r in sp["rows"]]
    print(suite, name, "ref", ref, flush=True)
    for rep in range(4):
        its = []
        for s in sp["seeds"]:
            gr = bp.generate_ising(bp.IsingParams(n=sp["n"], c=sp["c"], seed=s))
            cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=low, high_p=1.0, max_iterations=sp["max_iterations"] * 10,
                                     time_limit=1e9, seed=s - sp["seeds"][0] + 1000 * rep)
            r = bp.run_ex(gr, cfg, beliefs=False)
            its.append(r.iterations if r.converged else -1)
        print(suite, name, "dev rep", rep, its, flush=True)
