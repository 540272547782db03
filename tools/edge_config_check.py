"""Edge-case configurations against the oracle on small models: extreme p /
low_p / high_p / thresholds, splash depth 0 / 1, iteration caps 0 / 1 / 2,
large epsilon.  Deterministic schedulers (LBP, RBP, RS) must match the
reference's verdict and iteration count (RBP / RS within 1 at fp32 ties);
every converged pair of runs must agree on marginals within 1e-4 (5e-3 at
epsilon >= 1e-3, where the stopping point is eps-dependent)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from tests.helpers import Stream, flatten, oracle_config, random_graph  # noqa: E402

orc = po.load()


def rg():
    cards, un, edges = random_graph(Stream(orc, 3), 40, 3, 0.08)
    a = flatten(cards, un, edges)
    return bp.PairwiseMRF.from_arrays(*a), po.Graph.from_arrays(orc, *a)


models = [("ising20", lambda: (bp.generate_ising(bp.IsingParams(n=20, c=1.5, seed=4)), po.Graph.ising(orc, 20, 1.5, 4))),
          ("potts12_q3", lambda: (bp.generate_potts(12, 3, 1.0, 2), po.Graph.potts(orc, 12, 3, 1.0, 2))),
          ("random40", rg)]
K = bp.SchedulerKind
configs = [("rbp p=1", dict(kind=K.rbp, p=1.0)), ("rbp p=1e-6", dict(kind=K.rbp, p=1e-6)),
           ("rs p=1 h2", dict(kind=K.rs, p=1.0, splash_depth=2)), ("rs p=1e-6 h2", dict(kind=K.rs, p=1e-6, splash_depth=2)),
           ("rs h0", dict(kind=K.rs, p=0.2, splash_depth=0)), ("rs h1", dict(kind=K.rs, p=0.2, splash_depth=1)),
           ("rnbp low=0.01", dict(kind=K.rnbp, low_p=0.01)), ("rnbp low=1", dict(kind=K.rnbp, low_p=1.0)),
           ("rnbp high=0.5", dict(kind=K.rnbp, low_p=0.3, high_p=0.5)),
           ("rnbp thr=0", dict(kind=K.rnbp, low_p=0.5, edge_ratio_threshold=0.0)),
           ("rnbp thr=1", dict(kind=K.rnbp, low_p=0.5, edge_ratio_threshold=1.0)),
           ("lbp cap0", dict(kind=K.lbp, max_iterations=0)), ("lbp cap1", dict(kind=K.lbp, max_iterations=1)),
           ("rbp cap2", dict(kind=K.rbp, p=0.3, max_iterations=2)), ("rnbp cap1", dict(kind=K.rnbp, max_iterations=1)),
           ("rs cap0", dict(kind=K.rs, p=0.3, max_iterations=0)),
           ("lbp eps0.5", dict(kind=K.lbp, epsilon=0.5)), ("rnbp eps0.5", dict(kind=K.rnbp, epsilon=0.5)),
           ("rbp eps1e-3", dict(kind=K.rbp, p=0.2, epsilon=1e-3))]
bad = 0
for mname, mk in models:
    dg, og = mk()
    for cname, kw in configs:
        kw = dict(kw)
        kw.setdefault("max_iterations", 3000)
        cfg = bp.SchedulerConfig(seed=7, **kw)
        try:
            o = po.run(og, oracle_config(cfg))
        except Exception as e:  # noqa: BLE001
            oerr = type(e).__name__ + ": " + str(e)
            o = None
        try:
            r = bp.run(dg, cfg)
            derr = None
        except Exception as e:  # noqa: BLE001
            derr = type(e).__name__ + ": " + str(e)
            r = None
        if o is None or r is None:
            same = (o is None) == (r is None)
            bad += not same
            print(f"{mname:11s} {cname:14s} oracle {'ERR ' + oerr if o is None else 'ok'} | device {'ERR ' + derr if r is None else 'ok'} {'' if same else '<-- MISMATCH'}")
            continue
        det = kw["kind"] != K.rnbp
        tol_it = 0 if kw["kind"] == K.lbp else 1
        both = r.converged and o.converged
        diff = float(np.max(np.abs(r.beliefs.values - o.beliefs))) if (both or r.iterations == o.iterations) else float("nan")
        btol = 5e-3 if cfg.epsilon >= 1e-3 else 1e-4
        flag = r.converged != o.converged or (det and abs(r.iterations - o.iterations) > tol_it) or (both and diff > btol)
        if det and not both and r.iterations == o.iterations and kw["kind"] == K.lbp:
            flag = flag or diff > 1e-5
        bad += flag
        print(f"{mname:11s} {cname:14s} device {r.converged!s:5s} {r.iterations:5d} upd {r.messages_updated_total:9d} | "
              f"oracle {o.converged!s:5s} {o.iterations:5d} upd {o.messages_updated_total:9d} | diff {diff:.1e} "
              f"{'<-- MISMATCH' if flag else ''}")
print("mismatches", bad)
