"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself
(oracle/_ref/libbpsched_ref.so, compiled from /root/reference by
oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --suite    # + 100x100 convergence suite (minutes)

The fixtures are committed so the oracle and the GPU tests are pinned to the
reference's outputs even where /root/reference is absent (the GPU box)."""
import argparse
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def small_cases(ref):
    cases = []
    for kind in ("lbp", "rbp", "rs", "rnbp", "srbp"):
        for (n, c, seed) in ((6, 2.5, 2), (8, 2.5, 800), (10, 2.0, 11)):
            g = po.Graph.ising(ref, n, c, seed)
            cfg = po.make_config(kind, p=0.25, max_iterations=3000 if kind == "srbp" else 300, seed=17,
                                 low_p=0.7)
            r = po.run(g, cfg)
            cases.append({
                "graph": {"kind": "ising", "n": n, "c": c, "seed": seed},
                "config": {"kind": kind, "p": 0.25, "max_iterations": int(cfg.max_iterations), "seed": 17,
                           "low_p": 0.7},
                "converged": r.converged, "iterations": r.iterations,
                "messages_updated_total": r.messages_updated_total,
                "trace_signature_sha": hashlib.sha256(r.signature().encode()).hexdigest()[:32],
                "trace_head": r.trace[:10].tolist(),
                "beliefs": r.beliefs.tolist() if r.beliefs.size <= 200 else None,
                "beliefs_sha": h(r.beliefs),
            })
    for (length, c, seed) in ((10, 2.0, 10), (33, 2.0, 33)):
        g = po.Graph.chain(ref, length, c, seed)
        r = po.run(g, po.make_config("lbp", max_iterations=length + 5))
        cases.append({"graph": {"kind": "chain", "n": length, "c": c, "seed": seed},
                      "config": {"kind": "lbp", "max_iterations": length + 5},
                      "converged": r.converged, "iterations": r.iterations,
                      "messages_updated_total": r.messages_updated_total,
                      "trace_signature_sha": hashlib.sha256(r.signature().encode()).hexdigest()[:32],
                      "trace_head": r.trace[:10].tolist(), "beliefs": r.beliefs.tolist(),
                      "beliefs_sha": h(r.beliefs)})
    return cases


def instance_hashes(ref):
    out = []
    for (n, c, seed) in ((3, 2.5, 0), (30, 2.5, 7), (100, 2.5, 500)):
        a = po.Graph.ising(ref, n, c, seed).arrays()
        out.append({"kind": "ising", "n": n, "c": c, "seed": seed, "unary_sha": h(a.unary),
                    "endpoints_sha": h(a.endpoints.astype(np.uint32)), "tables_sha": h(a.tables),
                    "unary_head": a.unary[:6].tolist(), "tables_head": a.tables[:8].tolist()})
    return out


def suite(ref, workers):
    """BASELINE config 1: 100x100 Ising C=2.5 seeds 500-524, eps 1e-5, cap 10k."""
    rows = []
    for s in range(500, 525):
        g = po.Graph.ising(ref, 100, 2.5, s)
        row = {"seed": s}
        for name, kw in (("lbp", dict()), ("rnbp_low0.5", dict(low_p=0.5, high_p=1.0, seed=s - 500)),
                         ("rnbp_low0.7", dict(low_p=0.7, high_p=1.0, seed=s - 500))):
            kind = "lbp" if name == "lbp" else "rnbp"
            r = po.run(g, po.make_config(kind, max_iterations=10000, time_limit=1e9, worker_count=workers, **kw),
                       trace_cap=1)
            row[name] = {"converged": r.converged, "iterations": r.iterations, "wall_time": r.wall_time,
                         "beliefs_sha": h(r.beliefs)}
            if r.converged:
                row[name]["beliefs_head"] = r.beliefs[:20].tolist()
        print(s, {k: (v["converged"], v["iterations"]) for k, v in row.items() if k != "seed"}, flush=True)
        rows.append(row)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--suite", action="store_true")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    ref = po.load("ref")
    mt = {str(seed): [int(x) for x in po.mt_draws(ref, seed, 8)[0]] for seed in (0, 5489, 17)}
    raw, _ = po.mt_draws(ref, 5489, 10000)
    fx = {"generated_by": "tests/golden/make_golden.py from oracle/_ref (the reference compiled from /root/reference)",
          "mt19937_64": mt, "mt19937_64_5489_10000th": int(raw[-1]),
          "instances": instance_hashes(ref), "runs": small_cases(ref)}
    with open(os.path.join(HERE, "reference_small.json"), "w") as f:
        json.dump(fx, f, indent=1)
    print("wrote reference_small.json")
    if a.suite:
        rows = suite(ref, a.workers)
        with open(os.path.join(HERE, "reference_suite_100x100.json"), "w") as f:
            json.dump({"generated_by": "tests/golden/make_golden.py --suite (reference, oracle/_ref)",
                       "config": "Ising 100x100 C=2.5, eps 1e-5, cap 10000, RnBP high_p 1.0 thr 0.9 seed = s-500",
                       "workers": a.workers, "rows": rows}, f, indent=1)
        print("wrote reference_suite_100x100.json")


if __name__ == "__main__":
    main()
