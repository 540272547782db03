"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself
(oracle/_ref/libbpsched_ref.so, compiled from /root/reference by
oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --suite    # + the convergence suites (minutes)

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


SUITES = {
    # BASELINE config 1 / acceptance criteria 5-6 (acceptance.cpp:282-351): 100x100
    # Ising C=2.5 seeds 500-524, eps 1e-5; an iteration cap instead of the 60 s limit
    "ising100": dict(n=100, c=2.5, seeds=range(500, 525), cap=10000,
                     runs=(("lbp", dict()), ("rnbp_low0.5", dict(low_p=0.5)), ("rnbp_low0.7", dict(low_p=0.7)))),
    # acceptance criterion 7 (acceptance.cpp:353-378): 30x30 C=3 seeds 700-709, LBP vs RnBP low_p 0.1
    "hard30": dict(n=30, c=3.0, seeds=range(700, 710), cap=20000,
                   runs=(("lbp", dict()), ("rnbp_low0.1", dict(low_p=0.1)))),
}


RNBP_REPLICATES = 4  # RnBP is randomized: replicate k uses seed = instance index + 1000 k


def suite(ref, workers, name):
    """Converged flags, iterations, reference wall times and (converged runs)
    the full marginals P(x = 1) per vertex as float32 (for the 1e-4 check).
    RnBP runs are repeated with RNBP_REPLICATES seeds (the convergence
    fraction of a randomized scheduler at a cap is a random variable);
    replicate 0 is the acceptance suite's own seed (acceptance.cpp:50-61)."""
    sp = SUITES[name]
    rows, marg = [], {}
    for s in sp["seeds"]:
        g = po.Graph.ising(ref, sp["n"], sp["c"], s)
        row = {"seed": s}
        for run_name, kw in sp["runs"]:
            kind = "lbp" if run_name == "lbp" else "rnbp"
            reps, conv = [], []
            for k in range(RNBP_REPLICATES if kind == "rnbp" else 1):
                extra = dict(high_p=1.0, edge_ratio_threshold=0.9, seed=s - sp["seeds"][0] + 1000 * k) \
                    if kind == "rnbp" else {}
                r = po.run(g, po.make_config(kind, max_iterations=sp["cap"], time_limit=1e9, worker_count=workers,
                                             **kw, **extra), trace_cap=1)
                reps.append({"converged": r.converged, "iterations": r.iterations, "wall_time": r.wall_time,
                             "messages_updated_total": r.messages_updated_total, "beliefs_sha": h(r.beliefs)})
                if r.converged:
                    conv.append(r.beliefs[1::2].copy())
            row[run_name] = dict(reps[0])
            if len(reps) > 1:
                row[run_name]["replicates"] = [{"converged": x["converged"], "iterations": x["iterations"]}
                                               for x in reps]
            # the distinct fixed points the converged replicates reached (max
            # marginal difference < 1e-2 = same fixed point), one stored
            # representative each, and the spread of converged marginals
            # within a fixed point (the reference's own run-to-run precision)
            clusters = []
            for b in conv:
                for cl in clusters:
                    if np.max(np.abs(cl[0] - b)) < 1e-2:
                        cl.append(b)
                        break
                else:
                    clusters.append([b])
            spread = 0.0
            for j, cl in enumerate(clusters):
                marg[f"{run_name}_{s}_fp{j}"] = cl[0].astype(np.float32)
                for a in range(len(cl)):
                    for b in range(a + 1, len(cl)):
                        spread = max(spread, float(np.max(np.abs(cl[a] - cl[b]))))
            row[run_name]["fixed_points"] = len(clusters)
            row[run_name]["spread"] = spread
        print(name, s, {k: [x["iterations"] if x["converged"] else -1 for x in v.get("replicates", [v])]
                        for k, v in row.items() if k != "seed"}, flush=True)
        rows.append(row)
    return rows, marg


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
        out, marg = {}, {}
        for name in SUITES:
            rows, m = suite(ref, a.workers, name)
            sp = SUITES[name]
            out[name] = {"n": sp["n"], "c": sp["c"], "seeds": list(sp["seeds"]), "max_iterations": sp["cap"],
                         "epsilon": 1e-5, "rows": rows}
            marg.update({f"{name}/{k}": v for k, v in m.items()})
        with open(os.path.join(HERE, "reference_suites.json"), "w") as f:
            json.dump({"generated_by": "tests/golden/make_golden.py --suite (the reference, oracle/_ref)",
                       "rnbp": "high_p 1.0, edge_ratio_threshold 0.9, seed = instance index (acceptance.cpp:50-61) "
                               "+ 1000 k for replicate k",
                       "workers": a.workers, "suites": out}, f, indent=1)
        np.savez_compressed(os.path.join(HERE, "reference_suites_marginals.npz"), **marg)
        print("wrote reference_suites.json, reference_suites_marginals.npz")


if __name__ == "__main__":
    main()
