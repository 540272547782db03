"""Time every BASELINE.json config on one GPU (one JSON line per run).

    python tools/configs_probe.py [--only er,potts,...] [--timing]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--only", default="")
ap.add_argument("--timing", action="store_true")
ap.add_argument("--big", action="store_true", help="include the 16384^2 grid")
ap.add_argument("--skip-rs", action="store_true")
a = ap.parse_args()
only = set(x for x in a.only.split(",") if x)


def emit(name, g, cfg, **extra):
    bp.run_ex(g, cfg, beliefs=False)  # warm (graph capture, allocation)
    r = bp.run_ex(g, cfg, beliefs=False)
    out = {"config": name, "kind": str(cfg.kind), "converged": r.converged, "iterations": r.iterations,
           "device_ms": round(r.device_ms, 3), "wall_s": round(r.wall_time, 4),
           "updates": r.messages_updated_total, "updates_per_s": r.messages_updated_total / (r.device_ms / 1e3),
           "evals": r.message_evaluations, "ms_per_iter": round(r.device_ms / max(r.iterations, 1), 4),
           "launches": r.gpu_launches, "splashes": r.splashes, "splash_rounds": r.splash_rounds}
    out.update(extra)
    if a.timing:
        rk = bp.run_ex(g, cfg, beliefs=False, kernel_timing=True)
        out["kernels"] = {k: (round(v["ms"], 3), v["launches"]) for k, v in rk.kernel_stats.items() if v["launches"]}
    print(json.dumps(out), flush=True)


def want(x):
    return not only or x in only


if want("ising1000"):
    t = time.time()
    g = bp.generate_ising(bp.IsingParams(n=1000, c=2.5, seed=0))
    gen = time.time() - t
    for kind, kw in (("lbp", {}), ("rnbp", dict(low_p=0.5)), ("rbp", dict(p=1 / 256)), ("rs", dict(p=1 / 256)))[: 3 if a.skip_rs else 4]:
        emit("ising1000_c2.5", g, bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(kind), max_iterations=10000,
                                                     time_limit=1e9, **kw), generate_s=round(gen, 3))
    del g
if want("er"):
    t = time.time()
    g = bp.generate_er(1_000_000, 2_000_000, 2.5, 0)
    gen = time.time() - t
    for p in (1 / 128, 1 / 256):
        emit("er1M_deg4", g, bp.SchedulerConfig(kind=bp.SchedulerKind.rs, p=p, splash_depth=2, max_iterations=20,
                                                time_limit=1e9), p=p, generate_s=round(gen, 3))
    emit("er1M_deg4", g, bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=20, time_limit=1e9))
    del g
if want("potts"):
    t = time.time()
    g = bp.generate_potts(4096, 8, 2.5, 0)
    gen = time.time() - t
    emit("potts4096_q8", g, bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=20, time_limit=1e9),
         generate_s=round(gen, 3))
    for lp in (0.1, 0.5, 1.0):
        emit("potts4096_q8", g, bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=lp, max_iterations=20,
                                                   time_limit=1e9), low_p=lp)
    del g
if want("ising4096"):
    g = bp.generate_ising(bp.IsingParams(n=4096, c=2.5, seed=0))
    emit("ising4096", g, bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=50, time_limit=1e9))
    emit("ising4096", g, bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=50,
                                            time_limit=1e9))
    del g
if a.big and want("ising16k"):
    t = time.time()
    g = bp.generate_ising(bp.IsingParams(n=16384, c=2.5, seed=0))
    gen = time.time() - t
    emit("ising16384", g, bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=20, time_limit=1e9),
         generate_s=round(gen, 3), device_bytes=g.device_bytes)
    emit("ising16384", g, bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=20,
                                             time_limit=1e9))
