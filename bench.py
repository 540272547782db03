#!/usr/bin/env python
"""Benchmark of the BP message-scheduling hot path (BASELINE.json configs[1]).

Workload ("step"): one complete bpsched::run (schedulers.cpp:293-353) of RnBP
(low_p 0.5, high_p 1.0, EdgeRatio threshold 0.9, epsilon 1e-5, 10,000-iteration
cap) on the 1000 x 1000 Ising grid, C = 2.5, generated bit-identically to the
reference's generate_ising (seed = step index + rank * 1000).

  value  = committed edge-message updates / second (sum |F| / device time of the
           runs, graph resident in HBM, CUDA events on the engine stream)
  e2e    = the same metric through the public API with host buffers: every step
           uploads the graph from host arrays in build_graph's input layout
           (bp_graph_create: validation, CSR, H2D), runs, and copies the beliefs
           back (D2H)

At N > 1 GPUs every rank runs its own instances (weak scaling, replicas), and
the row-band partitioned LBP on the 16384^2 grid (BASELINE config 5, one band
per GPU, NCCL halo exchange) is reported beside it under "partitioned_16k".
Extra keys: LBP / RBP on the workload instance, the 100^2 C=2.5 convergence
suite (seeds 500-524), the HBM roofline of the LBP sweep on 16384^2.  The
reference arm (--impl reference) times the reference's own bpsched::run compiled
from /root/reference (oracle/_ref) on the host cores on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_GRID = 1000
C_COUPLING = 2.5
CAP = 10000
METRIC = "edge-message updates/sec (RnBP, Ising 1000x1000 C=2.5, run to convergence or 10k-iteration cap)"
UNIT = "updates/s"
REF_SAMPLE_ITERS = 5   # bounded CPU sample: reference run capped at 5 iterations
BIG_N = 16384          # BASELINE config 5
BIG_ITERS = 30         # fixed LBP window on the big grid
BIG_RNBP_ITERS = 10    # fixed RnBP window on the big grid (N > 1)


def rnbp_kw(seed):
    return dict(low_p=0.5, high_p=1.0, edge_ratio_threshold=0.9, epsilon=1e-5, max_iterations=CAP,
                time_limit=1e9, seed=seed)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region:
    ONE `nvidia-smi --query-gpu=... -lms 200` process (the profiling recipe's
    clocks line), started before the region and stopped after it by its own
    handle.  (Spawning nvidia-smi per sample initialises NVML each time and
    can stall the run's host round trips.)"""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "200"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        time.sleep(0.25)  # at least one sample after the region on short runs
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except Exception:
            self._p.kill()
            out, _ = self._p.communicate()
        for line in (out or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[4 + i].strip() == "Active"})
        loaded = [x for x in sm if mx and x > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def flush_l2(torch, buf):
    buf.zero_()  # 256 MiB > 126 MB L2
    torch.cuda.synchronize()


# Algorithmic bytes, binary Ising lattice, compressed
# layout (one fp32 log2-odds per message, one fp32 coupling per edge):
#   LBP sweep: per vertex read its 2 edge pairs (16 B) + write 4 messages (16 B)
#              + 2 couplings (8 B) + unary (4 B) = 44 B
#   touched refresh (update class): per vertex unary 4 B (+ 4 B list id); per
#              message edge pair 8 B + coupling 4 B + candidate 4 B + residual 8 B
# reference fp32 layout: 30 B per directed edge per LBP sweep.
def lbp_sweep_bytes(vertices):
    return 44 * vertices


def refresh_bytes(visits, evals):
    return 8 * visits + 24 * evals


def run_b200(args):
    import torch

    import paper_1909_11469_b200 as bp

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    K, W = args.steps, args.warmup

    graphs = {}

    def graph_for(seed):
        if seed not in graphs:
            graphs[seed] = bp.generate_ising(bp.IsingParams(n=N_GRID, c=C_COUPLING, seed=seed), device=local)
        return graphs[seed]

    seeds = [rank * 1000 + s for s in range(K)]
    for s in seeds:
        graph_for(s)
    kind = bp.SchedulerKind.rnbp
    for w in range(W):  # warmup (graph capture, allocation, first-touch)
        bp.run(graph_for(seeds[w % K]), bp.SchedulerConfig(kind=kind, **rnbp_kw(seeds[w % K])))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    results = []
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        dev_ms = 0.0
        for s in seeds:
            flush_l2(torch, flush)
            r = bp.run(graph_for(s), bp.SchedulerConfig(kind=kind, **rnbp_kw(s)))
            dev_ms += r.device_ms
            results.append(r)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if dist:
        dist.barrier()
    updates = sum(r.messages_updated_total for r in results)
    t_dev = dev_ms / 1e3
    if dist:
        tt = torch.tensor([t_dev, float(updates)], dtype=torch.float64, device="cuda")
        mx = tt.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        t_dev = float(mx[0])
        updates = float(tt[1])
    value = updates / t_dev
    ms_per_step = t_dev / K * 1e3
    launches = sum(r.gpu_launches for r in results)

    # ---- e2e: public API with host buffers (graph upload + run + beliefs D2H)
    e2e_updates, e2e_t = 0, 0.0
    h2d = d2h = 0
    host_arrays = {s: bp.generate_ising_arrays(bp.IsingParams(n=N_GRID, c=C_COUPLING, seed=s))
                   for s in seeds[: min(K, 5)]}
    e2e_steps = []
    # one untimed call first: process-level first use of the host-array path
    # (module loading of its kernels, host thread pool start-up)
    cards, un, ep, tb = host_arrays[seeds[0]]
    bp.run(bp.PairwiseMRF.from_arrays(cards, un, ep, tb, device=local),
           bp.SchedulerConfig(kind=kind, **dict(rnbp_kw(seeds[0]), max_iterations=10)))
    for s in seeds[: min(K, 5)]:
        cards, un, ep, tb = host_arrays[s]
        flush_l2(torch, flush)
        t1 = time.perf_counter()
        g = bp.PairwiseMRF.from_arrays(cards, un, ep, tb, device=local)
        r = bp.run(g, bp.SchedulerConfig(kind=kind, **rnbp_kw(s)))
        _ = r.beliefs.values.sum()
        dt = time.perf_counter() - t1
        e2e_t += dt
        e2e_steps.append(round(dt * 1e3, 3))
        e2e_updates += r.messages_updated_total
        h2d = cards.nbytes + un.nbytes + ep.nbytes + tb.nbytes
        d2h = r.beliefs.values.nbytes + 32 * len(r.trace)
        del g
    if dist:
        tt = torch.tensor([e2e_t, float(e2e_updates)], dtype=torch.float64, device="cuda")
        mx = tt.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        e2e_t, e2e_updates = float(mx[0]), float(tt[1])

    # ---- partitioned 16K^2 LBP (config 5): every rank, a band each
    part = _partitioned_big(bp, torch, dist, ws, rank, local)

    out = {}
    if rank == 0:
        peak, peak_src = measured_peaks()
        # ---- dominant kernel of the workload (instrumented run: CUDA events per launch)
        g0 = graph_for(seeds[0])
        ri = bp.run_ex(g0, bp.SchedulerConfig(kind=kind, **rnbp_kw(seeds[0])), kernel_timing=True)
        ks = ri.kernel_stats
        tot_ms = sum(v["ms"] for v in ks.values()) or 1.0
        dom = max(ks, key=lambda k: ks[k]["ms"])
        if dom == "persist":
            dom_bytes = ks["persist"]["bytes"]
            dom_name = "k_rnbp_persist (RnBP candidate-list iterations, cooperative grid of one CTA per SM, one 16-CTA cluster for lists under 2048 entries)"
        else:
            dom_bytes = refresh_bytes(ri.vertex_visits, ri.message_evaluations)
            dom_name = f"{dom} kernels"
        dom_ms = ks[dom]["ms"]
        achieved = dom_bytes / (dom_ms / 1e3) / 1e9 if dom_ms else 0.0
        shares = {k: round(v["ms"] / tot_ms, 4) for k, v in ks.items() if v["launches"]}

        # ---- other schedulers on the workload instance + convergence suite
        extra = {}
        for name, cfg in (("lbp", bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=CAP, time_limit=1e9)),
                          ("rbp", bp.SchedulerConfig(kind=bp.SchedulerKind.rbp, p=1 / 256, max_iterations=CAP,
                                                     time_limit=1e9)),
                          ("rs", bp.SchedulerConfig(kind=bp.SchedulerKind.rs, p=1 / 256, max_iterations=200,
                                                    time_limit=1e9))):
            bp.run(g0, cfg)
            rr = bp.run(g0, cfg)
            extra[name] = {"value": rr.messages_updated_total / (rr.device_ms / 1e3), "unit": UNIT,
                           "iterations": rr.iterations, "converged": rr.converged,
                           "ms": round(rr.device_ms, 3), "ms_per_iteration": round(rr.device_ms / max(1, rr.iterations), 4)}
        suite = _convergence_suite(bp, local)

        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (base-2 log-odds messages)",
            "data": "synthetic (generate_ising, bit-identical to the reference generator)",
            "config": {"workload": "ising1000_c2.5_rnbp", "n": N_GRID, "c": C_COUPLING, "scheduler": "rnbp",
                       "low_p": 0.5, "high_p": 1.0, "edge_ratio_threshold": 0.9, "epsilon": 1e-5,
                       "max_iterations": CAP, "seeds": f"rank*1000 + 0..{K - 1}",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU",
                       "l2": "flushed between timed steps (256 MiB write)"},
            "steps_detail": [{"seed": s, "converged": r.converged, "iterations": r.iterations,
                              "updates": r.messages_updated_total, "ms": round(r.device_ms, 3)}
                             for s, r in zip(seeds, results)],
            "time_to_convergence_s": _ttc(results),
            "wall_s": wall,
            "gpu_launches": launches,
            "e2e": {"value": e2e_updates / e2e_t if e2e_t else None, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": min(K, 5), "steps_ms": e2e_steps,
                    "includes": "bp_graph_create from host arrays (validation + CSR + H2D) + run + beliefs D2H"},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _read_traffic(dom), "peak_source": peak_src,
                         "algorithmic_bytes": dom_bytes, "kernel_ms": dom_ms, "launches": ks[dom]["launches"],
                         "kernel_shares": shares,
                         "regime": "latency-bound: the 1000^2 working set (~70 MB) is L2-resident and the "
                                   "candidate-list iterations move ~3k messages each; roofline_hbm is the "
                                   "HBM-bound kernel (LBP sweep, 16384^2)"},
            "schedulers": extra,
            "convergence_suite_100x100": suite,
            "clocks": clk.summary(),
        }
        out["roofline_hbm"] = _hbm_roofline(bp, torch, local, peak, peak_src)
        if part:
            out["partitioned_16k"] = part
        if ws == 1:
            out["cpu_baseline"] = _cpu_baseline(sample_iters=REF_SAMPLE_ITERS)
        print(json.dumps(out))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def _hbm_roofline(bp, torch, device, peak, peak_src):
    """LBP sweep on the 16384^2 grid (config 5, working set >> L2): CUDA-event time
    of the update launches of a fixed window, algorithmic bytes per section 5."""
    g = bp.generate_ising(bp.IsingParams(n=BIG_N, c=C_COUPLING, seed=0), device=device)
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=BIG_ITERS, time_limit=1e9)
    bp.run_ex(g, cfg, beliefs=False)
    r = bp.run_ex(g, cfg, beliefs=False, kernel_timing=True)
    k = r.kernel_stats["update"]
    sweeps = r.iterations + 1
    V = g.num_vertices()
    nbytes = lbp_sweep_bytes(V) * sweeps
    ach = nbytes / (k["ms"] / 1e3) / 1e9
    ref_bytes = 30 * g.num_directed_edges() * sweeps
    out = {"kernel": "k_vertex_update<Count> lattice tiles (LBP sweep), Ising 16384^2", "bound": "hbm",
           "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "peak_source": peak_src,
           "algorithmic_bytes": nbytes, "bytes_per_vertex": 44, "kernel_ms": k["ms"], "launches": k["launches"],
           "sweeps": sweeps, "ms_per_sweep": k["ms"] / sweeps,
           "updates_per_s": r.messages_updated_total / (r.device_ms / 1e3),
           "effective_reference_layout_GBps": ref_bytes / (k["ms"] / 1e3) / 1e9,
           "traffic": _read_traffic("lbp16k")}
    del g
    torch.cuda.empty_cache()
    return out


def _partitioned_big(bp, torch, dist, ws, rank, local):
    """Row-band partitioned LBP on the 16384^2 grid: one band per rank, NCCL halo
    exchange + count all-reduce each iteration (paper_1909_11469_b200.parallel).
    Strong scaling: the grid is fixed.  At N = 1 the same window runs on the
    whole grid (one band)."""
    if ws == 1:
        return None
    from paper_1909_11469_b200 import parallel as par

    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=10 ** 9, time_limit=1e9)
    band = par.BandLBP(BIG_N, C_COUPLING, 0, rank, ws, cfg, local)
    ex = par.NcclExchange(rank, ws)
    with torch.cuda.stream(band.stream):
        for _ in range(3):  # warmup
            band.sweep()
            ex(band)
            band.finish()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st0 = band.status()
        e0.record(band.stream)
        for _ in range(BIG_ITERS):
            band.sweep()
            ex(band)
            band.finish()
        e1.record(band.stream)
        torch.cuda.synchronize()
    st1 = band.status()
    ms = e0.elapsed_time(e1)
    upd = st1.messages_updated_total - st0.messages_updated_total
    del band
    # RnBP on the same bands: a fixed window of the run loop (host polls the
    # all-reduced sums every iteration; Philox keyed by global edge ids)
    rcfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=BIG_RNBP_ITERS, time_limit=1e9)
    rb = [par.BandRnBP(BIG_N, C_COUPLING, 0, rank, ws, rcfg, local)]
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    rst = par.run_band_rnbp(rb, par.NcclComm(rank, ws), BIG_RNBP_ITERS)
    torch.cuda.synchronize()
    rms = (time.perf_counter() - t0) * 1e3
    tt = torch.tensor([ms, float(upd), rms], dtype=torch.float64, device="cuda")
    mx = tt.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(tt, op=dist.ReduceOp.SUM)
    ms_max, upd_sum, rms_max = float(mx[0]), float(tt[1]), float(mx[2])
    return {"config": f"Ising {BIG_N}^2 C={C_COUPLING}, row bands x{ws}, NCCL halo + all-reduce per iteration",
            "lbp": {"iterations": BIG_ITERS, "ms_max_over_ranks": ms_max, "updates": upd_sum,
                    "value": upd_sum / (ms_max / 1e3), "unit": UNIT, "timing": "CUDA events on the band stream"},
            "rnbp": {"iterations": rst.iterations, "ms_max_over_ranks": rms_max,
                     "updates": rst.messages_updated_total,
                     "value": rst.messages_updated_total / (rms_max / 1e3), "unit": UNIT,
                     "timing": "host clock incl. init (per-iteration host poll of the all-reduced sums)"},
            "scaling": "strong"}


def _ttc(results):
    conv = [r.wall_time for r in results if r.converged]
    return {"converged_steps": len(conv), "steps": len(results),
            "median_s": statistics.median(conv) if conv else None}


def _read_traffic(key):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def _convergence_suite(bp, device):
    """BASELINE config 1: Ising 100^2 C=2.5, seeds 500-524, eps 1e-5, cap 10k."""
    out = {}
    for name, cfg_kw in (("lbp", dict(kind=bp.SchedulerKind.lbp)),
                         ("rnbp_low0.5", dict(kind=bp.SchedulerKind.rnbp, low_p=0.5, high_p=1.0)),
                         ("rnbp_low0.7", dict(kind=bp.SchedulerKind.rnbp, low_p=0.7, high_p=1.0))):
        conv, times, iters = 0, [], []
        t0 = time.perf_counter()
        for s in range(500, 525):
            g = bp.generate_ising(bp.IsingParams(n=100, c=2.5, seed=s), device=device)
            kw = dict(cfg_kw)
            if kw["kind"] == bp.SchedulerKind.rnbp:
                kw["seed"] = s - 500
            r = bp.run(g, bp.SchedulerConfig(max_iterations=CAP, time_limit=1e9, **kw))
            conv += r.converged
            if r.converged:
                times.append(r.wall_time)
                iters.append(r.iterations)
        out[name] = {"converged": conv, "of": 25, "median_time_s": statistics.median(times) if times else None,
                     "median_iterations": statistics.median(iters) if iters else None,
                     "suite_wall_s": round(time.perf_counter() - t0, 3)}
    return out


def _cpu_baseline(sample_iters):
    """The reference's bpsched::run (oracle/_ref, compiled from /root/reference)
    on this host, bounded sample of the workload."""
    from oracle import pyoracle as po
    try:
        ref = po.load("ref")
        kind = "reference"
    except FileNotFoundError:
        ref = po.load("orc")
        kind = "port"
    cores = os.cpu_count() or 1
    g = po.Graph.ising(ref, N_GRID, C_COUPLING, 0)
    cfg = po.make_config("rnbp", low_p=0.5, high_p=1.0, edge_ratio_threshold=0.9, epsilon=1e-5,
                         max_iterations=sample_iters, time_limit=1e9, seed=0, worker_count=cores)
    r = po.run(g, cfg)
    return {"value": r.messages_updated_total / r.wall_time, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"RnBP Ising {N_GRID}^2 C={C_COUPLING} seed 0, first {sample_iters} iterations "
                      f"(EngineState ctor + loop, {r.wall_time:.2f} s, {r.messages_updated_total} updates)",
            "wall_s": r.wall_time}


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import pyoracle as po
    try:
        ref = po.load("ref")
        kind = "reference"
    except FileNotFoundError:
        ref = po.load("orc")
        kind = "port"
    cores = os.cpu_count() or 1
    K, W = args.steps, args.warmup
    graphs = [po.Graph.ising(ref, N_GRID, C_COUPLING, s) for s in range(min(K, 2))]

    def cfg(s):
        return po.make_config("rnbp", low_p=0.5, high_p=1.0, edge_ratio_threshold=0.9, epsilon=1e-5,
                              max_iterations=REF_SAMPLE_ITERS, time_limit=1e9, seed=s, worker_count=cores)
    for w in range(W):
        po.run(graphs[w % len(graphs)], cfg(w))
    upd, t = 0, 0.0
    for k in range(K):
        r = po.run(graphs[k % len(graphs)], cfg(k))
        upd += r.messages_updated_total
        t += r.wall_time
    v = upd / t
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
           "ms_per_step": t / K * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic (generate_ising)",
           "config": {"workload": "ising1000_c2.5_rnbp", "n": N_GRID, "c": C_COUPLING, "scheduler": "rnbp",
                      "low_p": 0.5, "sample_iterations": REF_SAMPLE_ITERS},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                            "sample": f"first {REF_SAMPLE_ITERS} RnBP iterations per step (incl. EngineState ctor)"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
