"""Digest of an ncu --set full report for profiles/: the details page (one line
per metric) plus the kernel's DRAM traffic per launch; --traffic KEY also
records dram__bytes_read.sum + dram__bytes_write.sum under KEY in
profiles/traffic.json (bench.py reports it as roofline.traffic)."""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def scale_of(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6,
            "GB": 1e9}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--traffic", default=None)
    a = ap.parse_args()
    rows = ncu_csv(a.rep, "--page", "details")
    h = rows[0]
    ik, isec, iname, iunit, ival = (h.index("Kernel Name"), h.index("Section Name"), h.index("Metric Name"),
                                     h.index("Metric Unit"), h.index("Metric Value"))
    lines, kernel = [], None
    for r in rows[1:]:
        if kernel != r[ik]:
            kernel = r[ik]
            lines.append(f"Kernel: {kernel[:130]}")
        lines.append(f"{r[isec][:30]:30s} {r[iname][:50]:50s} {r[ival]:>14s} {r[iunit]}")
    # summary block: the numbers the roofline / stall discussion cites
    full = ncu_csv(a.rep, "--page", "raw")
    fh, fu = full[0], full[1]
    summary = []
    for r in full[2:]:
        def val(name):
            if name not in fh:
                return None
            try:
                return float(r[fh.index(name)].replace(",", ""))
            except ValueError:
                return None
        kname = r[fh.index("Kernel Name")][:100] if "Kernel Name" in fh else "?"
        dur = val("gpu__time_duration.sum")
        dram = (val("dram__bytes_read.sum") or 0) * scale_of(fu[fh.index("dram__bytes_read.sum")]) + \
               (val("dram__bytes_write.sum") or 0) * scale_of(fu[fh.index("dram__bytes_write.sum")])
        dur_s = (dur or 0) * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
                              "second": 1.0, "s": 1.0}.get(
            fu[fh.index("gpu__time_duration.sum")], 1e-9)
        stalls = []
        for i, n in enumerate(fh):
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i].replace(",", "")), n[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot_st = sum(x for x, _ in stalls) or 1.0
        summary.append(f"SUMMARY {kname}")
        summary.append(f"  duration {dur_s * 1e6:.2f} us, DRAM bytes {dram:.4g}, DRAM {dram / dur_s / 1e9 if dur_s else 0:.1f} GB/s")
        for label, name in (("L2 hit rate %", "lts__t_sector_hit_rate.pct"),
                            ("DRAM throughput % of peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                            ("IPC (executed, per SM)", "sm__inst_executed.avg.per_cycle_active"),
                            ("issue slots busy %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
                            ("achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
                            ("registers / thread", "launch__registers_per_thread"),
                            ("grid size", "launch__grid_size"), ("block size", "launch__block_size")):
            v = val(name)
            if v is not None:
                summary.append(f"  {label}: {v:g}")
        summary.append("  warp stall cycles per issued instruction (top 6 of {:.1f}): ".format(tot_st) +
                       ", ".join(f"{n} {x:.2f} ({100 * x / tot_st:.0f}%)" for x, n in stalls[:6]))
    lines = summary + [""] + lines
    raw = ncu_csv(a.rep, "--page", "raw", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum")
    hh = raw[0]
    units = raw[1] if len(raw) > 1 else []
    rd = hh.index("dram__bytes_read.sum")
    wr = hh.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot = []
    for r in raw[2:]:
        b = float(r[rd].replace(",", "")) * scale.get(units[rd], 1) + float(r[wr].replace(",", "")) * scale.get(
            units[wr], 1)
        tot.append(b)
    lines.append(f"dram__bytes_read.sum + dram__bytes_write.sum per launch: {[round(t) for t in tot]}")
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.traffic and tot:
        p = os.path.join(ROOT, "profiles", "traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        d[a.traffic] = sum(tot) / len(tot)
        d["note"] = "dram__bytes_read.sum + dram__bytes_write.sum per launch from ncu --set full (profiles/r01_ncu_*.txt)"
        json.dump(d, open(p, "w"), indent=1)
    print(f"{a.out}: {len(lines)} lines, traffic {tot}")


if __name__ == "__main__":
    main()
