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
