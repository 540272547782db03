"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    seq = []
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
              "second": 1e6, "s": 1e6}[r[ui]]
        name = r[ki].split("(")[0].replace("void ", "").replace("bpb::", "")
        seq.append((name, v))
    return seq


if __name__ == "__main__":
    seq = load(sys.argv[1])
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    seq = seq[skip:]
    agg = collections.defaultdict(list)
    for n, v in seq:
        agg[n].append(v)
    tot = sum(v for _, v in seq)
    print(f"launches {len(seq)}  total {tot:.1f} us")
    for n, vs in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(vs):10.1f} us {100*sum(vs)/tot:5.1f}%  n={len(vs):5d} avg={sum(vs)/len(vs):8.2f} us  min={min(vs):7.2f}  {n}")
