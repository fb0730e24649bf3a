"""Aggregate an ncu --csv launch list (gpu__time_duration per kernel)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    idi = h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
              "second": 1e6, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
        per[r[idi]][r[mi]] = v
        names[r[idi]] = r[ki]
    return per, names


if __name__ == "__main__":
    per, names = load(sys.argv[1])
    skip = sys.argv[2] if len(sys.argv) > 2 else "distribution_elementwise"
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for k, m in per.items():
        n = names[k]
        if skip and skip in n:
            continue
        key = n.split("(")[0][:70]
        t = m.get("gpu__time_duration.sum", 0.0)
        agg[key][0] += 1
        agg[key][1] += t
        agg[key][2] += m.get("dram__bytes_read.sum", 0.0)
        tot += t
    for key, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = (b / n) / (t / n * 1e-6) / 1e9 if b else 0.0
        print(f"{t:10.1f} us {100 * t / tot:5.1f}% n={n:5d} avg={t / n:8.2f} us  {gbs:7.0f} GB/s(read)  {key}")
    print(f"total {tot / 1e3:.3f} ms")
