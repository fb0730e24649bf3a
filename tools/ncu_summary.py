"""Summarise an .ncu-rep (raw page) into the few metrics we track."""
import csv
import subprocess
import sys

WANT = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes.sum.per_second",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_shared_mem"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    units = r[1]
    res = []
    for row in r[2:]:
        d = {}
        for w in WANT:
            for i, name in enumerate(h):
                if name == w or name.endswith("." + w) or name.endswith(w):
                    d[w] = (row[i], units[i])
                    break
        res.append(d)
    return res


if __name__ == "__main__":
    for d in rows(sys.argv[1]):
        print("; ".join(f"{k.split('.')[0] if k != 'Kernel Name' else 'kernel'}={v[0]}{(' ' + v[1]) if v[1] else ''}"
                        if k not in ("Kernel Name",) else f"kernel={v[0][:50]}" for k, v in d.items()))
