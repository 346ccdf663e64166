"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (dev tool).

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/<name>.txt
"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr_i]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hdr_i + 1:]:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            agg[r[ik]].append(float(r[iv].replace(",", "")))
    unit_ns = 1.0  # ncu reports gpu__time_duration.sum in ns (or us); normalised below
    unit = h[iv + 1] if len(h) > iv + 1 else ""
    tot = sum(sum(v) for v in agg.values())
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none ({path}); cold-cache, serialised launches")
    print("# count      mean    total    share  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):7d} {sum(v)/len(v):9.1f} {sum(v):9.1f} {100*sum(v)/tot:6.1f}%  {k[:110]}")


if __name__ == "__main__":
    main(sys.argv[1])
