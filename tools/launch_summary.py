"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py gpurun_out/launches_r1e.csv > profiles/r1_bench_launches.txt
ncu serialises launches and runs them cold, so compare shares, not absolute times.
"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
         "second": 1e6, "s": 1e6}


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        d = dict(zip(hdr, r))
        if len(r) != len(hdr) or d["Metric Name"] != "gpu__time_duration.sum":
            continue
        us = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
        a = agg.setdefault(d["Kernel Name"].split("(")[0], [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot / 1e3:.3f} ms total")
    print(f"# {'launches':>8} {'total us':>12} {'share':>7}  kernel")
    for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {c:8d} {us:12.1f} {100 * us / tot:6.2f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
