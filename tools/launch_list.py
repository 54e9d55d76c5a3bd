"""Per-kernel totals of an ncu launch list (`--metrics gpu__time_duration.sum
--csv --log-file X`), over launches [first, last) -- the profiles/ launch
tables.

    python tools/launch_list.py gpurun_out/launches.csv 700 1000 "header line" > profiles/x.txt
"""
import csv
import sys
from collections import OrderedDict


def main():
    path, first, last = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    header = sys.argv[4] if len(sys.argv) > 4 else ""
    rows = [r for r in csv.reader(open(path)) if r and r[0] not in ("==PROF==",)]
    hdr = next(r for r in rows if "Kernel Name" in r)
    ki, ii = hdr.index("Kernel Name"), hdr.index("ID")
    vi, ui, mi = hdr.index("Metric Value"), hdr.index("Metric Unit"), hdr.index("Metric Name")
    agg = OrderedDict()
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        i = int(r[ii])
        if not first <= i < last:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        us = v / 1000.0 if u in ("nsecond", "ns") else (v * 1000.0 if u in ("msecond", "ms") else v)
        name = r[ki].split("(")[0][:60]
        if "FillFunctor" in name:   # bench.py's untimed L2 flush between steps
            continue
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    tot = sum(t for _, t in agg.values())
    if header:
        print(header)
    print("# per-launch times are cold-cache and serialised; compare SHARES with the bench line")
    print(f"# {'kernel':60s} {'launches':>9s} {'total_us':>10s} {'share':>7s}")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:62s} {n:9d} {t:10.1f} {t / tot:7.3f}")


if __name__ == "__main__":
    main()
