"""Summarise an `ncu --set full` capture into the text kept under profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep "title" [launch] > profiles/x.txt

`launch` picks one launch of a multi-launch capture (default 0); the header
then also lists every launch's duration and DRAM bytes and their mean.

Prints duration, DRAM bytes (the roofline `traffic`), pipe utilisations, L1/L2
behaviour, occupancy and the top warp-stall reasons by SASS instruction.
"""

import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
    li = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units, v = rows[0], rows[1], rows[2 + li]
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    print(f"# {title}")
    print(f"# kernel: {name[:160]}")
    if len(rows) > 3:
        def f(r, k):
            return float(r[h.index(k)].replace(",", ""))
        per = [(f(r, "gpu__time_duration.sum"), f(r, "dram__bytes_read.sum") + f(r, "dram__bytes_write.sum"))
               for r in rows[2:]]
        print(f"# {len(per)} launches (duration {units[h.index('gpu__time_duration.sum')]}, "
              f"DRAM read+write {units[h.index('dram__bytes_read.sum')]}):")
        for i, (t, b) in enumerate(per):
            print(f"#   launch {i}: {t:10.2f} {b:10.2f}")
        print(f"#   mean:     {sum(t for t, _ in per) / len(per):10.2f} {sum(b for _, b in per) / len(per):10.2f}")
        print(f"# launch {li} in detail:")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"{k:70s} {v[i]:>16s} {units[i]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass",
                                          "--launch-skip", str(li), "--launch-count", "1"))))
    if len(src) > 2:
        sh = src[1]
        si, ws = sh.index("Source"), sh.index("Warp Stall Sampling (All Samples)")
        cols = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
        data = []
        for r in src[2:]:
            try:
                data.append((int(r[ws] or 0), r[si].strip(), {c: int(r[sh.index(c)] or 0) for c in cols}))
            except (ValueError, IndexError):
                pass
        tot = sum(d[0] for d in data) or 1
        agg = {}
        for d in data:
            for c, x in d[2].items():
                agg[c] = agg.get(c, 0) + x
        print("# warp-stall samples by reason (share of all samples)")
        for c, x in sorted(agg.items(), key=lambda t: -t[1])[:6]:
            print(f"  {c:24s} {x / tot:6.1%}")
        print("# top SASS instructions by stall samples")
        for d in sorted(data, key=lambda t: -t[0])[:8]:
            top = max(d[2].items(), key=lambda t: t[1])[0] if d[2] else ""
            print(f"  {d[0] / tot:6.1%}  {d[1][:64]:64s} {top}")


if __name__ == "__main__":
    main()
