"""Summarise an ncu report (--set full) or a launch-list CSV into markdown.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep  > profiles/rNN/<name>.md
    python tools/ncu_summary.py --launches gpurun_out/launches.csv > profiles/rNN/launches.md
"""

import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Frequency", "Memory Throughput",
        "DRAM Throughput", "Compute (SM) Throughput", "Registers Per Thread", "Block Size", "Grid Size",
        "Achieved Occupancy", "Theoretical Occupancy", "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__warps_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "lts__t_bytes.sum", "smsp__inst_executed.sum"]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize(rep):
    print(f"# ncu summary: `{rep}`\n")
    rows = ncu_csv(rep, "details")
    if rows:
        hdr = rows[0]
        ik, iname, iunit, ival = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"),
                                  hdr.index("Metric Value"))
        by = collections.OrderedDict()
        for r in rows[1:]:
            if r[iname] in KEYS and (r[ik], r[iname]) not in by:
                by[(r[ik], r[iname])] = f"{r[ival]} {r[iunit]}".strip()
        kern = None
        for (k, name), v in by.items():
            if k != kern:
                print(f"\n## `{k}`\n\n| metric | value |\n|---|---|")
                kern = k
            print(f"| {name} | {v} |")
    raw = ncu_csv(rep, "raw")
    if len(raw) > 2:
        hdr = raw[0]
        print("\n### raw counters\n\n| counter | value |\n|---|---|")
        for key in RAW:
            if key in hdr:
                i = hdr.index(key)
                for r in raw[2:]:
                    print(f"| {key} | {r[i]} {raw[1][i]} |")
    src = ncu_csv(rep, "source")
    if len(src) > 2:
        hdr = src[1]
        reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        agg = collections.Counter()
        for r in src[2:]:
            for h in reasons:
                v = r[hdr.index(h)]
                if v:
                    try:
                        agg[h] += float(v)
                    except ValueError:
                        pass
        tot = sum(agg.values()) or 1.0
        print("\n### warp-stall samples (all warps)\n\n| reason | samples | share |\n|---|---|---|")
        for h, v in agg.most_common(10):
            print(f"| {h} | {v:.0f} | {v / tot:.1%} |")


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[start + 1:]:
        if len(r) > iv and r[iv]:
            v = float(r[iv].replace(",", ""))
            tot[r[ik]] += v
            cnt[r[ik]] += 1
    s = sum(tot.values()) or 1.0
    print(f"# launch list: `{path}` (gpu__time_duration.sum, ns; cold-cache, serialised)\n")
    print("| kernel | launches | total ns | share |\n|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| `{k[:90]}` | {cnt[k]} | {v:.0f} | {v / s:.1%} |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        summarize(sys.argv[1])
