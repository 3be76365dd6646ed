"""Summarise ncu reports / launch lists into profiles/*.md (run here, no GPU needed)."""
import collections
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "DRAM Frequency", "SM Frequency",
        "Elapsed Cycles", "SM Active Cycles", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Achieved Active Warps Per SM",
        "Eligible Warps Per Scheduler", "Issued Warp Per Scheduler", "L2 Hit Rate", "Grid Size",
        "Block Size", "Dynamic Shared Memory Per Block", "Cluster Size"]


def details(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "details", "--csv"], text=True)
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    res = collections.OrderedDict()
    name = None
    for row in r[1:]:
        d = dict(zip(h, row))
        name = d["Kernel Name"]
        if d["Metric Name"] in KEYS and d["Metric Name"] not in res:
            res[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rr = list(csv.reader(raw.splitlines()))
    hh = rr[0]
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if m in hh:
            res[m] = f"{rr[2][hh.index(m)]} {rr[1][hh.index(m)]}"
    return name, res


def stalls(rep, top=12):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                                   "sass"], text=True)
    rows = [r for r in csv.reader(out.splitlines()) if len(r) > 5 and r[0].startswith("0x")]
    tot = sum(int(x[2]) for x in rows) or 1
    lines = []
    for x in sorted(rows, key=lambda x: -int(x[2]))[:top]:
        lines.append(f"| `{x[1].strip()[:60]}` | {int(x[2])} | {100 * int(x[2]) / tot:.1f}% |")
    return lines


def launches(csvfile):
    rows = list(csv.reader(open(csvfile)))
    hdr = None
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg[d["Kernel Name"]][(d["Metric Name"], d["Metric Unit"])].append(
                float(d["Metric Value"].replace(",", "")))
    lines = ["| kernel | launches | metric | mean |", "|---|---|---|---|"]
    for k, v in agg.items():
        for (m, u), x in v.items():
            lines.append(f"| `{k[:70]}` | {len(x)} | {m} | {sum(x) / len(x):,.1f} {u} |")
    return lines


if __name__ == "__main__":
    out = sys.argv[1]
    parts = []
    for arg in sys.argv[2:]:
        if arg.endswith(".csv"):
            parts.append(f"## Launch list `{arg.split('/')[-1]}` (ncu, serialised, cold caches)\n")
            parts += launches(arg)
        else:
            name, res = details(arg)
            parts.append(f"\n## `{arg.split('/')[-1]}` -- {name[:100]}\n")
            parts.append("| metric | value |\n|---|---|")
            parts += [f"| {k} | {v} |" for k, v in res.items()]
            parts.append("\nTop stall lines (warp-stall samples):\n\n| SASS | samples | share |\n|---|---|---|")
            parts += stalls(arg)
        parts.append("")
    open(out, "w").write("\n".join(parts) + "\n")
    print(open(out).read())
