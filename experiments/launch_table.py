"""Summarise an ncu --metrics launch list (csv) per kernel: launches, mean duration,
mean DRAM bytes, tensor-pipe and xu-pipe activity."""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    per[r[ki].split("(")[0][:70]][r[mi]].append(v)
print(f"{'kernel':70s} {'n':>4s} {'us':>9s} {'MB':>9s} {'tensor%':>8s} {'xu%':>6s}")
for k, m in sorted(per.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
    t = m["gpu__time_duration.sum"]
    b = [x + y for x, y in zip(m.get("dram__bytes_read.sum", [0] * len(t)), m.get("dram__bytes_write.sum", [0] * len(t)))]
    tp = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", [0])
    xu = m.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", [0])
    print(f"{k:70s} {len(t):4d} {sum(t)/len(t)/1e3:9.1f} {sum(b)/len(b)/1e6:9.1f} {sum(tp)/len(tp):8.1f} {sum(xu)/len(xu):6.1f}")
