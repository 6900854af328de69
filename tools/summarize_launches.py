"""Summarise an ncu launch list (gpu__time_duration + dram bytes) per kernel.

    python tools/summarize_launches.py gpurun_out/keystep_launches.csv > profiles/....txt

Writes a per-kernel table and, for the tcgen05 GEMM family, a JSON line with
per-key-step DRAM traffic used by bench.py's roofline.traffic.
"""
import csv
import json
import sys
from collections import defaultdict

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
data = rows[hi + 1:]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
launch = defaultdict(dict)
names = {}
for r in data:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    name = r[ki].split("(")[0]
    if name.startswith(("void at::", "at::")):
        continue  # torch's own setup kernels (weight conversion), not the step
    launch[r[ii]][r[mi]] = v
    names[r[ii]] = name
agg = defaultdict(lambda: defaultdict(float))
for lid, m in launch.items():
    n = names[lid]
    a = agg[n]
    a["calls"] += 1
    for k, v in m.items():
        a[k] += v
tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
print(f"# {path}: {len(launch)} launches, {tot / 1e6:.3f} ms total (ncu: serialised, cold cache)")
print(f"# {'ms':>9} {'share':>6} {'calls':>5} {'DRAM GB':>8} {'GB/s':>7}  kernel")
for n, a in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    t = a["gpu__time_duration.sum"]
    b = a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)
    print(f"  {t / 1e6:9.3f} {100 * t / tot:5.1f}% {int(a['calls']):5d} {b / 1e9:8.3f} {b / t:7.0f}  {n}")
g = [a for n, a in agg.items() if "tc_gemm_kernel" in n]
if g:
    b = sum(a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0) for a in g)
    print(json.dumps({"gemm_dram_bytes_per_key_step": b, "gemm_launches": int(sum(a["calls"] for a in g)),
                      "gemm_ncu_ms": sum(a["gpu__time_duration.sum"] for a in g) / 1e6}))
