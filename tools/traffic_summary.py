"""Per-class DRAM bytes from the ncu CSV of the bench's profiling pass
(tools/gpu/r02_traffic.sh: kernels renamed after their NVTX class range) ->
profiles/traffic_r02.json. Each class gets its measured DRAM bytes per class
bracket (the unit bench.py's events time and roofline.achieved counts), next
to the bracket count the plain run printed.

    python tools/traffic_summary.py gpurun_out/traffic_all.csv gpurun_out/traffic_plain.log > profiles/traffic_r02.json
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if "Kernel Name" in r][0]
ki, mi, ui, vi, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0,
         "nsecond": 1e-3, "msecond": 1e3}
per = collections.defaultdict(dict)
for r in rows:
    if len(r) != len(hdr) or r is hdr or r[ui] not in scale:
        continue
    per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * scale[r[ui]]
    per[r[idi]]["name"] = r[ki]
counts = {}
for line in open(sys.argv[2]):
    if line.startswith("{") and "class_launches" in line:
        counts = json.loads(line)["class_launches"]
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
kern = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in per.values():
    cls, _, kname = d["name"].partition("/")  # --print-nvtx-rename kernel: "<class range>/<kernel>"
    kname = kname.replace("void ", "").split("(")[0].split("<")[0].replace("ce::", "").strip()
    by = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    us = d.get("gpu__time_duration.sum", 0.0)
    for t in (tot[cls], kern[(cls, kname)]):
        t[0] += 1
        t[1] += by
        t[2] += us
classes = {}
for name, (kernels, by, us) in sorted(tot.items()):
    n = counts.get(name)
    classes[name] = {"kernels": kernels, "dram_bytes_total": by, "us_serial_cold": us, "class_launches": n,
                     "dram_bytes_per_launch": by / n if n else None,
                     "by_kernel": {k: {"launches": v[0], "dram_bytes": v[1], "us": v[2]}
                                   for (c, k), v in sorted(kern.items()) if c == name}}
print(json.dumps({"source": sys.argv[1], "rule": "ncu dram__bytes_read.sum + dram__bytes_write.sum summed over "
                  "the kernels inside each class's NVTX range, divided by the class brackets of the same pass",
                  "classes": classes}, indent=1))
